// Predictor stage, bf16 tcgen05/TMEM path (placeholder until the kernel lands).
#include <cuda_runtime.h>

#include "sp_internal.h"

namespace sp {

bool pack_bf16_model(const sp_mlp_desc &, const std::vector<double> *, const std::vector<double> *,
                     std::vector<uint16_t> &, std::vector<float> &, float &) {
  return false;
}

int launch_predict_tcgen05(const MlpBf16 &, const sp_features &, float *, float *, int, void *) {
  return (int)cudaErrorNotSupported;
}

}  // namespace sp
