bash tools/gpu_ab.sh gpurun_out/r02af cfg2 cur ns cur ns
