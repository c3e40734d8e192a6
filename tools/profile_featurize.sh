#!/usr/bin/env bash
# ncu captures of the standalone HBM-bound feature kernels (the two-call path,
# bench.py --fused off): featurize_uniform_cross on cfg5 and cfg3,
# featurize_splitk_cross on split-K.  Output: gpurun_out/prof_feat/
set -u
OUT=gpurun_out/prof_feat
mkdir -p $OUT
for w in cfg5 cfg3; do
  timeout 900 ncu --set full --clock-control none -k regex:featurize_uniform_cross -s 2 -c 1 -o $OUT/uniform_$w \
    python bench.py --workload $w --fused off --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/uniform_$w.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:featurize_splitk_cross -s 2 -c 1 -o $OUT/splitk \
  python bench.py --workload splitk --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/splitk.log 2>&1
ls -la $OUT
