#!/usr/bin/env bash
# Collects the ncu evidence for one round (run under gpurun, 1 GPU):
#   1. launch list with device times (--metrics gpu__time_duration.sum, cold-cache, serialised)
#   2. one `ncu --set full` capture each of the feature kernel and the tcgen05 predictor
# at the exact bench.py workload, then summarises them into profiles/ (tools/ncu_summary.py).
# Usage: tools/profile_round.sh r01 [workload]   (output: gpurun_out/prof_<r>_<workload>)
set -euo pipefail
R=${1:-r01}
W=${2:-cfg2}
OUT=gpurun_out/prof_${R}_$W
mkdir -p "$OUT"
BENCH="python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" $BENCH \
  > "$OUT/launches_bench.log" 2>&1 || true
FEAT=attn_schedule_cross
SKIP=3; COUNT=1; PSKIP=3
case "$W" in
  cfg2) ;;
  cfg4) SKIP=6; COUNT=2; PSKIP=20 ;;  # a step: 2 attention launches (one per serving model)
  splitk) FEAT=featurize_splitk_cross ;;
  *) FEAT=uniform_prepass ;;  # uniform families run the fused pass: pre-pass + predict_tcgen05_fused
esac
ncu --set full --clock-control none --import-source on -k regex:$FEAT -s $SKIP -c $COUNT -o "$OUT/featurize" $BENCH \
  > "$OUT/featurize.log" 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:predict_tcgen05 -s $PSKIP -c 1 -o "$OUT/predict" $BENCH \
  > "$OUT/predict.log" 2>&1 || true
ls -la "$OUT"
