# A/B timing of variants/lib_<name>.so: tools/gpu_ab.sh outdir workload name...
out=$1; w=$2; shift 2
mkdir -p $out
for v in "$@"; do
  if [ $v = default ]; then unset SYNPERF_LIB; else export SYNPERF_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/time_stages.py --reps 10 --workload $w > $out/stages_${w}_$v.txt 2>&1
done
unset SYNPERF_LIB
tail -n 1 $out/stages_${w}_*.txt
