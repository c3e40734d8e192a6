# A/B driver: tools/ab_run.sh outdir "workloads" variants...  (variant "cur" = the in-tree library)
out=$1; ws=$2; shift 2
mkdir -p $out
if [ -z "$NOTEST" ]; then timeout 600 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; tail -3 $out/pytest.txt; fi
for w in $ws; do for rep in 1 2; do for v in "$@"; do
 if [ $v = cur ]; then unset SYNPERF_LIB; else export SYNPERF_LIB=variants/lib_$v.so; fi
 timeout 300 python tools/time_stages.py --reps 10 --fused --workload $w 2>&1 | tail -1 | sed "s/^/$w $v /"
done; done; done
unset SYNPERF_LIB
