# A/B of attention variants: parity (attention tests) + cfg2 featurize/fused + cfg4 step
for v in "$@"; do
 if [ $v = cur ]; then unset SYNPERF_LIB; else export SYNPERF_LIB=variants/lib_$v.so; fi
 r=$(timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_e2e.py tests/test_gpu_range.py -q -x -k "attention or compose or plan or range" 2>&1 | tail -1)
 t2=$(timeout 300 python tools/time_stages.py --reps 10 --fused --workload cfg2 2>&1 | tail -1 | sed 's/.*featurize/featurize/')
 t4=$(timeout 300 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms_per_step'])")
 echo "$v | $r | cfg2 $t2 | cfg4 $t4"
done
unset SYNPERF_LIB
