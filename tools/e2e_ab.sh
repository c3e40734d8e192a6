timeout 900 python -m pytest tests/test_gpu_e2e.py -q -x 2>&1 | tail -2
for v in preve2e cur preve2e cur; do
 if [ $v = cur ]; then unset SYNPERF_LIB; else export SYNPERF_LIB=variants/lib_$v.so; fi
 timeout 300 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], [ (k['name'], round(k['ms'],3)) for k in d.get('kernels',[]) if 'expand' in k['name']] if isinstance(d.get('kernels'), list) else d.get('kernels',{}).get('e2e_expand'))"
done
