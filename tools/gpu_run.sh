mkdir -p gpurun_out/r02j
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02j/pytest.txt 2>&1
tail -n 5 gpurun_out/r02j/pytest.txt
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/r02j/bench_cfg2.json 2> gpurun_out/r02j/bench_cfg2.err
timeout 600 python bench.py --steps 5 --no-cpu-baseline --workload cfg3 > gpurun_out/r02j/bench_cfg3.json 2> gpurun_out/r02j/bench_cfg3.err
timeout 600 python bench.py --steps 5 --no-cpu-baseline --workload cfg5 > gpurun_out/r02j/bench_cfg5.json 2> gpurun_out/r02j/bench_cfg5.err
for w in cfg2 cfg3 cfg5; do python -c "
import json; d=json.loads(open('gpurun_out/r02j/bench_$w.json').read().strip().splitlines()[-1]); print('$w', '%.4g'%d['value'], d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'])"; done
