mkdir -p gpurun_out/r02l
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/r02l/pytest.txt 2>&1
tail -n 3 gpurun_out/r02l/pytest.txt
for c in 1 4; do for w in cfg2 cfg3; do
timeout 600 python bench.py --steps 5 --no-cpu-baseline --workload $w --chunks $c > gpurun_out/r02l/bench_${w}_c$c.json 2> gpurun_out/r02l/bench_${w}_c$c.err
python -c "
import json; d=json.loads(open('gpurun_out/r02l/bench_${w}_c$c.json').read().strip().splitlines()[-1]); print('$w c$c', '%.4g'%d['value'], d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], d['stage_ms'], d['gpu_launches'])" || tail -5 gpurun_out/r02l/bench_${w}_c$c.err
done; done
