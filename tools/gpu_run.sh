mkdir -p gpurun_out/r02x
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -k "tcgen05_parity or full_size or equals_two or planner_and" > gpurun_out/r02x/pytest.txt 2>&1; tail -n 3 gpurun_out/r02x/pytest.txt; grep "fp16 " gpurun_out/r02x/pytest.txt | head
bash tools/gpu_ab.sh gpurun_out/r02x cfg2 head default
bash tools/gpu_ab.sh gpurun_out/r02x cfg3 head default
timeout 600 python bench.py --steps 10 > gpurun_out/r02x/bench_cfg2.json 2> gpurun_out/r02x/bench_cfg2.err
python -c "
import json; d=json.loads(open('gpurun_out/r02x/bench_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', '%.4g'%d['value'], d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], d.get('parity'))"
