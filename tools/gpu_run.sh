mkdir -p gpurun_out/r02w
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02w/pytest.txt 2>&1; tail -n 4 gpurun_out/r02w/pytest.txt
timeout 600 python bench.py > gpurun_out/r02w/bench_cfg2.json 2> gpurun_out/r02w/bench_cfg2.err
python -c "
import json; d=json.loads(open('gpurun_out/r02w/bench_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', '%.4g'%d['value'], d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], d.get('parity'), d['roofline'])"
