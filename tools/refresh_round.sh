mkdir -p gpurun_out/r
(time python -m pytest tests -m gpu -q) > gpurun_out/r/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r/smoke.log 2>&1
for w in cfg2 cfg1 cfg3 cfg4 cfg5 scaledmm splitk; do
  timeout 600 python bench.py --workload $w > gpurun_out/r/bench_$w.json 2> gpurun_out/r/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r/bench_reference.json 2> gpurun_out/r/bench_reference.err
tail -2 gpurun_out/r/pytest.log; tail -1 gpurun_out/r/smoke.log
for w in cfg2 cfg1 cfg3 cfg4 cfg5 scaledmm splitk; do python -c "
import json; d=json.loads(open('gpurun_out/r/bench_$w.json').read().strip().splitlines()[-1]); print('$w', '%.3g'%d['value'], '%.3f'%d['ms_per_step'], d['roofline']['kernel'], '%.3f'%(d['roofline']['frac'] or 0), '%.3g'%d['e2e']['value'], d['clocks']['sm_mhz'])"; done
