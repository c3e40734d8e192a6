#!/usr/bin/env bash
# Round evidence on one GPU box: ncu launch lists + full captures (profile_round.sh)
# for the BASELINE workloads, every bench line, the reference arm, GPU tests, smoke.
# Usage: tools/round_evidence.sh r02   (outputs under gpurun_out/)
R=${1:-r02}
mkdir -p gpurun_out/ev_$R
(time timeout 1500 python -m pytest tests -m gpu -q) > gpurun_out/ev_$R/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/ev_$R/smoke.log 2>&1
for w in cfg2 cfg3 cfg4 cfg5; do timeout 1200 bash tools/profile_round.sh $R $w > gpurun_out/ev_$R/prof_$w.log 2>&1; done
for w in cfg2 cfg1 cfg3 cfg4 cfg5 scaledmm splitk; do
  timeout 900 python bench.py --workload $w > gpurun_out/ev_$R/bench_$w.json 2> gpurun_out/ev_$R/bench_$w.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ev_$R/bench_reference.json 2> gpurun_out/ev_$R/bench_reference.err
tail -2 gpurun_out/ev_$R/pytest.log; tail -1 gpurun_out/ev_$R/smoke.log
for w in cfg2 cfg1 cfg3 cfg4 cfg5 scaledmm splitk; do python -c "
import json; d=json.loads(open('gpurun_out/ev_$R/bench_$w.json').read().strip().splitlines()[-1]); print('$w', '%.4g'%d['value'], '%.3f'%d['ms_per_step'], d['roofline']['kernel'], d['roofline'].get('frac'), 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'], (d.get('parity') or {}).get('pass'))" || tail -3 gpurun_out/ev_$R/bench_$w.err; done
tail -c 400 gpurun_out/ev_$R/bench_reference.json
