timeout 1500 python -m pytest tests -m gpu -q -x > /tmp/pt.txt 2>&1; tail -n 2 /tmp/pt.txt
for v in default default; do for w in cfg2 cfg3; do timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 1 > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$v $w', d['ms_per_step'], {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done; done
