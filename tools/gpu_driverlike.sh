#!/bin/bash
# what the driver runs at round end, on a fresh box
O=gpurun_out/r02_driverlike; mkdir -p $O
python -m pytest tests/ -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log; tail -2 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log; cat $O/smoke.log
python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?"
python bench.py --gpus 1 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
python -c "
import json
d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); r=json.loads(open('$O/bench_ref.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'executed_frac', d['roofline']['executed_frac'], 'traffic', d['roofline']['traffic'], 'launches', d['gpu_launches'], 'clocks', d['clocks'])
print('ref', r['value'], r['cpu_baseline']['cores'], 'ratio e2e', d['e2e']['value']/r['value'])
print(sorted(d.keys()))"
