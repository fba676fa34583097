#!/bin/bash
O=gpurun_out/r02_e2e; mkdir -p $O
python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['value'], d['e2e'], d['roofline']['executed_frac'], d['roofline']['frac'])"
python bench.py --workload c5 > $O/bench_c5.json 2> $O/bench_c5.err; python -c "
import json; d=json.load(open('$O/bench_c5.json')); print('c5', d['value'], d['e2e']['value'], d['e2e']['steps'], d['roofline']['executed_frac'])"
python bench.py --workload c4 > $O/bench_c4.json 2> $O/bench_c4.err; python -c "
import json; d=json.load(open('$O/bench_c4.json')); print('c4', d['value'], d['e2e']['value'], d['e2e']['steps'], d['roofline']['executed_frac'])"
tail -3 $O/bench_c3.err
