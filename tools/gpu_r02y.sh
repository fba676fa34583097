#!/bin/bash
# C1 / C2 streamed e2e vs stream depth and cluster size (bench.py e2e key)
O=gpurun_out/r02_depth; mkdir -p $O
for w in c1 c2; do
for d in 4 6 8 12; do for cl in 0 3; do
  [ $w = c2 ] && [ $cl = 3 ] && continue
  TNRD_STREAM_DEPTH=$d TNRD_CLUSTER_SIZE=$cl python bench.py --workload $w --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('$w depth $d cl $cl: value %.1f e2e %.1f lat %.3f' % (d['value'], d['e2e']['value'], d['e2e_latency']['ms']))"
done; done; done | tee $O/depth_sweep.txt
TNRD_AUTO_CLUSTER=0 python bench.py --workload c1 --no-cpu-baseline > $O/b.json 2> $O/b.err; python -c "
import json; d=json.load(open('$O/b.json')); print('c1 split (TNRD_AUTO_CLUSTER=0): value %.1f e2e %.1f lat %.3f' % (d['value'], d['e2e']['value'], d['e2e_latency']['ms']))" | tee -a $O/depth_sweep.txt
