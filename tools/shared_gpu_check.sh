#!/bin/bash
# Functional check of bench.py's N > 1 path (torchrun, barriers, max-over-
# ranks reductions, per-rank shards, C4's per-stage halo exchange, and the
# `verify` output check against an N = 1 recomputation) on a ONE-GPU box:
# TNRD_BENCH_SHARED_GPU=1 puts every rank on cuda:0 with gloo (C4's halo
# rows host-staged).  Lines are marked not_a_measurement; the N-GPU numbers
# come from the driver's scaling run.
# Usage (under gpurun): bash tools/shared_gpu_check.sh <outdir>
O=gpurun_out/${1:-r02_nproc}
mkdir -p $O
export TNRD_BENCH_SHARED_GPU=1
P=29500
for spec in "2 c3" "8 c3" "2 c4" "8 c4" "2 c5" "8 c5" "2 c2"; do
  set -- $spec; P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P \
     bench.py --gpus $1 --workload $2 --steps 3 --warmup 3 > $O/n$1_$2.json 2> $O/n$1_$2.err
  echo "n$1 $2 EXIT $? verify=$(python -c "import json,sys; d=json.loads(open('$O/n$1_$2.json').read().strip().splitlines()[-1]); print(d.get('verify',{}).get('ok'), d.get('verify',{}).get('checked'))" 2>/dev/null)" >> $O/summary.txt
done
cat $O/summary.txt
