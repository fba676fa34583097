#!/bin/bash
O=gpurun_out/r02_adj; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_adj.py -x -q -p no:cacheprovider > $O/pytest_adj.log 2>&1; echo "pytest rc $?" >> $O/pytest_adj.log; tail -30 $O/pytest_adj.log
for k in 0 12; do
  TNRD_STAGE_KERNEL=$k timeout 300 python tools/batch_perf.py c3 > $O/batch_mode$k.txt 2>&1; echo "== mode $k"; cat $O/batch_mode$k.txt
done
