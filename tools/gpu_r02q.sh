#!/bin/bash
# cluster kernel: tests, grid sweep, TM variants, phase trace
O=gpurun_out/r02_cluster; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cluster.py -q > $O/pytest_cluster.log 2>&1
echo "pytest rc=$?" >> $O/pytest_cluster.log
tail -5 $O/pytest_cluster.log
timeout 900 python tools/grid_sweep.py c3 > $O/grid_sweep_c3.txt 2>&1; cat $O/grid_sweep_c3.txt
timeout 600 python tools/grid_sweep.py c5 > $O/grid_sweep_c5.txt 2>&1; cat $O/grid_sweep_c5.txt
for v in cltm0 cltm1; do
  TNRD_LIB_PATH=build_variants/libtnrd_$v.so timeout 300 python tools/cluster_perf.py 2>&1 | grep "c2 B=1\|c1 B=1" | grep "auto\|cl=4\|cl=6" > $O/cluster_perf_$v.txt
  echo "== $v"; cat $O/cluster_perf_$v.txt
done
export TNRD_LIB_PATH=build_variants/libtnrd_phase.so
for a in "c3 32 4" "c5 8 4" "c2 1 10" "c4 1 4"; do timeout 300 python tools/phase_trace.py $a; done > $O/phase_trace.txt 2>&1
cat $O/phase_trace.txt
