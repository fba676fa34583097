#!/bin/bash
O=gpurun_out/r02_probe; mkdir -p $O
# tests on the tree, then the bounds build, phase trace, the no-backward ceiling probe
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
bash tools/bounds_run.sh r02_bounds
export TNRD_LIB_PATH=build_variants/libtnrd_phase.so
for a in "c3 32 4" "c5 8 4" "c2 1 10" "c4 1 4"; do timeout 300 python tools/phase_trace.py $a; done > $O/phase_trace_edge.txt 2>&1
cat $O/phase_trace_edge.txt
for v in tree nobwd; do
  if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
  timeout 300 python tools/batch_perf.py c3 > $O/batch_$v.txt 2>&1
  timeout 300 python tools/batch_perf.py c5 >> $O/batch_$v.txt 2>&1
  echo "== $v"; cat $O/batch_$v.txt
done
unset TNRD_LIB_PATH
timeout 900 python tools/grid_sweep.py c3 > $O/grid_sweep_c3.txt 2>&1; cat $O/grid_sweep_c3.txt
