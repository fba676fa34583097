#!/bin/bash
O=gpurun_out/r02_m9; mkdir -p $O
for i in 1 2; do
for v in tree m9rf6; do
  if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
  timeout 300 python tools/batch_perf.py c5 > $O/batch_${v}_$i.txt 2>&1
  echo "== $v"; cat $O/batch_${v}_$i.txt
done
done
unset TNRD_LIB_PATH
