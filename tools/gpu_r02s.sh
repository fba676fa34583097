#!/bin/bash
# EDGE backward (no fix-up pass on tile-aligned edges): tests, A/B bits + perf vs the fix_phi build
O=gpurun_out/r02_edge; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc $?" >> $O/pytest_gpu.log
tail -12 $O/pytest_gpu.log
timeout 300 python tools/ab_outputs.py $O/out_tree.npz > $O/ab.log 2>&1
TNRD_LIB_PATH=build_variants/libtnrd_noedge.so timeout 300 python tools/ab_outputs.py $O/out_noedge.npz >> $O/ab.log 2>&1
python tools/ab_compare.py $O/out_tree.npz $O/out_noedge.npz > $O/ab_bits_edge_vs_fixphi.txt 2>&1; tail -45 $O/ab_bits_edge_vs_fixphi.txt
rm -f $O/out_tree.npz $O/out_noedge.npz
for i in 1 2; do
  for v in tree noedge; do
    if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
    timeout 300 python tools/quick_perf.py > $O/perf_${v}_$i.txt 2>&1
    timeout 300 python tools/batch_perf.py c3 > $O/batch_${v}_$i.txt 2>&1
  done
done
unset TNRD_LIB_PATH
for v in tree noedge; do echo "== $v"; cat $O/perf_${v}_1.txt $O/perf_${v}_2.txt $O/batch_${v}_1.txt $O/batch_${v}_2.txt; done > $O/perf_all.txt
cat $O/perf_all.txt
