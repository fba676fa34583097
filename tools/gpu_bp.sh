# batch_perf.py for several variants (two rounds).  Usage: bash tools/gpu_bp.sh <outdir> <variant>...
O=gpurun_out/$1; shift; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2; do
for v in "$@"; do
  if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
  python tools/batch_perf.py c3 > $O/bp_${v}_$i.txt 2>&1
  python tools/batch_perf.py c5 >> $O/bp_${v}_$i.txt 2>&1
done; done
unset TNRD_LIB_PATH
for v in "$@"; do echo "== $v"; cat $O/bp_${v}_1.txt $O/bp_${v}_2.txt | sed 's/sm_mhz.*//' | sort -k2 -V; done > $O/all.txt
