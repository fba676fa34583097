# quick_perf of several library variants on one box (two rounds, interleaved).
# Usage: bash tools/gpu_variants.sh <outdir> <name>...   (build_variants/libtnrd_<name>.so; "tree" = in-tree)
O=gpurun_out/$1; shift; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2; do
  for v in "$@"; do
    if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
    timeout 300 python tools/quick_perf.py > $O/perf_${v}_$i.txt 2>&1
  done
done
unset TNRD_LIB_PATH
for v in "$@"; do echo "== $v"; cat $O/perf_${v}_1.txt $O/perf_${v}_2.txt; done > $O/all.txt
