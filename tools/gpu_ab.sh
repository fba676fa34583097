# A/B of a variant library against the in-tree one: output bits + quick perf.
# Usage: bash tools/gpu_ab.sh <outdir> <variant .so>
O=gpurun_out/$1; mkdir -p $O; B=$2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TNRD_LIB_PATH=$B timeout 300 python tools/ab_outputs.py $O/base.npz > $O/ab_base.log 2>&1
timeout 300 python tools/ab_outputs.py $O/new.npz > $O/ab_new.log 2>&1
python tools/ab_compare.py $O/base.npz $O/new.npz > $O/ab_compare.txt 2>&1
rm -f $O/base.npz $O/new.npz
for i in 1 2; do
  TNRD_LIB_PATH=$B timeout 300 python tools/quick_perf.py > $O/perf_base_$i.txt 2>&1
  timeout 300 python tools/quick_perf.py > $O/perf_new_$i.txt 2>&1
done
