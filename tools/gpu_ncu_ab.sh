# ncu --set full of the C3 tile kernel for the in-tree and a variant library.
# Usage: bash tools/gpu_ncu_ab.sh <outdir> <variant .so> [workload] [batch] [kernel regex]
O=gpurun_out/$1; mkdir -p $O; B=$2; W=${3:-c3}; N=${4:-32}; K=${5:-stage_kernel_pt}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in base new; do
  if [ $v = base ]; then export TNRD_LIB_PATH=$B; else unset TNRD_LIB_PATH; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 \
      -o $O/$v python tools/prof_one.py $W $N > $O/ncu_$v.log 2>&1
  python tools/ncu_summary.py $O/$v.ncu-rep > $O/summary_$v.txt 2>&1
  python tools/ncu_sass_stats.py $O/$v.ncu-rep $((N*512*512)) >> $O/summary_$v.txt 2>&1
done
unset TNRD_LIB_PATH
