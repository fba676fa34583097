O=gpurun_out/r02i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2; do
for v in base tree; do
  if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
  python tools/batch_perf.py c3 > $O/bp_${v}_$i.txt 2>&1
  python tools/batch_perf.py c5 >> $O/bp_${v}_$i.txt 2>&1
done; done
unset TNRD_LIB_PATH
for f in $O/bp_*; do echo "== $f"; cat $f; done > $O/all.txt
