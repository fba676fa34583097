bash tools/gpu_variants.sh r02h tree m9rf3 m9rf4
O=gpurun_out/r02h
# split kernel: scalar (tree) vs TM2 variant, ncu full
for v in tree splittm2; do
  if [ $v = tree ]; then unset TNRD_LIB_PATH; else export TNRD_LIB_PATH=build_variants/libtnrd_$v.so; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:stage_kernel_split -s 5 -c 1 \
      -o $O/split_$v python tools/prof_one.py c2 1 > $O/ncu_split_$v.log 2>&1
  python tools/ncu_summary.py $O/split_$v.ncu-rep > $O/summary_split_$v.txt 2>&1
  python tools/ncu_sass_stats.py $O/split_$v.ncu-rep $((512*512)) >> $O/summary_split_$v.txt 2>&1
done
unset TNRD_LIB_PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c2.csv python tools/prof_one.py c2 1 > /dev/null 2>&1
tools/probes/mma_rate_probe > $O/mma_rate.txt 2>&1
