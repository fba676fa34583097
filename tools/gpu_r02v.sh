#!/bin/bash
O=gpurun_out/r02_adj; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_adj.py -x -q -p no:cacheprovider > $O/pytest_adj.log 2>&1; echo "pytest rc $?" >> $O/pytest_adj.log; tail -4 $O/pytest_adj.log
TNRD_STAGE_KERNEL=12 timeout 300 python tools/batch_perf.py c3 > $O/batch_mode12.txt 2>&1; cat $O/batch_mode12.txt
TNRD_STAGE_KERNEL=12 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_adj.csv python tools/prof_one.py c3 64 > $O/ncu_launch.log 2>&1
python tools/launch_times.py $O/launches_adj.csv | tee $O/launch_times_adj.txt
TNRD_STAGE_KERNEL=12 ncu --set full --import-source on --clock-control none -k regex:adj_kernel -s 6 -c 1 -o $O/adj python tools/prof_one.py c3 64 > $O/ncu_adj.log 2>&1
python tools/ncu_summary.py $O/adj.ncu-rep > $O/ncu_summary_adj.txt 2>&1; python tools/ncu_sass_stats.py $O/adj.ncu-rep $((64*512*512)) >> $O/ncu_summary_adj.txt 2>&1
ncu -i $O/adj.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
for k in ('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tensor.sum','sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'):
    for i,n in enumerate(h):
        if n==k: print(k, v[i])
for i,n in enumerate(h):
    if 'tensor' in n: print(n, v[i])
" >> $O/ncu_summary_adj.txt 2>&1
rm -f $O/*.ncu-rep
cat $O/ncu_summary_adj.txt
