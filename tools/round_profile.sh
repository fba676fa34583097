#!/bin/bash
# One round's measurement set on a GPU box (run under gpurun): GPU tests,
# smoke, bench lines of every workload + the reference arm, the ncu launch
# list of the default bench command, ncu --set full captures of the top
# kernels (summaries + executed.json / traffic.json inputs).
# Usage: bash tools/round_profile.sh <outdir under gpurun_out/> [notest]
set -u
O=gpurun_out/$1
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ "${2:-}" != notest ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest.log 2>&1
  echo "pytest rc $?" >> $O/pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
fi
python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --workload c2 > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --workload c4 > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --workload c5 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/launches_c3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c2.csv \
    python tools/prof_one.py c2 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:stage_kernel_pt -s 2 -c 1 \
    -o $O/c3_tile python tools/prof_one.py c3 256 > $O/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:stage_kernel_cl -s 10 -c 1 \
    -o $O/c2_cluster python tools/prof_one.py c2 1 > $O/ncu_c2.log 2>&1
ncu --set full --clock-control none -k regex:stage_kernel_pt -s 2 -c 1 \
    -o $O/c4_tile python tools/prof_one.py c4 1 > $O/ncu_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:stage_kernel_pt -s 2 -c 1 \
    -o $O/c5_tile python tools/prof_one.py c5 32 > $O/ncu_c5.log 2>&1
ncu --set full --clock-control none -k regex:stage_kernel -s 10 -c 1 \
    -o $O/c1_cluster python tools/prof_one.py c1 1 > $O/ncu_c1.log 2>&1
# per pixel of ONE launch: C3 / C5 launches cover half the batch (batch fork)
PX_C3=$((128*512*512)); PX_C2=$((512*512)); PX_C4=$((16384*16384)); PX_C5=$((16*1024*1024)); PX_C1=$((256*256))
for r in c2_cluster:$PX_C2 c3_tile:$PX_C3 c4_tile:$PX_C4 c5_tile:$PX_C5 c1_cluster:$PX_C1; do
    n=${r%%:*}; px=${r#*:}
    python tools/ncu_summary.py $O/$n.ncu-rep > $O/ncu_summary_$n.txt 2>&1
    python tools/ncu_sass_stats.py $O/$n.ncu-rep $px >> $O/ncu_summary_$n.txt 2>&1
done
python tools/launch_times.py $O/launches_c3.csv > $O/launch_times_c3.txt 2>&1
python tools/launch_times.py $O/launches_c2.csv > $O/launch_times_c2.txt 2>&1
python tools/make_executed.py $O > $O/executed_update.txt 2>&1
rm -f $O/*.ncu-rep
ls -la $O
