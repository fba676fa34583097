#!/bin/bash
# auto = cluster kernels on small grids: full GPU suite, smoke, bench c2/c1/c3
O=gpurun_out/r02_cluster; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=8 > $O/pytest_gpu.log 2>&1
echo "pytest rc $?" >> $O/pytest_gpu.log
tail -25 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; cat $O/smoke.log
python bench.py --workload c2 > $O/bench_c2.json 2> $O/bench_c2.err; cut -c1-400 $O/bench_c2.json
python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; cut -c1-400 $O/bench_c1.json
python tools/cluster_perf.py 2>&1 | grep "auto  \|cl=auto" > $O/cluster_perf_auto.txt; cat $O/cluster_perf_auto.txt
