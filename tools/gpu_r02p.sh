#!/bin/bash
# cluster kernel: tests + perf
mkdir -p gpurun_out/r02_cluster
timeout 900 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/r02_cluster/pytest_cluster.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_cluster/pytest_cluster.log
tail -15 gpurun_out/r02_cluster/pytest_cluster.log
timeout 600 python tools/cluster_perf.py > gpurun_out/r02_cluster/cluster_perf.txt 2>&1
cat gpurun_out/r02_cluster/cluster_perf.txt
