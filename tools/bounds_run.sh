#!/bin/bash
# Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
# the GPU test suite on a -DTNRD_BOUNDS build (every run-time shared-memory
# index and image coordinate of the stage kernels checked against its buffer,
# tnrd_stage.cuh TNRD_ASSERT); tests/conftest.py reads the violation counters
# at session end.  Usage (under gpurun): bash tools/bounds_run.sh <outdir under gpurun_out/>
O=gpurun_out/$1; mkdir -p $O
[ -f build_variants/libtnrd_bounds.so ] || bash tools/build_variant.sh bounds -DTNRD_BOUNDS > $O/build_bounds.log 2>&1
export TNRD_LIB_PATH=build_variants/libtnrd_bounds.so TNRD_BOUNDS_REPORT=$O/bounds_report.txt
rm -f $TNRD_BOUNDS_REPORT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --deselect tests/test_abi_cpu.py > $O/pytest_bounds.log 2>&1
echo "pytest rc $?" >> $O/pytest_bounds.log
tail -6 $O/pytest_bounds.log; cat $O/bounds_report.txt
