#!/bin/bash
# Build the library WITH the opt-in tensor-core / dataflow stage kernels
# (-DTNRD_EXPERIMENTS: tnrd_stage_tc.cuh, tnrd_stage_tc3.cuh,
# tnrd_stage_zf.cuh, tnrd_stage_fused.cuh) into
# paper_1702_07482_b200/libtnrd_exp.so.  The shipped libtnrd.so leaves them
# out.  Use it with TNRD_LIB_PATH, e.g.
#   TNRD_LIB_PATH=$PWD/paper_1702_07482_b200/libtnrd_exp.so python -m pytest tests/test_gpu_tc.py -m gpu
set -e
cd "$(dirname "$0")/.."
CSRC=paper_1702_07482_b200/csrc
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -shared -Xcompiler -fPIC \
     -Xcompiler -fvisibility=hidden -DTNRD_EXPERIMENTS \
     -o paper_1702_07482_b200/libtnrd_exp.so $CSRC/*.cu
