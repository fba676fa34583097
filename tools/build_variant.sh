#!/bin/bash
# Build a variant of libtnrd.so with extra -D flags into build_variants/.
# Usage: tools/build_variant.sh <name> [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_variants
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -shared -Xcompiler -fPIC \
     -Xcompiler -fvisibility=hidden "$@" -o build_variants/libtnrd_$name.so \
     paper_1702_07482_b200/csrc/tnrd_capi.cu paper_1702_07482_b200/csrc/tnrd_probe.cu
