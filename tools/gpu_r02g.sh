bash tools/gpu_variants.sh r02g tree c5tm3 splittm2 splittm3
mkdir -p gpurun_out/r02g
for v in c5tm3 splittm2 splittm3; do
  TNRD_LIB_PATH=build_variants/libtnrd_$v.so timeout 300 python tools/ab_outputs.py /tmp/$v.npz > /dev/null 2>&1
done
TNRD_LIB_PATH=build_variants/libtnrd_base.so timeout 300 python tools/ab_outputs.py /tmp/base.npz > /dev/null 2>&1
for v in c5tm3 splittm2 splittm3; do python tools/ab_compare.py /tmp/base.npz /tmp/$v.npz > gpurun_out/r02g/bits_$v.txt 2>&1; done
