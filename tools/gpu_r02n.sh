O=gpurun_out/r02n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TNRD_LIB_PATH=build_variants/libtnrd_trace.so python tools/split_trace.py 0 c2 > $O/trace_c2.txt 2>&1
TNRD_LIB_PATH=build_variants/libtnrd_trace.so TRACE_OUT=$O/trace.npy python tools/split_trace.py 0 c2 > /dev/null 2>&1
bash tools/gpu_variants.sh r02n tree nomap
