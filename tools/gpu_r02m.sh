O=gpurun_out/r02m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TNRD_LIB_PATH=build_variants/libtnrd_base.so timeout 300 python tools/ab_outputs.py /tmp/base.npz > /dev/null 2>&1
timeout 300 python tools/ab_outputs.py /tmp/new.npz > $O/ab_new.log 2>&1
python tools/ab_compare.py /tmp/base.npz /tmp/new.npz > $O/bits.txt 2>&1
TNRD_LIB_PATH=build_variants/libtnrd_trace.so python tools/split_trace.py 0 c2 > $O/trace_c2.txt 2>&1
bash tools/gpu_variants.sh r02m tree nomap
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "split or tiles or param_taps or contract or batch_fork or scene or strips" > $O/pytest.log 2>&1
echo "pytest rc $?" >> $O/pytest.log
