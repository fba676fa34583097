set -x
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/pytest.log 2>&1
echo "pytest rc $?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -3 $O/pytest.log
