# quick GPU check: probes + a test subset.  Usage: bash tools/gpu_quick.sh <outdir> [pytest -k expr]
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
[ -x tools/probes/ffma2_probe ] && tools/probes/ffma2_probe > $O/ffma2_probe.txt 2>&1
if [ -n "$2" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$2" > $O/pytest.log 2>&1
  echo "pytest rc $?" >> $O/pytest.log
fi
