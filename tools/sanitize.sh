# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over a selection of GPU tests
# usage: bash tools/sanitize.sh TAG "pytest -k expression"
TAG=$1; K=$2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" -p no:cacheprovider > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "passed|failed|SUMMARY" $OUT/$tool.log | tail -2
done
