set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_shim.py -q -m gpu > $O/shim.log 2>&1; echo "shim rc=$?"; tail -2 $O/shim.log
./oracle/_ref/shim_driver
for tool in racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > $O/san_$tool.txt 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 $O/san_$tool.txt
done
