# compute-sanitizer evidence: logs under gpurun_out/sanitize_<tool>.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
