# compute-sanitizer runs of the small end-to-end driver (GPU box); logs under gpurun_out/
mkdir -p gpurun_out
python tools/sanitize_driver.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/san_plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -2 | tr '\n' ' ')"
done
