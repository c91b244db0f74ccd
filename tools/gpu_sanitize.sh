mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
