timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/sanitize_racecheck.txt
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
