#!/bin/bash
# compute-sanitizer over tools/sanitize.py (memcheck, synccheck, initcheck, racecheck)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  echo "== $tool" >> $O/sanitize.txt
  timeout 1500 $S --tool $tool python tools/sanitize.py 2>&1 | tail -4 >> $O/sanitize.txt
done
echo "== initcheck (--check-api-memory-access no)" >> $O/sanitize.txt
timeout 1500 $S --tool initcheck --check-api-memory-access no python tools/sanitize.py 2>&1 | tail -4 >> $O/sanitize.txt
echo "== racecheck" >> $O/sanitize.txt
timeout 2400 $S --tool racecheck python tools/sanitize.py 2>&1 | grep -E "Race reported|RACECHECK SUMMARY|sanitize workload" | sort | uniq -c | head -20 >> $O/sanitize.txt
