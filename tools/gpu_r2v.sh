#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2v; mkdir -p $O
CS=compute-sanitizer
{ echo "== memcheck"; timeout 1200 $CS --tool memcheck python tools/sanitize.py 2>&1 | tail -3
  echo "== racecheck"; timeout 1800 $CS --tool racecheck python tools/sanitize.py 2>&1 | grep -E "RACECHECK SUMMARY|Race reported|workload done|fixups" | sort | uniq -c | head -20
  echo "== synccheck"; timeout 1200 $CS --tool synccheck python tools/sanitize.py 2>&1 | tail -3
  echo "== initcheck (--check-api-memory-access no)"; timeout 1200 $CS --tool initcheck --check-api-memory-access no python tools/sanitize.py 2>&1 | tail -3
} > $O/sanitizer.txt 2>&1
