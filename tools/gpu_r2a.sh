#!/bin/bash
# round 2, session A: full GPU suite, bench, K1C under ncu (cooperative vs not)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2a/smi.txt
nproc >> gpurun_out/r2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 -s > gpurun_out/r2a/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a/pytest.log
timeout 600 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
echo "bench rc=$?" >> gpurun_out/r2a/bench.err
for v in coop nocoop; do
  if [ $v = nocoop ]; then export MXP_LIB_PATH=$PWD/tools/_variants/libmxp_nocoop.so; fi
  timeout 300 python tools/c2_once.py c2 3 > gpurun_out/r2a/plain_$v.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/r2a/ncu_launch_$v.csv python tools/c2_once.py c2 3 > gpurun_out/r2a/ncu_launch_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/r2a/ncu_launch_$v.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1c -c 1 \
     -o gpurun_out/r2a/prof_k1c_$v python tools/c2_once.py c2 2 > gpurun_out/r2a/ncu_full_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/r2a/ncu_full_$v.log
done
unset MXP_LIB_PATH
