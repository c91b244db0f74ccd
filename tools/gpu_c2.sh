mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/c2_launches.csv python bench.py --workload c2 --quick --steps 3 --warmup 1 > /dev/null 2>&1; echo rc=$?
