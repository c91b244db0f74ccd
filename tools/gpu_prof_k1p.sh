mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1p_gemm -s 3 -c 1 -o gpurun_out/prof_k1p python bench.py --workload c5 --steps 1 --warmup 0 --quick > gpurun_out/ncu_k1p.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_k1p.log
