# one GPU call: smoke, tests, bench, ncu launch list + full capture of the top kernels
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --quick > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_batched -s 1 -c 1 -o gpurun_out/prof_k3 python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_k3.log 2>&1; echo "ncu k3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1p_gemm -s 3 -c 1 -o gpurun_out/prof_k1p python bench.py --workload c5 --steps 1 --warmup 0 --quick > gpurun_out/ncu_k1p.log 2>&1; echo "ncu k1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f64_gemm -s 3 -c 1 -o gpurun_out/prof_f64 python bench.py --workload c4 --steps 1 --warmup 0 --quick > gpurun_out/ncu_f64.log 2>&1; echo "ncu f64 rc=$?"
ls -la gpurun_out
