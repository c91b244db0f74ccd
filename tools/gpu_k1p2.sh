timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
for w in c5 c4 c2; do timeout 300 python bench.py --workload $w --quick --steps 3 --warmup 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'])"; done
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1p_gemm -s 3 -c 1 -o gpurun_out/prof_k1p python bench.py --workload c5 --steps 1 --warmup 0 --quick > gpurun_out/ncu_k1p.log 2>&1; echo "ncu rc=$?"
