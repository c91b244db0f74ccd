# One ncu --set full capture per secondary kernel (K1P, K2 f64, K1 cluster split-K, K3B),
# each a single launch in steady state; summarise here with tools/ncu_summary.py.
mkdir -p gpurun_out
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:k1p_gemm -s 3 -c 1 -o gpurun_out/prof_k1p -f python bench.py --workload c5 --steps 1 --warmup 0 --quick --no-extras > gpurun_out/ncu_k1p.log 2>&1; echo "k1p rc=$?"
$NCU -k regex:f64_gemm -s 3 -c 1 -o gpurun_out/prof_f64 -f python bench.py --workload c4 --steps 1 --warmup 0 --quick --no-extras > gpurun_out/ncu_f64.log 2>&1; echo "f64 rc=$?"
MXP_K1C=0 $NCU -k regex:k1_gemm -s 6 -c 1 -o gpurun_out/prof_k1 -f python bench.py --workload c2 --steps 1 --warmup 0 --quick --no-extras > gpurun_out/ncu_k1.log 2>&1; echo "k1 rc=$?"
$NCU -k regex:k3b_batched -c 1 -o gpurun_out/prof_k3b -f python -c "
import sys, math, torch; sys.path.insert(0, '.')
import paper_1204_3052_b200 as mx
eng = mx.Engine(0); n, B, k = 128, 8192, 1000
a = torch.empty((B, n, n), dtype=torch.float32, device='cuda'); o = torch.empty_like(a)
eng.random_device(a.data_ptr(), n, B, seed0=42, scale=math.sqrt(12.0 / n))
eng.power_batched_device(a.data_ptr(), o.data_ptr(), n, B, k); eng.synchronize(); print('k3b ok')
" > gpurun_out/ncu_k3b.log 2>&1; echo "k3b rc=$?"
ls -la gpurun_out/*.ncu-rep
