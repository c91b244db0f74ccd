timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -4
BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-extras 2>&1 | tail -2 | cut -c1-600
