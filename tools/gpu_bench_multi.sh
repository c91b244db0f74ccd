#!/bin/bash
# the driver's multi-rank invocations on a one-GPU box (BENCH_SHARE_GPU=1: every
# rank on GPU 0, gloo): our arm self-launched with --gpus 2, the torchrun form,
# the C5 fused row-sharded workload, and the reference arm under torchrun
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
export BENCH_SHARE_GPU=1
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/share2.json 2> $O/share2.err; echo "rc=$?" >> $O/share2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > $O/torchrun2.json 2> $O/torchrun2.err; echo "rc=$?" >> $O/torchrun2.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workload c5 > $O/c5_share2.json 2> $O/c5_share2.err; echo "rc=$?" >> $O/c5_share2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/ref2.json 2> $O/ref2.err; echo "rc=$?" >> $O/ref2.err
unset BENCH_SHARE_GPU
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref1.json 2> $O/ref1.err; echo "rc=$?" >> $O/ref1.err
