#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2g; mkdir -p $O
timeout 600 python tools/c3_shard_time.py > $O/c3_shard.txt 2>&1; echo "rc=$?" >> $O/c3_shard.txt
python - > $O/mc_attr.txt 2>&1 <<'PY'
import ctypes
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(dev), 0)
for name, attr in (("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                   ("HANDLE_TYPE_POSIX_FD_SUPPORTED", 103)):
    v = ctypes.c_int(-1)
    rc = cuda.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, attr, rc, v.value)
PY
nvidia-smi topo -m >> $O/mc_attr.txt 2>&1
BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --workload c5 --steps 2 --warmup 1 --quick > $O/c5_share2.json 2> $O/c5_share2.err; echo "rc=$?" >> $O/c5_share2.err
