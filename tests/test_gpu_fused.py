"""Fused row-sharded exchange (CTA-pair epilogue stores into every rank's
buffers over CUDA IPC, flag barrier in peer memory) — two ranks sharing one
B200 (the box has one GPU): the IPC mappings, peer stores, row offsets and the
cross-process barrier are exercised exactly as across GPUs.  The result must be
BITWISE the single-GPU chain."""

import os
import socket

import numpy as np
import pytest

import oracle



def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, ks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_1204_3052_b200 as mx
    from paper_1204_3052_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        eng = mx.Engine(0)
        eng.set_f32_datapath("3xtf32")  # the row shards' datapath: bitwise comparable
        a_np = oracle.scaled_input(n, np.float32, 42)
        a = torch.from_numpy(a_np).cuda()
        res = {}
        for k in ks:
            got = D.exponentiate_row_sharded_fused(a, k, engine=eng).cpu().numpy()
            res[k] = (got.tobytes(), eng.power(a_np, k).tobytes() if rank == 0 else None)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n", [(2, 1024), (4, 1024), (3, 1500)])
def test_fused_exchange_ranks_one_gpu_bitwise(world, n):
    """2 and 4 ranks (power-of-two row blocks) and 3 ranks on a padded order
    (1500 -> 3 x 512 rows): peer stores and the flag barrier with npeers > 2."""
    import torch.multiprocessing as mp

    ks = (16, 13)  # 13: plan with MULTIPLY_BASE steps
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, ks, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for k in ks:
        single = results[0][k][1]
        for r in range(world):
            assert results[r][k][0] == single, (k, r)
    if n <= 1024:
        ref = oracle.exponentiate(oracle.scaled_input(n, np.float32, 42), 13)
        got = np.frombuffer(results[1][13][0], dtype=np.float32).reshape(n, n)
        assert oracle.compare(got, ref)[2] <= 16 * 5 * np.sqrt(n) * 2.0 ** -24


def _worker_k1ph(rank, world, port, n, ks, cancel, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_1204_3052_b200 as mx
    from paper_1204_3052_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        eng = mx.Engine(0)  # default datapath: K1PH at these sizes
        if cancel:
            rng = np.random.default_rng(5)
            nil = np.zeros((n, n))
            nil[: n // 2, n // 2:] = rng.uniform(-1, 1, (n // 2, n // 2))
            a_np = (nil + 1e-6 * rng.uniform(-1, 1, (n, n))).astype(np.float32)
        else:
            a_np = oracle.scaled_input(n, np.float32, 42)
        a = torch.from_numpy(a_np).cuda()
        ctx = D.RowShardedK1PH(n, a.device, engine=eng)
        res = {}
        try:
            for k in ks:
                got = ctx.power(a, k).cpu().numpy()
                res[k] = (got.tobytes(), eng.power(a_np, k).tobytes() if rank == 0 else None,
                          ctx.last_fallback)
        finally:
            ctx.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,cancel", [(2, 1024, False), (4, 2048, False), (3, 1500, False),
                                            (2, 1024, True)])
def test_k1ph_row_shards_ranks_one_gpu_bitwise(world, n, cancel):
    """RowShardedK1PH (one process per rank sharing the B200): K1PH row-block
    GEMMs, maxima into every rank's state over CUDA IPC, rows split into every
    rank's planes, flag barriers — BITWISE the single-GPU K1PH chain; a
    cancelling input falls back to the 3xTF32 fused exchange on every rank,
    bitwise the single-GPU chain's own recomputation."""
    import torch.multiprocessing as mp

    ks = (6,) if cancel else (16, 13, 2)  # 2: a one-step plan (the first step is the last)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_k1ph, args=(r, world, port, n, ks, cancel, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for k in ks:
        single = results[0][k][1]
        for r in range(world):
            assert results[r][k][0] == single, (k, r)
            assert results[r][k][2] == cancel, (k, r)


def test_fused_layout():
    from paper_1204_3052_b200 import distributed as D

    assert D.fused_layout(8192, 8) == (8192, 1024)
    assert D.fused_layout(1000, 2) == (1024, 512)
    n_p, rows = D.fused_layout(3000, 4)
    assert rows % 256 == 0 and n_p == 4 * rows and n_p >= 3000


@pytest.mark.gpu
def test_fused_exchange_nvls_multicast_single_rank_bitwise():
    """The NVLS variant (mxp_mc_*: a multicast object with this GPU's memory
    bound to it; the epilogue's multimem.st goes through the switch) on one
    rank: BITWISE the single-GPU chain.  The box has one GPU, so this is the
    whole multicast machinery with a team of one; ranks sharing a GPU cannot
    join one multicast team (they take the IPC path above)."""
    import torch
    import torch.distributed as dist

    import paper_1204_3052_b200 as mx
    from paper_1204_3052_b200 import distributed as D

    eng = mx.Engine(0)
    eng.set_f32_datapath("3xtf32")
    if not eng.mc_supported():
        pytest.skip("no NVLS multicast on this device")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        for n in (1024, 2000):
            a_np = oracle.scaled_input(n, np.float32, 42)
            a = torch.from_numpy(a_np).cuda()
            try:
                chain = D.RowShardedFused(n, a.device, engine=eng, multicast=True)
            except RuntimeError as exc:
                # the one-GPU sandbox reports MULTICAST_SUPPORTED but refuses
                # cuMulticastCreate (profiles/r02_mc_probe.txt)
                pytest.skip(f"multicast object refused here: {exc}")
            try:
                assert chain.multicast
                for k in (16, 13):
                    got = chain.power(a, k)
                    torch.cuda.synchronize()
                    assert got.cpu().numpy().tobytes() == eng.power(a_np, k).tobytes(), (n, k)
            finally:
                chain.close()
    finally:
        dist.destroy_process_group()
