"""Multi-process host logic of the multi-GPU paths, world_size 2 on the gloo
backend (CPU).  The device compute is replaced by the oracle (test
infrastructure), which makes the sharded chains BITWISE comparable with the
unsharded oracle chain: row sharding and batch sharding must not change a
single element's arithmetic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1204_3052_b200 import distributed as D


class OracleOps:
    """CPU stand-in for EngineOps (same call signatures)."""

    def gemm_rows(self, a_rows, b, out):
        a = a_rows.numpy()
        bb = b.numpy()
        full = np.zeros((bb.shape[0], bb.shape[0]), dtype=bb.dtype)
        full[: a.shape[0]] = a
        out.copy_(torch.from_numpy(oracle.matmul_rows(full, bb, 0, a.shape[0], 1)))

    def power_batched(self, a, k, out):
        out.copy_(torch.from_numpy(oracle.exponentiate_batched(a.numpy(), k, 1)))

    def prepare_rhs(self, b):
        self._b = b.numpy().copy()

    def gemm_rows_prepared(self, a_rows, out):
        self.gemm_rows(a_rows, torch.from_numpy(self._b), out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, k, dtype, q, chunks=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = torch.from_numpy(oracle.scaled_input(n, dtype, 42))
        out = D.exponentiate_row_sharded(a, k, ops=OracleOps(), chunks=chunks)
        # batched: 5 matrices sharded unevenly over the ranks
        batch = torch.from_numpy(oracle.scaled_batch(16, 5, np.float32, 7))
        lo, hi = D.shard_range(5, rank, world)
        local = D.exponentiate_batched_sharded(batch[lo:hi].contiguous(), 13, ops=OracleOps())
        gathered = D.gather_batched(local, 5)
        if rank == 0:
            q.put((out.numpy().tobytes(), gathered.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,dtype,chunks", [(64, 13, np.float32, None), (37, 1000, np.float32, 3),
                                              (48, 257, np.float64, 2), (9, 2, np.float32, None),
                                              (70, 7, np.float32, 4)])
def test_row_and_batch_sharding_bitwise(n, k, dtype, chunks):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, dtype, q, chunks))
             for r in range(world)]
    for p in procs:
        p.start()
    got_rows, got_batch = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = oracle.scaled_input(n, dtype, 42)
    ref = oracle.exponentiate(a, k, 1)
    if k >= 1000:  # scaled input overflows at k=1000: compare non-finite patterns exactly too
        assert np.frombuffer(got_rows, dtype=dtype).tobytes() == ref.tobytes()
    assert got_rows == ref.tobytes()
    batch = oracle.scaled_batch(16, 5, np.float32, 7)
    assert got_batch == oracle.exponentiate_batched(batch, 13, 1).tobytes()


def test_shard_range_covers_exactly():
    for total in (0, 1, 5, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    assert D.padded_rows(8192, 8) == 1024 and D.padded_rows(37, 2) == 19
    # C5 layout: 8 ranks x 4 chunks of 256 rows (CTA-pair tiles), no padding
    assert D.chunk_layout(8192, 8) == (4, 256, 8192)
    ck, c, n_p = D.chunk_layout(37, 2, 3)
    assert ck == 3 and n_p == c * 2 * 3 and n_p >= 37
