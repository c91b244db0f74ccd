"""Multi-GPU execution: one process per GPU, torch.distributed for plumbing.

Two strategies:

* ``exponentiate_batched_sharded`` — independent matrices (config 3): rank r
  takes the contiguous slice ``shard_range(batch, r, world)``; no collective
  on the data path, results are bitwise the single-GPU ones.
* ``exponentiate_row_sharded`` — one large matrix (config 5): each rank owns
  a set of row chunks of the running power.  Each step prepares the
  right-hand side once (RHS = P for SQUARE, the replicated base A for
  MULTIPLY_BASE, accumulator on the left as in expo.py:133-136), then computes
  its chunks ``P'[rows, :] = P[rows, :] @ RHS`` one after the other and
  all-gathers every chunk (NCCL over NVLink, ``async_op``) as soon as it is
  computed, so the exchange of chunk j overlaps the MMAs of chunk j+1; only
  the last chunk's gather is exposed.  Chunks are interleaved over the ranks
  (rank r's chunk j = global rows [(j W + r) c, +c)) so each chunk's gather
  lands in one contiguous slab of P'.  Every element keeps its full-K dot
  product on one GPU, so the result is bitwise equal to the single-GPU chain.

The per-step compute is injectable (``ops``) so the host-side sharding and
collective logic is tested with the gloo backend on CPU (tests/
test_distributed.py); on B200s the default ops call the C ABI
(mxp_gemm_rows / mxp_power_batched_device) on the engine's CUDA stream,
which is also the stream the NCCL all-gather is issued on.
"""

from __future__ import annotations

import math
from typing import Optional

from .expo import Step, plan_exponentiation


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, end) slice of `total` units for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def padded_rows(n: int, world: int) -> int:
    """Rows per rank when n is padded to a multiple of `world` (zero padding keeps
    the top-left n x n block of every power exact)."""
    return math.ceil(n / world)


class EngineOps:
    """Device ops over the C ABI, on the engine's stream (torch tensors in HBM)."""

    def __init__(self, engine):
        self.eng = engine

    def stream(self):
        import torch

        return torch.cuda.ExternalStream(self.eng.stream)

    def gemm_rows(self, a_rows, b, out):
        from . import _lib

        mode = _lib.MXP_F32 if str(b.dtype) == "torch.float32" else _lib.MXP_F64
        self.eng.gemm_rows_device(a_rows.data_ptr(), b.data_ptr(), out.data_ptr(), b.shape[0],
                                  a_rows.shape[0], mode)

    def prepare_rhs(self, b):
        from . import _lib

        mode = _lib.MXP_F32 if str(b.dtype) == "torch.float32" else _lib.MXP_F64
        self._n, self._mode = b.shape[0], mode
        self.eng.gemm_prepare_rhs_device(b.data_ptr(), b.shape[0], mode)

    def gemm_rows_prepared(self, a_rows, out):
        self.eng.gemm_rows_prepared_device(a_rows.data_ptr(), out.data_ptr(), self._n,
                                           a_rows.shape[0], self._mode)

    def power_batched(self, a, k, out):
        from . import _lib

        mode = _lib.MXP_F32 if str(a.dtype) == "torch.float32" else _lib.MXP_F64
        self.eng.power_batched_device(a.data_ptr(), out.data_ptr(), a.shape[1], a.shape[0], k, mode)


def _all_gather_slab(slab, local, group, dist, async_op):
    """slab[(r*c):(r+1)*c] <- local of rank r, on every rank (NCCL: one
    all_gather_into_tensor; gloo: the list form)."""
    if dist.get_backend(group) == "nccl":
        return dist.all_gather_into_tensor(slab, local, group=group, async_op=async_op)
    world = dist.get_world_size(group)
    return dist.all_gather(list(slab.chunk(world, dim=0)), local, group=group, async_op=async_op)


def chunk_layout(n: int, world: int, chunks: Optional[int] = None) -> tuple[int, int, int]:
    """(chunks per rank, rows per chunk, padded n) for the row-sharded chain.
    Rows per chunk are a multiple of 256 (the CTA-pair tile) when n allows."""
    if chunks is None:
        chunks = 4 if n >= 1024 * world else (2 if n >= 512 * world else 1)
    align = 256 if n >= 256 * world * chunks else 1
    c = math.ceil(n / (world * chunks * align)) * align
    return chunks, c, c * world * chunks


def exponentiate_row_sharded(a, power: int, group=None, ops=None, chunks: Optional[int] = None):
    """A^power for one n x n matrix with its rows sharded over the group.

    `a` is the full base matrix (torch tensor, replicated on every rank, on
    this rank's device).  Returns the full A^power on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = plan_exponentiation(power)
    n = a.shape[0]
    if power == 0:
        return torch.eye(n, dtype=a.dtype, device=a.device)
    if power == 1:
        return a.clone()
    ck, c, n_p = chunk_layout(n, world, chunks)
    slab = world * c
    if ops is None:
        from .engine import default_engine

        ops = EngineOps(default_engine(a.device.index or 0))
    stream = ops.stream() if hasattr(ops, "stream") else None
    caller = torch.cuda.current_stream(a.device) if stream is not None else None
    if stream is not None:
        stream.wait_stream(caller)  # `a` may still be in flight on the caller's stream
    ctx = torch.cuda.stream(stream) if stream is not None else _nullcontext()
    with ctx:
        base = torch.zeros((n_p, n_p), dtype=a.dtype, device=a.device)
        base[:n, :n] = a  # zero padding never mixes into the top-left n x n block
        full = base.clone()
        nxt = torch.empty_like(full)
        local = [torch.empty((c, n_p), dtype=a.dtype, device=a.device) for _ in range(ck)]
        for step in plan.steps:
            ops.prepare_rhs(full if step is Step.SQUARE else base)
            pending = []
            for j in range(ck):
                g0 = (j * world + rank) * c  # this rank's chunk j
                ops.gemm_rows_prepared(full[g0:g0 + c], local[j])
                # issued behind chunk j on the compute stream; chunk j+1's MMAs
                # are enqueued right away and overlap the transfer
                pending.append(_all_gather_slab(nxt[j * slab:(j + 1) * slab], local[j], group, dist,
                                                async_op=True))
            for work in pending:
                work.wait()  # the next step reads every row of P'
            full, nxt = nxt, full
        result = full[:n, :n].contiguous()
    if stream is not None:
        caller.wait_stream(stream)  # the result is complete before the caller reads it
        result.record_stream(caller)
    return result


def fused_layout(n: int, world: int) -> tuple[int, int]:
    """(padded n, rows per rank) for the fused exchange: 256-row CTA-pair row
    blocks per rank and n_p >= 1024 (the CTA-pair kernel's range)."""
    blk = 256 * world
    n_p = max(math.ceil(1024 / blk), math.ceil(n / blk)) * blk  # every rank: 256-row blocks
    return n_p, n_p // world


class RowShardedFused:
    """The fused row-sharded chain for one n x n FP32 matrix shape on a group:
    every rank's CTA-pair epilogue stores its new rows (tf32 hi/lo planes; fp32
    at the last step) straight into every rank's buffers over NVLink (CUDA IPC
    mappings), tile by tile, so the transfer overlaps the other tiles' MMAs; a
    flag barrier in peer memory orders the steps.  No collective library on
    the data path.  Bitwise equal to the single-GPU chain (same CTA-pair
    kernel, same per-element order).  Buffers and peer mappings are set up
    once (collective over the group) and reused by every ``power`` call;
    ``close`` (also collective) unmaps them."""

    _SHARED = ("p0_hi", "p0_lo", "p1_hi", "p1_lo", "out", "flags")
    _MC = ("p0_hi", "p0_lo", "p1_hi", "p1_lo", "out")  # one multicast group, five n_p^2 slots

    def __init__(self, n: int, device, group=None, engine=None, multicast=None):
        """multicast: True = NVLS multicast stores (one store per tile reaches
        every rank through the switch), False = per-peer stores over CUDA IPC,
        None = multicast when every rank has its own multicast-capable GPU."""
        import torch
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self.n_p, self.rows = fused_layout(n, self.world)
        if engine is None:
            from .engine import default_engine

            engine = default_engine(torch.device(device).index or 0)
        self.eng = engine
        n_p = self.n_p
        plane = n_p * n_p * 4
        self.buf = {k: torch.empty((n_p, n_p), dtype=torch.int32, device=device)
                    for k in ("base_hi", "base_lo")}
        self.buf["flags"] = torch.zeros(self.world, dtype=torch.int32, device=device)
        self.base = torch.zeros((n_p, n_p), dtype=torch.float32, device=device)
        # every rank on its own GPU, all of them multicast-capable?
        dev = torch.device(device)
        uuid = str(getattr(torch.cuda.get_device_properties(dev), "uuid", dev.index))
        caps = [None] * self.world
        dist.all_gather_object(caps, (uuid, self.eng.mc_supported()), group=group)
        possible = len({c[0] for c in caps}) == self.world and all(c[1] for c in caps)
        if multicast and not possible:
            raise RuntimeError("NVLS multicast needs one multicast-capable GPU per rank")
        self.multicast = possible if multicast is None else bool(multicast)
        self.mc = None
        if self.multicast:
            # rank 0 creates the multicast object, everyone imports / adds its
            # device, then (the team complete) binds its own memory to it
            info = [None]
            if self.rank == 0:
                try:
                    self.mc, handle, size = self.eng.mc_create(self.world, len(self._MC) * plane)
                    info = [(handle, size)]
                except Exception as exc:  # noqa: BLE001 - reported below, on every rank
                    info = [str(exc)]
            dist.broadcast_object_list(info, src=0, group=group)
            if isinstance(info[0], str):
                if multicast:
                    raise RuntimeError(f"NVLS multicast unavailable: {info[0]}")
                self.multicast = False  # the driver refused the multicast object: peer stores
                self.mc_error = info[0]
        if self.multicast:
            if self.rank != 0:
                self.mc = self.eng.mc_import(info[0][0], info[0][1])
            dist.barrier(group=group)
            uc, mcp = self.eng.mc_bind(self.mc)
            self.local = {k: uc + i * plane for i, k in enumerate(self._MC)}
            self.mcast = {k: mcp + i * plane for i, k in enumerate(self._MC)}
            self.local["flags"] = self.buf["flags"].data_ptr()
            shared = ("flags",)
        else:
            for k in ("p0_hi", "p0_lo", "p1_hi", "p1_lo"):
                self.buf[k] = torch.empty((n_p, n_p), dtype=torch.int32, device=device)
            self.buf["out"] = torch.empty((n_p, n_p), dtype=torch.float32, device=device)
            self.local = {k: self.buf[k].data_ptr() for k in self._SHARED}
            shared = self._SHARED
        torch.cuda.synchronize(device)
        mine = {k: self.eng.ipc_get_handle(self.local[k]) for k in shared}
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.opened = []
        self.peer = {k: [] for k in shared}
        for r in range(self.world):
            for k in shared:
                if r == self.rank:
                    self.peer[k].append(self.local[k])
                else:
                    ptr = self.eng.ipc_open_handle(everyone[r][k])
                    self.opened.append(ptr)
                    self.peer[k].append(ptr)
        self.epoch = 0
        dist.barrier(group=group)  # every rank's buffers exist and are mapped

    def power(self, a, power: int):
        """A^power (a: n x n float32 on this rank's device, replicated); the full
        result on every rank.  Collective: every rank calls it with the same power."""
        import torch

        n, n_p, rows, eng = self.n, self.n_p, self.rows, self.eng
        if power == 0:
            return torch.eye(n, dtype=a.dtype, device=a.device)
        if power == 1:
            return a.clone()
        plan = plan_exponentiation(power)
        b = self.buf
        ext = torch.cuda.ExternalStream(eng.stream)
        ext.wait_stream(torch.cuda.current_stream(a.device))  # `a` is ready
        # nobody may overwrite a peer's buffers while that peer still copies the
        # previous call's result out of them
        self.epoch += 1
        eng.peer_barrier(self.rank, self.peer["flags"], self.epoch)
        with torch.cuda.stream(ext):
            self.base[:n, :n] = a  # zero padding never mixes into the top-left n x n block
        eng.split_planes_device(self.base.data_ptr(), b["base_hi"].data_ptr(),
                                b["base_lo"].data_ptr(), n_p)
        eng.split_planes_device(self.base.data_ptr(), self.local["p0_hi"], self.local["p0_lo"], n_p)
        cur, nxt = "p0", "p1"
        r0 = self.rank * rows
        for s, step in enumerate(plan.steps):
            last = s == len(plan.steps) - 1
            if step is Step.SQUARE:
                b_hi, b_lo = self.local[cur + "_hi"], self.local[cur + "_lo"]
            else:
                b_hi, b_lo = b["base_hi"].data_ptr(), b["base_lo"].data_ptr()
            if self.multicast:
                eng.gemm_rows_planes_mc(
                    n_p, rows, r0, self.local[cur + "_hi"], self.local[cur + "_lo"], b_hi, b_lo,
                    None if last else self.mcast[nxt + "_hi"],
                    None if last else self.mcast[nxt + "_lo"], self.mcast["out"] if last else None)
            else:
                eng.gemm_rows_planes_peers(
                    n_p, rows, r0, self.local[cur + "_hi"], self.local[cur + "_lo"], b_hi, b_lo,
                    None if last else self.peer[nxt + "_hi"],
                    None if last else self.peer[nxt + "_lo"], self.peer["out"] if last else None)
            # all ranks' rows have landed everywhere (and nobody still reads the
            # buffer the next step overwrites) before anyone goes on
            self.epoch += 1
            eng.peer_barrier(self.rank, self.peer["flags"], self.epoch)
            cur, nxt = nxt, cur
        with torch.cuda.stream(ext):
            out = torch.empty((n, n), dtype=a.dtype, device=a.device)
        # the top-left n x n block of the (n_p-strided) result, on the engine stream
        eng.copy2d_device(out.data_ptr(), n * 4, self.local["out"], n_p * 4, n * 4, n)
        caller = torch.cuda.current_stream(a.device)
        caller.wait_stream(ext)
        out.record_stream(caller)
        return out

    def close(self):
        self.eng.synchronize()
        self.dist.barrier(group=self.group)  # nobody unmaps what a peer still writes through
        for ptr in self.opened:
            self.eng.ipc_close_handle(ptr)
        self.opened = []
        if self.mc is not None:
            self.eng.mc_destroy(self.mc)
            self.mc = None


class RowShardedK1PH:
    """The row-sharded chain on the K1PH datapath (scaled fp16x2 planes, one
    exponent per matrix, DESIGN.md §3 K1PH) for one n x n FP32 shape on a
    group, one process per GPU.  Per plan step every rank computes its
    256-row blocks of the product in fp32 with the K1PH row-block GEMM, folds
    their max into every rank's chain state (system-scope atomicMax through
    CUDA IPC mappings), and after a flag barrier splits its rows at the now
    global exact scale straight into every rank's next planes (peer stores:
    the split is the all-gather); a second barrier closes the step.  Every
    element is computed on one rank with the single-GPU kernel, k-order and
    scale, so the result is bitwise the single-GPU K1PH chain.  A chain whose
    product loses dynamic range (every rank sees the same flag) is recomputed
    collectively on the 3xTF32 fused exchange (RowShardedFused), bitwise the
    single-GPU chain's own recomputation.  Set up once (collective), reused
    by ``power``; ``close`` is collective too."""

    _SHARED = ("p0_h0", "p0_h1", "p1_h0", "p1_h1", "out", "state", "flags")

    def __init__(self, n: int, device, group=None, engine=None):
        import torch
        import torch.distributed as dist

        self.dist, self.group, self.device = dist, group, device
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self.n_p, self.rows = fused_layout(n, self.world)
        if engine is None:
            from .engine import default_engine

            engine = default_engine(torch.device(device).index or 0)
        self.eng = engine
        n_p = self.n_p
        b = {k: torch.empty((n_p, n_p), dtype=torch.int16, device=device)
             for k in ("base_h0", "base_h1", "p0_h0", "p0_h1", "p1_h0", "p1_h1")}
        b["out"] = torch.empty((n_p, n_p), dtype=torch.float32, device=device)
        b["rows"] = torch.empty((self.rows, n_p), dtype=torch.float32, device=device)
        b["state"] = torch.zeros(engine.k1ph_state_bytes(), dtype=torch.uint8, device=device)
        b["flags"] = torch.zeros(self.world, dtype=torch.int32, device=device)
        self.buf = b
        self.local = {k: b[k].data_ptr() for k in b}
        torch.cuda.synchronize(device)
        mine = {k: engine.ipc_get_handle(self.local[k]) for k in self._SHARED}
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.opened = []
        self.peer = {k: [] for k in self._SHARED}
        for r in range(self.world):
            for k in self._SHARED:
                if r == self.rank:
                    self.peer[k].append(self.local[k])
                else:
                    ptr = engine.ipc_open_handle(everyone[r][k])
                    self.opened.append(ptr)
                    self.peer[k].append(ptr)
        self.epoch = 0
        self.last_fallback = False
        dist.barrier(group=group)

    def _barrier(self):
        self.epoch += 1
        self.eng.peer_barrier(self.rank, self.peer["flags"], self.epoch)

    def power(self, a, power: int):
        """A^power (a: n x n float32 on this rank's device, replicated); the full
        result on every rank.  Collective: every rank calls it with the same power."""
        import torch

        n, n_p, rows, eng, loc = self.n, self.n_p, self.rows, self.eng, self.local
        if power == 0:
            return torch.eye(n, dtype=a.dtype, device=a.device)
        if power == 1:
            return a.clone()
        a = a.contiguous()
        plan = plan_exponentiation(power)
        ext = torch.cuda.ExternalStream(eng.stream)
        ext.wait_stream(torch.cuda.current_stream(a.device))  # `a` is ready
        self._barrier()  # peers are done with the previous call's buffers
        with torch.cuda.stream(ext):
            self.buf["state"].zero_()
        eng.k1ph_split_base(n, n_p, a.data_ptr(), loc["base_h0"], loc["base_h1"], loc["state"])
        self._barrier()  # every state is reset before peers' maxima arrive
        r0 = self.rank * rows
        cur, cur_i, nxt = "base", 0, "p0"
        for s, step in enumerate(plan.steps):
            last = s == len(plan.steps) - 1
            rhs, rhs_i = (cur, cur_i) if step is Step.SQUARE else ("base", 0)
            oi = s + 1
            eng.k1ph_gemm_rows(n_p, rows, r0, loc[cur + "_h0"], loc[cur + "_h1"], loc[rhs + "_h0"],
                               loc[rhs + "_h1"], loc["rows"], n_p, n if last else n_p, loc["state"],
                               cur_i, rhs_i, -1 if last else oi)
            if last:
                # this rank's rows of the result into every rank's `out`
                h = min(rows, n - r0)
                if h > 0:
                    for dst in self.peer["out"]:
                        eng.copy2d_device(dst + r0 * n_p * 4, n_p * 4, loc["rows"], n_p * 4, n * 4, h)
                self._barrier()
                break
            eng.k1ph_max_to_peers(loc["state"], oi, self.peer["state"])
            self._barrier()  # the max is global on every rank
            eng.k1ph_split_rows_peers(n, n_p, rows, r0, loc["rows"], loc["state"], oi, cur_i, rhs_i,
                                      self.peer[nxt + "_h0"], self.peer[nxt + "_h1"])
            self._barrier()  # every rank's rows of the next planes have landed
            cur, cur_i = nxt, oi
            nxt = "p1" if nxt == "p0" else "p0"
        self.last_fallback = eng.k1ph_read_flag(loc["state"])  # (the same on every rank)
        if self.last_fallback:
            ctx = RowShardedFused(n, a.device, group=self.group, engine=eng, multicast=False)
            try:
                return ctx.power(a, power)
            finally:
                ctx.close()
        with torch.cuda.stream(ext):
            out = torch.empty((n, n), dtype=a.dtype, device=a.device)
        eng.copy2d_device(out.data_ptr(), n * 4, loc["out"], n_p * 4, n * 4, n)
        caller = torch.cuda.current_stream(a.device)
        caller.wait_stream(ext)
        out.record_stream(caller)
        return out

    def close(self):
        self.eng.synchronize()
        self.dist.barrier(group=self.group)  # nobody unmaps what a peer still writes through
        for ptr in self.opened:
            self.eng.ipc_close_handle(ptr)
        self.opened = []


def exponentiate_row_sharded_k1ph(a, power: int, group=None, engine=None):
    """A^power for one n x n FP32 matrix with its rows sharded over the group
    on the K1PH datapath (see RowShardedK1PH); the full result on every rank."""
    import torch

    if a.dtype != torch.float32:
        raise ValueError("the K1PH row shards run the FP32 chain")
    if power in (0, 1):
        return torch.eye(a.shape[0], dtype=a.dtype, device=a.device) if power == 0 else a.clone()
    ctx = RowShardedK1PH(a.shape[0], a.device, group=group, engine=engine)
    try:
        return ctx.power(a, power)
    finally:
        ctx.close()


def exponentiate_row_sharded_fused(a, power: int, group=None, engine=None):
    """A^power for one n x n FP32 matrix with its rows sharded over the group and
    the exchange fused into the GEMM epilogue (see RowShardedFused).  `a` is
    the full base matrix (replicated, on this rank's device); the full A^power
    is returned on every rank."""
    import torch

    if a.dtype != torch.float32:
        raise ValueError("the fused exchange runs the FP32 (3xTF32) chain")
    if power in (0, 1):
        return torch.eye(a.shape[0], dtype=a.dtype, device=a.device) if power == 0 else a.clone()
    ctx = RowShardedFused(a.shape[0], a.device, group=group, engine=engine)
    try:
        return ctx.power(a, power)
    finally:
        ctx.close()


def exponentiate_batched_sharded(a_local, power: int, ops=None):
    """A_i^power for this rank's shard (independent matrices, no collective)."""
    import torch

    if ops is None:
        from .engine import default_engine

        ops = EngineOps(default_engine(a_local.device.index or 0))
    stream = ops.stream() if hasattr(ops, "stream") else None
    if stream is None:
        out = torch.empty_like(a_local)
        ops.power_batched(a_local, power, out)
        return out
    caller = torch.cuda.current_stream(a_local.device)
    stream.wait_stream(caller)
    with torch.cuda.stream(stream):
        out = torch.empty_like(a_local)
    ops.power_batched(a_local, power, out)
    a_local.record_stream(stream)
    caller.wait_stream(stream)
    out.record_stream(caller)
    return out


def gather_batched(local, total: int, group=None):
    """Concatenate every rank's shard (uneven shards allowed) on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_range(total, r, world)[1] - shard_range(total, r, world)[0] for r in range(world)]
    width = max(sizes)
    padded = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False
