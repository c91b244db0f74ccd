#!/usr/bin/env python
"""Benchmark: effective TFLOP/s (2 n^3 * multiplies / s) and matrices/s for A^k.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...      # the reference CPU path (oracle port)

With ``--gpus N > 1`` and no torchrun environment the script re-launches
itself under ``torch.distributed.run`` with N ranks (one per GPU); under
torchrun ``WORLD_SIZE`` must equal ``--gpus``.

Workload (BASELINE.json configs; the metric is quoted "at 1/2/4/8 B200",
which is config 3's batch-sharded form):  c3 = 65536 x 128x128 FP32 A^64,
inputs fl(random_matrix(128, F64, 42+i) * sqrt(12/128)) generated on device.
The 65536 matrices are sharded over the ranks (rank r takes
``shard_range(65536, r, N)``, seeds 42+i of its own slice; strong scaling, no
collective on the data path); ``weak_scaling`` reports 65536 per rank beside
it.  ``--workload c5`` runs the 8192^2 A^1024 chain, row-sharded over the
ranks with the exchange fused into the GEMM epilogue.  A "step" is one pass
of the chain over the batch: ONE launch of the persistent sm_100a kernel for
c3.  Inputs (4.3 GB) exceed the 126 MB L2, so no flush is needed between
steps.

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = ("effective TFLOP/s (2N^3·mults/s) and matrices/s for A^k at 1/2/4/8 B200 "
          "vs CPU ref")

WORKLOADS = {
    "c3": dict(name="batched 65536 x 128x128 FP32 (split-fp32 tensor cores) A^64", n=128, batch=65536, k=64,
               dtype="f32"),
    "c2": dict(name="512x512 FP32 (3xTF32) A^1000", n=512, batch=1, k=1000, dtype="f32"),
    # K1PH (scaled fp16x2 planes, 3xTF32 recomputation on range loss), on one
    # GPU or row-sharded over N GPUs (RowShardedK1PH)
    "c5": dict(name="8192x8192 FP32 (split-fp32 tensor cores) A^1024", n=8192, batch=1, k=1024,
               dtype="f32"),
    "c4": dict(name="4096x4096 FP64 (DMMA) A^257", n=4096, batch=1, k=257, dtype="f64"),
    "c1": dict(name="64x64 FP32 (split-fp32 tensor cores) A^16", n=64, batch=1, k=16, dtype="f32"),
}


def mults(k: int) -> int:
    return k.bit_length() - 1 + bin(k).count("1") - 1 if k >= 1 else 0


def flops(w: dict, batch: int | None = None) -> float:
    return 2.0 * w["n"] ** 3 * mults(w["k"]) * (w["batch"] if batch is None else batch)


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Same rule as paper_1204_3052_b200.distributed.shard_range (kept import-free
    here so --plan-only runs without the package's native library)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during a region."""

    BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.002):
        self.samples = []
        self.power_mw = []
        self.power_limit_w = None
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            try:
                self.power_limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self._h) / 1e3
            except Exception:  # noqa: BLE001
                pass
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self._nv = None
        self.period = period

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                try:
                    self.power_mw.append(nv.nvmlDeviceGetPowerUsage(self._h))
                except Exception:  # noqa: BLE001
                    pass
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:  # noqa: BLE001
                try:
                    self.reasons |= int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h))
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        reasons = [name for bit, name in self.BITS.items() if self.reasons & bit]
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": reasons, "samples": len(self.samples)}
        if self.power_mw:
            out["power_w"] = statistics.median(self.power_mw) / 1e3
            out["power_limit_w"] = self.power_limit_w
        return out


# ----------------------------------------------------------------------------- peaks
def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except OSError:
        return {}


def library_gemm_peak_tflops(device, dtype_name: str) -> float:
    """cuBLAS GEMM 8192^3, best of 10: the TF32 (3xTF32 denominator) and FP64
    (DMMA denominator) peaks the driver's MEASURED_PEAKS.json does not carry.
    A library GEMM is used only as a peak reference, never on the measured path."""
    import torch

    dt = torch.float32 if dtype_name == "tf32" else torch.float64
    torch.backends.cuda.matmul.allow_tf32 = dtype_name == "tf32"
    n = 8192
    a = torch.randn(n, n, device=device, dtype=dt)
    b = torch.randn(n, n, device=device, dtype=dt)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10 if dtype_name == "tf32" else 5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def int8_peak_tops(device) -> float:
    """cuBLASLt int8 GEMM (torch._int_mm) 8192^3, best of 10: the denominator for
    the exact modular mode's INT8 limb datapath (library used as a reference)."""
    import torch

    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=device)
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=device)
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def run_mod(eng, n: int = 4096, k: int = 257, p: int = 2**31 - 1, steps: int = 5) -> dict:
    """The exact modular mode: A^k mod p for an n x n uint32 matrix on the
    INT8 limb datapath (K5I), device-resident, CUDA-event timed."""
    import numpy as np
    import torch

    a = np.random.default_rng(42).integers(0, p, size=(n, n), dtype=np.int64).astype(np.uint32)
    d_in, d_out = eng.alloc(a.nbytes), eng.alloc(a.nbytes)
    eng.upload(d_in, a)
    for _ in range(2):
        eng.power_mod_device(d_in, d_out, n, k, p)
    eng.synchronize()
    launches = eng.last_stats.launches
    stream = torch.cuda.ExternalStream(eng.stream)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        eng.power_mod_device(d_in, d_out, n, k, p)
    end.record(stream)
    end.synchronize()
    ms = start.elapsed_time(end) / steps
    eng.free(d_in)
    eng.free(d_out)
    return {"workload": f"{n}x{n} uint32 residues mod {p} A^{k} (exact, INT8 limb GEMMs)",
            "ms": ms, "launches": launches,
            "TOP/s": 2.0 * n ** 3 * mults(k) / (ms / 1e3) / 1e12,
            "note": "effective 2 n^3 m integer multiply-adds (mod p); the datapath runs 16 "
                    "byte-limb GEMMs per product"}


def ncu_traffic(kernel: str):
    """dram bytes per launch from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data.get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- CPU
def cpu_sample(w: dict, budget_s: float = 12.0, threads: int | None = None,
               one_core: bool = True) -> dict:
    """Time the oracle port (CPU restatement of the reference's naive chain,
    bit-identical to it) on a bounded sample of the workload."""
    import numpy as np

    import oracle

    # every host core this process may run on (torchrun sets OMP_NUM_THREADS=1
    # for its ranks; the reference arm runs on rank 0 alone and uses them all)
    if threads is None:
        threads = max(oracle.max_threads(), len(os.sched_getaffinity(0)))
    n, k = w["n"], w["k"]
    dt = np.float32 if w["dtype"] == "f32" else np.float64
    m = mults(k)
    if w["batch"] > 1:
        # whole chains of independent matrices (seeds 42, 43, ...), in chunks,
        # until the budget is spent or the whole batch is done
        chunk = max(threads * 16, 64)
        done, dt_s = 0, 0.0
        while done < w["batch"] and dt_s < budget_s:
            cnt = min(chunk, w["batch"] - done)
            stack = oracle.scaled_batch(n, cnt, dt, 42 + done)
            t0 = time.perf_counter()
            oracle.exponentiate_batched(stack, k, threads)
            dt_s += time.perf_counter() - t0
            done += cnt
        count = done
        fl = 2.0 * n ** 3 * m * count
        whole = " (the whole batch)" if count == w["batch"] else ""
        sample = (f"{count} full A^{k} chains of {n}x{n}{whole} (seeds 42..{41 + count}) on "
                  f"{threads} threads")
        per_unit_s = dt_s / count
        full_s = per_unit_s * w["batch"]
    elif n <= 1024:
        a = oracle.scaled_input(n, dt, 42)
        t0 = time.perf_counter()
        oracle.exponentiate(a, k, threads)
        dt_s = time.perf_counter() - t0
        fl = 2.0 * n ** 3 * m
        sample = f"one full A^{k} chain of {n}x{n} on {threads} threads"
        full_s = dt_s
    else:
        # rows of one multiply, extrapolated to m multiplies (labelled)
        a = oracle.scaled_input(n, dt, 42)
        rows = 16
        t0 = time.perf_counter()
        oracle.matmul_rows(a, a, 0, rows, threads)
        dt_s = time.perf_counter() - t0
        rows = max(16, min(n, int(rows * budget_s / max(dt_s, 1e-3))))
        t0 = time.perf_counter()
        oracle.matmul_rows(a, a, 0, rows, threads)
        dt_s = time.perf_counter() - t0
        fl = 2.0 * n * n * rows
        sample = (f"{rows} rows of one {n}x{n} multiply on {threads} threads, extrapolated "
                  f"x{n / rows:.0f} rows x{m} multiplies")
        full_s = dt_s * (n / rows) * m
    res = {"value": fl / dt_s / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "port",
           "sample": sample, "sample_seconds": dt_s, "est_full_workload_seconds": full_s,
           "matrices_per_s": w["batch"] / full_s if w["batch"] > 1 else 1.0 / full_s}
    if threads > 1 and one_core:
        # BASELINE.md §3 asks for the 1-core figure beside the N-core one
        one = cpu_sample(w, budget_s=min(budget_s, 3.0), threads=1, one_core=False)
        res["one_core"] = {k: one[k] for k in ("value", "unit", "cores", "sample",
                                               "sample_seconds", "est_full_workload_seconds")}
    return res


# ----------------------------------------------------------------------------- GPU
def device_workload(eng, w: dict, batch: int | None = None, seed0: int = 42):
    """Allocate the workload's buffers, generate its inputs on the device and
    return (d_in, d_out, step): ``step()`` enqueues exactly the call the
    bench times (one ``mxp_power_batched_device`` over the whole batch for a
    batched config, one ``mxp_power_device`` chain otherwise).  The GPU
    parity tests import this function, so the launch they check against the
    oracle is the launch measured here."""
    from paper_1204_3052_b200 import _lib

    n, k = w["n"], w["k"]
    B = w["batch"] if batch is None else batch
    mode = _lib.MXP_F32 if w["dtype"] == "f32" else _lib.MXP_F64
    es = 4 if w["dtype"] == "f32" else 8
    nbytes = n * n * max(B, 1) * es
    d_in = eng.alloc(nbytes)
    d_out = eng.alloc(nbytes)
    eng.random_device(d_in, n, B, seed0, -0.5, 0.5, math.sqrt(12.0 / n), mode)
    batched = w["batch"] > 1

    def step():
        if batched:
            eng.power_batched_device(d_in, d_out, n, B, k, mode)
        else:
            eng.power_device(d_in, d_out, n, k, mode)

    return d_in, d_out, step


def run_row_sharded(eng, w: dict, steps: int, warmup: int, dist, sample=True):
    """C5 on N GPUs: one matrix, rows sharded, the exchange fused into the
    CTA-pair GEMM epilogue (peer stores + flag barrier).  Strong scaling."""
    import torch

    from paper_1204_3052_b200 import distributed as D

    n, k = w["n"], w["k"]
    a = torch.empty((n, n), dtype=torch.float32, device="cuda")
    eng.random_device(a.data_ptr(), n, 1, 42, -0.5, 0.5, math.sqrt(12.0 / n))
    eng.synchronize()
    # buffers + peer mappings, once: K1PH row shards at the K1PH sizes (C5),
    # else the 3xTF32 fused exchange
    chain = (D.RowShardedK1PH(n, a.device, engine=eng) if k1ph_runs(w)
             else D.RowShardedFused(n, a.device, engine=eng))
    for _ in range(warmup):
        chain.power(a, k)
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device()) if sample else None
    if sampler:
        sampler.__enter__()
    stream = torch.cuda.ExternalStream(eng.stream)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        chain.power(a, k)
    end.record(stream)
    end.synchronize()
    if sampler:
        sampler.__exit__()
    chain.close()
    ms = start.elapsed_time(end) / steps
    return ms, mults(k) + 1, (sampler.summary() if sampler else None)


def run_device(eng, w: dict, steps: int, warmup: int, seed0: int, dist=None, sample=True,
               batch: int | None = None):
    """Device-resident inputs, CUDA-event timing on the engine's stream."""
    import torch

    d_in, d_out, step = device_workload(eng, w, batch, seed0)
    for _ in range(warmup):
        step()
    eng.synchronize()
    launches = eng.last_stats.launches
    stream = torch.cuda.ExternalStream(eng.stream)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device()) if sample else None
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    if sampler:
        sampler.__enter__()
    start.record(stream)
    for _ in range(steps):
        step()
    end.record(stream)
    end.synchronize()
    if sampler:
        sampler.__exit__()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = start.elapsed_time(end) / steps
    clocks = sampler.summary() if sampler else None
    if clocks is not None and w["batch"] > 1:
        # the SM clock inside the last timed launch (clock64 / globaltimer of
        # CTA 0): NVML's samples can miss or smear a few-ms kernel
        try:
            mhz, kms = eng.last_kernel_clock()
            clocks["sm_mhz_in_kernel"] = mhz
            clocks["in_kernel_ms"] = kms
            clocks["sm_mhz_source"] = "NVML median over the timed region; sm_mhz_in_kernel from the kernel"
        except Exception:  # noqa: BLE001 - K3B launches carry no stamps
            pass
        # board power under a sustained run of the same step (untimed, ~1.5 s:
        # NVML's power counter averages over far longer than the timed region)
        sus = ClockSampler(torch.cuda.current_device(), period=0.01)
        sus.__enter__()
        t_end = time.perf_counter() + 1.5
        while time.perf_counter() < t_end:
            for _ in range(10):
                step()
            eng.synchronize()
        sus.__exit__()
        ss = sus.summary()
        try:
            mhz, _kms = eng.last_kernel_clock()
        except Exception:  # noqa: BLE001
            mhz = None
        clocks["sustained"] = {"seconds": 1.5, "power_w": ss.get("power_w"),
                               "power_limit_w": ss.get("power_limit_w"),
                               "sm_mhz_in_kernel": mhz, "reasons": ss.get("reasons")}
    eng.free(d_in)
    eng.free(d_out)
    return ms, launches, clocks


def run_e2e(eng, w: dict, batch: int, seed0: int, steps: int = 3, pinned: bool = True) -> dict:
    """Same metric through the public host API: host input -> H2D -> chain ->
    D2H into the host output, every step.  ``pinned``: engine-allocated pinned
    buffers; else ordinary (pageable) numpy arrays, the drop-in
    ``exponentiate_batched(np.ndarray)`` call a user makes."""
    import numpy as np

    import paper_1204_3052_b200 as mx
    from paper_1204_3052_b200 import _lib

    n, k = w["n"], w["k"]
    dt = np.float32 if w["dtype"] == "f32" else np.float64
    mode = _lib.MXP_F32 if w["dtype"] == "f32" else _lib.MXP_F64
    batched = w["batch"] > 1
    shape = (batch, n, n) if batched else (n, n)
    if pinned:
        host_in = eng.pinned_array(shape, dt)
        host_out = eng.pinned_array(shape, dt)
    else:
        host_in = np.empty(shape, dt)
        host_out = None
    d = eng.alloc(host_in.nbytes)
    eng.random_device(d, n, batch, seed0, -0.5, 0.5, math.sqrt(12.0 / n), mode)
    eng.download(host_in, d)
    eng.free(d)

    from paper_1204_3052_b200.engine import default_engine

    user_eng = eng if pinned else default_engine(eng.device)  # the engine the public API uses

    def call():
        if batched:
            if pinned:
                eng.power_batched(host_in, k, out=host_out)
            else:
                mx.exponentiate_batched(host_in, k, device=eng.device)
        elif pinned:
            host_out[...] = eng.power(host_in, k)
        else:
            mx.exponentiate(host_in, k, mx.b200_backend(eng.device))

    call()  # warm (allocations, graph capture)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    st = user_eng.last_stats
    med = statistics.median(times)
    res = {"value": flops(w, batch) / med / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": int(st.h2d_bytes), "d2h_bytes_per_step": int(st.d2h_bytes),
           "ms_per_step": med * 1e3, "matrices_per_s": batch / med,
           "host_memory": "pinned (engine-allocated)" if pinned else "pageable numpy arrays",
           "timing": f"host wall clock around the synchronous public call, median of {steps}"}
    if pinned:
        eng.host_free(host_in.ctypes.data)
        eng.host_free(host_out.ctypes.data)
    return res


# ----------------------------------------------------------------------------- launch
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(n: int) -> int:
    """Re-run this script under torch.distributed.run with n ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def plan_only(args, w, world, rank) -> None:
    """The launch and sharding plan without touching a GPU (tests/test_bench.py
    runs it on CPU with gloo): every rank reports its slice, rank 0 prints."""
    import torch.distributed as tdist

    if world > 1:
        tdist.init_process_group("gloo")
    batched = w["batch"] > 1
    lo, hi = shard_range(w["batch"], rank, world) if batched else (0, 1)
    mine = {"rank": rank, "shard": [lo, hi], "seed0": 42 + lo}
    everyone = [mine]
    if world > 1:
        everyone = [None] * world
        tdist.all_gather_object(everyone, mine)
    if rank == 0:
        print(json.dumps({"plan_only": True, "n_gpus": world, "workload": w["name"],
                          "global_batch": w["batch"], "ranks": everyone}))
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def k1ph_runs(w: dict, world: int = 1) -> bool:
    """Whether a single-matrix f32 chain runs K1PH (kernels_f16x2.cu): the
    CTA-pair sizes and n > 1408, on one GPU or row-sharded (RowShardedK1PH)."""
    n_pad = -(-w["n"] // 128) * 128
    return (w["dtype"] == "f32" and w["batch"] == 1
            and ((n_pad >= 1024 and n_pad % 256 == 0) or w["n"] > 1408))


def roofline_of(w: dict, batched: bool, rank_fl: float, ms: float, launches: int, value: float,
                world: int, peaks: dict, tf32) -> dict:
    """The bench line's roofline object for the kernel that runs workload w:
    rank_fl algorithmic flops of this rank's step, ms its device time,
    launches the engine's kernel launches per step (value: whole-job rate)."""
    # Roofline denominator = the datapath the kernel runs on.  C3 (K3H) forms
    # each fp32 product from three fp16 tensor-core products (scaled fp16x2
    # split), so its effective peak is the dense 16-bit tensor peak / 3
    # (MEASURED_PEAKS bf16; fp16 runs at the same rate).  The K1/K1P chains
    # (C2, C5) run 3xTF32: cuBLAS TF32 measured here / 3.
    bf16 = peaks.get("bf16_tflops")
    if k1ph_runs(w, world):
        # K1PH: three fp16 products per fp32 product, like K3H
        if bf16:
            peak, src = bf16 / 3.0, "MEASURED_PEAKS bf16 dense burst (fp16 same rate) / 3 products"
        else:
            peak, src = 2250.0 / 3.0, "fallback: nominal 2.25 PF dense fp16 / 3 products"
        kernel = "k1ph_gemm_f16x2"
    elif batched and w["dtype"] == "f32":
        if bf16:
            peak, src = bf16 / 3.0, "MEASURED_PEAKS bf16 dense burst (fp16 same rate) / 3 products"
        else:
            peak, src = 2250.0 / 3.0, "fallback: nominal 2.25 PF dense fp16 / 3 products"
        kernel = "k3h_batched_power"
    else:
        if tf32:
            peak, src = tf32 / 3.0, f"cuBLAS TF32 8192^3 measured in this run ({tf32:.0f} TFLOP/s) / 3"
        elif bf16:
            peak, src = bf16 / 6.0, "MEASURED_PEAKS bf16 burst / 2 (tf32) / 3"
        else:
            peak, src = 1590.0 / 6.0, "fallback 1.59 PF bf16 / 6"
        # the kernel that runs the chain's multiplies
        n_pad = -(-w["n"] // 128) * 128
        if w["dtype"] == "f64":
            kernel = "f64_gemm_kernel"
        elif w["n"] <= 128:
            kernel = "k3h_batched_power"
        elif n_pad >= 1024 and n_pad % 256 == 0:
            kernel = "k1p_gemm_3xtf32"
        elif n_pad in (256, 384, 512, 640, 768, 896, 1152, 1408):
            kernel = "k1c_chain_3xtf32"
        else:
            kernel = "k1_gemm_3xtf32"
    # A batched step is ONE K3H launch doing all the work plus the K3B fixup
    # pass, which returns at once on an empty list (0 matrices on this input;
    # ~4 us, overlapped with K3H's tail by programmatic dependent launch).  The
    # K3H launch time is therefore taken as the whole step time: a lower bound
    # on the kernel's rate, never an inflated one.
    kernel_ms = ms
    achieved = rank_fl / (kernel_ms / 1e3) / 1e12 if batched else value / world
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": ncu_traffic(kernel),
                "kernel": kernel, "peak_source": src,
                "per_gpu": True,
                "algorithmic_flops_per_launch": rank_fl if batched else rank_fl / max(launches, 1),
                "kernel_time": ("step time: the K3H launch + the empty K3B fixup pass"
                                if batched else "chain time / launches"),
                "bf16_measured_peak": bf16,
                "bf16_measured_peak_sustained": peaks.get("bf16_tflops_sustained"),
                "frac_vs_sustained": (achieved / (peaks["bf16_tflops_sustained"] / 3.0)
                                      if peaks.get("bf16_tflops_sustained") and batched
                                      else None),
                "tf32_cublas_measured": tf32,
                "vs_3xtf32_effective_peak": achieved / (tf32 / 3.0) if tf32 else None}
    return roofline


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary configs")
    ap.add_argument("--quick", action="store_true",
                    help="device timing only (no e2e / CPU baseline / peak GEMM): for ncu runs")
    ap.add_argument("--plan-only", action="store_true",
                    help="print the rank/shard plan and exit (no GPU needed)")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch one rank "
                         "per GPU (or omit torchrun and let --gpus launch the ranks)")
    if args.plan_only:
        plan_only(args, w, world, rank)
        return

    batched = w["batch"] > 1
    lo, hi = shard_range(w["batch"], rank, world) if batched else (0, 1)
    config = {"workload": w["name"], "n": w["n"], "k": w["k"],
              "multiplies_per_matrix": mults(w["k"]), "global_batch": w["batch"],
              "batch_per_gpu": hi - lo, "shard": [lo, hi],
              "input": "fl(random_matrix(n, F64, 42+i) * sqrt(12/n)) generated on device",
              "l2": "inputs larger than L2 (no flush needed)" if batched else
                    "single matrix chain, L2-resident by design (graph replay)",
              "parallelism": (f"batch-sharded x{world}: rank r runs matrices shard_range(65536, r, "
                              f"{world}) (no collective)") if world > 1 else "1 GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        samples = []
        for i in range(args.warmup + args.steps):
            r = cpu_sample(w, budget_s=2.0, one_core=False)
            if i >= args.warmup:
                samples.append(r)
        val = statistics.median(s["value"] for s in samples)
        cpu = dict(samples[-1])
        cpu["value"] = val
        config["batch_per_gpu"] = w["batch"]
        config["shard"] = [0, w["batch"]]
        config["parallelism"] = "host CPU (rank 0 only)"
        print(json.dumps({"metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": statistics.median(s["sample_seconds"] for s in samples) * 1e3,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": w["dtype"], "data": "synthetic (SURVEY §8(d) recipe)",
                          "config": config, "cpu_baseline": cpu,
                          "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    import torch

    dist = None
    nccl_nranks = None
    # Test knob: BENCH_SHARE_GPU=1 maps every rank onto the visible GPUs
    # round-robin and uses gloo, so the multi-rank path (per-rank shards,
    # barriers, max over ranks) runs on a one-GPU box (numbers meaningless).
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as tdist

        if share:
            tdist.init_process_group("gloo")
        else:
            # NCCL's init log carries "nranks N" for every communicator: the
            # driver's evidence that N ranks ran
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout keeps the one JSON line
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
        one = torch.ones(1, device="cuda") if not share else torch.ones(1)
        dist.all_reduce(one)
        nccl_nranks = int(one.item())
        if nccl_nranks != world:
            raise SystemExit(f"communicator has {nccl_nranks} ranks, expected {world}")

    import paper_1204_3052_b200 as mx

    eng = mx.Engine(local)
    row_sharded = dist is not None and not batched and w["n"] >= 1024 and w["dtype"] == "f32"
    if row_sharded:  # one matrix over N GPUs (C5): fused exchange, strong scaling
        ms, launches, clocks = run_row_sharded(eng, w, args.steps, args.warmup, dist)
        config["parallelism"] = f"row-sharded x{world} (exchange fused into the GEMM epilogue)"
    else:
        ms, launches, clocks = run_device(eng, w, args.steps, args.warmup, seed0=42 + lo,
                                          dist=dist, batch=hi - lo)

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], device="cuda") if not share else torch.tensor([v])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    fl = flops(w)  # the whole job: all 65536 matrices (or the one matrix)
    value = fl / (ms / 1e3) / 1e12

    weak = None
    if dist is not None and batched and not args.quick:
        # secondary: every rank runs a full 65536-matrix batch of its own
        wms, _, _ = run_device(eng, w, args.steps, args.warmup, seed0=42 + rank * w["batch"],
                               dist=dist, sample=False)
        wms = max_over_ranks(wms)
        weak = {"batch_per_gpu": w["batch"], "global_batch": w["batch"] * world,
                "ms_per_step": wms, "value": world * fl / (wms / 1e3) / 1e12, "unit": "TFLOP/s"}

    # e2e through the public host API on every rank (its own shard; max over ranks)
    e2e = e2e_pageable = None
    if not args.quick:
        for pinned in (True, False):
            try:
                r = run_e2e(eng, w, hi - lo, 42 + lo, steps=3 if pinned else 1, pinned=pinned)
            except Exception as exc:  # noqa: BLE001
                r = {"value": None, "error": str(exc)}
            if dist is not None:
                worst = max_over_ranks(r.get("ms_per_step") or float("inf"))
                if r.get("ms_per_step"):
                    r["ms_per_step"] = worst
                    r["value"] = fl / (worst / 1e3) / 1e12
                    r["matrices_per_s"] = w["batch"] / (worst / 1e3)
                    r["timing"] += f"; max over {world} ranks"
                    for key in ("h2d_bytes_per_step", "d2h_bytes_per_step"):
                        r[key + "_per_rank"] = r[key]
                        r[key] = int(max_over_ranks(float(r[key])) * world) if batched else r[key]
            if pinned:
                e2e = r
            else:
                e2e_pageable = r

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    tf32 = None
    if not args.quick:
        try:
            tf32 = library_gemm_peak_tflops(torch.device("cuda", local), "tf32")
        except Exception:  # noqa: BLE001
            tf32 = None
    roofline = roofline_of(w, batched, flops(w, hi - lo), ms, launches, value, world, peaks, tf32)
    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None,
           "dtype": ("f32 (split-fp32: scaled fp16x2, tcgen05)" if batched else
                     "f32 (3xTF32 tcgen05)") if w["dtype"] == "f32" else "f64 (DMMA)",
           "data": "synthetic (SURVEY §8(d) recipe, device SplitMix64)", "config": config,
           "matrices_per_s": w["batch"] / (ms / 1e3),
           "roofline": roofline, "clocks": clocks,
           "gpu_launches": args.steps * launches}
    if nccl_nranks is not None:
        out["comm"] = {"backend": "gloo (BENCH_SHARE_GPU test mode)" if share else "nccl",
                       "nranks": nccl_nranks}
    if weak is not None:
        out["weak_scaling"] = weak
    if args.quick:
        print(json.dumps(out))
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    out["e2e"] = e2e
    out["e2e_pageable"] = e2e_pageable
    if world == 1:
        try:
            out["cpu_baseline"] = cpu_sample(w)
        except Exception as exc:  # noqa: BLE001
            out["cpu_baseline"] = {"value": None, "error": str(exc)}
        if not args.no_extras:
            try:
                f64 = library_gemm_peak_tflops(torch.device("cuda", local), "f64")
            except Exception:  # noqa: BLE001
                f64 = None
            roofline["f64_cublas_measured"] = f64
            extras = {}
            for key in ("c1", "c2", "c4", "c5"):
                if key == args.workload:
                    continue
                wx = WORKLOADS[key]
                try:
                    xms, xl, _ = run_device(eng, wx, 3 if wx["n"] >= 4096 else 20, 2, 42,
                                            sample=False)
                    tf = flops(wx) / (xms / 1e3) / 1e12
                    ex = {"workload": wx["name"], "ms": xms, "launches": xl, "TFLOP/s": tf}
                    if wx["dtype"] == "f64" and f64:
                        ex["frac"] = tf / f64
                        ex["peak"] = f"cuBLAS DGEMM 8192^3 measured in this run ({f64:.1f} TFLOP/s)"
                    elif k1ph_runs(wx) and peaks.get("bf16_tflops"):
                        ex["frac"] = tf / (peaks["bf16_tflops"] / 3.0)
                        ex["peak"] = (f"MEASURED_PEAKS bf16 dense burst / 3 products "
                                      f"({peaks['bf16_tflops'] / 3.0:.0f} TFLOP/s): K1PH, scaled fp16x2")
                        if tf32:
                            ex["vs_3xtf32_effective_peak"] = tf / (tf32 / 3.0)
                    elif wx["n"] > 128 and tf32:
                        ex["frac"] = tf / (tf32 / 3.0)
                        ex["peak"] = f"cuBLAS TF32 8192^3 / 3 ({tf32 / 3.0:.0f} TFLOP/s)"
                    extras[key] = ex
                except Exception as exc:  # noqa: BLE001
                    extras[key] = {"error": str(exc)}
            try:
                mod = run_mod(eng)
                try:
                    i8 = int8_peak_tops(torch.device("cuda", local))
                    mod["frac"] = mod["TOP/s"] / (i8 / 16.0)
                    mod["peak"] = (f"cuBLASLt int8 8192^3 measured in this run ({i8:.0f} TOP/s) / 16 "
                                   "limb GEMMs")
                except Exception as exc:  # noqa: BLE001
                    mod["peak_error"] = str(exc)
                extras["mod"] = mod
            except Exception as exc:  # noqa: BLE001
                extras["mod"] = {"error": str(exc)}
            out["other_configs"] = extras
    print(json.dumps(out))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
