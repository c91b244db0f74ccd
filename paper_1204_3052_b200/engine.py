"""B200 engine: a thin, typed wrapper over the C ABI (include/matexpo_b200.h).

One `Engine` = one device handle = one CUDA stream + workspace + graph cache
(the reference's "one device instance is one serialized queue",
gpu-backend/src/device.ts:6-8).  Host-array entry points copy in once and
out once; the `*_device` entry points take raw device pointers (e.g. from
torch tensors) and enqueue asynchronously on the engine's stream.

Every call goes to hand-written sm_100a kernels; if the extension is not
built or no B200 is present the call raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Optional

import numpy as np

from . import _lib
from . import errors as E

_MODES = {np.dtype(np.float32): _lib.MXP_F32, np.dtype(np.float64): _lib.MXP_F64}


def _mode_of(arr: np.ndarray) -> int:
    try:
        return _MODES[arr.dtype]
    except KeyError:
        raise E.ShapeError(f"unsupported element dtype {arr.dtype}") from None


def _ptr(arr: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(arr.ctypes.data)


class Engine:
    """A device handle.  Use one Engine per thread (or guard it)."""

    def __init__(self, device: int = 0):
        L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(L.mxp_create(int(device), ctypes.byref(h)), "mxp_create")
        self._L = L
        self._h = h
        self.device = int(device)
        self.last_stats = _lib.Stats()
        self._lock = threading.Lock()

    # ------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if self._h:
            self._L.mxp_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    @property
    def stream(self) -> int:
        """The engine's cudaStream_t as an integer (for torch.cuda.ExternalStream)."""
        s = ctypes.c_void_p()
        _lib.check(self._L.mxp_get_stream(self._h, ctypes.byref(s)), "mxp_get_stream")
        return int(s.value or 0)

    @property
    def num_sms(self) -> int:
        v = ctypes.c_int()
        _lib.check(self._L.mxp_num_sms(self._h, ctypes.byref(v)), "mxp_num_sms")
        return v.value

    def synchronize(self) -> None:
        _lib.check(self._L.mxp_synchronize(self._h), "mxp_synchronize")

    def debug_inject_fault(self, step: int) -> None:
        """Test hook: chains captured from now on trap at plan step `step` (-1
        disables).  The trap kills the CUDA context (use a throw-away process)."""
        _lib.check(self._L.mxp_debug_inject_fault(self._h, int(step)), "mxp_debug_inject_fault")

    # ------------------------------------------------------------ errors
    @staticmethod
    def _raise_chain(status: int, stats: _lib.Stats, plan: str, what: str) -> None:
        """Map a failed chain to BackendStepError (errors.py:43-49) when the
        failing plan step is known, else to the status' exception."""
        if status == _lib.MXP_OK:
            return
        step = stats.failed_step
        if status in (_lib.MXP_E_CUDA, _lib.MXP_E_NCCL) and 0 <= step < len(plan):
            name = "SQUARE" if plan[step] == "S" else "MULTIPLY_BASE"
            cause = E.DeviceError(_lib.last_error())
            raise E.BackendStepError(step, name, cause) from cause
        _lib.check(status, what)

    # ------------------------------------------------------------ host API
    def power(self, a: np.ndarray, k: int) -> np.ndarray:
        """A^k for one n x n float32/float64 array (one upload, one readback)."""
        a = np.ascontiguousarray(a)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise E.ShapeError(f"expected a square 2-D array, got shape {a.shape}")
        mode = _mode_of(a)
        out = np.empty_like(a)
        st = _lib.Stats()
        rc = self._L.mxp_power(self._h, mode, a.shape[0], int(k), _ptr(a), _ptr(out),
                               ctypes.byref(st))
        self.last_stats = st
        self._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power")
        return out

    def power_batched(self, a: np.ndarray, k: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """A_i^k for a (batch, n, n) stack; chunked H2D | compute | D2H pipeline."""
        a = np.ascontiguousarray(a)
        if a.ndim != 3 or a.shape[1] != a.shape[2]:
            raise E.ShapeError(f"expected a (batch, n, n) array, got shape {a.shape}")
        mode = _mode_of(a)
        if out is None:
            out = np.empty_like(a)
        elif (not isinstance(out, np.ndarray) or out.shape != a.shape or out.dtype != a.dtype
              or not out.flags.c_contiguous or not out.flags.writeable):
            raise E.ShapeError(f"out must be a writeable C-contiguous {a.dtype} array of shape "
                               f"{a.shape}")
        st = _lib.Stats()
        rc = self._L.mxp_power_batched(self._h, mode, a.shape[1], a.shape[0], int(k), _ptr(a),
                                       _ptr(out), ctypes.byref(st))
        self.last_stats = st
        self._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power_batched")
        return out

    def multiply(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """C = A * B (one product; 2 uploads + 1 readback like gpuMatmul, host.ts:67-95)."""
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise E.ShapeError(f"expected a square 2-D array, got shape {a.shape}")
        if a.shape != b.shape:
            raise E.ShapeError(f"matrix orders differ: {a.shape[0]} vs {b.shape[0]}")
        if a.dtype != b.dtype:
            raise E.ShapeError(f"matrix dtypes differ: {a.dtype} vs {b.dtype}")
        mode = _mode_of(a)
        out = np.empty_like(a)
        st = _lib.Stats()
        rc = self._L.mxp_multiply(self._h, mode, a.shape[0], _ptr(a), _ptr(b), _ptr(out),
                                  ctypes.byref(st))
        self.last_stats = st
        _lib.check(rc, "mxp_multiply")
        return out

    def power_mod(self, a: np.ndarray, k: int, p: int) -> np.ndarray:
        """(A^k) mod p, exact, uint32 residues."""
        a = np.ascontiguousarray(a, dtype=np.uint32)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise E.ShapeError(f"expected a square 2-D array, got shape {a.shape}")
        if not 2 <= int(p) < 2 ** 31:
            raise E.ValidationError(f"modulus must satisfy 2 <= p < 2^31, got {p}")
        out = np.empty_like(a)
        st = _lib.Stats()
        rc = self._L.mxp_power_mod(self._h, a.shape[0], int(k), int(p), _ptr(a), _ptr(out),
                                   ctypes.byref(st))
        self.last_stats = st
        self._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power_mod")
        return out

    def repeated_power(self, a: np.ndarray, k: int) -> np.ndarray:
        """A^k by k-1 successive device multiplies acc = acc * A (the REPEATED
        strategy / F64 oracle of expo.py:142-156 and bench.py:178-180, on the
        device: one upload, k-1 GEMM launches over ping-pong buffers, one readback)."""
        if k < 1:
            raise E.UnsupportedPowerError(f"repeated baseline needs power >= 1, got {k}")
        a = np.ascontiguousarray(a)
        mode = _mode_of(a)
        n = a.shape[0]
        d_a, d_x, d_y = self.alloc(a.nbytes), self.alloc(a.nbytes), self.alloc(a.nbytes)
        try:
            self.upload(d_a, a)
            self.upload(d_x, a)
            for _ in range(k - 1):
                self.gemm_device(d_x, d_a, d_y, n, mode)
                d_x, d_y = d_y, d_x
            out = np.empty_like(a)
            self.download(out, d_x)
            return out
        finally:
            self.free(d_a)
            self.free(d_x)
            self.free(d_y)

    # ------------------------------------------------------------ device API
    def power_device(self, d_in: int, d_out: int, n: int, k: int, mode: int = _lib.MXP_F32) -> None:
        st = _lib.Stats()
        rc = self._L.mxp_power_device(self._h, mode, n, k, ctypes.c_void_p(d_in),
                                      ctypes.c_void_p(d_out), ctypes.byref(st))
        self.last_stats = st
        self._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power_device")

    def power_batched_device(self, d_in: int, d_out: int, n: int, batch: int, k: int,
                             mode: int = _lib.MXP_F32) -> None:
        st = _lib.Stats()
        rc = self._L.mxp_power_batched_device(self._h, mode, n, batch, k, ctypes.c_void_p(d_in),
                                              ctypes.c_void_p(d_out), ctypes.byref(st))
        self.last_stats = st
        self._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power_batched_device")

    def power_mod_device(self, d_in: int, d_out: int, n: int, k: int, p: int) -> None:
        st = _lib.Stats()
        rc = self._L.mxp_power_mod_device(self._h, n, k, p, ctypes.c_void_p(d_in),
                                          ctypes.c_void_p(d_out), ctypes.byref(st))
        self.last_stats = st
        self._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power_mod_device")

    def gemm_device(self, d_a: int, d_b: int, d_c: int, n: int, mode: int = _lib.MXP_F32) -> None:
        _lib.check(self._L.mxp_gemm(self._h, mode, n, ctypes.c_void_p(d_a), ctypes.c_void_p(d_b),
                                    ctypes.c_void_p(d_c)), "mxp_gemm")

    def gemm_prepare_rhs_device(self, d_b: int, n: int, mode: int = _lib.MXP_F32) -> None:
        _lib.check(self._L.mxp_gemm_prepare_rhs(self._h, mode, n, ctypes.c_void_p(d_b)),
                   "mxp_gemm_prepare_rhs")

    def gemm_rows_prepared_device(self, d_a: int, d_c: int, n: int, rows: int,
                                  mode: int = _lib.MXP_F32) -> None:
        _lib.check(self._L.mxp_gemm_rows_prepared(self._h, mode, n, rows, ctypes.c_void_p(d_a),
                                                  ctypes.c_void_p(d_c)), "mxp_gemm_rows_prepared")

    # ------------------------------------------------------------ fused row-sharded exchange
    def ipc_get_handle(self, d_ptr: int) -> bytes:
        buf = ctypes.create_string_buffer(_lib.MXP_IPC_HANDLE_BYTES)
        _lib.check(self._L.mxp_ipc_get_handle(self._h, ctypes.c_void_p(d_ptr), buf),
                   "mxp_ipc_get_handle")
        return buf.raw

    def ipc_open_handle(self, handle: bytes) -> int:
        out = ctypes.c_void_p()
        _lib.check(self._L.mxp_ipc_open_handle(self._h, handle, ctypes.byref(out)),
                   "mxp_ipc_open_handle")
        return out.value

    def ipc_close_handle(self, d_ptr: int) -> None:
        _lib.check(self._L.mxp_ipc_close_handle(self._h, ctypes.c_void_p(d_ptr)),
                   "mxp_ipc_close_handle")

    def split_planes_device(self, d_a: int, d_hi: int, d_lo: int, n: int) -> None:
        _lib.check(self._L.mxp_split_planes(self._h, n, ctypes.c_void_p(d_a), ctypes.c_void_p(d_hi),
                                            ctypes.c_void_p(d_lo)), "mxp_split_planes")

    @staticmethod
    def _ptr_array(ptrs):
        if ptrs is None:
            return None
        return (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(p) for p in ptrs])

    def gemm_rows_planes_peers(self, n: int, rows: int, row0: int, a_hi: int, a_lo: int,
                               b_hi: int, b_lo: int, peer_hi, peer_lo, peer_f32=None) -> None:
        npeers = len(peer_f32 if peer_f32 is not None else peer_hi)
        _lib.check(self._L.mxp_gemm_rows_planes_peers(
            self._h, n, rows, row0, ctypes.c_void_p(a_hi), ctypes.c_void_p(a_lo),
            ctypes.c_void_p(b_hi), ctypes.c_void_p(b_lo), npeers, self._ptr_array(peer_hi),
            self._ptr_array(peer_lo), self._ptr_array(peer_f32)), "mxp_gemm_rows_planes_peers")

    # ------------------------------------------------------------ K1PH row shards (multi-process)
    @staticmethod
    def k1ph_state_bytes() -> int:
        b = ctypes.c_size_t()
        _lib.check(_lib.load().mxp_k1ph_state_bytes(ctypes.byref(b)), "mxp_k1ph_state_bytes")
        return b.value

    def k1ph_split_base(self, n_true: int, n: int, d_a: int, h0: int, h1: int, state: int) -> None:
        _lib.check(self._L.mxp_k1ph_split_base(self._h, n_true, n, ctypes.c_void_p(d_a),
                                               ctypes.c_void_p(h0), ctypes.c_void_p(h1),
                                               ctypes.c_void_p(state)), "mxp_k1ph_split_base")

    def k1ph_gemm_rows(self, n: int, rows: int, row0: int, x_h0: int, x_h1: int, y_h0: int,
                       y_h1: int, out: int, ld_out: int, n_out: int, state: int, xi: int, yi: int,
                       oi: int) -> None:
        _lib.check(self._L.mxp_k1ph_gemm_rows(
            self._h, n, rows, row0, ctypes.c_void_p(x_h0), ctypes.c_void_p(x_h1),
            ctypes.c_void_p(y_h0), ctypes.c_void_p(y_h1), ctypes.c_void_p(out), ld_out, n_out,
            ctypes.c_void_p(state), xi, yi, oi), "mxp_k1ph_gemm_rows")

    def k1ph_max_to_peers(self, state: int, i: int, peer_states) -> None:
        _lib.check(self._L.mxp_k1ph_max_to_peers(self._h, ctypes.c_void_p(state), i, len(peer_states),
                                                 self._ptr_array(peer_states)), "mxp_k1ph_max_to_peers")

    def k1ph_split_rows_peers(self, n_true: int, n: int, rows: int, row0: int, rows_f32: int,
                              state: int, i: int, xi: int, yi: int, peer_h0, peer_h1) -> None:
        _lib.check(self._L.mxp_k1ph_split_rows_peers(
            self._h, n_true, n, rows, row0, ctypes.c_void_p(rows_f32), ctypes.c_void_p(state), i,
            xi, yi, len(peer_h0), self._ptr_array(peer_h0), self._ptr_array(peer_h1)),
            "mxp_k1ph_split_rows_peers")

    def k1ph_read_flag(self, state: int) -> bool:
        c = ctypes.c_int()
        _lib.check(self._L.mxp_k1ph_read_flag(self._h, ctypes.c_void_p(state), ctypes.byref(c)),
                   "mxp_k1ph_read_flag")
        return bool(c.value)

    def copy2d_device(self, dst: int, dpitch: int, src: int, spitch: int, width: int,
                      rows: int) -> None:
        """rows x width bytes, device to device, on the engine's stream."""
        _lib.check(self._L.mxp_copy2d_device(self._h, ctypes.c_void_p(dst), dpitch,
                                             ctypes.c_void_p(src), spitch, width, rows),
                   "mxp_copy2d_device")

    # ------------------------------------------------------------ NVLS multicast exchange
    def mc_supported(self) -> bool:
        ok = ctypes.c_int()
        _lib.check(self._L.mxp_mc_supported(self._h, ctypes.byref(ok)), "mxp_mc_supported")
        return bool(ok.value)

    def mc_create(self, nranks: int, nbytes: int):
        """(mc object, exported 64-byte handle, granted size) — the creator's side."""
        buf = ctypes.create_string_buffer(_lib.MXP_MC_HANDLE_BYTES)
        mc = ctypes.c_void_p()
        _lib.check(self._L.mxp_mc_create(self._h, int(nranks), int(nbytes), buf, ctypes.byref(mc)),
                   "mxp_mc_create")
        size = ctypes.c_size_t()
        _lib.check(self._L.mxp_mc_size(mc, ctypes.byref(size)), "mxp_mc_size")
        return mc, buf.raw, size.value

    def mc_import(self, handle: bytes, nbytes: int):
        mc = ctypes.c_void_p()
        _lib.check(self._L.mxp_mc_import(self._h, handle, int(nbytes), ctypes.byref(mc)),
                   "mxp_mc_import")
        return mc

    def mc_bind(self, mc):
        """(local unicast pointer, multicast pointer) of this rank's bound copy."""
        uc, mcp = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(self._L.mxp_mc_bind(mc, ctypes.byref(uc), ctypes.byref(mcp)), "mxp_mc_bind")
        return uc.value, mcp.value

    def mc_destroy(self, mc) -> None:
        _lib.check(self._L.mxp_mc_destroy(mc), "mxp_mc_destroy")

    def gemm_rows_planes_mc(self, n: int, rows: int, row0: int, a_hi: int, a_lo: int, b_hi: int,
                            b_lo: int, mc_hi=None, mc_lo=None, mc_f32=None) -> None:
        _lib.check(self._L.mxp_gemm_rows_planes_mc(
            self._h, n, rows, row0, ctypes.c_void_p(a_hi), ctypes.c_void_p(a_lo),
            ctypes.c_void_p(b_hi), ctypes.c_void_p(b_lo), ctypes.c_void_p(mc_hi),
            ctypes.c_void_p(mc_lo), ctypes.c_void_p(mc_f32)), "mxp_gemm_rows_planes_mc")

    def peer_barrier(self, rank: int, peer_flags, epoch: int) -> None:
        _lib.check(self._L.mxp_peer_barrier(self._h, rank, len(peer_flags),
                                            self._ptr_array(peer_flags), epoch & 0xFFFFFFFF),
                   "mxp_peer_barrier")

    def gemm_rows_device(self, d_a: int, d_b: int, d_c: int, n: int, rows: int,
                         mode: int = _lib.MXP_F32) -> None:
        """C[rows x n] = A[rows x n] * B[n x n] on device (row block of one multiply)."""
        _lib.check(self._L.mxp_gemm_rows(self._h, mode, n, rows, ctypes.c_void_p(d_a),
                                         ctypes.c_void_p(d_b), ctypes.c_void_p(d_c)),
                   "mxp_gemm_rows")

    def random_device(self, d_out: int, n: int, batch: int = 1, seed0: int = 0,
                      lo: float = -0.5, hi: float = 0.5, scale: float = 0.0,
                      mode: int = _lib.MXP_F32) -> None:
        _lib.check(self._L.mxp_random_device(self._h, mode, n, batch,
                                             ctypes.c_uint64(seed0 & (2**64 - 1)), lo, hi, scale,
                                             ctypes.c_void_p(d_out)), "mxp_random_device")

    def set_f32_datapath(self, datapath: str) -> None:
        """FP32 chains at the CTA-pair sizes (n_pad % 256 == 0, n_pad >= 1024):
        "auto" = K1PH (scaled fp16x2, 3xTF32 recomputation when a product
        loses dynamic range), "3xtf32" = always 3xTF32 (the row-sharded
        multi-GPU chains' datapath)."""
        codes = {"auto": 0, "3xtf32": 1}
        if datapath not in codes:
            raise ValueError(f"unknown f32 datapath {datapath!r} (auto | 3xtf32)")
        _lib.check(self._L.mxp_set_f32_datapath(self._h, codes[datapath]), "mxp_set_f32_datapath")

    def last_f32_fallback(self) -> bool:
        """Whether the last K1PH chain was recomputed on 3xTF32 (dynamic range)."""
        c = ctypes.c_int()
        _lib.check(self._L.mxp_last_f32_fallback(self._h, ctypes.byref(c)), "mxp_last_f32_fallback")
        return bool(c.value)

    def last_small_fixups(self) -> int:
        """Matrices of the last n <= 128 launch that K3B recomputed (dynamic range)."""
        c = ctypes.c_int64()
        _lib.check(self._L.mxp_last_small_fixups(self._h, ctypes.byref(c)), "mxp_last_small_fixups")
        return c.value

    def last_kernel_clock(self):
        """(sm_mhz, kernel_ms) of the last batched K3H launch, measured in the
        kernel (clock64 / globaltimer of CTA 0)."""
        mhz, ms = ctypes.c_double(), ctypes.c_double()
        _lib.check(self._L.mxp_last_kernel_clock(self._h, ctypes.byref(mhz), ctypes.byref(ms)),
                   "mxp_last_kernel_clock")
        return mhz.value, ms.value

    def splitmix64_device(self, d_out: int, seed: int, count: int) -> None:
        _lib.check(self._L.mxp_splitmix64_device(self._h, ctypes.c_uint64(seed & (2**64 - 1)),
                                                 int(count), ctypes.c_void_p(d_out)),
                   "mxp_splitmix64_device")

    # ------------------------------------------------------------ memory
    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _lib.check(self._L.mxp_alloc(self._h, nbytes, ctypes.byref(p)), "mxp_alloc")
        return int(p.value)

    def free(self, ptr: int) -> None:
        _lib.check(self._L.mxp_free(self._h, ctypes.c_void_p(ptr)), "mxp_free")

    def host_alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _lib.check(self._L.mxp_host_alloc(self._h, nbytes, ctypes.byref(p)), "mxp_host_alloc")
        return int(p.value)

    def host_free(self, ptr: int) -> None:
        _lib.check(self._L.mxp_host_free(self._h, ctypes.c_void_p(ptr)), "mxp_host_free")

    def pinned_array(self, shape, dtype) -> np.ndarray:
        """A numpy view of freshly allocated pinned host memory (freed with the engine
        process; call host_free(arr.ctypes.data) to release early)."""
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        ptr = self.host_alloc(nbytes)
        buf = (ctypes.c_char * nbytes).from_address(ptr)
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def upload(self, d_dst: int, host: np.ndarray) -> None:
        host = np.ascontiguousarray(host)
        _lib.check(self._L.mxp_upload(self._h, ctypes.c_void_p(d_dst), _ptr(host), host.nbytes),
                   "mxp_upload")

    def download(self, host: np.ndarray, d_src: int) -> np.ndarray:
        _lib.check(self._L.mxp_download(self._h, _ptr(host), ctypes.c_void_p(d_src), host.nbytes),
                   "mxp_download")
        return host


def plan_string(k: int) -> str:
    """The plan as 'S'/'M' characters, from the C ABI (expo.py:60-75)."""
    L = _lib.load()
    buf = ctypes.create_string_buffer(256)
    cnt = ctypes.c_int64()
    _lib.check(L.mxp_plan(int(k), buf, 256, ctypes.byref(cnt)), "mxp_plan")
    return buf.raw[: cnt.value].decode()


_engines: dict = {}
_engines_lock = threading.Lock()


def default_engine(device: Optional[int] = None) -> Engine:
    """Per-(thread, device) engine, created lazily."""
    if device is None:
        device = 0
    key = (threading.get_ident(), device)
    with _engines_lock:
        eng = _engines.get(key)
        if eng is None:
            eng = Engine(device)
            _engines[key] = eng
        return eng


def power_multi(a: np.ndarray, k: int, devices=None, out: Optional[np.ndarray] = None) -> np.ndarray:
    """A^k on several GPUs of this process (``mxp_power_multi``): a (batch, n, n)
    stack is split into contiguous batch shards (no communication); a single
    n x n FP32 matrix (n > 128) is row-sharded with each step's rows stored by
    the GEMM epilogue into every device's planes over NVLink.  ``devices``: a
    list of device ordinals (may repeat), an int N (devices 0..N-1), or None
    (every visible device)."""
    a = np.ascontiguousarray(a)
    if a.ndim not in (2, 3) or a.shape[-1] != a.shape[-2]:
        raise E.ShapeError(f"expected an (n, n) or (batch, n, n) array, got shape {a.shape}")
    if isinstance(devices, int):
        devices = list(range(devices))
    devs = [int(d) for d in devices] if devices is not None else list(range(device_count()))
    if not devs:
        raise E.DeviceUnavailableError("no CUDA device available")
    mode = _mode_of(a)
    if out is None:
        out = np.empty_like(a)
    elif (not isinstance(out, np.ndarray) or out.shape != a.shape or out.dtype != a.dtype
          or not out.flags.c_contiguous or not out.flags.writeable):
        raise E.ShapeError(f"out must be a writeable C-contiguous {a.dtype} array of shape {a.shape}")
    batch = a.shape[0] if a.ndim == 3 else 1
    if batch == 0:
        return out
    L = _lib.load()
    arr = (ctypes.c_int * len(devs))(*devs)
    st = _lib.Stats()
    rc = L.mxp_power_multi(len(devs), arr, mode, a.shape[-1], batch, int(k), _ptr(a), _ptr(out),
                           ctypes.byref(st))
    power_multi.last_stats = st
    Engine._raise_chain(rc, st, plan_string(k) if k >= 0 else "", "mxp_power_multi")
    return out


def release_multi() -> None:
    """Destroy the internal per-device handles of ``power_multi``."""
    _lib.check(_lib.load().mxp_multi_release(), "mxp_multi_release")


def device_count() -> int:
    L = _lib.load()
    c = ctypes.c_int()
    rc = L.mxp_device_count(ctypes.byref(c))
    return c.value if rc == _lib.MXP_OK else 0
