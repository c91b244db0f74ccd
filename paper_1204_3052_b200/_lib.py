"""ctypes binding of the C ABI in include/matexpo_b200.h.

The library is the in-tree `libmatexpo_b200.so` (built by
paper_1204_3052_b200/build.py).  If it is missing the product path raises
ExtensionNotBuiltError — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors as E

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MXP_LIB_PATH") or os.path.join(HERE, "libmatexpo_b200.so")

MXP_OK = 0
MXP_E_VALIDATION = 1
MXP_E_UNSUPPORTED = 2
MXP_E_DEVICE_UNAVAILABLE = 3
MXP_E_CUDA = 4
MXP_E_NCCL = 5

MXP_F32 = 0
MXP_F64 = 1
MXP_U32_MOD = 2

MXP_KERNEL_K3H = 0
MXP_KERNEL_K3B = 1

# Every symbol the header declares (tests/test_abi.py checks the .so exports them).
EXPORTS = (
    "mxp_version", "mxp_device_count", "mxp_create", "mxp_destroy", "mxp_get_stream",
    "mxp_synchronize", "mxp_num_sms", "mxp_alloc", "mxp_free", "mxp_host_alloc", "mxp_gemm_rows",
    "mxp_host_free", "mxp_upload", "mxp_download", "mxp_plan", "mxp_gemm", "mxp_multiply",
    "mxp_power_device", "mxp_power", "mxp_power_batched_device", "mxp_power_batched",
    "mxp_power_mod_device", "mxp_power_mod", "mxp_random_device", "mxp_last_error",
    "mxp_status_string", "mxp_gemm_prepare_rhs", "mxp_gemm_rows_prepared",
    "mxp_ipc_get_handle", "mxp_ipc_open_handle", "mxp_ipc_close_handle", "mxp_split_planes",
    "mxp_gemm_rows_planes_peers", "mxp_peer_barrier", "mxp_debug_inject_fault",
    "mxp_splitmix64_device", "mxp_last_kernel_clock",
    "mxp_small_kernel_for", "mxp_mc_supported", "mxp_mc_create", "mxp_mc_import",
    "mxp_mc_size", "mxp_mc_bind", "mxp_mc_destroy", "mxp_gemm_rows_planes_mc",
    "mxp_copy2d_device", "mxp_last_small_fixups", "mxp_power_multi", "mxp_multi_release",
    "mxp_set_f32_datapath", "mxp_last_f32_fallback",
    "mxp_k1ph_state_bytes", "mxp_k1ph_split_base", "mxp_k1ph_gemm_rows", "mxp_k1ph_max_to_peers",
    "mxp_k1ph_split_rows_peers", "mxp_k1ph_read_flag",
)
MXP_IPC_HANDLE_BYTES = 72
MXP_MC_HANDLE_BYTES = 64


class Stats(ctypes.Structure):
    """mxp_stats."""

    _fields_ = [
        ("multiply_count", ctypes.c_int64),
        ("square_count", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("h2d", ctypes.c_int64),
        ("d2h", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("failed_step", ctypes.c_int64),
        ("device_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libmatexpo_b200.so (raises ExtensionNotBuiltError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise E.ExtensionNotBuiltError(
                f"{LIB_PATH} not found; build it with `python -m paper_1204_3052_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, c_int, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        P = ctypes.POINTER
        sig = {
            "mxp_version": [P(c_int), P(c_int)],
            "mxp_device_count": [P(c_int)],
            "mxp_create": [c_int, P(vp)],
            "mxp_destroy": [vp],
            "mxp_get_stream": [vp, P(vp)],
            "mxp_synchronize": [vp],
            "mxp_num_sms": [vp, P(c_int)],
            "mxp_alloc": [vp, sz, P(vp)],
            "mxp_free": [vp, vp],
            "mxp_host_alloc": [vp, sz, P(vp)],
            "mxp_host_free": [vp, vp],
            "mxp_upload": [vp, vp, vp, sz],
            "mxp_download": [vp, vp, vp, sz],
            "mxp_plan": [i64, ctypes.c_char_p, i64, P(i64)],
            "mxp_gemm": [vp, c_int, i64, vp, vp, vp],
            "mxp_gemm_rows": [vp, c_int, i64, i64, vp, vp, vp],
            "mxp_gemm_prepare_rhs": [vp, c_int, i64, vp],
            "mxp_gemm_rows_prepared": [vp, c_int, i64, i64, vp, vp],
            "mxp_ipc_get_handle": [vp, vp, vp],
            "mxp_ipc_open_handle": [vp, vp, ctypes.POINTER(vp)],
            "mxp_ipc_close_handle": [vp, vp],
            "mxp_split_planes": [vp, i64, vp, vp, vp],
            "mxp_gemm_rows_planes_peers": [vp, i64, i64, i64, vp, vp, vp, vp, c_int,
                                           ctypes.POINTER(vp), ctypes.POINTER(vp),
                                           ctypes.POINTER(vp)],
            "mxp_peer_barrier": [vp, c_int, c_int, ctypes.POINTER(vp), ctypes.c_uint32],
            "mxp_multiply": [vp, c_int, i64, vp, vp, vp, P(Stats)],
            "mxp_power_device": [vp, c_int, i64, i64, vp, vp, P(Stats)],
            "mxp_power": [vp, c_int, i64, i64, vp, vp, P(Stats)],
            "mxp_power_batched_device": [vp, c_int, i64, i64, i64, vp, vp, P(Stats)],
            "mxp_power_batched": [vp, c_int, i64, i64, i64, vp, vp, P(Stats)],
            "mxp_power_mod_device": [vp, i64, i64, ctypes.c_uint32, vp, vp, P(Stats)],
            "mxp_power_mod": [vp, i64, i64, ctypes.c_uint32, vp, vp, P(Stats)],
            "mxp_random_device": [vp, c_int, i64, i64, ctypes.c_uint64, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_double, vp],
            "mxp_last_error": [ctypes.c_char_p, sz],
            "mxp_status_string": [c_int],
            "mxp_debug_inject_fault": [vp, i64],
            "mxp_splitmix64_device": [vp, ctypes.c_uint64, i64, vp],
            "mxp_last_kernel_clock": [vp, P(ctypes.c_double), P(ctypes.c_double)],
            "mxp_small_kernel_for": [i64, i64, P(c_int)],
            "mxp_mc_supported": [vp, P(c_int)],
            "mxp_mc_create": [vp, c_int, sz, vp, P(vp)],
            "mxp_mc_import": [vp, vp, sz, P(vp)],
            "mxp_mc_size": [vp, P(sz)],
            "mxp_mc_bind": [vp, P(vp), P(vp)],
            "mxp_mc_destroy": [vp],
            "mxp_gemm_rows_planes_mc": [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp],
            "mxp_copy2d_device": [vp, vp, sz, vp, sz, sz, sz],
            "mxp_last_small_fixups": [vp, P(i64)],
            "mxp_set_f32_datapath": [vp, c_int],
            "mxp_k1ph_state_bytes": [P(sz)],
            "mxp_k1ph_split_base": [vp, i64, i64, vp, vp, vp, vp],
            "mxp_k1ph_gemm_rows": [vp, i64, i64, i64, vp, vp, vp, vp, vp, i64, i64, vp, c_int, c_int,
                                   c_int],
            "mxp_k1ph_max_to_peers": [vp, vp, c_int, c_int, P(vp)],
            "mxp_k1ph_split_rows_peers": [vp, i64, i64, i64, i64, vp, vp, c_int, c_int, c_int, c_int,
                                          P(vp), P(vp)],
            "mxp_k1ph_read_flag": [vp, vp, P(c_int)],
            "mxp_last_f32_fallback": [vp, P(c_int)],
            "mxp_power_multi": [c_int, P(c_int), c_int, i64, i64, i64, vp, vp, P(Stats)],
            "mxp_multi_release": [],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = c_int
        L.mxp_status_string.restype = ctypes.c_char_p
        _lib = L
        return L


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().mxp_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


_STATUS_EXC = {
    MXP_E_VALIDATION: E.ValidationError,
    MXP_E_UNSUPPORTED: E.UnsupportedError,
    MXP_E_DEVICE_UNAVAILABLE: E.DeviceUnavailableError,
    MXP_E_CUDA: E.DeviceError,
    MXP_E_NCCL: E.DeviceError,
}


def check(status: int, what: str = "") -> None:
    """Raise the matexpo-style exception for a non-OK status."""
    if status == MXP_OK:
        return
    exc = _STATUS_EXC.get(status, E.DeviceError)
    msg = last_error()
    raise exc(f"{what}: {msg}" if what else msg)


def small_kernel_for(n: int, k: int) -> str:
    """'k3h' or 'k3b': the persistent kernel an n <= 128 fp32 chain of power k
    runs on (the accuracy router, mxp_small_kernel_for)."""
    v = ctypes.c_int()
    check(load().mxp_small_kernel_for(int(n), int(k), ctypes.byref(v)), "mxp_small_kernel_for")
    return "k3h" if v.value == MXP_KERNEL_K3H else "k3b"
