"""The C-ABI library loads here (no GPU) and exports every symbol the header
declares; host-side entry points that need no device behave like the reference."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1204_3052_b200 import _lib, build
import paper_1204_3052_b200 as mx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "matexpo_b200.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"MXP_API\s+[\w\s\*]+?\b(mxp_\w+)\s*\(", text)))


def test_header_symbols_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (mxp_\w+)", out))
    assert set(syms) <= exported, set(syms) - exported
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s)


def test_only_abi_symbols_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    text_syms = set(re.findall(r" T (\w+)", out))
    assert all(s.startswith("mxp_") for s in text_syms), text_syms


def test_plan_through_abi(lib):
    for k in list(range(0, 300)) + [1000, 1024, 257, 2**40 + 5, 2**62 + 2**61 + 1]:
        assert mx.engine.plan_string(k) == mx.plan_exponentiation(k).as_string(), k
    buf = ctypes.create_string_buffer(8)
    cnt = ctypes.c_int64()
    assert lib.mxp_plan(-1, buf, 8, ctypes.byref(cnt)) == _lib.MXP_E_VALIDATION
    assert "power must be >= 0" in _lib.last_error()


def test_status_strings(lib):
    assert lib.mxp_status_string(0) == b"MXP_OK"
    assert lib.mxp_status_string(_lib.MXP_E_CUDA) == b"MXP_E_CUDA"
    major, minor = ctypes.c_int(), ctypes.c_int()
    assert lib.mxp_version(ctypes.byref(major), ctypes.byref(minor)) == 0


def test_no_device_is_reported_not_faked(lib):
    """Without a GPU the engine refuses loudly (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    assert lib.mxp_create(0, ctypes.byref(h)) == _lib.MXP_E_DEVICE_UNAVAILABLE
    with pytest.raises(mx.DeviceUnavailableError):
        mx.Engine(0)
    with pytest.raises(mx.DeviceUnavailableError):
        mx.exponentiate(mx.Matrix([[1.0, 1.0], [1.0, 0.0]]), 10, mx.b200_backend())


def test_null_handle_validation(lib):
    st = _lib.Stats()
    rc = lib.mxp_power(None, 0, 4, 3, None, None, ctypes.byref(st))
    assert rc == _lib.MXP_E_VALIDATION


def test_sass_uses_tcgen05_and_dmma(lib):
    """The built cubins really contain tcgen05 MMAs (UTCHMMA), TMA loads,
    TMEM loads and DMMA — i.e. the tensor-core paths are what ships."""
    res = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True)
    if res.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = res.stdout
    assert re.search(r"UTC\w*MMA", sass)
    assert "UTMALDG" in sass
    assert "LDTM" in sass
    assert "DMMA" in sass


def test_small_kernel_router_both_sides_of_threshold():
    """The K3H -> K3B accuracy router (kernels_tf32.cu k3_route): K3B exactly
    when the predicted accumulated truncation bias (k-1)(2.5e-8 + 1.05e-9 n)
    exceeds 60% of the tolerance 16 m(k) sqrt(n) 2^-24.  Host-only."""
    import math

    def predicted(n, k):
        m = k.bit_length() - 1 + bin(k).count("1") - 1
        bias = (k - 1) * (2.5e-8 + 1.05e-9 * n)
        return "k3b" if bias > 0.6 * 16 * m * math.sqrt(n) * 2.0 ** -24 else "k3h"

    seen = set()
    for n in (1, 2, 7, 64, 100, 127, 128):
        for k in list(range(2, 70)) + [255, 256, 257, 383, 384, 385, 511, 512, 1000, 1024, 4096]:
            got = _lib.small_kernel_for(n, k)
            assert got == predicted(n, k), (n, k)
            seen.add(got)
    assert seen == {"k3h", "k3b"}
    # the configs: C1 (64^2 A^16) and C3 (128^2 A^64) run on K3H
    assert _lib.small_kernel_for(64, 16) == "k3h" and _lib.small_kernel_for(128, 64) == "k3h"
    # at n = 128 the switch sits between k = 383 and 384
    assert _lib.small_kernel_for(128, 383) == "k3h" and _lib.small_kernel_for(128, 384) == "k3b"


def test_power_multi_validation_without_device(lib):
    """mxp_power_multi validates before touching a device and, with no GPU,
    reports the device as unavailable (no CPU fallback)."""
    import numpy as np
    import torch

    st = _lib.Stats()
    a = np.zeros((4, 4), np.float32)
    out = np.empty_like(a)
    p = ctypes.c_void_p(a.ctypes.data)
    q = ctypes.c_void_p(out.ctypes.data)
    assert lib.mxp_power_multi(0, None, 0, 4, 1, 3, p, q, ctypes.byref(st)) == _lib.MXP_E_VALIDATION
    assert lib.mxp_power_multi(9, None, 0, 4, 1, 3, p, q, ctypes.byref(st)) == _lib.MXP_E_VALIDATION
    assert lib.mxp_power_multi(1, None, 0, 4, 1, -1, p, q, ctypes.byref(st)) == _lib.MXP_E_VALIDATION
    assert lib.mxp_power_multi(1, None, 7, 4, 1, 3, p, q, ctypes.byref(st)) == _lib.MXP_E_VALIDATION
    assert lib.mxp_power_multi(1, None, 0, 4, 1, 3, None, q, ctypes.byref(st)) == _lib.MXP_E_VALIDATION
    with pytest.raises(ValueError):
        mx.exponentiate_multi(a, -1, [0])
    with pytest.raises(mx.ShapeError):
        mx.exponentiate_multi(np.zeros((4, 5), np.float32), 3, [0])
    if not torch.cuda.is_available():
        devs = (ctypes.c_int * 2)(0, 0)
        rc = lib.mxp_power_multi(2, devs, 0, 4, 1, 3, p, q, ctypes.byref(st))
        assert rc == _lib.MXP_E_DEVICE_UNAVAILABLE
        with pytest.raises(mx.DeviceUnavailableError):
            mx.exponentiate_multi(a, 3, [0, 0])
