"""How fast can pageable numpy buffers be pinned in place (cudaHostRegister)
compared with copying them through the engine's staging ring?"""
import ctypes
import time

import numpy as np
import torch

torch.cuda.init()
rt = torch.cuda.cudart()
for gb in (0.5, 4.0):
    n = int(gb * (1 << 30))
    a = np.empty(n, np.uint8)
    a[::4096] = 1  # touch
    t0 = time.perf_counter()
    r = rt.cudaHostRegister(a.ctypes.data, n, 0)
    t1 = time.perf_counter()
    r2 = rt.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    b = np.empty(n, np.uint8)  # untouched
    t3 = time.perf_counter()
    r3 = rt.cudaHostRegister(b.ctypes.data, n, 0)
    t4 = time.perf_counter()
    rt.cudaHostUnregister(b.ctypes.data)
    c = np.empty_like(a)
    t5 = time.perf_counter()
    np.copyto(c, a)
    t6 = time.perf_counter()
    print(f"{gb} GB: register touched {t1-t0:.3f}s ({r}), unregister {t2-t1:.3f}s, "
          f"register untouched {t4-t3:.3f}s ({r3}), numpy copy {t6-t5:.3f}s")
