"""PCIe duplex throughput with 1, 2 and 4 copy streams per direction (4 GiB each
way, 64 MB chunks round-robin over the streams): does more than one DMA queue
per direction beat the single-stream duplex rate the e2e path runs at?"""
import time

import torch

n = 1 << 30  # 4 GiB of float32
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
chunk = 16 << 20  # elements (64 MB)


def run(k):
    ins = [torch.cuda.Stream() for _ in range(k)]
    outs = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, o in enumerate(range(0, n, chunk)):
        with torch.cuda.stream(ins[i % k]):
            d_a[o:o + chunk].copy_(h_in[o:o + chunk], non_blocking=True)
        with torch.cuda.stream(outs[i % k]):
            h_out[o:o + chunk].copy_(d_b[o:o + chunk], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for k in (1, 2, 4, 1, 2, 4):
    dt = run(k)
    print(f"{k} stream(s) per direction: {8 / dt:.1f} GB/s duplex ({dt * 1e3:.0f} ms for 4+4 GiB)")
