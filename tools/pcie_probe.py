import torch, time
n = 1 << 30  # 4 GiB of float32 = 1G elements
h_in = torch.empty(n, dtype=torch.float32).pin_memory(); h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda"); d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t0
for _ in range(2):
    a = t(lambda: d_a.copy_(h_in, non_blocking=True))
    b = t(lambda: h_out.copy_(d_b, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    c = t(both)
print(f"H2D {4/a:.1f} GB/s  D2H {4/b:.1f} GB/s  both {8/c:.1f} GB/s total ({c*1e3:.0f} ms for 4+4 GiB)")
