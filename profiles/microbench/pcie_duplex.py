import torch, time
n = 1_540_000_000 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    tb = t(both)
    print(f"H2D {1.54/th:.1f} GB/s  D2H {1.54/td:.1f} GB/s  both {2*1.54/tb:.1f} GB/s total ({tb*1e3:.1f} ms)")
