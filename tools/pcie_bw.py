"""Pinned-host PCIe bandwidth on the GPU box: H2D of the Wan2.1-14B Q/K/V bytes
(2.32 GB) alone, D2H of O (0.77 GB) alone, and both concurrently -- the bound
of bench.py's e2e number. Usage: python tools/pcie_bw.py"""
import torch, time
n = 2322432000 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
ho = torch.empty(n // 3, dtype=torch.bfloat16).pin_memory()
do = torch.empty(n // 3, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"H2D alone: {n*2/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms for 2.32 GB)")
t = time.perf_counter()
for _ in range(3):
    ho.copy_(do, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"D2H alone: {n*2/3/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms for 0.77 GB)")
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"H2D 2.32 GB + D2H 0.77 GB concurrent: {dt*1e3:.1f} ms")
