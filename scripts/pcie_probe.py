"""Measure pinned H2D / D2H bandwidth alone and concurrently (PCIe ceiling of e2e)."""
import time
import torch

n = 1 << 27  # 1 GiB of fp64
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d(); d2h()


b = n * 8
print(f"H2D {b / t(h2d) / 1e9:.1f} GB/s  D2H {b / t(d2h) / 1e9:.1f} GB/s  "
      f"concurrent {2 * b / t(both) / 1e9:.1f} GB/s total")
import subprocess
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
print(subprocess.run(["bash", "-c", "nproc; lscpu | grep -E 'Model name|NUMA|Socket'; free -g | head -2"], capture_output=True, text=True).stdout)
