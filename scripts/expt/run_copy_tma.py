"""TMA bulk copy (global->smem->global) vs the BS1 kernel, n = 1e8 / 4e8 doubles."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402

SO = os.path.join(ROOT, "gpurun_out", "copy_tma.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", SO,
                os.path.join(os.path.dirname(os.path.abspath(__file__)), "copy_tma.cu")], check=True)
L = ctypes.CDLL(SO)
L.copy_tma.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
for n in (100_000_000, 400_000_000):
    n -= n % 4096
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    runs = {"bs1 (LDG/STG)": lambda: sb.bs1_copy(x, y)}
    for v, name in ((0, "16K x 8"), (1, "32K x 6"), (2, "8K x 16"), (3, "16K x 12")):
        for grid in (148, 296):
            runs[f"tma {name} grid {grid}"] = (lambda v=v, grid=grid: L.copy_tma(v, x.data_ptr(), y.data_ptr(), 8 * n, grid, st))
    for name, fn in runs.items():
        y.zero_()
        fn()
        torch.cuda.synchronize()
        ok = torch.equal(x, y)
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"n={n:.1e} {name:28s} {16 * n / ms / 1e6:.0f} GB/s ok={ok}", flush=True)
    del x, y
    torch.cuda.empty_cache()
