"""BS5: product lattice kernel (TMA ring or SB200_NO_TMA=1 register lattice) vs the plain-stream ceiling."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2009_10917_b200 import kernels as KN  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(ROOT, "gpurun_out", "bs5_ceiling.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                "-o", SO, os.path.join(HERE, "bs5_ceiling.cu")], check=True)
L = ctypes.CDLL(SO)
L.bs5_ceiling.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_double,
                                                                    ctypes.c_void_p, ctypes.c_void_p]
tag = "no-tma" if os.environ.get("SB200_NO_TMA") == "1" else "tma"
for n in (int(1e8), int(4e8)):
    p, ap, x, r = (torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(4))
    res = torch.empty(1, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    runs = {f"lattice-{tag}": lambda: KN.bs5_fused_cg_update_async(1e-3, p, ap, x, r, out=res)}
    if tag == "tma":
        runs["stream-u2"] = lambda: L.bs5_ceiling(2, p.data_ptr(), ap.data_ptr(), x.data_ptr(), r.data_ptr(), n,
                                                  1e-3, res.data_ptr(), st)
        runs["stream-u4"] = lambda: L.bs5_ceiling(4, p.data_ptr(), ap.data_ptr(), x.data_ptr(), r.data_ptr(), n,
                                                  1e-3, res.data_ptr(), st)
    for name, fn in runs.items():
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"n={n:.0e} {name:16s} {48 * n / ms / 1e6:.0f} GB/s", flush=True)
    del p, ap, x, r
    torch.cuda.empty_cache()
