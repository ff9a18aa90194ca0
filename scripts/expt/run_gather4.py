"""TMA gather4 vs LSU gathers over BS6 column orders (probe)."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402

SO = os.path.join(ROOT, "gpurun_out", "g4.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", SO, os.path.join(os.path.dirname(os.path.abspath(__file__)), "gather4_probe.cu"),
                "-lcuda"], check=True)
L = ctypes.CDLL(SO)
L.probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                    ctypes.c_int, ctypes.c_void_p]
for K, p in [(463, 1), (232, 2), (66, 7)]:
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    ci = op.col_ids_dev
    n = ci.shape[0]
    q = torch.empty(n + 2, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for mode, grid in ((0, 148 * 16), (0, 148 * 32), (1, 148 * 4), (1, 148 * 8), (1, 148 * 12)):
        rc = L.probe(mode, ci.data_ptr(), n, q.data_ptr(), n + 2, sink.data_ptr(), grid, st)
        torch.cuda.synchronize()
        if rc != 0:
            print(f"K={K} p={p} mode={mode} rc={rc}", flush=True)
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            L.probe(mode, ci.data_ptr(), n, q.data_ptr(), n + 2, sink.data_ptr(), grid, st)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"p={p} {'tma' if mode else 'ldg'} grid={grid} {ms:.3f} ms  {n / ms / 1e6:.1f} G entries/s "
              f"({12 * n / ms / 1e6:.0f} GB/s of ids+values)", flush=True)
    del mesh, op, ci, q
    torch.cuda.empty_cache()
