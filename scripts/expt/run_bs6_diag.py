"""Time the BS6 diagnosis variants (scripts/expt/bs6_diag.cu) on the box."""
import ctypes
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(ROOT, "gpurun_out", "diag_bs6.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                "-o", SO, os.path.join(HERE, "bs6_diag.cu")], check=True)
L = ctypes.CDLL(SO)
L.diag_bs6.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4 + \
    [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
NAMES = {0: "product", 1: "q-sequential", 2: "no-sums", 3: "q-seq+no-sums", 4: "stream ceiling"}

for K, p in [(66, 7), (463, 1), (31, 15)]:
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = torch.empty(mesh.nl + 2, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = sb.bs6_gather(op, q[:mesh.nl])
    plan = op.plan()
    nsb = plan.numel() // 2 - 1
    nbytes = bytes_moved("bs6", nl=mesh.nl, ng=mesh.ng)
    out = torch.empty(mesh.ng + 2, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for v in range(5):
        args = (v, plan.data_ptr(), nsb, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), q.data_ptr(),
                out.data_ptr(), mesh.nl, mesh.ng, st)
        assert L.diag_bs6(*args) == 0
        torch.cuda.synchronize()
        ok = torch.equal(out[:mesh.ng], ref) if v == 0 else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            L.diag_bs6(*args)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"K={K} p={p} {NAMES[v]:16s} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s ok={ok}", flush=True)
    del q, out, op, mesh, ref
    torch.cuda.empty_cache()
