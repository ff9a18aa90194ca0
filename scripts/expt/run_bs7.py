"""A/B timing of experimental BS7 variants (scripts/expt/bs7_expt.cu) on the box."""
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
SO = os.path.join(ROOT, "gpurun_out", "expt_bs7.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                "-o", SO, os.path.join(HERE, "bs7_expt.cu")], check=True)
L = ctypes.CDLL(SO)
L.expt_bs7.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_void_p]

for K, p in [(66, 7), (463, 1), (31, 15), (132, 3)]:
    mesh = sb.build_mesh(K, p)
    ids = sb.build_scatter_ids(mesh)
    qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = qg[mesh.local_to_global_dev.long()]
    nbytes = bytes_moved("bs7", nl=mesh.nl, ng=mesh.ng)
    ql = torch.empty(mesh.nl, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for variant in (0, 6, 8, 9, 10):
        per_sm = L.expt_bs7(variant, ids.ids.data_ptr(), mesh.nl, qg.data_ptr(), ql.data_ptr(), st)
        torch.cuda.synchronize()
        ok = torch.equal(ql, ref)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            L.expt_bs7(variant, ids.ids.data_ptr(), mesh.nl, qg.data_ptr(), ql.data_ptr(), st)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"K={K} p={p} variant={variant} ctas/SM={per_sm} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s ok={ok}",
              flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sb.bs7_scatter(ids, qg, ql)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"K={K} p={p} library {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
