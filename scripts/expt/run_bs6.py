"""A/B timing of experimental BS6 variants (scripts/expt/bs6_expt.cu) on the box."""
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
SO = os.path.join(ROOT, "gpurun_out", "expt_bs6.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                "-o", SO, os.path.join(HERE, "bs6_expt.cu")], check=True)
L = ctypes.CDLL(SO)
L.expt_bs6.argtypes = [ctypes.c_int] + [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4 + \
    [ctypes.c_int, ctypes.c_void_p]


def plan_for(op, G):
    nb = op.n_blocks
    nsb = (nb + G - 1) // G
    idx = torch.clamp(torch.arange(nsb + 1, device="cuda") * G, max=nb)
    r = op.block_starts_dev[idx].long()
    e = op.row_starts_dev[r]
    plan = torch.stack([r.int(), e.int()], 1).reshape(-1).contiguous()
    return plan, nsb


for K, p in [(66, 7), (463, 1), (31, 15)]:
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = sb.bs6_gather(op, q)
    nbytes = bytes_moved("bs6", nl=mesh.nl, ng=mesh.ng)
    out = torch.empty_like(ref)
    st = torch.cuda.current_stream()
    for variant, cap, cps in [(7, 512, 0), (12, 512, 0), (13, 512, 0), (14, 1024, 0), (11, 512, 0)]:
        plan, nsb = plan_for(op, max(1, cap // 512))
        per_sm = L.expt_bs6(variant, plan.data_ptr(), nsb, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(),
                            q.data_ptr(), out.data_ptr(), cps, st.cuda_stream)
        torch.cuda.synchronize()
        ok = torch.equal(out, ref) if variant not in (1, 11) else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            L.expt_bs6(variant, plan.data_ptr(), nsb, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(),
                       q.data_ptr(), out.data_ptr(), cps, st.cuda_stream)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"K={K} p={p} variant={variant} cap={cap} ctas/SM={per_sm} {ms:.3f} ms "
              f"{nbytes / ms / 1e6:.0f} GB/s ok={ok}", flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sb.bs6_gather(op, q, out)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"K={K} p={p} library {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
