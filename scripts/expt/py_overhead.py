"""Host-side cost per public call at tiny sizes (Python wrapper + ctypes), on the box."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200 import _lib, kernels as KN  # noqa: E402

x = torch.rand(1024, dtype=torch.float64, device="cuda")
y = torch.rand(1024, dtype=torch.float64, device="cuda")
res = torch.empty(1, dtype=torch.float64, device="cuda")
mesh = sb.build_mesh(2, 3)
op, ids = sb.build_gather(mesh), sb.build_scatter_ids(mesh)
q = torch.rand(mesh.nl, dtype=torch.float64, device="cuda")
qg = torch.rand(mesh.ng, dtype=torch.float64, device="cuda")
out = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
calls = {
    "raw ctypes sb_bs1_copy": lambda: L.sb_bs1_copy(x.data_ptr(), y.data_ptr(), 1024, st),
    "torch.cuda.current_stream()": lambda: torch.cuda.current_stream(x.device).cuda_stream,
    "bs1_copy": lambda: sb.bs1_copy(x, y),
    "bs2_axpy": lambda: sb.bs2_axpy(0.5, x, 0.25, y),
    "bs3_norm2_async": lambda: KN.bs3_norm2_async(x, out=res),
    "bs5_async": lambda: KN.bs5_fused_cg_update_async(0.1, x, y, x, y, out=res),
    "bs6_gather(op, q, out)": lambda: sb.bs6_gather(op, q, out),
    "bs7_scatter": lambda: sb.bs7_scatter(ids, qg, q),
    "torch y.copy_(x)": lambda: y.copy_(x),
}
for name, fn in calls.items():
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5000):
        fn()
    dt = (time.perf_counter() - t) / 5000
    torch.cuda.synchronize()
    print(f"{name:32s} {dt * 1e6:6.2f} us/call (host)", flush=True)
