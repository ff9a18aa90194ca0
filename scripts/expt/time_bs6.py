"""Time the product BS6 gather over N (SB200_BS6_V1=1 selects the one-deep kernel)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

tag = os.environ.get("SB200_BS6_CFG", "default")
orders = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 7, 10, 15]
for p in orders:
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    out = sb.bs6_gather(op, q)
    ref = torch.zeros_like(out).index_add_(0, mesh.local_to_global_dev.long(), q)  # order differs: check closeness
    err = ((out - ref).abs().max() / ref.abs().max()).item()
    nbytes = bytes_moved("bs6", nl=mesh.nl, ng=mesh.ng)
    for _ in range(3):
        sb.bs6_gather(op, q, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sb.bs6_gather(op, q, out)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{tag} N={p:2d} K={K} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s relerr={err:.1e}", flush=True)
    del mesh, op, q, out, ref
    torch.cuda.empty_cache()
