"""Time the product BS7 scatter over N (SB200_BS7_KERNEL selects a variant)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

tag = "k" + os.environ.get("SB200_BS7_KERNEL", "0")
orders = [int(a) for a in sys.argv[1:]] or list(range(1, 16))
for p in orders:
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    mesh = sb.build_mesh(K, p)
    ids = sb.build_scatter_ids(mesh)
    qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ql = torch.empty(mesh.nl, dtype=torch.float64, device="cuda")
    sb.bs7_scatter(ids, qg, ql)
    ok = torch.equal(ql, qg[mesh.local_to_global_dev.long()])
    nbytes = bytes_moved("bs7", nl=mesh.nl, ng=mesh.ng)
    for _ in range(3):
        sb.bs7_scatter(ids, qg, ql)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sb.bs7_scatter(ids, qg, ql)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{tag} N={p:2d} K={K} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s ok={ok}", flush=True)
    del mesh, ids, qg, ql
    torch.cuda.empty_cache()
