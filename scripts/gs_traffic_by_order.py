"""One BS6 and one BS7 launch per order N=1..15 at NG ~ 1e8 (run under ncu to
get DRAM bytes per launch vs the algorithmic bytes; see profiles/)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

for p in range(1, 16):
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    mesh = sb.build_mesh(K, p)
    op, ids = sb.build_gather(mesh), sb.build_scatter_ids(mesh)
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    out = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
    sb.bs6_gather(op, q, out)
    sb.bs7_scatter(ids, qg, q)
    torch.cuda.synchronize()
    print(f"N={p} K={K} nl={mesh.nl} ng={mesh.ng} bs6={bytes_moved('bs6', nl=mesh.nl, ng=mesh.ng)} "
          f"bs7={bytes_moved('bs7', nl=mesh.nl, ng=mesh.ng)}", flush=True)
    del mesh, op, ids, q, qg, out
    torch.cuda.empty_cache()
