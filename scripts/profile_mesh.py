"""Launch BS6 and BS7 on one mesh (for ncu):  python scripts/profile_mesh.py K p"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2009_10917_b200 as sb  # noqa: E402

K, p = int(sys.argv[1]), int(sys.argv[2])
mesh = sb.build_mesh(K, p)
op = sb.build_gather(mesh)
ids = sb.build_scatter_ids(mesh)
_ = ids.has_mask
q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1)
out = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
ql = torch.empty(mesh.nl, dtype=torch.float64, device="cuda")
for _ in range(2):
    sb.bs6_gather(op, q, out)
    sb.bs7_scatter(ids, qg, ql)
torch.cuda.synchronize()
print("K", K, "p", p, "NL", mesh.nl, "NG", mesh.ng)
