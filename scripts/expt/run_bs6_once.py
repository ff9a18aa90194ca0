"""One product BS6 call at C3 order N (argv[1], default 1) for ncu captures."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = int(sys.argv[2]) if len(sys.argv) > 2 else int(round((1e8 ** (1 / 3) - 1) / p))
mesh = sb.build_mesh(K, p)
op = sb.build_gather(mesh)
del mesh
q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
from paper_2009_10917_b200.gs import bs6_gather_into  # noqa: E402
for _ in range(3):
    bs6_gather_into(op, q, out)
torch.cuda.synchronize()
print("done", K, p)
