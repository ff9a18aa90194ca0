"""Small BS6/BS7/CG workload for compute-sanitizer memcheck."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200 import cg  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(4)
for K, p in ((1, 1), (3, 1), (4, 2), (3, 3), (2, 7), (2, 15)):
    m = sb.build_mesh(K, p)
    op = sb.build_gather(m)
    ids = sb.build_scatter_ids(m, mask={0, 5})
    qg = torch.rand(m.ng, dtype=torch.float64, device="cuda", generator=g)
    ql = torch.zeros(m.nl, dtype=torch.float64, device="cuda")
    sb.bs7_scatter(ids, qg, ql)
    out = sb.bs6_gather(op, ql)
    print(K, p, float(out.sum()), flush=True)
d = np.repeat([1.0, 2.0, 3.0], 8)
b = torch.rand(24, dtype=torch.float64, device="cuda", generator=g)
r = cg.cg_solve_device(sb.diagonal_operator(d), b, torch.zeros_like(b), eps=1e-20, max_iter=24, graph=True,
                       check_every=2)
print("cg", r.iterations, r.converged)
torch.cuda.synchronize()
print("done")
