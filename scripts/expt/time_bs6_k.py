"""BS6 GB/s at order N over several K (CUDA events, 20 calls after 3 warm-ups)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

p = int(sys.argv[1])
for K in [int(v) for v in sys.argv[2:]]:
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    out = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
    for _ in range(3):
        sb.bs6_gather(op, q, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sb.bs6_gather(op, q, out)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"N={p} K={K} {ms * 1e3:.1f} us {bytes_moved('bs6', nl=mesh.nl, ng=mesh.ng) / ms / 1e6:.0f} GB/s")
