"""Per-call timing of the public API on pinned host buffers (e2e breakdown)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2009_10917_b200 as sb  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda", 0)


def hvec(m):
    return torch.empty(m, dtype=torch.float64, device=dev).uniform_(-1, 1).cpu().pin_memory()


x, y, p, ap, r = (hvec(n) for _ in range(5))
mesh = sb.build_mesh(66, 7)
op = sb.build_gather(mesh)
ids = sb.build_scatter_ids(mesh)
q, qg = hvec(mesh.nl), hvec(mesh.ng)
ql = torch.zeros(mesh.nl, dtype=torch.float64).pin_memory()
calls = {
    "bs1": lambda: sb.bs1_copy(x, y),
    "bs2": lambda: sb.bs2_axpy(0.5, x, -0.25, y),
    "bs3": lambda: sb.bs3_norm2(x),
    "bs4": lambda: sb.bs4_dot(x, y),
    "bs5": lambda: sb.bs5_fused_cg_update(1e-3, p, ap, x, r),
    "bs6": lambda: sb.bs6_gather(op, q),
    "bs7": lambda: sb.bs7_scatter(ids, qg, ql),
}
for k, f in calls.items():
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    print(k, f"{(time.perf_counter() - t0) / 3 * 1e3:.1f} ms")
