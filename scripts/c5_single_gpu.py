"""BS6/BS7 bandwidth on the whole config-5 mesh (K=143, N=7: NG = 1.0e9) on ONE B200."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

mesh = sb.build_mesh(143, 7)
op, ids = sb.build_gather(mesh), sb.build_scatter_ids(mesh)
q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1)
out = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
res = {"K": 143, "order": 7, "nl": mesh.nl, "ng": mesh.ng}
for name, fn, nb in (("bs6", lambda: sb.bs6_gather(op, q, out), bytes_moved("bs6", nl=mesh.nl, ng=mesh.ng)),
                     ("bs7", lambda: sb.bs7_scatter(ids, qg, q), bytes_moved("bs7", nl=mesh.nl, ng=mesh.ng))):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[name] = {"ms": round(ms, 3), "GBps": round(nb / ms / 1e6, 1), "bytes": nb}
print(json.dumps(res))
