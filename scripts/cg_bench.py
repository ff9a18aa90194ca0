"""Host-scalar vs device-resident CG on the B200 (SURVEY 8(f) row 1 evidence).

A = Z^T diag(w) Z on an order-p hex mesh (BS7 scatter, weight, BS6 gather),
fixed iteration count (eps tiny, max_iter = iters) so all variants do the same
work; prints ms/iteration and the speed-up from dropping the two host syncs
per iteration (check_every) and the launch overhead (CUDA graph).
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200 import cg  # noqa: E402


def run(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return best, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--check-every", type=int, default=50)
    ap.add_argument("--cases", default="4,7;16,7;66,7")
    args = ap.parse_args()
    out = []
    for case in args.cases.split(";"):
        K, p = (int(v) for v in case.split(","))
        mesh = sb.build_mesh(K, p)
        op, ids = sb.build_gather(mesh), sb.build_scatter_ids(mesh)
        rng = np.random.default_rng([K, p])
        A = cg.gather_scatter_operator(op, ids, rng.uniform(1, 2, mesh.nl))
        b = torch.from_numpy(rng.uniform(-1, 1, mesh.ng)).cuda()
        x0 = torch.zeros_like(b)
        it = args.iters
        th, rh = run(lambda: cg.cg_solve(A, b, x0, 1e-300, it))
        td, rd = run(lambda: cg.cg_solve_device(A, b, x0, 1e-300, it, check_every=args.check_every))
        tg, rg = run(lambda: cg.cg_solve_device(A, b, x0, 1e-300, it, check_every=args.check_every, graph=True))
        same = torch.equal(rh.x, rd.x) and torch.equal(rh.x, rg.x) and rh.iterations == rd.iterations == rg.iterations
        rec = {"K": K, "p": p, "ng": mesh.ng, "nl": mesh.nl, "iterations": rh.iterations,
               "host_scalars_ms_per_iter": 1e3 * th / it, "device_ms_per_iter": 1e3 * td / it,
               "device_graph_ms_per_iter": 1e3 * tg / it, "speedup_device": th / td, "speedup_graph": th / tg,
               "bitwise_equal": bool(same)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del mesh, op, ids, A, b, x0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
