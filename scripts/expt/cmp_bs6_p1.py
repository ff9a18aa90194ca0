"""BS6 at p=1 over mesh sizes: super-block (planned) kernel vs the row-line-tiled kernel (default variant)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb
from paper_2009_10917_b200 import _lib

L = _lib.lib()
st = _lib.stream_handle()


def timed(f, reps=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps


for K in [int(k) for k in (sys.argv[1:] or "4 8 16 32 66 100 150 200 300 400 463".split())]:
    op = sb.build_gather(sb.build_mesh(K, 1))
    q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    a = torch.empty(op.ng, dtype=torch.float64, device="cuda")
    b = torch.empty(op.ng, dtype=torch.float64, device="cuda")
    plan = op.plan()
    fp = lambda: L.sb_bs6_gather_planned(plan.data_ptr(), op.n_blocks, op.nodes_per_block, op.row_starts_dev.data_ptr(),
                                         op.col_ids_dev.data_ptr(), op.ng, op.nl, q.data_ptr(), a.data_ptr(), None, 0, st)
    ft = lambda: L.sb_bs6_gather_tiled(*op.geometry, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng,
                                       op.nl, q.data_ptr(), b.data_ptr(), None, 0, st)
    nb = 12 * op.nl + 8 * op.ng + 4 * (op.ng + 1)
    tp, tt = timed(fp), timed(ft)
    torch.cuda.synchronize()
    print(f"K={K:4d} NG={op.ng:.2e}  planned {tp*1e3:8.1f} us {nb/tp/1e6:6.0f} GB/s   tiled {tt*1e3:8.1f} us "
          f"{nb/tt/1e6:6.0f} GB/s  bitwise={torch.equal(a, b)}", flush=True)
    del op, q, a, b, plan
