"""Time the tiled BS6 kernel's q-staging + row-sum traffic alone (SB200_BS6_TILE_KERNEL=p) vs the full kernel."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb
from paper_2009_10917_b200 import _lib

K = int(sys.argv[1]) if len(sys.argv) > 1 else 463
op = sb.build_gather(sb.build_mesh(K, 1))
q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
L = _lib.lib()
st = _lib.stream_handle()
for mode in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["t3", "4b"]):
    os.environ["SB200_BS6_TILE_KERNEL"] = mode
    f = lambda: L.sb_bs6_gather_tiled(*op.geometry, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng, op.nl, q.data_ptr(), out.data_ptr(), None, 0, st)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    full = 12 * op.nl + 8 * op.ng + 4 * (op.ng + 1)
    qo = 8 * op.nl + 8 * op.ng
    print(f"K={K} {mode}: {ms:.3f} ms  algorithmic {full / ms / 1e6:.0f} GB/s  q+out traffic {qo / ms / 1e6:.0f} GB/s")
