"""Partner-plan BS6 (sb_bs6_gather_partnered) vs the product gather over N; prints the paired fraction."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200 import _lib  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402

L = _lib.lib()
tag = f"mb{os.environ.get('SB200_BS6_PARTNER_MB', '12')}-swz{os.environ.get('SB200_BS6_PARTNER_SWZ', '1')}"
for p in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 7]:
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    plan = op.plan()
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = sb.bs6_gather(op, q)
    part = torch.empty(mesh.nl, dtype=torch.int8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = _lib.stream_handle()
    _lib.check(L.sb_bs6_make_partners(plan.data_ptr(), op.n_blocks, op.nodes_per_block, op.col_ids.data_ptr(),
                                      mesh.nl, part.data_ptr(), cnt.data_ptr(), st), "partners")
    out = torch.empty_like(ref)

    def run():
        _lib.check(L.sb_bs6_gather_partnered(plan.data_ptr(), op.n_blocks, op.nodes_per_block,
                                             op.row_starts.data_ptr(), op.col_ids.data_ptr(), part.data_ptr(),
                                             op.ng, op.nl, q.data_ptr(), out.data_ptr(), None, 0, st), "partnered")
    run()
    torch.cuda.synchronize()
    ok = torch.equal(out, ref)
    nbytes = bytes_moved("bs6", nl=mesh.nl, ng=mesh.ng)
    res = {}
    for name, fn in (("product", lambda: sb.bs6_gather(op, q, out)), ("partner", run)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        res[name] = nbytes / (e0.elapsed_time(e1) / 20) / 1e6
    print(f"{tag} N={p:2d} paired={cnt.item() / mesh.nl:.3f} product {res['product']:.0f} partner {res['partner']:.0f} "
          f"GB/s ok={ok}", flush=True)
    del mesh, op, q, ref, part, out
    torch.cuda.empty_cache()
