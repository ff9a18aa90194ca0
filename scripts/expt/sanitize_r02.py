"""Small workloads for compute-sanitizer over the round-2 BS6 kernels: the
TMA-tiled p=1 kernel (whole meshes, slabs with carry, a permuted CSR), the
z-sweep (p=1, p=2 row-lane and value-tile consumers) and the fused BS6 +
carry-halo kernel on emulated ranks."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200 import dist as D  # noqa: E402
from paper_2009_10917_b200.gs import bs6_gather_into, bs6_kernel_name  # noqa: E402
from paper_2009_10917_b200.mesh import build_slab_gather  # noqa: E402

which = sys.argv[1:] or ["tiled", "sweep", "halo"]
rng = np.random.default_rng(5)


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def q_of(n):
    return d(rng.uniform(-1, 1, n))


def run(op, q, carry=None):
    out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
    bs6_gather_into(op, q, out, carry)
    return float(out.sum())


if "tiled" in which:
    os.environ["SB200_BS6_TILED"] = "1"
    for K in (1, 2, 5, 33, 40):
        m = sb.build_mesh(K, 1)
        op = sb.build_gather(m)
        print("tiled", K, bs6_kernel_name(op, q_of(m.nl)), run(op, q_of(m.nl)), flush=True)
    part = D.SlabPartition(12, 1, 3)
    for r in range(3):
        z0, z1 = part.layers(r)
        c0, c1 = part.own_planes(r)
        op = build_slab_gather(12, 1, z0, z1, c0, c1)
        carry = q_of(part.plane) if r > 0 else None
        print("tiled slab", r, run(op, q_of(part.nl(r)), carry), flush=True)
    m = sb.build_mesh(9, 1)
    op = sb.build_gather(m)
    L = sb._lib.lib()
    perm = rng.permutation(m.nl).astype(np.int32)
    ci2 = d(perm[op.col_ids])
    out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
    q = q_of(m.nl)
    sb._lib.check(L.sb_bs6_gather_tiled(*op.geometry, op.row_starts_dev.data_ptr(), ci2.data_ptr(), op.ng, op.nl,
                                        q.data_ptr(), out.data_ptr(), None, 0, sb._lib.stream_handle()), "tiled")
    print("tiled permuted", float(out.sum()), flush=True)
    del os.environ["SB200_BS6_TILED"]

if "sweep" in which:
    os.environ["SB200_BS6_SWEEP"] = "1"
    for p in (1, 2):
        for K in (1, 3, 11, 17):
            m = sb.build_mesh(K, p)
            op = sb.build_gather(m)
            print("sweep", p, K, bs6_kernel_name(op, q_of(m.nl)), run(op, q_of(m.nl)), flush=True)
    os.environ["SB200_BS6_SWEEP_ROW2"] = "0"
    m = sb.build_mesh(11, 2)
    op = sb.build_gather(m)
    print("sweep p2 value tile", run(op, q_of(m.nl)), flush=True)
    del os.environ["SB200_BS6_SWEEP"], os.environ["SB200_BS6_SWEEP_ROW2"]

if "halo" in which:
    K, p, world = 8, 2, 3
    part = D.SlabPartition(K, p, world)
    own, send, outs = [], [], []
    for r in range(world):
        z0, z1 = part.layers(r)
        c0, c1 = part.own_planes(r)
        own.append(build_slab_gather(K, p, z0, z1, c0, c1))
        sp = part.send_plane(r)
        send.append(None if sp is None else build_slab_gather(K, p, z0, z1, sp, sp + 1))
        r0, r1 = part.row_span(r)
        outs.append(torch.empty(r1 - r0, dtype=torch.float64, device="cuda"))
    carry = [[torch.zeros(part.plane, dtype=torch.float64, device="cuda") for _ in (0, 1)] for _ in range(world)]
    sync = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]
    m = sb.build_mesh(K, p)
    for call in range(3):
        q = q_of(m.nl)
        for r in range(world):
            lo, hi = part.local_span(r)
            sendp = [t.data_ptr() for t in carry[r + 1]] if r + 1 < world else None
            carp = [t.data_ptr() for t in carry[r]] if r > 0 else None
            ready = sync[r + 1].data_ptr() if r + 1 < world else None
            ack = sync[r - 1].data_ptr() + 8 if r > 0 else None
            D.gather_halo_raw(send[r], own[r], q[lo:hi], outs[r].data_ptr(), sendp, carp,
                              part.plane if r > 0 else 0, sync[r].data_ptr(), ready, ack)
        print("halo call", call, sum(float(o.sum()) for o in outs), flush=True)
torch.cuda.synchronize()
print("done")
