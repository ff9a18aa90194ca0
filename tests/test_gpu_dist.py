"""dist.py building blocks on one GPU: slab operators, the carry composition run
rank by rank, the BS7 halo window, and the NCCL calls on a 1-rank group."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    _lib.lib()
    return sb


@pytest.mark.parametrize("K,p,world", [(9, 5, 3), (8, 7, 8), (6, 2, 2), (11, 1, 4)])
def test_sequential_ranks_bitexact(sb, K, p, world):
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200.gs import bs6_gather_into
    from paper_2009_10917_b200.mesh import build_slab_gather, build_slab_l2g
    part = D.SlabPartition(K, p, world)
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    gen = torch.Generator(device="cuda"); gen.manual_seed(K * 100 + p)
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
    qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
    full = sb.bs6_gather(op, q)
    carry = None
    for r in range(world):
        z0, z1 = part.layers(r)
        lo, hi = part.local_span(r)
        c0, c1 = part.own_planes(r)
        own = build_slab_gather(K, p, z0, z1, c0, c1)
        r0, r1 = part.row_span(r)
        out = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        bs6_gather_into(own, q[lo:hi], out, carry)
        assert torch.equal(out, full[r0:r1]), r
        sp = part.send_plane(r)
        if sp is not None:
            send = build_slab_gather(K, p, z0, z1, sp, sp + 1)
            carry = torch.empty(part.plane, dtype=torch.float64, device="cuda")
            bs6_gather_into(send, q[lo:hi], carry, None)
        # BS7 over the rank's read window
        a, b = part.read_span(r)
        l2g = build_slab_l2g(K, p, z0, z1)
        assert torch.equal(l2g, mesh.local_to_global_dev[lo:hi])
        ids = l2g - a
        ql = torch.zeros(hi - lo, dtype=torch.float64, device="cuda")
        D._gpu_scatter(ids, qg[a:b].clone(), ql)
        assert torch.equal(ql, qg[mesh.local_to_global_dev[lo:hi].long()])


def test_nccl_one_rank_group(sb):
    import torch.distributed as dist
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200 import kernels as KN
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        x = torch.empty(3_000_001, dtype=torch.float64, device=dev).uniform_(-1, 1)
        red = D.DistReducer(1, dev)
        got = float(red.combine(KN.bs3_norm2_async(x))[0])
        assert got == sb.bs3_norm2(x)  # +0.0 + v == v
        part = D.SlabPartition(5, 3, 1)
        g = D.DistGather.build(part, 0, dev)
        mesh = sb.build_mesh(5, 3)
        q = torch.empty(mesh.nl, dtype=torch.float64, device=dev).uniform_(-1, 1)
        out = torch.empty(mesh.ng, dtype=torch.float64, device=dev)
        g.gather(q, out)
        assert torch.equal(out, sb.bs6_gather(sb.build_gather(mesh), q))
        sc = D.DistScatter.build(part, 0, dev)
        sc.window.uniform_(-1, 1)
        ql = torch.zeros(mesh.nl, dtype=torch.float64, device=dev)
        sc.scatter(ql)
        assert torch.equal(ql, sc.window[mesh.local_to_global_dev.long()])
    finally:
        dist.destroy_process_group()


def test_bench_context_fused_combine_one_rank(sb):
    """BenchContext on a 1-rank NCCL group picks the fused in-kernel combine
    (lsa.py) and its BS3/BS4/BS5 results equal the all-gather path's."""
    import types
    import torch.distributed as dist
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200 import kernels as KN
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        args = types.SimpleNamespace(K=6, order=3)
        ctx = D.BenchContext(0, 1, args, dev, use_lsa=True)  # (bench default: NCCL collectives)
        assert ctx.lsa is not None, ctx.collective
        cfg = KN.ReductionConfig()
        x, y, p, ap, r = (torch.empty(2_000_003, dtype=torch.float64, device=dev).uniform_(-1, 1)
                          for _ in range(5))
        w = types.SimpleNamespace(x=x, y=y, p=p, ap=ap, r=r, cfg=cfg,
                                  res=torch.empty(1, dtype=torch.float64, device=dev), sb=sb)
        ctx.call(w, "bs3")
        assert w.res.item() == KN.bs3_norm2_async(x, cfg).item()
        ctx.call(w, "bs4")
        assert w.res.item() == 0.0 + KN.bs4_dot_async(x, y, cfg).item()
        x0, r0 = x.clone(), r.clone()
        ctx.call(w, "bs5")
        got = w.res.item()
        want = KN.bs5_fused_cg_update_async(1e-3, p, ap, x0, r0, cfg).item()
        assert got == want and torch.equal(x, x0) and torch.equal(r, r0)
        ctx.lsa.close()
    finally:
        dist.destroy_process_group()
