"""BS6 + the multi-GPU carry halo in ONE launch (sb_bs6_gather_halo, SURVEY
8(f) row 3).  One GPU per gpurun call, so the slab ranks run one after
another on it: each rank's send partials go into the next rank's carry
buffer, flags in device memory order the hand-off (ready / ack / the
device-side call count), and every rank's rows must equal the single-GPU
gather bit for bit -- over several calls (both carry buffers, the ack wait
from the third call on), inside a CUDA graph replayed with new inputs, and
through the NVLink (LSA) mapping of a symmetric window."""

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


class Ranks:
    """Per-rank slab operators and halo state on one GPU (plain device buffers)."""

    def __init__(self, K, p, world):
        from paper_2009_10917_b200 import dist as D
        from paper_2009_10917_b200.mesh import build_slab_gather
        self.part = D.SlabPartition(K, p, world)
        self.world, self.K, self.p = world, K, p
        plane = self.part.plane
        self.own, self.send, self.out = [], [], []
        for r in range(world):
            z0, z1 = self.part.layers(r)
            c0, c1 = self.part.own_planes(r)
            self.own.append(build_slab_gather(K, p, z0, z1, c0, c1))
            sp = self.part.send_plane(r)
            self.send.append(None if sp is None else build_slab_gather(K, p, z0, z1, sp, sp + 1))
            r0, r1 = self.part.row_span(r)
            self.out.append(torch.full((r1 - r0,), float("nan"), dtype=torch.float64, device="cuda"))
        self.carry = [[torch.full((plane,), float("nan"), dtype=torch.float64, device="cuda") for _ in (0, 1)]
                      for _ in range(world)]
        self.sync = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]

    def ptrs(self, r):
        """(send buffers, carry buffers, sync, peer_ready, peer_ack) addresses of rank r."""
        send = [t.data_ptr() for t in self.carry[r + 1]] if r + 1 < self.world else None
        carry = [t.data_ptr() for t in self.carry[r]] if r > 0 else None
        ready = self.sync[r + 1].data_ptr() if r + 1 < self.world else None
        ack = self.sync[r - 1].data_ptr() + 8 if r > 0 else None
        return send, carry, self.sync[r].data_ptr(), ready, ack

    def call(self, q):
        from paper_2009_10917_b200 import dist as D
        for r in range(self.world):
            lo, hi = self.part.local_span(r)
            send, carry, sync, ready, ack = self.ptrs(r)
            D.gather_halo_raw(self.send[r], self.own[r], q[lo:hi], self.out[r].data_ptr(), send, carry,
                              self.part.plane if r > 0 else 0, sync, ready, ack)

    def check(self, full):
        for r in range(self.world):
            r0, r1 = self.part.row_span(r)
            assert torch.equal(self.out[r], full[r0:r1]), r


def _q(n, seed):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    return torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)


@pytest.mark.parametrize("K,p,world", [(6, 1, 2), (9, 2, 3), (8, 7, 2), (12, 3, 4), (10, 1, 5), (7, 5, 7)])
def test_fused_halo_emulated_ranks_bitexact(sb, K, p, world):
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    R = Ranks(K, p, world)
    for call in range(5):  # epochs 0..4: both carry buffers, ack waits from call 2 on
        q = _q(mesh.nl, 100 * K + call)
        R.call(q)
        R.check(sb.bs6_gather(op, q))
    for r in range(world):
        s = R.sync[r].tolist()
        assert s[2] == 5 and s[3] == 0 and s[4] == 0, (r, s)      # call count, counters reset
        assert s[0] == (5 if r > 0 else 0) and s[1] == (5 if r < world - 1 else 0), (r, s)


def test_fused_halo_inside_cuda_graph(sb):
    """The call parity lives in device memory: replays of one captured chain
    alternate the carry buffers correctly (the host-side epoch of the r01 path
    was frozen into a graph)."""
    K, p, world = 8, 2, 3
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    R = Ranks(K, p, world)
    q = _q(mesh.nl, 7)
    R.call(q)  # builds the plans (host syncs) before capture
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        R.call(q)
    torch.cuda.current_stream().wait_stream(side)
    for rep in range(4):
        q.copy_(_q(mesh.nl, 50 + rep))
        g.replay()
        torch.cuda.synchronize()
        R.check(sb.bs6_gather(op, q))
    assert all(int(R.sync[r][2]) == 5 for r in range(world))


@pytest.mark.parametrize("K,p,world", [(6, 1, 3), (8, 7, 2)])
def test_fused_halo_through_lsa_window(sb, K, p, world):
    """The ranks' carry buffers and sync words in ONE symmetric window of a
    one-rank LSA team; every store into a 'peer' goes through the NVLink (LSA)
    mapping of the window, every load through the local address."""
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200 import lsa as LSA
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    R = Ranks(K, p, world)
    nb = 8 * R.part.plane
    stride = 2 * nb + 64
    ctx = LSA.LsaReducer(1, 0, "cuda:0", unique_id=LSA.LsaReducer.unique_id())
    try:
        ctx.halo_window(world * stride)

        def loc(off):
            return ctx.halo_pointers(off, 0)[0]

        def rem(off):
            return ctx.halo_pointers(off, 0)[1]

        for call in range(4):
            q = _q(mesh.nl, 900 + call)
            for r in range(world):
                lo, hi = R.part.local_span(r)
                b = r * stride
                send = [rem((r + 1) * stride + e * nb) for e in (0, 1)] if r + 1 < world else None
                carry = [loc(b + e * nb) for e in (0, 1)] if r > 0 else None
                ready = rem((r + 1) * stride + 2 * nb) if r + 1 < world else None
                ack = rem((r - 1) * stride + 2 * nb + 8) if r > 0 else None
                D.gather_halo_raw(R.send[r], R.own[r], q[lo:hi], R.out[r].data_ptr(), send, carry,
                                  R.part.plane if r > 0 else 0, loc(b + 2 * nb), ready, ack)
            R.check(sb.bs6_gather(op, q))
    finally:
        ctx.close()


def test_fused_halo_rejects_bad_arguments(sb):
    from paper_2009_10917_b200 import _lib
    from paper_2009_10917_b200 import dist as D
    R = Ranks(6, 2, 2)
    q = _q(R.part.nl(1), 3)
    send, carry, sync, ready, ack = R.ptrs(1)
    with pytest.raises(ValueError):  # a carry without buffers
        D.gather_halo_raw(None, R.own[1], q, R.out[1].data_ptr(), None, None, 5, sync, None, ack)
    with pytest.raises(ValueError):  # peer_ready without a send operator
        D.gather_halo_raw(None, R.own[1], q, R.out[1].data_ptr(), None, carry, R.part.plane, sync,
                          R.sync[0].data_ptr(), ack)
    _ = _lib
