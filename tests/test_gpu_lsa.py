"""Fused BS3/BS4/BS5 + cross-rank combine over NVLink peer memory (lsa.py,
csrc/sb_lsa.cu).  One GPU per gpurun call, so this runs the one-rank team:
the kernel still stores into the (own) symmetric window through the LSA
mapping, passes the LSA barrier and sums the slots -- the result must equal
dist.DistReducer's rank-order sum (0.0 + v) bit for bit.  The multi-rank
ordering/epoch logic is covered by test_dist_gloo.py's reference semantics."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lsa():
    from paper_2009_10917_b200 import lsa as LSA
    try:
        r = LSA.LsaReducer(1, 0, "cuda:0", unique_id=LSA.LsaReducer.unique_id())
    except LSA.LsaUnavailable as e:  # pragma: no cover - depends on the box's NCCL
        pytest.fail(f"fused path unavailable: {e}")
    yield r
    r.close()


def _v(n, seed):
    return torch.from_numpy(np.random.default_rng(seed).uniform(-1, 1, n)).cuda()


@pytest.mark.parametrize("n", [0, 1, 4097, 1_000_003, 20_000_000])
def test_lsa_reductions_equal_plain(lsa, n):
    from paper_2009_10917_b200 import kernels as KN
    from paper_2009_10917_b200.kernels import ReductionConfig
    for cfg in (ReductionConfig(), ReductionConfig(64, 7), ReductionConfig(1024, 1184), ReductionConfig(2048, 3)):
        x, y, p, ap = (_v(n, s) for s in range(4))
        want3 = KN.bs3_norm2_async(x, cfg).item()
        want4 = KN.bs4_dot_async(x, y, cfg).item()
        assert lsa.bs3_norm2(x, cfg).item() == 0.0 + want3
        got4 = lsa.bs4_dot(x, y, cfg).item()
        assert got4 == 0.0 + want4 and np.signbit(got4) == np.signbit(0.0 + want4)
        x2, y2 = x.clone(), y.clone()
        want5 = KN.bs5_fused_cg_update_async(0.375, p, ap, x, y, cfg).item()
        got5 = lsa.bs5_fused_cg_update(0.375, p, ap, x2, y2, cfg).item()
        assert got5 == 0.0 + want5
        assert torch.equal(x2, x) and torch.equal(y2, y)


def test_lsa_many_calls_alternate_epochs(lsa):
    from paper_2009_10917_b200 import kernels as KN
    x = _v(300_001, 9)
    want = KN.bs3_norm2_async(x).item()
    outs = [lsa.bs3_norm2(x) for _ in range(9)]
    torch.cuda.synchronize()
    assert all(o.item() == want for o in outs)


def test_lsa_inside_cuda_graph_not_required_but_stream_ordered(lsa):
    """Back-to-back fused calls on one stream with no host sync in between."""
    from paper_2009_10917_b200 import kernels as KN
    xs = [_v(100_000 + i, 20 + i) for i in range(6)]
    res = [lsa.bs3_norm2(x) for x in xs]
    want = [KN.bs3_norm2_async(x).item() for x in xs]
    assert [r.item() for r in res] == want


@pytest.mark.parametrize("K,p,world", [(9, 5, 3), (8, 7, 2), (6, 1, 3)])
def test_carry_halo_through_lsa_window_bitexact(lsa, K, p, world):
    """The slab ranks run one after another on this GPU; each send-plane
    gather writes through the NVLink (LSA) mapping of the halo window (peer =
    self here), the barrier orders it, and the next rank's own gather reads
    the carry from the window: bitwise the single-GPU gather."""
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200.mesh import build_slab_gather
    part = D.SlabPartition(K, p, world)
    mesh = sb.build_mesh(K, p)
    gen = torch.Generator(device="cuda"); gen.manual_seed(K + 10 * p)
    q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
    full = sb.bs6_gather(sb.build_gather(mesh), q)
    if not hasattr(lsa, "_halo_ok"):
        lsa.halo_window(2 * 8 * 4_000_000)
        lsa._halo_ok = True
    nb = 8 * part.plane
    for r in range(world):
        z0, z1 = part.layers(r)
        lo, hi = part.local_span(r)
        c0, c1 = part.own_planes(r)
        e = r & 1
        carry_local, _ = lsa.halo_pointers(((r + 1) & 1) * nb, 0)   # written by rank r-1 (epoch of r-1)
        r0, r1 = part.row_span(r)
        out = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        D.gather_raw(build_slab_gather(K, p, z0, z1, c0, c1), q[lo:hi], out.data_ptr(),
                     carry_local if r > 0 else None, part.plane if r > 0 else 0)
        assert torch.equal(out, full[r0:r1]), r
        sp = part.send_plane(r)
        if sp is not None:
            _, remote = lsa.halo_pointers(e * nb, 0)
            D.gather_raw(build_slab_gather(K, p, z0, z1, sp, sp + 1), q[lo:hi], remote, None, 0)
            lsa.barrier()


@pytest.mark.parametrize("K,p,world", [(7, 3, 3), (6, 7, 2), (5, 1, 4)])
def test_bs7_halo_through_lsa_window_bitexact(lsa, K, p, world):
    """BS7 over slabs with the one-plane halo put through the LSA mapping of
    the halo window (peer = self) and the split scatter (own rows + halo)."""
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200.mesh import build_slab_l2g
    part = D.SlabPartition(K, p, world)
    mesh = sb.build_mesh(K, p)
    gen = torch.Generator(device="cuda"); gen.manual_seed(3 * K + p)
    qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
    want = qg[mesh.local_to_global_dev.long()]
    if not hasattr(lsa, "_halo_ok"):
        lsa.halo_window(2 * 8 * 4_000_000)
        lsa._halo_ok = True
    L = _lib.lib()
    st = _lib.stream_handle()
    plane = part.plane
    for r in range(world):
        z0, z1 = part.layers(r)
        lo, hi = part.local_span(r)
        a, b = part.read_span(r)
        ids = build_slab_l2g(K, p, z0, z1) - a
        ql = torch.zeros(hi - lo, dtype=torch.float64, device="cuda")
        if r < world - 1:
            own = part.ng_own(r)
            a1, _ = part.read_span(r + 1)
            loc, rem = lsa.halo_pointers((r & 1) * 8 * plane, 0)
            src = qg[a1:a1 + plane].clone()   # rank r+1's bottom plane
            _lib.check(L.sb_bs1_copy(src.data_ptr(), rem, plane, st), "put")
            lsa.barrier()
            win = qg[a:a + own].clone()
            _lib.check(L.sb_bs7_scatter_split(ids.data_ptr(), ids.shape[0], win.data_ptr(), own, loc, plane,
                                              ql.data_ptr(), 0, st), "split")
        else:
            win = qg[a:b].clone()
            _lib.check(L.sb_bs7_scatter(ids.data_ptr(), ids.shape[0], win.data_ptr(), win.shape[0],
                                        ql.data_ptr(), 0, st), "scatter")
        assert torch.equal(ql, want[lo:hi]), r


@pytest.mark.parametrize("K,p,world", [(6, 3, 3), (5, 1, 4)])
def test_bs7_halo_buffer_parity_on_device_under_graph_replay(lsa, K, p, world):
    """The BS7 halo's two buffers alternate on a call counter in device memory
    (sb_bs7_halo_put / sb_lsa_barrier_advance / sb_bs7_scatter_split_pair):
    emulated ranks on this GPU, one captured call replayed 5 times (an odd
    count per replay, which a host-side parity would freeze) -- every replay
    bitwise, the counters at the call count, and the buffer written last
    alternating."""
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200.mesh import build_slab_l2g
    part = D.SlabPartition(K, p, world)
    mesh = sb.build_mesh(K, p)
    if not hasattr(lsa, "_halo_ok"):
        lsa.halo_window(2 * 8 * 4_000_000)
        lsa._halo_ok = True
    L = _lib.lib()
    plane, nb = part.plane, 8 * part.plane
    stride = 2 * nb + 64
    base = 8 * 1_000_000  # clear of the other tests' halo buffers

    ptr = {}  # (halo_pointers is not capturable: resolve every address up front)
    for r in range(world):
        for off in (r * stride, r * stride + nb, r * stride + 2 * nb):
            ptr[off] = lsa.halo_pointers(base + off, 0)

    def loc(off):
        return ptr[off][0]

    def rem(off):
        return ptr[off][1]

    counters = [loc(r * stride + 2 * nb) for r in range(world)]
    for r in range(world):  # fresh counters (the window is shared with other tests)
        torch.cuda.synchronize()
        _lib.check(L.sb_bs1_copy(torch.zeros(1, dtype=torch.float64, device="cuda").data_ptr(), counters[r], 1,
                                 _lib.stream_handle()), "zero")
    qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
    ids, ql, own = [], [], []
    for r in range(world):
        z0, z1 = part.layers(r)
        lo, hi = part.local_span(r)
        a, b = part.read_span(r)
        ids.append(build_slab_l2g(K, p, z0, z1) - a)
        ql.append(torch.zeros(hi - lo, dtype=torch.float64, device="cuda"))
        own.append(torch.empty(part.ng_own(r) if r < world - 1 else b - a, dtype=torch.float64, device="cuda"))

    def call():
        st = _lib.stream_handle()
        for r in range(world):  # rank r's bottom plane -> rank r-1's halo buffer (rank r's parity)
            a, _ = part.read_span(r)
            own[r].copy_(qg[a:a + own[r].shape[0]])
            if r > 0:
                b0 = (r - 1) * stride
                _lib.check(L.sb_bs7_halo_put(own[r].data_ptr(), rem(b0), rem(b0 + nb), plane, counters[r], st),
                           "put")
        for r in range(world):
            lsa.barrier_advance(counters[r])
        for r in range(world):
            n = ids[r].shape[0]
            if r < world - 1:
                b0 = r * stride
                _lib.check(L.sb_bs7_scatter_split_pair(ids[r].data_ptr(), n, own[r].data_ptr(), own[r].shape[0],
                                                       loc(b0), loc(b0 + nb), plane, counters[r],
                                                       ql[r].data_ptr(), 0, st), "split pair")
            else:
                _lib.check(L.sb_bs7_scatter(ids[r].data_ptr(), n, own[r].data_ptr(), own[r].shape[0],
                                            ql[r].data_ptr(), 0, st), "scatter")

    gen = torch.Generator(device="cuda"); gen.manual_seed(K + p)
    qg.uniform_(-1, 1, generator=gen)
    call()  # eager call 0 (buffer 0)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        call()
    torch.cuda.current_stream().wait_stream(side)
    l2g = mesh.local_to_global_dev.long()
    for rep in range(5):
        qg.uniform_(-1, 1, generator=gen)
        g.replay()
        torch.cuda.synchronize()
        want = qg[l2g]
        for r in range(world):
            lo, hi = part.local_span(r)
            assert torch.equal(ql[r], want[lo:hi]), (rep, r)
        calls = rep + 2  # the eager call, the capture run none: replays only
        for r in range(world):
            cnt = torch.empty(1, dtype=torch.int64, device="cuda")
            _lib.check(L.sb_bs1_copy(counters[r], cnt.data_ptr(), 1, _lib.stream_handle()), "read")
            assert int(cnt.item()) == calls, (rep, r, int(cnt.item()))
        # the buffer the last put wrote holds rank 1's bottom plane, the other one an older plane
        a1, _ = part.read_span(1)
        last = torch.empty(plane, dtype=torch.float64, device="cuda")
        _lib.check(L.sb_bs1_copy(loc(((calls - 1) & 1) * nb), last.data_ptr(), plane, _lib.stream_handle()), "rd")
        torch.cuda.synchronize()
        assert torch.equal(last, qg[a1:a1 + plane]), rep


@pytest.mark.parametrize("fused,graph", [(True, False), (False, False), (True, True)])
def test_device_cg_with_fused_combine_one_rank(lsa, fused, graph):
    """cg_solve_device with the multi-GPU reductions (sb_lsa_cg_*) on a one-rank
    team reproduces the single-GPU device CG (and so the reference) bit for bit."""
    from paper_2009_10917_b200 import cg
    rng = np.random.default_rng(17)
    d = torch.from_numpy(rng.uniform(1, 50, 20_000)).cuda()
    b = torch.from_numpy(rng.uniform(-1, 1, 20_000)).cuda()
    A = cg.diagonal_operator(d)
    want = cg.cg_solve_device(A, b, torch.zeros_like(b), 1e-20, 300, fused=fused, relative=True)
    got = cg.cg_solve_device(A, b, torch.zeros_like(b), 1e-20, 300, fused=fused, relative=True,
                             check_every=8, graph=graph, lsa=lsa)
    assert got.iterations == want.iterations and got.final_rr == want.final_rr
    assert torch.equal(got.x, want.x)


def test_dist_mass_operator_and_cg_one_rank(lsa):
    """dist.DistMassOperator (BS7 + NVLink halo, weight, BS6 + NVLink carry) on a
    one-rank partition equals cg.gather_scatter_operator, and the fully
    device-resident CG through it (lsa-combined scalars) equals the
    single-GPU device CG bit for bit."""
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import cg
    from paper_2009_10917_b200 import dist as D
    from paper_2009_10917_b200 import lsa as LSA
    K, p = 5, 3
    mesh = sb.build_mesh(K, p)
    rng = np.random.default_rng(21)
    w = rng.uniform(1, 2, mesh.nl)
    A1 = cg.gather_scatter_operator(sb.build_gather(mesh), sb.build_scatter_ids(mesh), w)
    # a fresh context: the halo window is allocated once per context
    ctx = LSA.LsaReducer(1, 0, "cuda:0", unique_id=LSA.LsaReducer.unique_id())
    try:
        Ad = D.DistMassOperator(D.SlabPartition(K, p, 1), 0, "cuda:0", w, ctx)
        x = torch.from_numpy(rng.uniform(-1, 1, mesh.ng)).cuda()
        assert torch.equal(Ad(x), A1(x))
        b = torch.from_numpy(rng.uniform(-1, 1, mesh.ng)).cuda()
        want = cg.cg_solve_device(A1, b, torch.zeros_like(b), 1e-22, 500, relative=True)
        got = cg.cg_solve_device(Ad, b, torch.zeros_like(b), 1e-22, 500, relative=True, lsa=ctx, check_every=8)
        assert got.iterations == want.iterations and torch.equal(got.x, want.x)
        # captured iterations, an odd number per replay (every halo parity is device-side)
        got = cg.cg_solve_device(Ad, b, torch.zeros_like(b), 1e-22, 500, relative=True, lsa=ctx, check_every=7,
                                 graph=True)
        assert got.iterations == want.iterations and torch.equal(got.x, want.x)
    finally:
        ctx.close()


def test_abort_is_local_and_leaves_the_device_usable():
    """LsaReducer.abort (the fallback when peers disagree) tears a context
    down without collective calls; a fresh context then works normally."""
    from paper_2009_10917_b200 import lsa as LSA
    r = LSA.LsaReducer(1, 0, "cuda:0", unique_id=LSA.LsaReducer.unique_id())
    r.abort()
    assert r.handle is None
    r2 = LSA.LsaReducer(1, 0, "cuda:0", unique_id=LSA.LsaReducer.unique_id())
    x = _v(4097, 21)
    import paper_2009_10917_b200 as sb
    assert r2.bs3_norm2(x) == 0.0 + sb.bs3_norm2(x)
    r2.close()


def test_lsa_parity_is_device_side_across_graph_replays(lsa):
    """An odd number of fused reductions captured in a CUDA graph: the slot
    parity comes from the window's call counter, so replays keep alternating
    and every result still equals the plain rank-order sum."""
    import paper_2009_10917_b200 as sb
    x = _v(100_003, 5)
    want = 0.0 + sb.bs3_norm2(x)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    lsa.bs3_norm2(x, out=out)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(3):
            lsa.bs3_norm2(x, out=out)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert float(out.item()) == want
