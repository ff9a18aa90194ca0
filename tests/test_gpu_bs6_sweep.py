"""z-sweep BS6 (csrc/sb_gs_sweep.cu, the p <= 2 fast path) vs the oracle's
row-wise gather (oracle/sb_oracle.c, restating gs.py:10-39): bitwise on whole
meshes, slabs with carry-in, CSRs whose columns leave the staged runs
(global fallback), long / empty rows (direct warp-steps), odd-length tails,
every ring depth and prefetch setting, and C3's full size at N = 1 and 2."""

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


@pytest.fixture(autouse=True)
def sweep_on(monkeypatch):
    monkeypatch.setenv("SB200_BS6_SWEEP", "1")  # opt-in while slower than the super-block kernel


@pytest.fixture
def tune(sb):
    from paper_2009_10917_b200 import _lib
    L = _lib.lib()

    def set_(slots=0, pfd=-1, waves=0, swz=-1, h=0):
        _lib.check(L.sb_bs6_sweep_tune(slots, pfd, waves, swz, h), "tune")
    yield set_
    set_()


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def h(t):
    return t.cpu().numpy()


def sweep(geo, rs, ci, ng, nl, q, carry=None):
    """One direct sb_bs6_gather_sweep call."""
    from paper_2009_10917_b200 import _lib
    L = _lib.lib()
    out = torch.full((ng,), float("nan"), dtype=torch.float64, device="cuda")
    nc = 0 if carry is None else int(carry.shape[0])
    _lib.check(L.sb_bs6_gather_sweep(*geo, rs.data_ptr(), ci.data_ptr(), ng, nl, q.data_ptr(), out.data_ptr(),
                                     None if carry is None else carry.data_ptr(), nc, _lib.stream_handle()),
               "sweep")
    return out


def expect(oracle, rs, ci, q, carry=None):
    want = oracle.bs6_gather(h(rs), h(ci), h(q))
    if carry is not None:  # rows < len(carry) start from the carry instead of +0.0
        rs_, ci_, qq, c = h(rs), h(ci), h(q), h(carry)
        for r in range(c.shape[0]):
            acc = c[r]
            for j in range(rs_[r], rs_[r + 1]):
                acc = acc + qq[ci_[j]]
            want[r] = acc
    return want


@pytest.mark.parametrize("K,p", [(1, 1), (2, 1), (3, 1), (5, 1), (16, 1), (33, 1), (45, 1),
                                 (1, 2), (2, 2), (3, 2), (7, 2), (16, 2), (30, 2)])
def test_sweep_whole_mesh_bitwise(sb, oracle, K, p):
    from paper_2009_10917_b200.gs import sweep_geometry
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng([K, p, 71]).uniform(-1, 1, mesh.nl))
    assert sweep_geometry(op, q) == (K, p, 0, K, 0, K * p + 1)  # the public call takes the sweep
    out = sb.bs6_gather(op, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q))


@pytest.mark.parametrize("K", [1, 2, 5, 11, 16, 31])
def test_sweep_p2_value_tile_consumer(sb, oracle, monkeypatch, K):
    """p = 2 through the p = 1 (value-tile) consumer instead of the default
    row-lane one (SB200_BS6_SWEEP_ROW2=0): same bits."""
    monkeypatch.setenv("SB200_BS6_SWEEP_ROW2", "0")
    mesh = sb.build_mesh(K, 2)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng([K, 77]).uniform(-1, 1, mesh.nl))
    out = sweep(op.geometry, op.row_starts_dev, op.col_ids_dev, op.ng, op.nl, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q))


@pytest.mark.parametrize("slots,pfd,waves,swz,rows", [(3, 0, 1, -1, 0), (3, 4, 64, 0, 7), (5, 1, 2, 1, 16),
                                                   (8, 16, 8, -1, 8), (4, 0, 1000, 1, 7), (3, 2, 3, -1, 16)])
@pytest.mark.parametrize("K,p", [(13, 1), (11, 2), (34, 1)])
def test_sweep_ring_and_prefetch_settings(sb, oracle, tune, K, p, slots, pfd, waves, swz, rows):
    tune(slots, pfd, waves, swz, rows)
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng([K, p, 72]).uniform(-1, 1, mesh.nl))
    out = sweep(op.geometry, op.row_starts_dev, op.col_ids_dev, op.ng, op.nl, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q))


@pytest.mark.parametrize("K,p,world", [(8, 1, 2), (9, 2, 3), (12, 1, 4), (40, 1, 3), (21, 2, 2)])
def test_sweep_slabs_with_carry(sb, oracle, K, p, world):
    """Slab operators (dist.py partition), incl. the carry-seeded first plane
    and the one-plane send operators."""
    from paper_2009_10917_b200.dist import SlabPartition
    from paper_2009_10917_b200.gs import bs6_gather_into, sweep_geometry
    from paper_2009_10917_b200.mesh import build_slab_gather
    part = SlabPartition(K, p, world)
    rng = np.random.default_rng([K, p, world, 73])
    for rank in range(world):
        z0, z1 = part.layers(rank)
        c0, c1 = part.own_planes(rank)
        q = d(rng.uniform(-1, 1, part.nl(rank)))
        ops = [build_slab_gather(K, p, z0, z1, c0, c1)]
        if part.send_plane(rank) is not None:
            sp = part.send_plane(rank)
            ops.append(build_slab_gather(K, p, z0, z1, sp, sp + 1))
        for op in ops:
            assert sweep_geometry(op, q) is not None
            carry = d(rng.uniform(-1, 1, part.plane)) if rank > 0 and op is ops[0] else None
            out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
            bs6_gather_into(op, q, out, carry)
            assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q, carry)), rank


def test_sweep_other_csr_same_rows(sb, oracle):
    """The geometry only steers staging: permuted columns (almost all outside
    the runs) still give the row-wise result of THEIR columns."""
    K, p = 9, 1
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    rng = np.random.default_rng(74)
    ci = h(op.col_ids_dev)
    perm = rng.permutation(ci.shape[0]).astype(np.int32)
    q = d(rng.uniform(-1, 1, mesh.nl))
    ci2 = d(perm[ci])
    out = sweep(op.geometry, op.row_starts_dev, ci2, op.ng, op.nl, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, ci2, q))


@pytest.mark.parametrize("p", [1, 2])
def test_sweep_long_and_empty_rows(sb, oracle, p):
    """Row lengths 0..40 with random columns: warp-steps above 256 entries sum
    from global memory, empty rows give +0.0 (or the carry)."""
    K = 6
    g = K * p + 1
    ng, nl = g ** 3, K ** 3 * (p + 1) ** 3
    rng = np.random.default_rng([p, 75])
    lens = rng.integers(0, 41, ng)
    short = rng.random(ng) < 0.6
    lens[short] = rng.integers(0, 9, int(short.sum()))
    rs = np.zeros(ng + 1, dtype=np.int32)
    rs[1:] = np.cumsum(lens)
    ci = rng.integers(0, nl, int(rs[-1])).astype(np.int32)
    q = d(rng.uniform(-1, 1, nl))
    carry = d(rng.uniform(-1, 1, g * g + 5))
    for c in (None, carry):
        out = sweep((K, p, 0, K, 0, g), d(rs), d(ci), ng, nl, q, c)
        assert np.array_equal(h(out), expect(oracle, d(rs), d(ci), q, c))


def test_sweep_odd_tails_and_offset_views(sb, oracle):
    """Odd NL (p = 2, odd K: the last run ends past the last 16 B unit) and a q
    view at an 8-byte offset (the public call falls back to the super-block
    kernel; the C entry point rejects it)."""
    from paper_2009_10917_b200 import _lib
    from paper_2009_10917_b200.gs import sweep_geometry
    for K in (1, 3, 5, 9):
        mesh = sb.build_mesh(K, 2)
        op = sb.build_gather(mesh)
        assert mesh.nl % 2 == 1
        base = torch.from_numpy(np.random.default_rng([K, 76]).uniform(-1, 1, mesh.nl + 1)).cuda()
        for q in (base[:mesh.nl].clone(), base[1:]):
            out = sb.bs6_gather(op, q)
            assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q)), K
        assert sweep_geometry(op, base[1:]) is None
        with pytest.raises(ValueError):
            sweep(op.geometry, op.row_starts_dev, op.col_ids_dev, op.ng, op.nl, base[1:])


def test_sweep_rejects_bad_geometry(sb):
    from paper_2009_10917_b200 import _lib
    mesh = sb.build_mesh(4, 1)
    op = sb.build_gather(mesh)
    q = torch.zeros(mesh.nl, dtype=torch.float64, device="cuda")
    for geo, ng, nl in [((4, 3, 0, 4, 0, 13), op.ng, op.nl),       # p > 2
                        ((4, 1, 0, 4, 0, 5), op.ng - 1, op.nl),     # ng mismatch
                        ((4, 1, 0, 4, 0, 5), op.ng, op.nl + 8),     # nl mismatch
                        ((4, 1, 2, 2, 0, 5), op.ng, op.nl),         # empty slab
                        ((4, 1, 0, 4, 3, 6), op.ng, op.nl)]:        # planes past the mesh
        with pytest.raises(ValueError):
            sweep(geo, op.row_starts_dev, op.col_ids_dev, ng, nl, q)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().sb_bs6_sweep_tune(2, -1, 0, -1, 0), "tune")


@pytest.mark.slow
@pytest.mark.parametrize("p", [1, 2])
def test_sweep_c3_full_size(sb, oracle, p):
    """C3 (NG ~ 1e8) at N = 1 (K = 463, NL = 7.9e8) and N = 2 (K = 232):
    the public call (sweep kernel) bitwise vs the OpenMP oracle."""
    from paper_2009_10917_b200.gs import sweep_geometry
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    oracle.set_threads(oracle.max_threads())
    try:
        mesh = sb.build_mesh(K, p)
        op = sb.build_gather(mesh)
        del mesh
        gen = torch.Generator(device="cuda")
        gen.manual_seed(4630 + p)
        q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        assert sweep_geometry(op, q) is not None
        out = h(sb.bs6_gather(op, q))
        want = oracle.bs6_gather(h(op.row_starts_dev), h(op.col_ids_dev), h(q))
        assert np.array_equal(out, want)
    finally:
        oracle.set_threads(1)
