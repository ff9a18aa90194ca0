"""TMA-staged BS6 (csrc/sb_gs_staged.cu) vs the oracle's row-wise gather
(oracle/sb_oracle.c, restating gs.py:10-39): bitwise, for the default tiles,
other tile shapes, slabs, carry-in, capacity overflow (direct tiles) and
columns outside the staged runs (global fallback)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def staged_on(monkeypatch):
    monkeypatch.setenv("SB200_BS6_STAGED", "1")  # the product default is the super-block kernel


@pytest.fixture(scope="module")
def sb():
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    _lib.lib()
    return sb


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def h(t):
    return t.cpu().numpy()


def staged_run(op, q, geo, tile=(0, 0, 0), carry=None, edit_info=None, edit_plan=None):
    """One sb_bs6_gather_staged call with an explicit tile / plan (bypassing the op cache)."""
    from paper_2009_10917_b200 import _lib
    L = _lib.lib()
    info = _lib.Bs6Staged()
    _lib.check(L.sb_bs6_staged_init(*geo, *tile, info), "init")
    if edit_info is not None:
        edit_info(info)
    plan = torch.empty(max(1, info.n_tiles * info.words_per_tile), dtype=torch.int32, device="cuda")
    _lib.check(L.sb_bs6_staged_make_plan(info, op.row_starts_dev.data_ptr(), plan.data_ptr(),
                                         _lib.stream_handle()), "plan")
    if edit_plan is not None:
        edit_plan(plan.view(-1, info.words_per_tile), info)
    out = torch.full((op.ng,), float("nan"), dtype=torch.float64, device="cuda")
    nc = 0 if carry is None else int(carry.shape[0])
    _lib.check(L.sb_bs6_gather_staged(info, plan.data_ptr(), op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(),
                                      op.ng, op.nl, q.data_ptr(), out.data_ptr(),
                                      None if carry is None else carry.data_ptr(), nc, _lib.stream_handle()),
               "gather")
    return out, info


def expect(oracle, op, q, carry=None):
    want = oracle.bs6_gather(h(op.row_starts_dev), h(op.col_ids_dev), h(q))
    if carry is not None:  # rows < len(carry) start from the carry instead of +0.0
        rs, ci, qq, c = h(op.row_starts_dev), h(op.col_ids_dev), h(q), h(carry)
        for r in range(c.shape[0]):
            acc = c[r]
            for j in range(rs[r], rs[r + 1]):
                acc = acc + qq[ci[j]]
            want[r] = acc
    return want


@pytest.mark.parametrize("K,p", [(1, 1), (2, 1), (3, 1), (5, 1), (16, 1), (45, 1),
                                 (1, 2), (2, 2), (3, 2), (7, 2), (30, 2)])
def test_staged_default_tiles_bitwise(sb, oracle, K, p):
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    assert op.staged() is not None
    q = d(np.random.default_rng([K, p, 61]).uniform(-1, 1, mesh.nl))
    out = sb.bs6_gather(op, q)
    assert np.array_equal(h(out), expect(oracle, op, q))


@pytest.mark.parametrize("p,tile", [(1, (1, 1, 8)), (1, (3, 3, 32)), (1, (2, 1, 64)), (1, (1, 2, 100)),
                                    (1, (2, 2, 1)), (2, (1, 1, 32)), (2, (2, 2, 32)), (2, (1, 2, 7)),
                                    (3, (1, 1, 32)), (4, (1, 1, 16))])
def test_staged_tile_shapes(sb, oracle, p, tile):
    K = 9
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng([K, p, 62]).uniform(-1, 1, mesh.nl))
    out, info = staged_run(op, q, (K, p, 0, K, 0, K * p + 1), tile)
    assert (info.ey, info.ez, info.w) == tile
    assert np.array_equal(h(out), expect(oracle, op, q))


@pytest.mark.parametrize("K,p,world", [(8, 1, 2), (9, 2, 3), (12, 1, 4)])
def test_staged_slabs_with_carry(sb, oracle, K, p, world):
    """Slab operators (dist.py partition) incl. the carry-seeded first plane."""
    from paper_2009_10917_b200.dist import SlabPartition
    from paper_2009_10917_b200.mesh import build_slab_gather
    part = SlabPartition(K, p, world)
    rng = np.random.default_rng([K, p, world])
    for rank in range(world):
        z0, z1 = part.layers(rank)
        c0, c1 = part.own_planes(rank)
        op = build_slab_gather(K, p, z0, z1, c0, c1)
        assert op.staged() is not None
        q = d(rng.uniform(-1, 1, part.nl(rank)))  # the slab's local DOFs (op.nl counts its entries)
        carry = d(rng.uniform(-1, 1, part.plane)) if rank > 0 else None
        out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
        from paper_2009_10917_b200.gs import bs6_gather_into
        bs6_gather_into(op, q, out, carry)
        assert np.array_equal(h(out), expect(oracle, op, q, carry)), rank


def test_staged_direct_tiles_when_caps_exceeded(sb, oracle):
    """A tile that does not fit the staging capacities is summed from global memory."""
    K, p = 11, 1
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng(63).uniform(-1, 1, mesh.nl))

    def shrink(info):
        info.q_cap = 64  # every interior tile overflows its q staging: the plan marks it direct
    out, _ = staged_run(op, q, (K, p, 0, K, 0, K * p + 1), edit_info=shrink)
    assert np.array_equal(h(out), expect(oracle, op, q))

    def flip(plan, info):  # a tile the plan stages but whose slices overflow the kernel's caps
        info.q_cap = 64
    out, _ = staged_run(op, q, (K, p, 0, K, 0, K * p + 1), edit_plan=flip)
    assert np.array_equal(h(out), expect(oracle, op, q))


def test_staged_columns_outside_runs(sb, oracle):
    """Runs removed from the plan: every entry takes the global-load fallback."""
    K, p = 10, 2
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng(64).uniform(-1, 1, mesh.nl))

    def drop_runs(plan, info):
        plan[:, 1] = 0
    out, _ = staged_run(op, q, (K, p, 0, K, 0, K * p + 1), edit_plan=drop_runs)
    assert np.array_equal(h(out), expect(oracle, op, q))

    def half_runs(plan, info):  # shorten every run: some entries staged, some not
        S, R = info.max_segments, info.max_runs
        o_ce = 9 + 7 * S + R  # table layout, csrc/sb_gs_staged.cu (hdr 8, koff S+1, 6 x S, cb R)
        ce = plan[:, o_ce:o_ce + R]
        ce -= 8 * (ce > 8).int()
    out, _ = staged_run(op, q, (K, p, 0, K, 0, K * p + 1), edit_plan=half_runs)
    assert np.array_equal(h(out), expect(oracle, op, q))


def test_staged_other_csr_same_rows(sb, oracle):
    """The plan only steers staging: a CSR with the same row structure but
    permuted columns still gives the row-wise result of ITS columns."""
    K, p = 6, 1
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    rng = np.random.default_rng(65)
    ci = h(op.col_ids_dev)
    perm = rng.permutation(ci.shape[0]).astype(np.int32)
    from paper_2009_10917_b200 import mesh as M
    op2 = M.GatherOp(ng=op.ng, row_starts=op.row_starts_dev, col_ids=d(perm[ci]), block_starts=op.block_starts_dev,
                     nodes_per_block=op.nodes_per_block, geometry=op.geometry)
    q = d(rng.uniform(-1, 1, mesh.nl))
    out = sb.bs6_gather(op2, q)
    assert np.array_equal(h(out), expect(oracle, op2, q))


def test_staged_unaligned_tails(sb, oracle):
    """Arrays whose lengths are not multiples of 16 B (odd NL at K=1..3, p=2)
    and a q view at an 8-byte offset (falls back to the super-block kernel)."""
    for K in (1, 3, 5):
        mesh = sb.build_mesh(K, 2)
        op = sb.build_gather(mesh)
        base = torch.from_numpy(np.random.default_rng([K, 66]).uniform(-1, 1, mesh.nl + 1)).cuda()
        for q in (base[:mesh.nl].clone(), base[1:]):
            out = sb.bs6_gather(op, q)
            assert np.array_equal(h(out), expect(oracle, op, q)), K


@pytest.mark.slow
@pytest.mark.parametrize("p", [1, 2])
def test_staged_c3_full_size(sb, oracle, p):
    """C3 (NG ~ 1e8) at N = 1 (K = 463, NL = 7.9e8) and N = 2: bitwise vs the OpenMP oracle."""
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    oracle.set_threads(oracle.max_threads())
    try:
        mesh = sb.build_mesh(K, p)
        op = sb.build_gather(mesh)
        del mesh
        assert op.staged() is not None
        gen = torch.Generator(device="cuda")
        gen.manual_seed(463 + p)
        q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        out = h(sb.bs6_gather(op, q))
        want = oracle.bs6_gather(h(op.row_starts_dev), h(op.col_ids_dev), h(q))
        assert np.array_equal(out, want)
    finally:
        oracle.set_threads(1)
