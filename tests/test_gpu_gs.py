"""BS6/BS7 and the operator builders on the B200 vs the reference's golden
arrays (bitwise) and the CPU oracle."""

import numpy as np
import pytest
import torch

from goldens import mesh_q_global, mesh_q_local, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    _lib.lib()
    return sb


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def h(t):
    return t.cpu().numpy()


def test_builders_and_kernels_vs_golden(sb, golden):
    for rec in golden["meshes"]:
        K, p, npb = rec["K"], rec["p"], rec["npb"]
        mesh = sb.build_mesh(K, p)
        assert mesh.nl == rec["nl"] and mesh.ng == rec["ng"]
        assert sha(h(mesh.local_to_global_dev)) == rec["l2g"], (K, p)
        op = sb.build_gather(mesh, npb)
        assert sha(h(op.row_starts_dev)) == rec["row_starts"], (K, p)
        assert sha(h(op.col_ids_dev)) == rec["col_ids"], (K, p)
        assert sha(h(op.block_starts_dev)) == rec["block_starts"], (K, p, npb)
        assert op.n_blocks == rec["n_blocks"]
        q = mesh_q_local(K, p, mesh.nl)
        out = sb.bs6_gather(op, d(q))
        assert sha(h(out)) == rec["bs6_out"], (K, p)
        ids = sb.build_scatter_ids(mesh)
        assert not ids.has_mask
        qg = mesh_q_global(K, p, mesh.ng)
        ql = torch.zeros(mesh.nl, dtype=torch.float64, device="cuda")
        sb.bs7_scatter(ids, d(qg), ql)
        assert sha(h(ql)) == rec["bs7_out"], (K, p)
        assert sha((sb.multiplicity(mesh))) == rec["mult"]
        assert sb.bytes_moved("bs6", nl=mesh.nl, ng=mesh.ng) == rec["bytes_bs6"]


def test_general_builder_path_matches(sb, golden):
    """A user-supplied l2g (not flagged structured) goes through the CUB path."""
    for rec in golden["meshes"][:12]:
        K, p, npb = rec["K"], rec["p"], rec["npb"]
        m = sb.build_mesh(K, p)
        mu = sb.MeshConnectivity(K=K, p=p, local_to_global=m.local_to_global_dev.clone())
        op = sb.build_gather(mu, npb)
        assert sha(h(op.row_starts_dev)) == rec["row_starts"]
        assert sha(h(op.col_ids_dev)) == rec["col_ids"]
        assert sha(h(op.block_starts_dev)) == rec["block_starts"]
        assert sha((sb.multiplicity(mu))) == rec["mult"]


def test_general_builder_random_map(sb, oracle):
    rng = np.random.default_rng(7)
    ng = 5000
    l2g = np.concatenate([np.arange(ng), rng.integers(0, ng, 20000)]).astype(np.int32)
    rng.shuffle(l2g)
    l2g_d = torch.from_numpy(l2g).cuda()
    from paper_2009_10917_b200 import mesh as M
    rs = torch.empty(ng + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(l2g.shape[0], dtype=torch.int32, device="cuda")
    from paper_2009_10917_b200 import _lib
    L = _lib.lib()
    tmp = torch.empty(int(L.sb_build_gather_general_temp_bytes(l2g.shape[0])), dtype=torch.uint8,
                      device="cuda")
    stats = torch.empty(2, dtype=torch.int64, device="cuda")
    _lib.check(L.sb_build_gather_general(l2g_d.data_ptr(), l2g.shape[0], ng,
                                         rs.data_ptr(), ci.data_ptr(), tmp.data_ptr(),
                                         tmp.shape[0], stats.data_ptr(),
                                         _lib.stream_handle()), "general")
    rs_o, ci_o, bst_o = oracle.build_gather(l2g, ng, 64)
    assert np.array_equal(h(rs), rs_o) and np.array_equal(h(ci), ci_o)
    assert np.array_equal(h(M._block_starts(rs, ng, 64)), bst_o)


def test_masks_vs_golden(sb, golden):
    for rec in golden["masks"]:
        K, p = rec["K"], rec["p"]
        mesh = sb.build_mesh(K, p)
        ids = sb.build_scatter_ids(mesh, mask=set(rec["mask"]))
        assert sha(h(ids.ids_dev)) == rec["ids"]
        assert ids.has_mask == rec["has_mask"]
        qg = np.random.default_rng([9, K, p]).uniform(-1, 1, mesh.ng)
        ql = torch.full((mesh.nl,), 99.0, dtype=torch.float64, device="cuda")
        sb.bs7_scatter(ids, d(qg), ql)
        assert sha(h(ql)) == rec["out"]


def test_gs_errors_and_identities(sb):
    mesh = sb.build_mesh(1, 1)
    op = sb.build_gather(mesh)
    q = d(np.arange(8.0))
    assert torch.equal(sb.bs6_gather(op, q), q)  # test_gs.py:23-26
    with pytest.raises(ValueError):
        sb.bs6_gather(op, d(np.zeros(9)))
    ids = sb.build_scatter_ids(mesh)
    with pytest.raises(ValueError):
        sb.bs7_scatter(ids, d(np.zeros(8)), d(np.zeros(9)))
    with pytest.raises(ValueError):
        sb.bs7_scatter(ids, d(np.zeros(4)), d(np.zeros(8)))
    with pytest.raises(ValueError):
        sb.build_gather(sb.build_mesh(2, 1), 7)  # test_mesh.py:173-176
    with pytest.raises(ValueError):
        sb.build_mesh(200, 7)
    with pytest.raises(ValueError):
        sb.build_mesh(0, 1)
    with pytest.raises(ValueError):
        sb.build_scatter_ids(mesh, mask={8})
    m = sb.build_mesh(2, 2)
    full = sb.build_scatter_ids(m, mask=set(range(m.ng)))
    assert bool((full.ids_dev == -1).all())
    ql = d(np.random.default_rng(3).uniform(-1, 1, m.nl))
    before = ql.clone()
    sb.bs7_scatter(full, d(np.ones(m.ng)), ql)
    assert torch.equal(ql, before)


@pytest.mark.parametrize("K,p", [(1, 1), (2, 1), (3, 2), (4, 3), (2, 7), (3, 15)])
def test_round_trip_and_linearity(sb, K, p):
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    ids = sb.build_scatter_ids(mesh)
    qg = d(np.random.default_rng([K, p]).uniform(-1, 1, mesh.ng))
    ql = torch.zeros(mesh.nl, dtype=torch.float64, device="cuda")
    sb.bs7_scatter(ids, qg, ql)
    m = sb.mesh.multiplicity_dev(mesh)
    assert torch.allclose(sb.bs6_gather(op, ql), m * qg, rtol=1e-13, atol=0)
    u = d(np.random.default_rng(3).uniform(-1, 1, mesh.nl))
    v = d(np.random.default_rng(4).uniform(-1, 1, mesh.nl))
    comb = sb.bs6_gather(op, 2.5 * u - 0.75 * v)
    sep = 2.5 * sb.bs6_gather(op, u) - 0.75 * sb.bs6_gather(op, v)
    assert torch.allclose(comb, sep, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("K,p,npb", [(40, 7, 512), (20, 3, 16), (12, 15, 4096), (30, 1, 8)])
def test_builders_vs_oracle_larger(sb, oracle, K, p, npb):
    mesh = sb.build_mesh(K, p)
    l2g = oracle.build_mesh(K, p)
    assert np.array_equal(h(mesh.local_to_global_dev), l2g)
    op = sb.build_gather(mesh, npb)
    rs, ci, bst = oracle.build_gather(l2g, mesh.ng, npb)
    assert np.array_equal(h(op.row_starts_dev), rs)
    assert np.array_equal(h(op.col_ids_dev), ci)
    assert np.array_equal(h(op.block_starts_dev), bst)
    q = np.random.default_rng([K, p]).uniform(-1, 1, mesh.nl)
    assert np.array_equal(h(sb.bs6_gather(op, d(q))), oracle.bs6_gather(rs, ci, q))


def test_c3_scale_bs6_bs7(sb, oracle):
    """C3 at N=7 (K=66, NG ~ 1e8): bitwise vs the row-wise oracle."""
    K, p = 66, 7
    oracle.set_threads(oracle.max_threads())
    try:
        mesh = sb.build_mesh(K, p)
        op = sb.build_gather(mesh)
        gen = torch.Generator(device="cuda"); gen.manual_seed(66)
        q = torch.empty(mesh.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        out = sb.bs6_gather(op, q)
        want = oracle.bs6_gather(h(op.row_starts_dev), h(op.col_ids_dev), h(q))
        assert np.array_equal(h(out), want)
        ids = sb.build_scatter_ids(mesh)
        qg = torch.empty(mesh.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        ql = torch.zeros(mesh.nl, dtype=torch.float64, device="cuda")
        sb.bs7_scatter(ids, qg, ql)
        assert torch.equal(ql, qg[mesh.local_to_global_dev.long()])
    finally:
        oracle.set_threads(1)


def test_reference_numpy_operator_drop_in(sb, golden):
    """The reference's numpy GatherOp-like objects are accepted (staged per call)."""
    import types
    arr = golden.arrays
    tag = "3_2_64"
    op = types.SimpleNamespace(ng=7 ** 3, row_starts=arr[f"rs_{tag}"], col_ids=arr[f"ci_{tag}"],
                               block_starts=arr[f"bst_{tag}"], nodes_per_block=64,
                               nl=arr[f"ci_{tag}"].shape[0])
    q = mesh_q_local(3, 2, op.nl)
    out = sb.bs6_gather(op, q)
    assert isinstance(out, np.ndarray)
    assert np.array_equal(out, arr[f"bs6_{tag}"])


@pytest.mark.parametrize("K,p,npb", [(20, 7, 512), (13, 2, 16), (7, 15, 2048), (25, 1, 64), (3, 3, 8),
                                     (80, 1, 512), (79, 1, 512), (64, 1, 256)])
def test_pipelined_bs6_matches_unplanned(sb, K, p, npb):
    """sb_bs6_gather_planned (persistent, cp.async pipeline) == sb_bs6_gather, with carry.
    The p = 1 meshes from K = 64 on take the 1024-entry (two plan
    super-blocks) kernel, odd and even plan lengths included."""
    import types
    from paper_2009_10917_b200.gs import bs6_gather_into
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh, npb)
    assert (op.plan() is not None) == (npb <= 512)
    plain = types.SimpleNamespace(ng=op.ng, nl=op.nl, row_starts=op.row_starts_dev, col_ids=op.col_ids_dev,
                                  block_starts=op.block_starts_dev, nodes_per_block=npb,
                                  n_blocks=op.n_blocks)
    q = d(np.random.default_rng([K, p, npb]).uniform(-1, 1, mesh.nl))
    carry = d(np.random.default_rng(1).uniform(-1, 1, min(mesh.ng, 1000)))
    for c in (None, carry):
        a = torch.empty(mesh.ng, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        bs6_gather_into(op, q, a, c)
        bs6_gather_into(plain, q, b, c)
        assert torch.equal(a, b)


@pytest.mark.parametrize("seed,ng,nl,hot", [(3, 7000, 30000, 300), (4, 2000, 2000, 0), (5, 50000, 180000, 490)])
def test_planned_bs6_general_operator(sb, oracle, seed, ng, nl, hot):
    """Pipelined BS6 on a non-mesh operator: empty rows, a row of `hot` entries
    (up to nodes_per_block), random columns -- bitwise the oracle gather."""
    from paper_2009_10917_b200 import _lib
    from paper_2009_10917_b200 import mesh as M
    from paper_2009_10917_b200.gs import bs6_gather_into
    rng = np.random.default_rng(seed)
    l2g = rng.integers(0, ng, nl).astype(np.int32)
    l2g[l2g == 17] = 18          # row 17 empty
    if hot:
        l2g[rng.choice(nl, hot, replace=False)] = 5   # one long row
    l2g_d = torch.from_numpy(l2g).cuda()
    L = _lib.lib()
    rs = torch.empty(ng + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(nl, dtype=torch.int32, device="cuda")
    tmp = torch.empty(int(L.sb_build_gather_general_temp_bytes(nl)), dtype=torch.uint8, device="cuda")
    stats = torch.empty(2, dtype=torch.int64, device="cuda")
    _lib.check(L.sb_build_gather_general(l2g_d.data_ptr(), nl, ng, rs.data_ptr(), ci.data_ptr(),
                                         tmp.data_ptr(), tmp.shape[0], stats.data_ptr(),
                                         _lib.stream_handle()), "general")
    npb = 512
    bst = M._block_starts(rs, ng, npb)
    op = M.GatherOp(ng=ng, row_starts=rs, col_ids=ci, block_starts=bst, nodes_per_block=npb)
    assert op.plan() is not None
    q = rng.uniform(-1, 1, nl)
    out = torch.empty(ng, dtype=torch.float64, device="cuda")
    bs6_gather_into(op, d(q), out)
    counts = np.bincount(l2g, minlength=ng)        # mesh.py:123-134 without the coverage check
    rs_o = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    ci_o = np.argsort(l2g, kind="stable").astype(np.int32)
    assert np.array_equal(h(rs), rs_o) and np.array_equal(h(ci), ci_o)
    want = oracle.bs6_gather(rs_o, ci_o, q)
    got = h(out)
    assert np.array_equal(got, want)
    assert got[17] == 0.0 and not np.signbit(got[17])


def test_planned_bs6_many_empty_rows_falls_back(sb, oracle):
    """A hand-built operator whose blocks hold > 512 (empty) rows must not use
    the super-block kernel's fixed row capacity -- result still bitwise."""
    from paper_2009_10917_b200 import mesh as M
    from paper_2009_10917_b200.gs import bs6_gather_into
    ng, nl = 5000, 3000
    rng = np.random.default_rng(9)
    l2g = np.sort(rng.choice(ng, nl, replace=False)).astype(np.int32)   # 2000 empty rows
    counts = np.bincount(l2g, minlength=ng)
    rs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    ci = np.argsort(l2g, kind="stable").astype(np.int32)
    bst, row = [0], 0
    while row < ng:  # mesh.py:136-143, the reference's greedy packing (empty rows included)
        nxt = min(max(int(np.searchsorted(rs, int(rs[row]) + 512, side="right")) - 1, row + 1), ng)
        bst.append(nxt)
        row = nxt
    op = M.GatherOp(ng=ng, row_starts=torch.from_numpy(rs).cuda(), col_ids=torch.from_numpy(ci).cuda(),
                    block_starts=torch.tensor(bst, dtype=torch.int32, device="cuda"), nodes_per_block=512)
    assert op._superblock_extent()[0] > 512 and op.plan() is None
    q = rng.uniform(-1, 1, nl)
    out = torch.empty(ng, dtype=torch.float64, device="cuda")
    bs6_gather_into(op, d(q), out)
    assert np.array_equal(h(out), oracle.bs6_gather(rs, ci, q))


@pytest.mark.parametrize("carry_rows", [0, 700])
def test_planned_bs6_abi_oversize_trailer(sb, oracle, carry_rows):
    """The C-ABI planned gather on an operator with > 512 (empty) rows per
    super-block: sb_bs6_make_plan flags it in the plan trailer and every
    kernel variant sums rows from global memory -- bitwise, carry included."""
    from paper_2009_10917_b200 import _lib
    ng, nl = 5000, 3000
    rng = np.random.default_rng(19)
    l2g = np.sort(rng.choice(ng, nl, replace=False)).astype(np.int32)
    rs = np.concatenate([[0], np.cumsum(np.bincount(l2g, minlength=ng))]).astype(np.int32)
    ci = np.argsort(l2g, kind="stable").astype(np.int32)
    bst = np.append(np.arange(0, ng, 16, dtype=np.int32), ng).astype(np.int32)  # hand-built: 16 rows per block
    npb = 8
    L = _lib.lib()
    size = int(L.sb_bs6_plan_size(bst.shape[0] - 1, npb))
    plan = torch.full((size,), -7, dtype=torch.int32, device="cuda")
    rs_d, ci_d, bst_d = (torch.from_numpy(a).cuda() for a in (rs, ci, bst))
    _lib.check(L.sb_bs6_make_plan(bst_d.data_ptr(), bst.shape[0] - 1, rs_d.data_ptr(), npb, plan.data_ptr(),
                                  _lib.stream_handle()), "plan")
    assert int(plan[-2].item()) == 1  # 64 blocks of 16 rows: 1024-row super-blocks
    q = rng.uniform(-1, 1, nl)
    carry = rng.uniform(-1, 1, carry_rows) if carry_rows else None
    want = oracle.bs6_gather(rs, ci, q)
    for r in range(carry_rows):
        acc = carry[r]
        for j in range(rs[r], rs[r + 1]):
            acc = acc + q[ci[j]]
        want[r] = acc
    q_d = d(q)
    carry_d = None if carry is None else d(carry)
    for cfg in ("lanes,0,12", "lanes,1,8", "pairs,1,12", "wide,1,6", None):
        import os
        if cfg:
            os.environ["SB200_BS6_CFG"] = cfg
        try:
            out = torch.full((ng,), float("nan"), dtype=torch.float64, device="cuda")
            _lib.check(L.sb_bs6_gather_planned(plan.data_ptr(), bst.shape[0] - 1, npb, rs_d.data_ptr(),
                                               ci_d.data_ptr(), ng, nl, q_d.data_ptr(), out.data_ptr(),
                                               None if carry_d is None else carry_d.data_ptr(), carry_rows,
                                               _lib.stream_handle()), "gather")
            assert np.array_equal(h(out), want), cfg
        finally:
            os.environ.pop("SB200_BS6_CFG", None)
