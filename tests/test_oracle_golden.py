"""Pin the CPU oracle (oracle/sb_oracle.c) to the unmodified reference.

Every expectation here comes from tests/golden/*, produced by running
/root/reference/pkg/src/streambench itself (tests/golden/make_golden.py).
No GPU needed.
"""

import numpy as np
import pytest

from goldens import acceptance_inputs, mesh_q_global, mesh_q_local, selftest_inputs, sha, unhex


def _cfg(key):
    bs, nb = key.split(",")
    return int(bs), int(nb)


@pytest.mark.parametrize("threads", [1, 4])
def test_vectors_selftest_sizes(golden, oracle, threads):
    oracle.set_threads(threads)
    try:
        for rec in golden["vectors"]:
            n = rec["n"]
            alpha, beta, x, y, p, ap = selftest_inputs(n)
            assert sha(np.concatenate([x, y, p, ap])) == rec["in_hash"], "numpy RNG stream drift"
            assert alpha == unhex(rec["alpha"]) and beta == unhex(rec["beta"])
            out = np.zeros(n)
            oracle.bs1_copy(x, out)
            assert np.array_equal(out, x)
            yy = y.copy()
            oracle.bs2_axpy(alpha, x, beta, yy)
            assert sha(yy) == rec["bs2_hash"], n
            for key, val in rec["norm2"].items():
                bs, nb = _cfg(key)
                assert oracle.bs3_norm2(x, bs, nb) == unhex(val), (n, key)
                assert oracle.bs4_dot(x, y, bs, nb) == unhex(rec["dot"][key]), (n, key)
                xx, rr = x.copy(), y.copy()
                got = oracle.bs5_fused_cg_update(alpha, p, ap, xx, rr, bs, nb)
                assert got == unhex(rec["bs5"][key]), (n, key)
                assert sha(xx) == rec["bs5_x"][key] and sha(rr) == rec["bs5_r"][key]
            if "fsum_norm2" in rec:
                assert oracle.fsum_norm2(x) == unhex(rec["fsum_norm2"])
                assert oracle.fsum_dot(x, y) == unhex(rec["fsum_dot"])
    finally:
        oracle.set_threads(1)


def test_vectors_acceptance_sizes(golden, oracle):
    assert len(golden["cfg_sweep"]) == 50
    for rec in golden["cfg_sweep"]:
        n = rec["n"]
        alpha, beta, x, y, p, ap = acceptance_inputs(n)
        assert sha(np.concatenate([x, y, p, ap])) == rec["in_hash"]
        yy = y.copy()
        oracle.bs2_axpy(alpha, x, beta, yy)
        assert sha(yy) == rec["bs2_hash"]
        assert oracle.bs3_norm2(x) == unhex(rec["norm2"])
        assert oracle.bs4_dot(x, y) == unhex(rec["dot"])
        xx, rr = x.copy(), y.copy()
        assert oracle.bs5_fused_cg_update(alpha, p, ap, xx, rr) == unhex(rec["bs5"])
        assert sha(xx) == rec["bs5_x"] and sha(rr) == rec["bs5_r"]


def test_hand_kats(oracle):
    # test_kernels.py:41-46, 76-79, 131-132, 159-160, 187-190
    x = np.array([1.0, 2.0, 3.0]); y = np.zeros(3)
    oracle.bs1_copy(x, y); assert np.array_equal(y, x)
    y = np.array([1.0]); oracle.bs2_axpy(2.0, np.array([1.0]), 3.0, y); assert y[0] == 5.0
    assert oracle.bs3_norm2(np.array([3.0, 4.0])) == 25.0
    assert oracle.bs4_dot(np.array([1.0, 2.0]), np.array([3.0, 4.0])) == 11.0
    x, r = np.array([0.0]), np.array([2.0])
    b = oracle.bs5_fused_cg_update(1.0, np.array([1.0]), np.array([2.0]), x, r)
    assert x[0] == 1.0 and r[0] == 0.0 and b == 0.0
    assert oracle.bs3_norm2(np.zeros(0)) == 0.0


def test_meshes_and_operators(golden, oracle):
    for rec in golden["meshes"]:
        K, p, npb = rec["K"], rec["p"], rec["npb"]
        l2g = oracle.build_mesh(K, p)
        assert l2g.shape[0] == rec["nl"] and sha(l2g) == rec["l2g"], (K, p)
        rs, ci, bst = oracle.build_gather(l2g, rec["ng"], npb)
        assert sha(rs) == rec["row_starts"], (K, p)
        assert sha(ci) == rec["col_ids"], (K, p)
        assert sha(bst) == rec["block_starts"] and bst.shape[0] - 1 == rec["n_blocks"], (K, p, npb)
        q = mesh_q_local(K, p, rec["nl"])
        assert sha(q) == rec["bs6_q_hash"]
        assert sha(oracle.bs6_gather(rs, ci, q)) == rec["bs6_out"], (K, p)
        qg = mesh_q_global(K, p, rec["ng"])
        assert sha(qg) == rec["bs7_qg_hash"]
        ql = np.zeros(rec["nl"])
        oracle.bs7_scatter(oracle.build_scatter_ids(l2g, rec["ng"]), qg, ql)
        assert sha(ql) == rec["bs7_out"], (K, p)
        assert sha(oracle.multiplicity(l2g, rec["ng"])) == rec["mult"]


def test_masks(golden, oracle):
    for rec in golden["masks"]:
        K, p = rec["K"], rec["p"]
        l2g = oracle.build_mesh(K, p)
        ng = (K * p + 1) ** 3
        ids = oracle.build_scatter_ids(l2g, ng, set(rec["mask"]))
        assert sha(ids) == rec["ids"]
        qg = np.random.default_rng([9, K, p]).uniform(-1, 1, ng)
        ql = np.full(l2g.shape[0], 99.0)
        oracle.bs7_scatter(ids, qg, ql)
        assert sha(ql) == rec["out"]


def test_builder_rejections(oracle):
    with pytest.raises(ValueError):
        oracle.build_mesh(0, 1)
    with pytest.raises(ValueError):
        oracle.build_mesh(200, 7)  # test_mesh.py:81-83
    l2g = oracle.build_mesh(2, 1)
    with pytest.raises(ValueError):
        oracle.build_gather(l2g, 27, 7)  # test_mesh.py:173-176


def test_carry_composition_bitexact(oracle):
    """z-slab carry reproduces the 1-rank gather bitwise."""
    K, p = 4, 3
    g = K * p + 1
    l2g = oracle.build_mesh(K, p)
    ng = g ** 3
    rs, ci, _ = oracle.build_gather(l2g, ng, 512)
    q = mesh_q_local(K, p, l2g.shape[0])
    full = oracle.bs6_gather(rs, ci, q)
    # two slabs: layers [0,2) and [2,4); interface plane c = 2p
    plane = g * g
    c_if = 2 * p
    # lower rank: partial sums of the interface plane from its own elements
    nl_lo = 2 * K * K * (p + 1) ** 3
    lo_rows = np.arange(c_if * plane, (c_if + 1) * plane)
    carry = np.zeros(plane)
    for k, r in enumerate(lo_rows):
        acc = 0.0
        for c in range(rs[r], rs[r + 1]):
            if ci[c] < nl_lo:
                acc += q[ci[c]]
        carry[k] = acc
    # upper rank: rows from plane c_if upward, seeded with the carry
    up_rows = np.arange(c_if * plane, ng)
    out_up = np.empty(up_rows.shape[0])
    for k, r in enumerate(up_rows):
        acc = carry[k] if k < plane else 0.0
        for c in range(rs[r], rs[r + 1]):
            if ci[c] >= nl_lo:
                acc += q[ci[c]]
        out_up[k] = acc
    assert np.array_equal(out_up, full[c_if * plane:])


# --- cg.py:27-72 (diagonal operators; tests/golden 'cg' records) -------------

def test_oracle_cg_matches_reference_golden(golden, oracle):
    from goldens import cg_inputs
    for rec in golden["cg"]:
        d, b, x0 = cg_inputs(rec)
        x, it, rr, conv = oracle.cg_solve_diag(d, b, x0, float.fromhex(rec["eps"]), rec["max_iter"],
                                          *rec["cfg"], fused=rec["fused"], relative=rec["relative"])
        assert it == rec["iterations"], rec
        assert rr.hex() == rec["final_rr"], rec
        assert conv == rec["converged"]
        assert sha(x) == rec["x_hash"], rec
