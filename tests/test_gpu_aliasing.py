"""Aliased arguments: the
reference's numpy semantics (kernels.py:90-132) for x is y, r is x, p is x,
... -- bitwise -- and overlapping-but-not-identical views."""

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


def ref_bs5(alpha, p, ap, x, r, oracle):
    """kernels.py:127-131 with one worker: x += alpha*p, then r -= alpha*ap, then the lattice."""
    x += alpha * p
    r -= alpha * ap
    return oracle.bs3_norm2(np.ascontiguousarray(r))


CASES = ["x_is_r", "p_is_x", "ap_is_x", "ap_is_r", "p_is_r", "all_same"]


def make(case, n, seed):
    rng = np.random.default_rng([n, seed])
    v = {k: rng.uniform(-1, 1, n) for k in ("p", "ap", "x", "r")}
    a, b = case.split("_is_") if "_is_" in case else (None, None)
    if case == "all_same":
        v = {k: v["x"] for k in v}
    else:
        v[a] = v[b]
    return v


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("where", ["cuda", "numpy"])
def test_bs5_aliased_matches_reference_order(sb, oracle, case, where):
    n, alpha = 100_003, 0.37
    hv = make(case, n, 1)
    names = ("p", "ap", "x", "r")
    # reference on host copies with the same aliasing structure
    hid = {}
    refv = {}
    for k in names:
        key = id(hv[k])
        if key not in hid:
            hid[key] = hv[k].copy()
        refv[k] = hid[key]
    want = ref_bs5(alpha, refv["p"], refv["ap"], refv["x"], refv["r"], oracle)
    if where == "cuda":
        did = {}
        dv = {}
        for k in names:
            key = id(hv[k])
            if key not in did:
                did[key] = torch.from_numpy(hv[k].copy()).cuda()
            dv[k] = did[key]
        got = sb.bs5_fused_cg_update(alpha, dv["p"], dv["ap"], dv["x"], dv["r"])
        gx, gr = dv["x"].cpu().numpy(), dv["r"].cpu().numpy()
    else:
        cid = {}
        cv = {}
        for k in names:
            key = id(hv[k])
            if key not in cid:
                cid[key] = hv[k].copy()
            cv[k] = cid[key]
        got = sb.bs5_fused_cg_update(alpha, cv["p"], cv["ap"], cv["x"], cv["r"])
        gx, gr = cv["x"], cv["r"]
    assert got == want
    assert np.array_equal(gx, refv["x"]) and np.array_equal(gr, refv["r"])


def test_bs5_partial_overlap_rejected(sb):
    buf = torch.zeros(1001, dtype=torch.float64, device="cuda")
    p = torch.ones(1000, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        sb.bs5_fused_cg_update(0.5, p, p.clone(), buf[:1000], buf[1:])


@pytest.mark.parametrize("shift", [1, 7, -3])
def test_bs1_bs2_partial_overlap_numpy_semantics(sb, shift):
    n = 50_000
    base = np.random.default_rng(5).uniform(-1, 1, n + 10)
    lo_x, lo_y = (0, shift) if shift > 0 else (-shift, 0)
    h = base.copy()
    h[lo_y:lo_y + n] = h[lo_x:lo_x + n].copy()  # numpy y[:] = x with overlap
    d = torch.from_numpy(base.copy()).cuda()
    sb.bs1_copy(d[lo_x:lo_x + n], d[lo_y:lo_y + n])
    assert np.array_equal(d.cpu().numpy(), h)
    h = base.copy()
    h[lo_y:lo_y + n] = 0.5 * h[lo_x:lo_x + n] + -0.25 * h[lo_y:lo_y + n]
    d = torch.from_numpy(base.copy()).cuda()
    sb.bs2_axpy(0.5, d[lo_x:lo_x + n], -0.25, d[lo_y:lo_y + n])
    assert np.array_equal(d.cpu().numpy(), h)


def test_bs2_x_is_y(sb):
    x = np.random.default_rng(6).uniform(-1, 1, 4097)
    want = 0.5 * x + 1.5 * x
    d = torch.from_numpy(x.copy()).cuda()
    sb.bs2_axpy(0.5, d, 1.5, d)
    assert np.array_equal(d.cpu().numpy(), want)
    h = x.copy()
    sb.bs2_axpy(0.5, h, 1.5, h)
    assert np.array_equal(h, want)
