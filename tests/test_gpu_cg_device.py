"""Device-resident CG: alpha, beta and the stopping test
on the GPU (sb_cg_*), checked bitwise against the reference's own CG results
(tests/golden 'cg' records, produced by running cg.py) and against the
host-scalar solver on the same operator."""

import numpy as np
import pytest
import torch

from goldens import cg_inputs, sha

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("graph,check_every", [(False, 1), (False, 7), (True, 16), (True, 5)])
def test_device_cg_matches_reference_golden(golden, graph, check_every):
    from paper_2009_10917_b200 import cg
    from paper_2009_10917_b200.kernels import ReductionConfig
    for rec in golden["cg"]:
        d, b, x0 = cg_inputs(rec)
        res = cg.cg_solve_device(cg.diagonal_operator(_dev(d)), _dev(b), _dev(x0), float.fromhex(rec["eps"]),
                                 rec["max_iter"], ReductionConfig(*rec["cfg"]), fused=rec["fused"],
                                 relative=rec["relative"], check_every=check_every, graph=graph)
        assert res.iterations == rec["iterations"], rec
        assert res.final_rr.hex() == rec["final_rr"], rec
        assert res.converged == rec["converged"]
        assert sha(res.x.cpu().numpy()) == rec["x_hash"], rec


def test_host_scalar_cg_matches_reference_golden(golden):
    from paper_2009_10917_b200 import cg
    from paper_2009_10917_b200.kernels import ReductionConfig
    for rec in golden["cg"]:
        d, b, x0 = cg_inputs(rec)
        res = cg.cg_solve(cg.diagonal_operator(_dev(d)), _dev(b), _dev(x0), float.fromhex(rec["eps"]),
                          rec["max_iter"], ReductionConfig(*rec["cfg"]), fused=rec["fused"],
                          relative=rec["relative"])
        assert (res.iterations, res.final_rr.hex()) == (rec["iterations"], rec["final_rr"])
        assert sha(res.x.cpu().numpy()) == rec["x_hash"]


@pytest.mark.parametrize("fused", [True, False])
def test_device_equals_host_dense(fused):
    from paper_2009_10917_b200 import cg
    a = cg.random_spd_matrix(96, seed=5)
    op = cg.dense_spd_operator(_dev(a))
    b = _dev(np.random.default_rng(6).uniform(-1, 1, 96))
    h = cg.cg_solve(op, b, torch.zeros_like(b), 1e-26, 500, fused=fused)
    for graph in (False, True):
        d = cg.cg_solve_device(op, b, torch.zeros_like(b), 1e-26, 500, fused=fused, check_every=4, graph=graph)
        assert d.iterations == h.iterations and d.final_rr == h.final_rr and d.converged == h.converged
        assert torch.equal(d.x, h.x)


def test_device_fused_equals_unfused():
    """test_cg.py:70-78 for the device solver."""
    from paper_2009_10917_b200 import cg
    a = cg.random_spd_matrix(120, seed=9)
    op = cg.dense_spd_operator(_dev(a))
    b = _dev(np.random.default_rng(10).uniform(-1, 1, 120))
    r1 = cg.cg_solve_device(op, b, torch.zeros_like(b), 1e-24, 300, fused=True)
    r2 = cg.cg_solve_device(op, b, torch.zeros_like(b), 1e-24, 300, fused=False)
    assert r1.iterations == r2.iterations and torch.equal(r1.x, r2.x)


def test_device_not_spd_same_error_as_host():
    from paper_2009_10917_b200 import cg
    b = _dev(np.random.default_rng(11).uniform(-1, 1, 300))
    with pytest.raises(cg.NotSPDError) as eh:
        cg.cg_solve(lambda v: -v, b, torch.zeros_like(b), 1e-20, 5)
    with pytest.raises(cg.NotSPDError) as ed:
        cg.cg_solve_device(lambda v: -v, b, torch.zeros_like(b), 1e-20, 5)
    assert str(eh.value) == str(ed.value)


def test_device_cg_edge_cases():
    from paper_2009_10917_b200 import cg
    b = _dev(np.random.default_rng(12).uniform(-1, 1, 64))
    with pytest.raises(ValueError):
        cg.cg_solve_device(lambda v: v, b, torch.zeros_like(b), 0.0, 5)
    with pytest.raises(ValueError):
        cg.cg_solve_device(lambda v: v, b, torch.zeros_like(b), 1e-10, 5, check_every=0)
    r = cg.cg_solve_device(lambda v: v, b, torch.zeros_like(b), 1e-10, 0)   # max_iter = 0
    h = cg.cg_solve(lambda v: v, b, torch.zeros_like(b), 1e-10, 0)
    assert (r.iterations, r.final_rr, r.converged) == (h.iterations, h.final_rr, h.converged) == (0, h.final_rr, False)
    r = cg.cg_solve_device(lambda v: v, b, torch.zeros_like(b), 1e-10, 50)  # identity: one iteration
    assert r.iterations == 1 and r.converged


@pytest.mark.parametrize("K,p", [(3, 3), (4, 2), (2, 7)])
def test_gather_scatter_operator_cg(K, p):
    """CG on A = Z^T diag(w) Z built from BS7 + BS6: device == host bitwise, and A x ~ b."""
    from paper_2009_10917_b200 import cg
    import paper_2009_10917_b200 as sb
    mesh = sb.build_mesh(K, p)
    op, ids = sb.build_gather(mesh), sb.build_scatter_ids(mesh)
    rng = np.random.default_rng([K, p, 3])
    A = cg.gather_scatter_operator(op, ids, rng.uniform(1, 2, mesh.nl))
    b = _dev(rng.uniform(-1, 1, mesh.ng))
    h = cg.cg_solve(A, b, torch.zeros_like(b), 1e-22, 2000, relative=True)
    d = cg.cg_solve_device(A, b, torch.zeros_like(b), 1e-22, 2000, relative=True, check_every=8, graph=True)
    assert h.converged and d.iterations == h.iterations and torch.equal(d.x, h.x)
    res = (A(d.x) - b).norm() / b.norm()
    assert res.item() < 1e-9


def test_host_array_operators_capturable():
    """Operators built from host numpy arrays (the reference's usage,
    cg.py:75-92) keep one device copy, so the CUDA-graph device CG can
    capture them; iterates equal the host-scalar solver's."""
    from paper_2009_10917_b200 import cg
    rng = np.random.default_rng(12)
    for op, n in ((cg.diagonal_operator(np.repeat([1.0, 2.0, 3.0], 8)), 24),
                  (cg.dense_spd_operator(cg.random_spd_matrix(40, seed=13)), 40)):
        b = _dev(rng.uniform(-1, 1, n))
        h = cg.cg_solve(op, b, torch.zeros_like(b), 1e-24, 200)
        d = cg.cg_solve_device(op, b, torch.zeros_like(b), 1e-24, 200, check_every=2, graph=True)
        assert d.iterations == h.iterations and torch.equal(d.x, h.x)
