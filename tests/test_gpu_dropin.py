"""Drop-in contract: reference-style numpy callers get the
reference's host types back, and the reference's own test suite (224 tests,
pkg/tests) passes against this package through the package-swap shim
(scripts/dropin/streambench) when it has been staged under
baseline/_ref/tests_ref (scripts/run_reference_tests.sh --stage)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_builders_hand_numpy_callers_numpy():
    import paper_2009_10917_b200 as sb
    mesh = sb.build_mesh(3, 2)
    op, ids = sb.build_gather(mesh), sb.build_scatter_ids(mesh, mask=[0, 5])
    for a in (mesh.local_to_global, op.row_starts, op.col_ids, op.block_starts, ids.ids):
        assert isinstance(a, np.ndarray) and a.dtype == np.int32
    for a in (mesh.local_to_global_dev, op.row_starts_dev, op.col_ids_dev, op.block_starts_dev, ids.ids_dev):
        assert isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.int32
    assert np.array_equal(mesh.local_to_global, mesh.local_to_global_dev.cpu().numpy())
    mult = sb.multiplicity(mesh)
    assert isinstance(mult, np.ndarray) and mult.dtype == np.float64
    # reference test_gs.py:32 mixes the two: gather of ones (numpy in -> numpy out) == multiplicity
    assert np.array_equal(sb.bs6_gather(op, np.ones(mesh.nl)), mult)
    v = sb.dvector(7)
    assert isinstance(v, np.ndarray) and v.dtype == np.float64 and not v.any()
    with pytest.raises(Exception):
        mesh.K = 4  # frozen, like the reference's dataclasses
    # operators built from numpy arrays (the reference's own objects' shape) upload on use
    op2 = sb.GatherOp(ng=op.ng, row_starts=op.row_starts, col_ids=op.col_ids, block_starts=op.block_starts,
                      nodes_per_block=op.nodes_per_block)
    q = np.random.default_rng(1).uniform(-1, 1, mesh.nl)
    assert np.array_equal(sb.bs6_gather(op2, q), sb.bs6_gather(op, q))


def test_cg_numpy_in_numpy_out():
    import paper_2009_10917_b200 as sb
    d = np.linspace(1.0, 4.0, 50)
    b = np.random.default_rng(2).uniform(-1, 1, 50)
    for op in (sb.diagonal_operator(d), lambda v: d * v):  # ours, and a plain numpy operator
        res = sb.cg_solve(op, b, np.zeros(50), 1e-24, 200)
        assert isinstance(res.x, np.ndarray) and res.converged
        assert np.allclose(d * res.x, b, rtol=0, atol=1e-10)


def test_reference_suite_through_the_shim():
    tests = os.path.join(ROOT, "baseline", "_ref", "tests_ref")
    if not os.path.isdir(tests):
        pytest.skip("reference tests not staged (scripts/run_reference_tests.sh --stage)")
    env = dict(os.environ, PYTHONPATH=os.path.join(ROOT, "scripts", "dropin") + os.pathsep + ROOT)
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "."], cwd=tests,
                          env=env, capture_output=True, text=True, timeout=900)
    tail = proc.stdout.strip().splitlines()[-1] if proc.stdout.strip() else proc.stderr[-2000:]
    assert proc.returncode == 0, tail
    assert "224 passed" in tail, tail
