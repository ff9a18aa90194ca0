"""Harness, CLI, selftest and CG on the B200 (harness.py / cli.py / selftest.py /
cg.py of the reference): sweeps validate against the device validators, write
the reference's CSV wire format, and fit with the reference's model."""

import json

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


@pytest.mark.parametrize("timer", ["host", "device", "graph"])
def test_run_sweep_all_tests(sb, timer):
    from paper_2009_10917_b200 import harness
    for test in ("bs1", "bs2", "bs3", "bs4", "bs5"):
        plan = harness.SweepPlan(test=test, sizes=[1, 1000, 131073, 2_000_000], trials=3, warmup=1)
        out = harness.run_sweep(plan, timer=timer)
        assert [s.n for s in out] == plan.sizes
        assert all(s.bandwidth > 0 and s.bytes == sb.bytes_moved(test, n=s.n) for s in out)
    for test in ("bs6", "bs7"):
        plan = harness.SweepPlan(test=test, sizes=[(2, 3), (5, 7)], trials=3, warmup=1)
        out = harness.run_sweep(plan, timer=timer)
        assert [(s.K, s.order) for s in out] == plan.sizes


@pytest.mark.parametrize("timer", ["host", "device"])
def test_run_sweep_sync_scalars(sb, timer):
    """sync_scalars=True reads every BS3-BS5 scalar back inside the timed
    batch (the reference API's float return); same samples, validated."""
    from paper_2009_10917_b200 import harness
    for test in ("bs3", "bs4", "bs5"):
        plan = harness.SweepPlan(test=test, sizes=[7, 131073], trials=3, warmup=1)
        out = harness.run_sweep(plan, timer=timer, sync_scalars=True)
        assert [s.n for s in out] == plan.sizes and all(s.bandwidth > 0 for s in out)


def test_sweep_failure_keeps_samples(sb, monkeypatch):
    """harness.py:256-267: a validation failure aborts with the samples so far."""
    from paper_2009_10917_b200 import harness
    monkeypatch.setattr(harness._VectorCase, "validate", lambda self, s: self.n < 500)
    plan = harness.SweepPlan(test="bs2", sizes=[10, 100, 1000], trials=2)
    with pytest.raises(harness.SweepError) as ei:
        harness.run_sweep(plan)
    assert [s.n for s in ei.value.samples] == [10, 100]


def test_cli_run_fit_roundtrip(sb, tmp_path):
    from paper_2009_10917_b200 import cli
    csv_path = tmp_path / "s.csv"
    rc = cli.main(["run", "--test", "bs1", "--min-bytes", "1e4", "--max-bytes", "4e8",
                   "--points", "12", "--trials", "5", "--timer", "device", "--out", str(csv_path)])
    assert rc == 0
    samples = cli.read_samples_csv(csv_path)
    assert len(samples) == 12 and all(s.test == "bs1" for s in samples)
    with open(csv_path) as f:
        assert f.readline().strip() == cli.CSV_HEADER
    fit_path = tmp_path / "fit.json"
    assert cli.main(["fit", str(csv_path), "--out", str(fit_path)]) == 0
    rep = json.load(open(fit_path))
    assert rep[0]["test"] == "bs1" and rep[0]["Wmax_Bps"] > 1e11
    rc = cli.main(["run", "--test", "bs7", "--kmin", "2", "--kmax", "4", "--order", "3",
                   "--trials", "3", "--format", "json", "--out", str(tmp_path / "m.json")])
    assert rc == 0 and len(json.load(open(tmp_path / "m.json"))) == 3


def test_selftest_and_fault_injection(sb, capsys):
    from paper_2009_10917_b200 import cli
    assert cli.main(["selftest"]) == 0
    out = capsys.readouterr().out
    assert "9 passed, 0 failed" in out
    assert cli.main(["selftest", "--inject-fault"]) == 1


def test_cg_fused_equals_unfused_bitwise(sb):
    """test_cg.py:70-78: fused and unfused CG produce bitwise-identical iterates."""
    from paper_2009_10917_b200 import cg
    a = cg.random_spd_matrix(200, seed=4)
    b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, 200)).cuda()
    op = cg.dense_spd_operator(a)
    r1 = cg.cg_solve(op, b, torch.zeros_like(b), eps=1e-24, max_iter=300, fused=True)
    r2 = cg.cg_solve(op, b, torch.zeros_like(b), eps=1e-24, max_iter=300, fused=False)
    assert r1.iterations == r2.iterations and r1.converged
    assert torch.equal(r1.x, r2.x) and r1.final_rr == r2.final_rr
    with pytest.raises(cg.NotSPDError):
        cg.cg_solve(lambda v: -v, b, torch.zeros_like(b), eps=1e-20, max_iter=5)
