"""Host-side logic of the B200 package (no GPU): byte accounting, model fit,
size schedules, CSV wire format, CLI flag handling, config validation, and the
C-ABI library's exported symbols.  Expectations come from the reference's own
tests and golden outputs."""

import ctypes
import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2009_10917_b200 as sb
from paper_2009_10917_b200 import _lib, cli, core, harness, model
from goldens import unhex

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# --- core.py (test_core.py) ---------------------------------------------------

def test_bytes_moved_kats():
    assert core.bytes_moved("bs1", n=1000) == 16000
    assert core.bytes_moved("bs5", n=1000) == 48000
    assert core.bytes_moved("bs6", nl=64, ng=27) == 1096
    assert core.bytes_moved("bs7", nl=64, ng=27) == 4 * 64 + 8 * 27 + 8 * 64
    assert [core.vector_bytes_per_element(t) for t in ("bs1", "bs2", "bs3", "bs4", "bs5")] == \
        [16, 24, 8, 16, 48]
    for t in ("bs1", "bs2", "bs3", "bs4", "bs5"):
        for n in [1, 17, 1000, 123456]:
            assert core.bytes_moved(t, n=2 * n) == 2 * core.bytes_moved(t, n=n)
    with pytest.raises(ValueError):
        core.bytes_moved("bs9", n=10)
    with pytest.raises(ValueError):
        core.bytes_moved("bs6", n=10)
    with pytest.raises(ValueError):
        core.bytes_moved("bs7", nl=10)
    with pytest.raises(ValueError):
        core.bytes_moved("bs1", n=-1)
    acct = core.ByteAccount.for_test("bs2", n=500)
    assert acct.test == "bs2" and acct.bytes == 24 * 500


def test_mesh_bytes_vs_golden(golden):
    for rec in golden["meshes"]:
        assert core.bytes_moved("bs6", nl=rec["nl"], ng=rec["ng"]) == rec["bytes_bs6"]
        assert core.bytes_moved("bs7", nl=rec["nl"], ng=rec["ng"]) == rec["bytes_bs7"]


def test_reduction_config_validation():
    for bad in (0, 1, 3, 24, 100):
        with pytest.raises(ValueError):
            sb.ReductionConfig(block_size=bad, n_blocks=4)
    with pytest.raises(ValueError):
        sb.ReductionConfig(block_size=4, n_blocks=0)
    assert sb.ReductionConfig() == sb.ReductionConfig(256, 512)


def test_public_names_match_reference():
    ref_all = ["BandwidthSample", "ByteAccount", "CGResult", "DVector", "GatherOp",
               "MeshConnectivity", "ModelFit", "ModelFitError", "NotSPDError", "ReductionConfig",
               "ScatterIds", "SweepError", "SweepPlan", "bs1_copy", "bs2_axpy", "bs3_norm2",
               "bs4_dot", "bs5_fused_cg_update", "bs6_gather", "bs7_scatter", "build_gather",
               "build_mesh", "build_scatter_ids", "bytes_moved", "cg_solve",
               "dense_spd_operator", "diagonal_operator", "dvector", "efficiency_point",
               "fit_model", "geometric_sizes", "max_workers", "multiplicity", "num_workers",
               "run_sweep", "set_num_workers", "w_eff"]
    assert sorted(sb.__all__) == sorted(ref_all)
    for name in ref_all:
        assert hasattr(sb, name), name


# --- model.py (test_model.py, golden fits) ----------------------------------

def test_model_fits_match_reference_bitwise(golden):
    G = golden["model"]
    t0, wmax = G["t0"], G["wmax"]
    sizes = G["sizes"]
    exact = [harness.BandwidthSample("bs1", int(b), (t0 + int(b) / wmax) * 20, 20, 0.0)
             for b in sizes]
    for name, weighted in (("exact", False), ("exact_w", True)):
        f = model.fit_model(exact, weighted=weighted)
        want = G["fits"][name]
        assert f.t0 == unhex(want["t0"]) and f.wmax == unhex(want["wmax"])
        assert f.r2 == unhex(want["r2"]) and f.n_points == want["n"]
    for seed in range(5):
        rng = np.random.default_rng([seed, 99])
        noisy = [harness.BandwidthSample("bs1", int(b), (t0 + int(b) / wmax)
                                         * (1 + 0.01 * rng.standard_normal()) * 20, 20, 0.0)
                 for b in sizes]
        for weighted in (False, True):
            f = model.fit_model(noisy, weighted=weighted)
            want = G["fits"][f"noisy{seed}_{int(weighted)}"]
            assert f.t0 == unhex(want["t0"]) and f.wmax == unhex(want["wmax"])
            assert f.r2 == unhex(want["r2"]) and f.clamped_t0 == want["clamped"]
    v100 = model.ModelFit(7.62e-6, 809e9, 1.0, 2)
    assert model.efficiency_point(v100) == unhex(G["b80_v100"])
    mi60 = model.ModelFit(16.99e-6, 843e9, 1.0, 2)
    assert model.efficiency_point(mi60) == unhex(G["b80_mi60"])
    assert model.w_eff(model.ModelFit(2.90e-6, 811e9, 1.0, 2), 0.1e9) == unhex(G["weff_v100_bs1"])


def test_model_errors_and_clamp():
    with pytest.raises(model.ModelFitError):
        model.fit_model([harness.BandwidthSample("bs1", 100, 1.0, 1, 0.0)] * 3)
    with pytest.raises(model.ModelFitError):
        model.fit_model([harness.BandwidthSample("bs1", 100, 2.0, 1, 0.0),
                         harness.BandwidthSample("bs1", 200, 1.0, 1, 0.0)])
    with pytest.warns(UserWarning):
        f = model.fit_model([harness.BandwidthSample("bs1", 100, 0.5, 1, 0.0),
                             harness.BandwidthSample("bs1", 200, 2.0, 1, 0.0)])
    assert f.clamped_t0 and f.t0 == 0.0
    fit = model.ModelFit(t0=0.0, wmax=8e11, r2=1.0, n_points=2)
    assert model.w_eff(fit, 0.0) == 8e11
    with pytest.raises(ValueError):
        model.w_eff(fit, -1.0)
    for bad in (0.0, 1.0, -0.1, 1.5):
        with pytest.raises(ValueError):
            model.efficiency_point(fit, bad)


# --- harness.py (test_harness.py) -------------------------------------------

def test_geometric_sizes_vs_golden(golden):
    for rec in golden["geometric"]:
        assert harness.geometric_sizes(*rec["args"]) == rec["sizes"], rec["args"]
    with pytest.raises(ValueError):
        harness.geometric_sizes(0, 10, 5)
    with pytest.raises(ValueError):
        harness.geometric_sizes(10, 5, 5)
    with pytest.raises(ValueError):
        harness.geometric_sizes(1, 10, 0)


def test_sweep_plan_validation():
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs8", sizes=[10])
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs1", sizes=[10, 10])
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs1", sizes=[10], trials=0)
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs1", sizes=[10], warmup=-1)
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs1", sizes=[0])
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs1", sizes=[10], seed=-3)
    harness.SweepPlan(test="bs6", sizes=[(2, 7), (3, 7)])
    with pytest.raises(ValueError):
        harness.SweepPlan(test="bs6", sizes=[(0, 7)])
    e = harness.SweepError("allocation failed", 10, [1, 2])
    assert e.samples == [1, 2] and "at size 10" in str(e)


# --- cli.py wire formats ----------------------------------------------------

def test_csv_rows_byte_identical(golden, tmp_path):
    assert cli.CSV_HEADER == golden["csv_header"]
    samples = []
    for rec in golden["csv"]:
        s = harness.BandwidthSample(rec["test"], rec["bytes"], 0.125, rec["trials"], 1.0 / 3.0,
                                    rec["n"], rec["order"], rec["K"], rec["nl"], rec["ng"])
        assert cli.sample_to_csv_row(s) == rec["row"]
        samples.append(s)
    path = tmp_path / "s.csv"
    with open(path, "w") as f:
        cli.write_samples_csv(samples, f)
    back = cli.read_samples_csv(path)
    assert back == samples
    buf = io.StringIO()
    cli.write_samples_json(samples, buf)
    assert len(json.loads(buf.getvalue())) == len(samples)


def test_cli_fit_and_usage_errors(tmp_path, capsys):
    t0, wmax = 5e-6, 8e11
    rows = [harness.BandwidthSample("bs1", b, (t0 + b / wmax) * 20, 20, b * 20 / ((t0 + b / wmax) * 20) / 1e9,
                                    n=b // 16) for b in (16000, 160000, 1600000, 16000000)]
    path = tmp_path / "sweep.csv"
    with open(path, "w") as f:
        cli.write_samples_csv(rows, f)
    out = tmp_path / "fit.json"
    assert cli.main(["fit", str(path), "--out", str(out)]) == 0
    rep = json.load(open(out))
    assert abs(rep[0]["T0_s"] - t0) / t0 < 1e-6 and abs(rep[0]["Wmax_Bps"] - wmax) / wmax < 1e-9
    assert cli.main(["fit", str(path), "--eff", "1.5"]) == 2
    bad = tmp_path / "bad.csv"
    bad.write_text("nope\n")
    assert cli.main(["fit", str(bad)]) == 1
    assert cli.main(["run", "--test", "bs1", "--min-bytes", "0"]) == 2
    assert cli.main(["run", "--test", "bs6", "--kmin", "5", "--kmax", "3"]) == 2
    assert cli.main(["run", "--test", "bs1", "--threads", "0"]) == 2
    with pytest.raises(SystemExit) as ei:
        cli.main(["run", "--test", "bs9"])
    assert ei.value.code == 2
    assert cli.main(["selftest", "--list"]) == 0
    assert "bs5_fused_update" in capsys.readouterr().out


# --- the C ABI library (no GPU: load + symbols only) -------------------------

def test_library_exports_every_header_symbol():
    path = _lib.LIB_PATH
    if not os.path.exists(path):
        from paper_2009_10917_b200 import build as B
        B.build()
    L = _lib.load_library(path)
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(L, name), f"{name} declared in include/sb200.h but not exported"
    assert set(_lib._SIGS) == set(syms), "ctypes signatures must mirror the header"
    assert L.sb_version() == 100
    assert L.sb_reduce_workspace_bytes(256, 512) >= 256 + 8 * 512
    assert L.sb_reduce_workspace_bytes(3, 512) == 0


def test_library_argument_validation_without_gpu():
    """Entry points reject bad arguments with SB_E_INVALID and a message
    before touching the device (the reference's ValueError cases)."""
    L = _lib.load_library(_lib.LIB_PATH)
    E = _lib.SB_E_INVALID
    assert L.sb_bs1_copy(None, None, -1, None) == E
    assert b"invalid" in L.sb_last_error()
    fake = 0x1000  # never dereferenced: the configuration is rejected first
    assert L.sb_bs3_norm2(fake, 10, 3, 512, fake, fake, None) == E            # block_size not a power of two
    assert b"power of two" in L.sb_last_error()
    assert L.sb_bs4_dot(fake, fake, 10, 256, 0, fake, fake, None) == E         # n_blocks < 1
    assert L.sb_bs6_plan_size(10, 513) == 0 and L.sb_bs6_plan_size(0, 512) == 0
    assert L.sb_bs6_gather_planned(None, 1, 512, None, None, 10, 10, None, None, None, 0, None) == E
    assert L.sb_bs7_scatter(None, 5, None, 5, None, 0, None) == E
    assert L.sb_bs7_scatter_split(None, 5, None, -1, None, 0, None, 0, None) == E
    assert L.sb_cg_begin(None, None, None, 1e-10, 5, None) == E
    assert L.sb_cg_pap(None, None, 10, 256, 512, None, None, None) == E
    assert L.sb_lsa_create(None, 0, 1, 0, None) == E
    assert L.sb_lsa_bs3_norm2(None, 10, 256, 512, None, None, None, None) == E
    assert L.sb_lsa_halo_window(None, 8) == E
    assert L.sb_sum_ordered(None, -1, None, None) == E


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    # DFMA is allowed only inside the device-CG control kernels, whose IEEE
    # division (alpha = rr/pAp, beta = rr_new/rr) is a correctly rounded
    # DFMA Newton sequence; every streaming kernel must be contraction-free.
    funcs, cur = {}, None
    for ln in sass.splitlines():
        if "Function :" in ln:
            cur = ln.split("Function :")[1].strip()
            funcs[cur] = []
        elif cur is not None:
            funcs[cur].append(ln)
    with_dfma = sorted(f for f, body in funcs.items() if any("DFMA" in x for x in body))
    assert funcs, "no SASS functions found"
    assert all("k_cg_check" in f or "k_cg_beta" in f for f in with_dfma), with_dfma


def test_kernel_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.SB200Unavailable):
        sb.bs3_norm2(np.ones(4))
