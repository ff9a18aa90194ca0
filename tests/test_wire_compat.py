"""the reference's own tools consume the B200 sweep output
unchanged -- `streambench fit` (cli.py) parses profiles/r01_sweep.csv (written
by scripts/sweep.py on the B200) and the plot frontend's readers
(pkg/frontend/src/streambench_plots/io.py) load both the CSV and the fit JSON.
Runs only where the reference tree exists (the build container)."""

import importlib.util
import json
import os
import subprocess
import sys

import pytest

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSV = os.path.join(ROOT, "profiles", "r01_sweep.csv")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")


def test_reference_cli_and_frontend_read_b200_sweep(tmp_path):
    env = dict(os.environ, PYTHONPATH=os.path.join(REF, "src"))
    out = subprocess.run([sys.executable, "-m", "streambench", "fit", CSV], capture_output=True, text=True,
                         env=env, cwd=str(tmp_path), timeout=120)
    assert out.returncode == 0, out.stderr
    fits = json.loads(out.stdout)
    tests = {f["test"] for f in fits}
    assert tests == {"bs1", "bs2", "bs3", "bs4", "bs5", "bs6", "bs7"}
    assert len([f for f in fits if f["test"] == "bs6"]) == 15  # one fit per order N=1..15
    fpath = tmp_path / "fits.json"
    fpath.write_text(out.stdout)
    spec = importlib.util.spec_from_file_location("sb_plots_io",
                                                  os.path.join(REF, "frontend/src/streambench_plots/io.py"))
    io = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(io)
    samples = io.read_samples(CSV)
    assert len(samples) == sum(1 for _ in open(CSV)) - 1
    assert len(io.read_fits(str(fpath))) == len(fits)
