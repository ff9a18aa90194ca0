"""bench.py --gpus 2 launches and times two ranks itself.
On a one-GPU box both ranks share cuda:0 over gloo (SB200_DIST_BACKEND=gloo,
host-staged exchanges): a functional check of the multi-rank bench path."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_line():
    env = dict(os.environ, SB200_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--dofs", "2e6", "--mesh-k", "12", "--order", "3"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["scaling"] == "weak"
    assert [x["rank"] for x in j["per_rank"]] == [0, 1]
    assert all(x["ms_per_step"] > 0 for x in j["per_rank"])
    assert j["ms_per_step"] == pytest.approx(max(x["ms_per_step"] for x in j["per_rank"]), rel=1e-3)
    assert "gloo" in j["config"]["collective"]
    assert j["aggregate_peak_GBps"] > 0 and j["value"] > 0
