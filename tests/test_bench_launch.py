"""bench.py owns its rank launch: `--gpus N` outside a
launcher starts N processes through torch.distributed.run; under a launcher
the world size must match --gpus.  CPU-only (--dry-run: rendezvous + pids,
no GPU work)."""

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=180):
    env = dict(os.environ, SB200_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, env=env,
                          timeout=timeout, cwd=ROOT)


def _json_line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_gpus2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    j = _json_line(r.stdout)
    assert j["n_gpus"] == 2 and j["self_launched"]
    pids = {x["pid"] for x in j["ranks"]}
    assert len(pids) == 2 and os.getpid() not in pids
    assert sorted(x["rank"] for x in j["ranks"]) == [0, 1]


def test_gpus1_runs_in_process():
    r = _run(["--gpus", "1", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    j = _json_line(r.stdout)
    assert j["n_gpus"] == 1 and not j["self_launched"]


def test_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "2", "--dry-run"], {"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=3" in r.stderr


def test_setup_deadline_gives_up():
    """The fused-collective setup runs under a deadline (dist._create_with_deadline)."""
    sys.path.insert(0, ROOT)
    from paper_2009_10917_b200.dist import _create_with_deadline

    t0 = time.perf_counter()
    obj, why = _create_with_deadline(lambda: time.sleep(30), 0.5, RuntimeError)
    assert obj is None and "did not finish" in why and time.perf_counter() - t0 < 5

    def refuse():
        raise RuntimeError("NCCL < 2.28")
    assert _create_with_deadline(refuse, 5, RuntimeError) == (None, "NCCL < 2.28")
    assert _create_with_deadline(lambda: 7, 5, RuntimeError) == (7, None)


def test_strong_scaling_sizes():
    """--strong: the global vector is split in rank chunks and the global mesh
    in slabs (C4: n = 1e9 on 8 GPUs; C5: K = 143, 18 x 7 + 17 layers)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2009_10917_b200.dist import SlabPartition, global_mesh_k
    from paper_2009_10917_b200.parallel import split_range
    a = bench.parse_args(["--gpus", "8", "--strong", "--dofs", "1e9", "--mesh-k", "143"])
    assert a.strong and int(a.n) == 10 ** 9 and a.K == 143
    assert global_mesh_k(143, 8, True) == 143 and global_mesh_k(66, 8, False) == 132
    assert [hi - lo for lo, hi in split_range(int(a.n), 8)] == [125_000_000] * 8
    part = SlabPartition(143, 7, 8)
    assert [z1 - z0 for z0, z1 in (part.layers(r) for r in range(8))] == [18] * 7 + [17]
    assert not bench.parse_args([]).strong
