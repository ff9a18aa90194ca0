"""Helpers shared by the oracle and GPU parity tests: load the golden fixtures
made by tests/golden/make_golden.py and regenerate their seeded inputs."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Golden:
    def __init__(self):
        with open(os.path.join(HERE, "golden.json")) as f:
            self.j = json.load(f)
        self.arrays = dict(np.load(os.path.join(HERE, "arrays.npz")))

    def __getitem__(self, k):
        return self.j[k]


_G = None


def load() -> Golden:
    global _G
    if _G is None:
        _G = Golden()
    return _G


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unhex(s: str) -> float:
    return float.fromhex(s)


def selftest_inputs(n: int):
    """golden 'vectors' records: rng([2024, n]); alpha,beta ~ U(-2,2); x; y; p; ap."""
    rng = np.random.default_rng([2024, n])
    alpha, beta = rng.uniform(-2, 2, 2)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    p, ap = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    return float(alpha), float(beta), x, y, p, ap


def acceptance_inputs(n: int):
    """golden 'cfg_sweep' records (test_acceptance.py:96-110 draw order)."""
    gen = np.random.default_rng([31337, n])
    x = gen.uniform(-1, 1, n)
    y = gen.uniform(-1, 1, n)
    alpha, beta = gen.uniform(-2, 2, 2)
    p, ap = gen.uniform(-1, 1, n), gen.uniform(-1, 1, n)
    return float(alpha), float(beta), x, y, p, ap


def mesh_q_local(K, p, nl):
    return np.random.default_rng([0, K, p]).uniform(-1, 1, nl)


def mesh_q_global(K, p, ng):
    return np.random.default_rng([0, K, p]).uniform(-1, 1, ng)


def cg_inputs(rec):
    """golden 'cg' records: rng(seed); d ~ U(lo, hi); b ~ U(-1, 1); x0 ~ U(-1, 1) or 0."""
    n = rec["n"]
    rng = np.random.default_rng(rec["seed"])
    lo, hi = rec["d_range"]
    d = rng.uniform(lo, hi, n)
    b = rng.uniform(-1, 1, n)
    x0 = rng.uniform(-1, 1, n) if rec["x0_nonzero"] else np.zeros(n)
    assert sha(np.concatenate([d, b, x0])) == rec["in_hash"], "numpy stream changed"
    return d, b, x0
