"""numpy restatement of the reference's CPU implementation of BS1-BS7.

TEST / BASELINE INFRASTRUCTURE ONLY (never imported by the product).  This is
the "reference arm" of bench.py: it reproduces how pkg/src/streambench runs
the hot path -- whole-array numpy expressions with materialised temporaries,
fanned out over contiguous spans on a thread pool (parallel.py:43-69) -- so
the CPU figure reflects the reference's own implementation strategy.  The C
restatement in sb_oracle.c is the fast exact checker; both are pinned to the
reference's golden vectors (tests/test_oracle_golden.py).

Cited reference lines are under /root/reference/pkg/src/streambench/.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


class Pool:
    """parallel.py:13-69: a worker count and contiguous, order-preserving spans."""

    def __init__(self, workers: int | None = None):
        self.workers = max(1, workers or os.cpu_count() or 1)
        self.ex = ThreadPoolExecutor(self.workers) if self.workers > 1 else None

    @staticmethod
    def spans(n: int, parts: int):
        parts = max(1, min(parts, n))
        q, extra = divmod(n, parts)
        out, lo = [], 0
        for i in range(parts):
            hi = lo + q + (i < extra)
            out.append((lo, hi))
            lo = hi
        return out

    def run(self, fn, n: int) -> None:
        if n <= 0:
            return
        sp = self.spans(n, self.workers)
        if self.ex is None or len(sp) == 1:
            fn(0, n)
            return
        for f in [self.ex.submit(fn, lo, hi) for lo, hi in sp]:
            f.result()

    def close(self):
        if self.ex is not None:
            self.ex.shutdown()


def bs1_copy(pool: Pool, x, y) -> None:
    """kernels.py:90-93."""
    def part(lo, hi):
        y[lo:hi] = x[lo:hi]
    pool.run(part, x.shape[0])


def bs2_axpy(pool: Pool, alpha, x, beta, y) -> None:
    """kernels.py:96-103: two rounded products, then a rounded add."""
    def part(lo, hi):
        y[lo:hi] = alpha * x[lo:hi] + beta * y[lo:hi]
    pool.run(part, x.shape[0])


def _fold(rows: np.ndarray) -> np.ndarray:
    """kernels.py:63-69: halve the last axis until two columns remain."""
    k = rows.shape[-1] >> 1
    while k > 1:
        rows[..., :k] += rows[..., k:2 * k]
        k >>= 1
    return rows[..., 0] + rows[..., 1]


def reduce_product(pool: Pool, u, v, bs=256, nb=512) -> float:
    """kernels.py:38-87: lattice accumulation, per-block tree, final block."""
    stride = bs * nb
    n = u.shape[0]
    lat = np.zeros(stride)

    def blocks(b_lo, b_hi):
        lo, hi = b_lo * bs, b_hi * bs
        seg = lat[lo:hi]
        off = 0
        while off + lo < n:
            a = off + lo
            b = min(off + hi, n)
            seg[:b - a] += u[a:b] * v[a:b]
            off += stride

    pool.run(blocks, nb)
    partials = _fold(lat.reshape(nb, bs))
    s = np.zeros(bs)
    for base in range(0, nb, bs):
        m = min(bs, nb - base)
        s[:m] += partials[base:base + m]
    return float(_fold(s))


def bs5_fused_cg_update(pool: Pool, alpha, p, ap, x, r, bs=256, nb=512) -> float:
    """kernels.py:117-132 (the reference's two passes: update, then norm)."""
    def part(lo, hi):
        x[lo:hi] += alpha * p[lo:hi]
        r[lo:hi] -= alpha * ap[lo:hi]
    pool.run(part, x.shape[0])
    return reduce_product(pool, r, r, bs, nb)


def bs6_gather(pool: Pool, row_starts, col_ids, block_starts, q) -> np.ndarray:
    """gs.py:10-39: per row block, step s adds every live row's s-th entry."""
    ng = row_starts.shape[0] - 1
    out = np.zeros(ng)

    def part(b_lo, b_hi):
        r_lo, r_hi = int(block_starts[b_lo]), int(block_starts[b_hi])
        if r_lo == r_hi:
            return
        first = row_starts[r_lo:r_hi].astype(np.int64)
        count = row_starts[r_lo + 1:r_hi + 1].astype(np.int64) - first
        view = out[r_lo:r_hi]
        for s in range(int(count.max())):
            live = count > s
            view[live] += q[col_ids[first[live] + s]]

    pool.run(part, block_starts.shape[0] - 1)
    return out


def bs7_scatter(pool: Pool, ids, q_global, q_local) -> None:
    """gs.py:42-61 (unmasked path; the range check is part of the call)."""
    if ids.size and int(ids.max()) >= q_global.shape[0]:
        raise ValueError("scatter id out of range")

    def part(lo, hi):
        q_local[lo:hi] = q_global[ids[lo:hi]]
    pool.run(part, ids.shape[0])
