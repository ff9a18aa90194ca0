"""Independent validators (reference.py of the reference package).

pkg/src/streambench/reference.py:1-69 supplies one-pass elementwise
references and compensated (math.fsum) reductions that the harness checks
each kernel against.  The same names and signatures here, for both kinds of
caller:

  * numpy (or CPU torch) arguments -- the reference's own definitions, on
    the host: reference-style code and the reference's test suite get exactly
    what they expect (numpy results, fsum reductions);
  * CUDA tensors -- the device counterparts the GPU harness uses, computed by
    a different method than the kernel under test:
      - copy / axpy / fused-update vectors: torch elementwise ops, one rounded
        operation per launch (bitwise the numpy temporaries);
      - norm2 / dot: double-double accumulation of the rounded products
        (sb_dot_compensated) -- error far below the 1e-12 tolerance, like fsum;
      - gather: torch index_add_ (the dense Z^T enumeration of
        reference.gather), compared with allclose like harness.py:211-215;
      - gather_rowwise: one masked torch step per row position, so every row
        is summed in stored column order (bitwise the sequential loop);
      - scatter: torch advanced indexing.

These are validation only; they are never timed.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib


def _dev(*arrays) -> bool:
    return any(isinstance(a, torch.Tensor) and a.is_cuda for a in arrays)


def _np(a):
    return a.numpy() if isinstance(a, torch.Tensor) else a


def copy(x):
    """reference.py:17-18."""
    return x.clone() if _dev(x) else _np(x).copy()


def axpy(alpha: float, x, beta: float, y):
    """reference.py:21-22: alpha*x + beta*y with two rounded products and a rounded add."""
    if _dev(x, y):
        return torch.add(torch.mul(x, alpha), torch.mul(y, beta))
    return alpha * _np(x) + beta * _np(y)


def _dd_dot(u: torch.Tensor, v: torch.Tensor) -> float:
    dev = u.device
    L = _lib.lib()
    with torch.cuda.device(dev):
        st = _lib.stream_handle(dev)
        ws = _lib.workspace(dev, st, 256, 592)
        res = torch.empty(1, dtype=torch.float64, device=dev)
        _lib.check(L.sb_dot_compensated(u.data_ptr(), v.data_ptr(), u.shape[0], ws.data_ptr(),
                                        res.data_ptr(), st), "dot_compensated")
        return float(res.item())


def norm2(x) -> float:
    """reference.py:25-26 (compensated sum of the rounded squares)."""
    if _dev(x):
        return _dd_dot(x, x)
    x = _np(x)
    return math.fsum((x * x).tolist())


def dot(x, y) -> float:
    """reference.py:29-30."""
    if _dev(x, y):
        return _dd_dot(x, y)
    return math.fsum((_np(x) * _np(y)).tolist())


def fused_cg_update(alpha, p, ap, x, r):
    """reference.py:33-38: unfused composition of the two axpy updates + norm."""
    x_new = axpy(alpha, p, 1.0, x)
    r_new = axpy(-alpha, ap, 1.0, r)
    return x_new, r_new, norm2(r_new)


def gather(local_to_global, ng: int, q_local):
    """reference.py:41-43: dense enumeration of Z^T (scatter-add)."""
    if _dev(local_to_global, q_local):
        out = torch.zeros(ng, dtype=torch.float64, device=q_local.device)
        out.index_add_(0, local_to_global.long(), q_local)
        return out
    return np.bincount(_np(local_to_global), weights=_np(q_local), minlength=ng)


def gather_rowwise(row_starts, col_ids, q_local):
    """reference.py:46-55: per-row CSR sum in stored column order from +0.0."""
    if _dev(row_starts, col_ids, q_local):
        rs = row_starts.long()
        lens = rs[1:] - rs[:-1]
        out = torch.zeros(lens.shape[0], dtype=torch.float64, device=q_local.device)
        for j in range(int(lens.max().item()) if lens.numel() else 0):
            rows = torch.nonzero(lens > j).squeeze(1)
            out[rows] = out[rows] + q_local[col_ids[rs[rows] + j].long()]
        return out
    row_starts, col_ids, q_local = _np(row_starts), _np(col_ids), _np(q_local)
    out = np.zeros(row_starts.shape[0] - 1, dtype=np.float64)
    for r in range(out.shape[0]):
        acc = 0.0
        for c in range(row_starts[r], row_starts[r + 1]):
            acc += q_local[col_ids[c]]
        out[r] = acc
    return out


def scatter(ids, q_global, q_local):
    """reference.py:58-63: masked copy-scatter on a copy."""
    if _dev(ids, q_global, q_local):
        out = q_local.clone()
        keep = ids >= 0
        out[keep] = q_global[ids[keep].long()]
        return out
    ids, q_global = _np(ids), _np(q_global)
    out = _np(q_local).copy()
    keep = ids >= 0
    out[keep] = q_global[ids[keep]]
    return out


def relative_error(value: float, truth: float) -> float:
    """reference.py:66-69."""
    if truth == 0.0:
        return abs(value)
    return abs(value - truth) / abs(truth)
