"""Independent validators used by the harness (the GPU counterpart of reference.py).

pkg/src/streambench/reference.py:1-69 supplies one-pass elementwise
references and compensated (math.fsum) reductions that the reference's
harness checks each kernel against.  Here they run on the device, by a
different method than the kernel under test:

  * copy / axpy / fused-update vectors: torch elementwise ops, one rounded
    operation per kernel launch (bitwise the numpy temporaries);
  * norm2 / dot: double-double accumulation of the rounded products
    (sb_dot_compensated) -- error far below the 1e-12 tolerance, like fsum;
  * gather: torch index_add_ (a scatter-add, i.e. the dense Z^T enumeration
    of reference.gather) compared with allclose like harness.py:211-215;
  * scatter: torch advanced indexing.

These are validation only; they are never timed.
"""

from __future__ import annotations

import torch

from . import _lib


def copy(x: torch.Tensor) -> torch.Tensor:
    """reference.py:17-18."""
    return x.clone()


def axpy(alpha: float, x: torch.Tensor, beta: float, y: torch.Tensor) -> torch.Tensor:
    """reference.py:21-22: alpha*x + beta*y with two rounded products and a rounded add."""
    return torch.add(torch.mul(x, alpha), torch.mul(y, beta))


def _dd_dot(u: torch.Tensor, v: torch.Tensor) -> float:
    dev = u.device
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    ws = _lib.workspace(dev, st, 256, 592)
    res = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(L.sb_dot_compensated(u.data_ptr(), v.data_ptr(), u.shape[0], ws.data_ptr(),
                                    res.data_ptr(), st), "dot_compensated")
    return float(res.item())


def norm2(x: torch.Tensor) -> float:
    """reference.py:25-26 (compensated sum of the rounded squares)."""
    return _dd_dot(x, x)


def dot(x: torch.Tensor, y: torch.Tensor) -> float:
    """reference.py:29-30."""
    return _dd_dot(x, y)


def fused_cg_update(alpha, p, ap, x, r):
    """reference.py:33-38: unfused composition of the two axpy updates + norm."""
    x_new = axpy(alpha, p, 1.0, x)
    r_new = axpy(-alpha, ap, 1.0, r)
    return x_new, r_new, norm2(r_new)


def gather(local_to_global: torch.Tensor, ng: int, q_local: torch.Tensor) -> torch.Tensor:
    """reference.py:41-43: dense enumeration of Z^T (scatter-add)."""
    out = torch.zeros(ng, dtype=torch.float64, device=q_local.device)
    out.index_add_(0, local_to_global.long(), q_local)
    return out


def scatter(ids: torch.Tensor, q_global: torch.Tensor, q_local: torch.Tensor) -> torch.Tensor:
    """reference.py:58-63: masked copy-scatter on a copy."""
    out = q_local.clone()
    keep = ids >= 0
    out[keep] = q_global[ids[keep].long()]
    return out


def relative_error(value: float, truth: float) -> float:
    """reference.py:66-69."""
    if truth == 0.0:
        return abs(value)
    return abs(value - truth) / abs(truth)
