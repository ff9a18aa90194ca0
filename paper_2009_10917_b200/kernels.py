"""BS1-BS5: copy, axpy, norm, dot, fused CG update on the B200.

Drop-in for pkg/src/streambench/kernels.py: same names, argument order,
in-place semantics, ReductionConfig validation and ValueError behaviour.
Every call runs one hand-written sm_100a kernel from libsb200.so
(include/sb200.h); reductions reproduce the reference lattice schedule
(kernels.py:38-87) bit for bit for any ReductionConfig.

Arguments may be CUDA float64 tensors (the fast path: no copies) or host
arrays (numpy / CPU torch), which are staged to the current device and, for
in-place outputs, written back -- so code written against the reference's
numpy API runs unchanged.

Reductions return a Python float like the reference (one device->host sync
per call).  The `*_async` variants return the 1-element device tensor
instead, for timed loops and device-resident solvers.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib, hoststream
from .core import DVector, check_same_length


@dataclass(frozen=True)
class ReductionConfig:
    """kernels.py:19-32: shape of the two-stage reduction (lattice, not CUDA, shape)."""

    block_size: int = 256
    n_blocks: int = 512

    def __post_init__(self):
        b = self.block_size
        if b < 2 or (b & (b - 1)) != 0:
            raise ValueError(f"block_size must be a power of two >= 2, got {b}")
        if self.n_blocks < 1:
            raise ValueError(f"n_blocks must be >= 1, got {self.n_blocks}")


DEFAULT_REDUCTION = ReductionConfig()

# A lattice shaped for the B200 rather than for the paper's GPUs: 1184 = 8 x 148
# CTAs of 256 slots fill every SM with two resident CTAs and give 303k
# independent in-order chains.  Parity is per config, so results are bitwise
# equal to the reference's kernels.bs3_norm2(x, B200_REDUCTION).
B200_REDUCTION = ReductionConfig(block_size=256, n_blocks=1184)


def _all_cuda(*vs) -> bool:
    return all(isinstance(v, torch.Tensor) and v.is_cuda for v in vs)


_F64 = torch.float64


def _fast_vecs(*vs):
    """Device of the arguments when they are all contiguous 1-D float64 CUDA
    tensors of one length on one device (the hot path), else None -- the
    caller then runs the full checks, which raise the reference's errors."""
    v0 = vs[0]
    if type(v0) is not torch.Tensor or not v0.is_cuda:
        return None
    dev, n = v0.device, v0.shape
    for v in vs:
        if (type(v) is not torch.Tensor or v.dtype is not _F64 or v.shape != n or len(n) != 1
                or not v.is_cuda or v.device != dev or not v.is_contiguous()):
            return None
    return dev


def _span(v):
    """(start, end) byte range of a vector's data, or None when unknown."""
    if isinstance(v, torch.Tensor):
        return (v.data_ptr(), v.data_ptr() + v.numel() * v.element_size()) if v.numel() else None
    try:
        import numpy as np
        a = np.asarray(v)
        if a.size == 0:
            return None
        lo, hi = np.byte_bounds(a) if hasattr(np, "byte_bounds") else np.lib.array_utils.byte_bounds(a)
        return (lo, hi)
    except Exception:  # noqa: BLE001 -- not array-like: no aliasing to report
        return None


def _aliasing(outs, ins) -> str:
    """How output vectors overlap the other arguments: "none", "same" (only
    identical vectors: same address and length), or "partial"."""
    kind = "none"
    allv = list(outs) + list(ins)
    for i, o in enumerate(outs):
        so = _span(o)
        if so is None:
            continue
        for j, v in enumerate(allv):
            if j == i:
                continue
            sv = _span(v)
            if sv is None or sv[1] <= so[0] or so[1] <= sv[0]:
                continue
            kind = "same" if (sv == so and kind != "partial") else "partial"
    return kind


def _stage_all(names, vs):
    dev = None
    for v in vs:
        if isinstance(v, torch.Tensor) and v.is_cuda:
            dev = v.device
            break
    return [_lib.stage(v, torch.float64, n, dev) for n, v in zip(names, vs)]


def _check_vec(v, name):
    if v.dtype != torch.float64:
        raise TypeError(f"{name}: expected float64, got {v.dtype}")
    if v.dim() != 1:
        raise ValueError(f"expected a 1-D vector, got shape {tuple(v.shape)}")
    if not v.is_contiguous():
        raise ValueError(f"{name}: vectors must be contiguous")


def _same_device(*vs) -> torch.device:
    dev = vs[0].device
    for v in vs[1:]:
        if v.device != dev:
            raise ValueError(f"vectors on different devices: {dev} vs {v.device}")
    return dev


def _result(dev, out):
    if out is None:
        return torch.empty(1, dtype=torch.float64, device=dev)
    if not (out.is_cuda and out.dtype is _F64 and out.numel() >= 1 and out.device == dev):
        raise ValueError("out must be a float64 device tensor on the inputs' device")
    return out


# ---- BS1 -------------------------------------------------------------------

@_lib.device_guard
def bs1_copy(x, y) -> None:
    """kernels.py:90-93: y = x (in place).  Overlapping (non-identical) x and
    y copy through a temporary, as numpy's slice assignment does."""
    dev = _fast_vecs(x, y)
    if dev is not None:
        px, py = x.data_ptr(), y.data_ptr()
        if px != py and abs(px - py) < 8 * x.shape[0]:
            x = x.clone()
        _lib.check(_lib.lib().sb_bs1_copy(x.data_ptr(), y.data_ptr(), x.shape[0], _lib.stream_handle(dev)),
                   "bs1_copy")
        return
    check_same_length(x, y)
    if _aliasing((y,), (x,)) == "partial":
        x = x.clone() if isinstance(x, torch.Tensor) else x.copy()
    if _all_cuda(x, y):
        _check_vec(x, "x"); _check_vec(y, "y")
        dev = _same_device(x, y)
        L = _lib.lib()
        _lib.check(L.sb_bs1_copy(x.data_ptr(), y.data_ptr(), x.shape[0], _lib.stream_handle(dev)),
                   "bs1_copy")
        return
    if hoststream.all_host(x, y):
        hx, hy = hoststream.as_host_tensor(x, "x"), hoststream.as_host_tensor(y, "y")
        hoststream.run(hx.shape[0], {"x": hx}, {"y": hy}, ("y",),
                       lambda d, lo, hi: bs1_copy(d["x"][lo:hi], d["y"][lo:hi]))
        return
    sx, sy = _stage_all(("x", "y"), (x, y))
    bs1_copy(sx.dev, sy.dev)
    sy.writeback()


# ---- BS2 -------------------------------------------------------------------

@_lib.device_guard
def bs2_axpy(alpha: float, x, beta: float, y) -> None:
    """kernels.py:96-103: y = alpha*x + beta*y, one rounded multiply-add pair per element.
    x may be y (elementwise); partially overlapping x and y go through a copy of x
    (the reference evaluates alpha*x into a temporary first)."""
    dev = _fast_vecs(x, y)
    if dev is not None:
        px, py = x.data_ptr(), y.data_ptr()
        if px != py and abs(px - py) < 8 * x.shape[0]:
            x = x.clone()
        _lib.check(_lib.lib().sb_bs2_axpy(float(alpha), x.data_ptr(), float(beta), y.data_ptr(), x.shape[0],
                                          _lib.stream_handle(dev)), "bs2_axpy")
        return
    check_same_length(x, y)
    if _aliasing((y,), (x,)) == "partial":
        x = x.clone() if isinstance(x, torch.Tensor) else x.copy()
    if _all_cuda(x, y):
        _check_vec(x, "x"); _check_vec(y, "y")
        dev = _same_device(x, y)
        L = _lib.lib()
        _lib.check(L.sb_bs2_axpy(float(alpha), x.data_ptr(), float(beta), y.data_ptr(), x.shape[0],
                                 _lib.stream_handle(dev)), "bs2_axpy")
        return
    if hoststream.all_host(x, y) and x is not y:
        hx, hy = hoststream.as_host_tensor(x, "x"), hoststream.as_host_tensor(y, "y")
        hoststream.run(hx.shape[0], {"x": hx, "y": hy}, {"y": hy}, (),
                       lambda d, lo, hi: bs2_axpy(alpha, d["x"][lo:hi], beta, d["y"][lo:hi]))
        return
    if x is y:
        sx = _lib.stage(x, torch.float64, "x")
        sy = sx
    else:
        sx, sy = _stage_all(("x", "y"), (x, y))
    bs2_axpy(alpha, sx.dev, beta, sy.dev)
    sy.writeback()


# ---- BS3 / BS4 / BS5 -------------------------------------------------------

def _cfg(cfg: ReductionConfig) -> ReductionConfig:
    if not isinstance(cfg, ReductionConfig):
        raise TypeError("cfg must be a ReductionConfig")
    return cfg


@_lib.device_guard
def bs3_norm2_async(x: DVector, cfg: ReductionConfig = DEFAULT_REDUCTION, out=None) -> torch.Tensor:
    """bs3_norm2 leaving the scalar on the device (no host sync)."""
    cfg = _cfg(cfg)
    dev = _fast_vecs(x)
    if dev is None:
        _check_vec(x, "x")
        dev = x.device
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    ws = _lib.workspace(dev, st, cfg.block_size, cfg.n_blocks)
    res = _result(dev, out)
    _lib.check(L.sb_bs3_norm2(x.data_ptr(), x.shape[0], cfg.block_size, cfg.n_blocks, ws.data_ptr(),
                              res.data_ptr(), st), "bs3_norm2")
    return res


@_lib.device_guard
def bs3_norm2(x, cfg: ReductionConfig = DEFAULT_REDUCTION) -> float:
    """kernels.py:106-108: sum(x[i]^2) via the fixed two-stage schedule."""
    if not _all_cuda(x):
        hx = hoststream.as_host_tensor(x, "x")
        return float(hoststream.run(hx.shape[0], {"x": hx}, {}, (),
                                    final_fn=lambda d: bs3_norm2_async(d["x"], cfg)).item())
    return float(bs3_norm2_async(x, cfg).item())


@_lib.device_guard
def bs4_dot_async(x: DVector, y: DVector, cfg: ReductionConfig = DEFAULT_REDUCTION,
                  out=None) -> torch.Tensor:
    cfg = _cfg(cfg)
    dev = _fast_vecs(x, y)
    if dev is None:
        check_same_length(x, y)
        _check_vec(x, "x"); _check_vec(y, "y")
        dev = _same_device(x, y)
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    ws = _lib.workspace(dev, st, cfg.block_size, cfg.n_blocks)
    res = _result(dev, out)
    _lib.check(L.sb_bs4_dot(x.data_ptr(), y.data_ptr(), x.shape[0], cfg.block_size, cfg.n_blocks,
                            ws.data_ptr(), res.data_ptr(), st), "bs4_dot")
    return res


@_lib.device_guard
def bs4_dot(x, y, cfg: ReductionConfig = DEFAULT_REDUCTION) -> float:
    """kernels.py:111-114: sum(x[i]*y[i]) via the fixed two-stage schedule."""
    check_same_length(x, y)
    if hoststream.all_host(x, y):
        hx, hy = hoststream.as_host_tensor(x, "x"), hoststream.as_host_tensor(y, "y")
        return float(hoststream.run(hx.shape[0], {"x": hx, "y": hy}, {}, (),
                                    final_fn=lambda d: bs4_dot_async(d["x"], d["y"], cfg)).item())
    if not _all_cuda(x, y):
        sx, sy = _stage_all(("x", "y"), (x, y))
        x, y = sx.dev, sy.dev
    return float(bs4_dot_async(x, y, cfg).item())


@_lib.device_guard
def bs5_fused_cg_update_async(alpha: float, p: DVector, ap: DVector, x: DVector, r: DVector,
                              cfg: ReductionConfig = DEFAULT_REDUCTION, out=None) -> torch.Tensor:
    cfg = _cfg(cfg)
    dev = _fast_vecs(p, ap, x, r)
    if dev is not None:
        n8 = 8 * x.shape[0]
        pp, pa, px, pr = p.data_ptr(), ap.data_ptr(), x.data_ptr(), r.data_ptr()
        if (abs(px - pr) < n8 or abs(px - pp) < n8 or abs(px - pa) < n8 or abs(pr - pp) < n8
                or abs(pr - pa) < n8):
            return _bs5_sequential(alpha, p, ap, x, r, cfg, out)
    elif _aliasing((x, r), (p, ap)) != "none":
        return _bs5_sequential(alpha, p, ap, x, r, cfg, out)
    if dev is None:
        check_same_length(p, ap, x, r)
        for v, nm in ((p, "p"), (ap, "ap"), (x, "x"), (r, "r")):
            _check_vec(v, nm)
        dev = _same_device(p, ap, x, r)
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    ws = _lib.workspace(dev, st, cfg.block_size, cfg.n_blocks)
    res = _result(dev, out)
    _lib.check(L.sb_bs5_fused_cg_update(float(alpha), p.data_ptr(), ap.data_ptr(), x.data_ptr(),
                                        r.data_ptr(), x.shape[0], cfg.block_size, cfg.n_blocks,
                                        ws.data_ptr(), res.data_ptr(), st), "bs5_fused_cg_update")
    return res


def _bs5_sequential(alpha, p, ap, x, r, cfg, out=None):
    """BS5 with aliased vectors: the reference's own order
    (kernels.py:127-131) -- x += alpha*p over the whole vector, then
    r -= alpha*ap, then the BS3 lattice over r -- as BS2, BS2, BS3 launches
    (bitwise the fused kernel when nothing aliases: (-alpha)*ap + r == r - alpha*ap).
    Only identical vectors may alias; partial overlaps are rejected."""
    if _aliasing((x, r), (p, ap)) == "partial":
        raise ValueError("bs5_fused_cg_update: vectors overlap without being identical")
    check_same_length(p, ap, x, r)
    bs2_axpy(alpha, p, 1.0, x)
    bs2_axpy(-alpha, ap, 1.0, r)
    if _all_cuda(r):
        return bs3_norm2_async(r, cfg, out)
    return torch.tensor([bs3_norm2(r, cfg)], dtype=torch.float64)


@_lib.device_guard
def bs5_fused_cg_update(alpha: float, p, ap, x, r,
                        cfg: ReductionConfig = DEFAULT_REDUCTION) -> float:
    """kernels.py:117-132: x += alpha*p; r -= alpha*ap; returns sum(r_new^2).

    Genuinely single-pass on the device (48 B/element), same lattice as BS3.
    Aliased arguments (x is r, p is x, ...) follow the reference's sequential
    order instead (_bs5_sequential).
    """
    check_same_length(p, ap, x, r)
    if _aliasing((x, r), (p, ap)) != "none":
        return float(_bs5_sequential(alpha, p, ap, x, r, _cfg(cfg)).item())
    if _all_cuda(p, ap, x, r):
        return float(bs5_fused_cg_update_async(alpha, p, ap, x, r, cfg).item())
    if hoststream.all_host(p, ap, x, r):
        # Chunked: per chunk the two rounded updates (bitwise BS5's vectors, SPEC
        # fusion equivalence); the scalar is the BS3 lattice over the assembled
        # r_new on the device -- bitwise the fused kernel's (test_kernels.py:194-199).
        h = {k: hoststream.as_host_tensor(v, k) for k, v in (("p", p), ("ap", ap), ("x", x), ("r", r))}

        def chunk(d, lo, hi):
            bs2_axpy(alpha, d["p"][lo:hi], 1.0, d["x"][lo:hi])
            bs2_axpy(-alpha, d["ap"][lo:hi], 1.0, d["r"][lo:hi])

        res = hoststream.run(h["x"].shape[0], h, {"x": h["x"], "r": h["r"]}, (), chunk,
                             final_fn=lambda d: bs3_norm2_async(d["r"], cfg))
        return float(res.item())
    staged = _stage_all(("p", "ap", "x", "r"), (p, ap, x, r))
    res = bs5_fused_cg_update_async(alpha, *(s.dev for s in staged), cfg)
    staged[2].writeback()
    staged[3].writeback()
    return float(res.item())
