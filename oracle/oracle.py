"""ctypes front end for the CPU parity oracle (oracle/sb_oracle.c).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg -- never from the product
package.  Pinned against golden vectors of the unmodified reference in
tests/test_oracle_golden.py (fixtures: tests/golden/, generator:
tests/golden/make_golden.py).

Each wrapper names the reference function it restates (paths relative to
/root/reference/pkg/src/streambench/).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sb_oracle.c")
_LIB = os.path.join(_HERE, "build", "libsboracle.so")

_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, OpenMP spans)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
           "-shared", "-o", _LIB, _SRC]
    subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_get_threads.restype = ctypes.c_int
        L.or_max_threads.restype = ctypes.c_int
        L.or_bs1_copy.argtypes = [_f64p, _f64p, _i64]
        L.or_bs2_axpy.argtypes = [ctypes.c_double, _f64p, ctypes.c_double, _f64p, _i64]
        L.or_reduce_product.argtypes = [_f64p, _f64p, _i64, _i64, _i64, _f64p]
        L.or_bs5_fused_cg_update.argtypes = [ctypes.c_double, _f64p, _f64p, _f64p, _f64p,
                                             _i64, _i64, _i64, _f64p]
        L.or_bs6_gather.argtypes = [_i32p, _i32p, _i64, _f64p, _f64p, _f64p, _i64]
        L.or_bs7_scatter.argtypes = [_i32p, _i64, _f64p, _f64p]
        L.or_build_mesh.argtypes = [_i64, _i64, _i32p]
        L.or_build_gather.argtypes = [_i32p, _i64, _i64, _i64, _i32p, _i32p, _i32p,
                                      ctypes.POINTER(ctypes.c_int64)]
        L.or_build_scatter_ids.argtypes = [_i32p, _i64, _u8p, _i32p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _f64(a):
    a = np.asarray(a)
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise TypeError("oracle expects contiguous float64 arrays")
    return a


def _i32(a):
    a = np.asarray(a)
    if a.dtype != np.int32 or not a.flags.c_contiguous:
        raise TypeError("oracle expects contiguous int32 arrays")
    return a


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def max_threads() -> int:
    return int(lib().or_max_threads())


# --- BS1-BS5 (kernels.py) ---------------------------------------------------

def bs1_copy(x, y) -> None:
    """kernels.py:90-93."""
    x, y = _f64(x), _f64(y)
    assert x.shape == y.shape
    lib().or_bs1_copy(_p(x, _f64p), _p(y, _f64p), x.shape[0])


def bs2_axpy(alpha, x, beta, y) -> None:
    """kernels.py:96-103 (two rounded products, one rounded add)."""
    x, y = _f64(x), _f64(y)
    assert x.shape == y.shape
    lib().or_bs2_axpy(float(alpha), _p(x, _f64p), float(beta), _p(y, _f64p), x.shape[0])


def reduce_product(u, v, block_size=256, n_blocks=512) -> float:
    """kernels.py:38-87 lattice -> tree -> final reduce."""
    u, v = _f64(u), _f64(v)
    assert u.shape == v.shape
    out = ctypes.c_double()
    rc = lib().or_reduce_product(_p(u, _f64p), _p(v, _f64p), u.shape[0], block_size,
                                 n_blocks, ctypes.byref(out))
    if rc:
        raise ValueError(f"oracle reduce_product failed rc={rc}")
    return out.value


def bs3_norm2(x, block_size=256, n_blocks=512) -> float:
    """kernels.py:106-108."""
    return reduce_product(x, x, block_size, n_blocks)


def bs4_dot(x, y, block_size=256, n_blocks=512) -> float:
    """kernels.py:111-114."""
    return reduce_product(x, y, block_size, n_blocks)


def bs5_fused_cg_update(alpha, p, ap, x, r, block_size=256, n_blocks=512) -> float:
    """kernels.py:117-132 (in place on x, r)."""
    p, ap, x, r = _f64(p), _f64(ap), _f64(x), _f64(r)
    out = ctypes.c_double()
    rc = lib().or_bs5_fused_cg_update(float(alpha), _p(p, _f64p), _p(ap, _f64p), _p(x, _f64p),
                                      _p(r, _f64p), x.shape[0], block_size, n_blocks,
                                      ctypes.byref(out))
    if rc:
        raise ValueError(f"oracle bs5 failed rc={rc}")
    return out.value


def cg_solve_diag(d, b, x0, eps, max_iter, block_size=256, n_blocks=512, fused=True, relative=False):
    """cg.py:27-72 with cg.py:75-82's diagonal operator (A v = d * v), on the
    kernels above.  Returns (x, iterations, final_rr, converged) or raises
    ValueError("not SPD ...") where the reference raises NotSPDError."""
    if eps <= 0:
        raise ValueError(f"eps must be positive, got {eps}")
    d, b = _f64(d), _f64(b)
    x = _f64(x0).copy()
    r = b.copy()
    bs2_axpy(-1.0, d * x, 1.0, r)
    p = r.copy()
    rr = bs3_norm2(r, block_size, n_blocks)
    tol = eps * bs3_norm2(b, block_size, n_blocks) if relative else eps
    it = 0
    while rr > tol and it < max_iter:
        ap = d * p
        pap = bs4_dot(p, ap, block_size, n_blocks)
        if pap <= 0.0:
            raise ValueError(f"not SPD: p . Ap = {pap} at iteration {it}")
        alpha = rr / pap
        if fused:
            rr_new = bs5_fused_cg_update(alpha, p, ap, x, r, block_size, n_blocks)
        else:
            bs2_axpy(alpha, p, 1.0, x)
            bs2_axpy(-alpha, ap, 1.0, r)
            rr_new = bs3_norm2(r, block_size, n_blocks)
        beta = rr_new / rr
        bs2_axpy(1.0, r, beta, p)
        rr = rr_new
        it += 1
    return x, it, rr, rr <= tol


# --- exact references (reference.py) ---------------------------------------

def fsum_norm2(x) -> float:
    """reference.py:25-26 (math.fsum of the rounded products)."""
    x = np.asarray(x, dtype=np.float64)
    return math.fsum((x * x).tolist())


def fsum_dot(x, y) -> float:
    """reference.py:29-30."""
    return math.fsum((np.asarray(x) * np.asarray(y)).tolist())


def relative_error(value: float, truth: float) -> float:
    """reference.py:66-69."""
    if truth == 0.0:
        return abs(value)
    return abs(value - truth) / abs(truth)


# --- BS6 / BS7 (gs.py) ------------------------------------------------------

def bs6_gather(row_starts, col_ids, q, carry=None) -> np.ndarray:
    """gs.py:10-39 (row-wise ascending sum from +0.0, or from carry[r])."""
    rs, ci, q = _i32(row_starts), _i32(col_ids), _f64(q)
    ng = rs.shape[0] - 1
    out = np.empty(ng, dtype=np.float64)
    if carry is None:
        lib().or_bs6_gather(_p(rs, _i32p), _p(ci, _i32p), ng, _p(q, _f64p), _p(out, _f64p),
                            None, 0)
    else:
        c = _f64(carry)
        lib().or_bs6_gather(_p(rs, _i32p), _p(ci, _i32p), ng, _p(q, _f64p), _p(out, _f64p),
                            _p(c, _f64p), c.shape[0])
    return out


def bs7_scatter(ids, q_global, q_local) -> None:
    """gs.py:42-61 (masked entries untouched)."""
    ids, qg, ql = _i32(ids), _f64(q_global), _f64(q_local)
    lib().or_bs7_scatter(_p(ids, _i32p), ids.shape[0], _p(qg, _f64p), _p(ql, _f64p))


# --- builders (mesh.py) -----------------------------------------------------

def build_mesh(K: int, p: int) -> np.ndarray:
    """mesh.py:73-97 -> local_to_global (int32, length K^3 (p+1)^3)."""
    nl = K ** 3 * (p + 1) ** 3 if K >= 1 and p >= 1 else 0
    l2g = np.empty(nl, dtype=np.int32)
    rc = lib().or_build_mesh(K, p, _p(l2g, _i32p))
    if rc:
        raise ValueError(f"build_mesh rejected K={K}, p={p}")
    return l2g


def build_gather(l2g, ng: int, nodes_per_block: int = 512):
    """mesh.py:113-147 -> (row_starts, col_ids, block_starts)."""
    l2g = _i32(l2g)
    nl = l2g.shape[0]
    rs = np.empty(ng + 1, dtype=np.int32)
    ci = np.empty(nl, dtype=np.int32)
    bs = np.empty(ng + 1, dtype=np.int32)
    nb = ctypes.c_int64()
    rc = lib().or_build_gather(_p(l2g, _i32p), nl, ng, nodes_per_block, _p(rs, _i32p),
                               _p(ci, _i32p), _p(bs, _i32p), ctypes.byref(nb))
    if rc:
        raise ValueError(f"build_gather failed rc={rc}")
    return rs, ci, bs[: nb.value + 1].copy()


def build_scatter_ids(l2g, ng: int, mask=None) -> np.ndarray:
    """mesh.py:100-110."""
    l2g = _i32(l2g)
    ids = np.empty_like(l2g)
    if mask:
        m = np.zeros(ng, dtype=np.uint8)
        m[np.asarray(sorted(mask), dtype=np.int64)] = 1
        lib().or_build_scatter_ids(_p(l2g, _i32p), l2g.shape[0], _p(m, _u8p), _p(ids, _i32p))
    else:
        lib().or_build_scatter_ids(_p(l2g, _i32p), l2g.shape[0], None, _p(ids, _i32p))
    return ids


def multiplicity(l2g, ng: int) -> np.ndarray:
    """mesh.py:150-153."""
    return np.bincount(np.asarray(l2g), minlength=ng).astype(np.float64)


def uniform(seed_seq, n):
    """harness.py:113-114 / test rand(): np.random.default_rng(seq).uniform(-1,1,n)."""
    return np.random.default_rng(seed_seq).uniform(-1.0, 1.0, n)
