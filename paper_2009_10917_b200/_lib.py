"""ctypes binding of libsb200.so (include/sb200.h) plus device-buffer plumbing.

This is the ONLY compute path of the package: there is no CPU fallback.  If
the library is missing or no CUDA device is visible, every kernel call raises
`SB200Unavailable` loudly.  PyTorch supplies device memory, streams and the
caching allocator; the kernels are ours.
"""

from __future__ import annotations

import ctypes
import functools
import os
import re
import threading

import numpy as np
import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libsb200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "sb200.h")

SB_OK, SB_E_INVALID, SB_E_CUDA, SB_E_RANGE = 0, 1, 2, 3


class SB200Unavailable(RuntimeError):
    """libsb200.so is not built or no CUDA device is present."""


class SB200Error(RuntimeError):
    """A CUDA-side failure reported by libsb200 (SB_E_CUDA)."""


_c_int, _c_i64, _c_dbl, _c_vp, _c_size = (ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                                          ctypes.c_void_p, ctypes.c_size_t)


# name -> (restype, argtypes); mirrors include/sb200.h
_SIGS = {
    "sb_version": (_c_int, []),
    "sb_last_error": (ctypes.c_char_p, []),
    "sb_device_info": (_c_int, [_c_int, _c_vp, _c_vp, _c_vp, _c_vp]),
    "sb_bs1_copy": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp]),
    "sb_bs2_axpy": (_c_int, [_c_dbl, _c_vp, _c_dbl, _c_vp, _c_i64, _c_vp]),
    "sb_reduce_workspace_bytes": (_c_size, [_c_i64, _c_i64]),
    "sb_bs3_norm2": (_c_int, [_c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "sb_bs4_dot": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "sb_bs5_fused_cg_update": (_c_int, [_c_dbl, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64,
                                        _c_i64, _c_vp, _c_vp, _c_vp]),
    "sb_sum_ordered": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp]),
    "sb_bs6_gather": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp,
                               _c_vp, _c_i64, _c_vp]),
    "sb_bs7_scatter": (_c_int, [_c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_int, _c_vp]),
    "sb_bs7_scatter_split": (_c_int, [_c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_int, _c_vp]),
    "sb_bs7_scatter_split_pair": (_c_int, [_c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_vp, _c_i64, _c_vp, _c_vp,
                                           _c_int, _c_vp]),
    "sb_bs7_halo_put": (_c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_vp, _c_vp]),
    "sb_build_l2g": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp]),
    "sb_build_gather_csr": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp,
                                     _c_vp, _c_vp]),
    "sb_build_block_starts": (_c_int, [_c_vp, _c_i64, _c_i64, _c_vp, _c_i64, _c_vp, _c_vp]),
    "sb_multiplicity": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp]),
    "sb_build_scatter_ids": (_c_int, [_c_vp, _c_i64, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "sb_ids_minmax": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp]),
    "sb_dot_compensated": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp, _c_vp]),
    "sb_build_gather_general_temp_bytes": (_c_size, [_c_i64]),
    "sb_build_gather_general": (_c_int, [_c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_size, _c_vp,
                                         _c_vp]),
    "sb_histogram": (_c_int, [_c_vp, _c_i64, _c_i64, _c_vp, _c_vp]),
    "sb_bs6_plan_size": (_c_i64, [_c_i64, _c_i64]),
    "sb_cg_begin": (_c_int, [_c_vp, _c_vp, _c_vp, _c_dbl, _c_i64, _c_vp]),
    "sb_cg_pap": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "sb_cg_update": (_c_int, [_c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp,
                              _c_vp]),
    "sb_cg_direction": (_c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_vp]),
    "sb_lsa_available": (_c_int, []),
    "sb_lsa_unique_id": (_c_int, [_c_vp, _c_size]),
    "sb_lsa_create": (_c_int, [_c_vp, _c_size, _c_int, _c_int, _c_vp]),
    "sb_lsa_destroy": (_c_int, [_c_vp]),
    "sb_lsa_abort": (_c_int, [_c_vp]),
    "sb_lsa_halo_window": (_c_int, [_c_vp, _c_size]),
    "sb_lsa_halo_pointers": (_c_int, [_c_vp, _c_size, _c_int, _c_vp, _c_vp]),
    "sb_lsa_barrier": (_c_int, [_c_vp, _c_vp]),
    "sb_lsa_barrier_advance": (_c_int, [_c_vp, _c_vp, _c_vp]),
    "sb_lsa_cg_pap": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "sb_lsa_cg_update": (_c_int, [_c_int, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp,
                                  _c_vp, _c_vp]),
    "sb_lsa_bs3_norm2": (_c_int, [_c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "sb_lsa_bs4_dot": (_c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "sb_lsa_bs5_fused_cg_update": (_c_int, [_c_dbl, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64,
                                            _c_vp, _c_vp, _c_vp, _c_vp]),
    "sb_bs6_gather_sweep": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_vp, _c_vp, _c_i64,
                                     _c_i64, _c_vp, _c_vp, _c_vp, _c_i64, _c_vp]),
    "sb_bs6_gather_halo": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_vp, _c_vp, _c_i64,
                                    _c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp]),
    "sb_bs6_planned_kernel": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_vp, _c_size]),
    "sb_bs6_gather_tiled": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_vp, _c_vp, _c_i64,
                                     _c_i64, _c_vp, _c_vp, _c_vp, _c_i64, _c_vp]),
    "sb_bs6_sweep_tune": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int]),
    "sb_bs6_make_plan": (_c_int, [_c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_vp]),
    "sb_bs6_gather_planned": (_c_int, [_c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_i64, _c_i64, _c_vp,
                                       _c_vp, _c_vp, _c_i64, _c_vp]),
}

_lib = None
_lock = threading.Lock()


def header_symbols() -> list[str]:
    """Function names declared in include/sb200.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", text)))


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen libsb200.so and declare every signature (no GPU needed)."""
    if not os.path.exists(path):
        raise SB200Unavailable(
            f"{path} is missing: build it with `python -m paper_2009_10917_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib() -> ctypes.CDLL:
    """The loaded library, requiring a CUDA device (raises otherwise)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not torch.cuda.is_available():
                    raise SB200Unavailable("no CUDA device visible: the sb200 kernels need a B200 "
                                           "(sm_100a); there is no CPU fallback")
                _lib = load_library(os.environ.get("SB200_LIB", LIB_PATH))  # (A/B builds)
    return _lib


def last_error() -> str:
    msg = lib().sb_last_error()
    return msg.decode() if msg else ""


def check(rc: int, name: str) -> None:
    if rc == SB_OK:
        return
    msg = last_error()
    if rc in (SB_E_INVALID, SB_E_RANGE):
        raise ValueError(f"{name}: {msg}")
    raise SB200Error(f"{name}: {msg}")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device: torch.device | None = None) -> int:
    """cudaStream_t of torch's current stream on `device` (the raw lookup is
    ~10x cheaper than building a torch.cuda.Stream object per call)."""
    if _raw_stream is not None:
        if device is None:
            return _raw_stream(torch.cuda.current_device())
        idx = device.index if isinstance(device, torch.device) else device
        return _raw_stream(torch.cuda.current_device() if idx is None else idx)
    return torch.cuda.current_stream(device).cuda_stream


# ---- reduction workspaces --------------------------------------------------
# One zero-initialised workspace per (device, stream, block_size, n_blocks);
# the kernels leave it zeroed, so calls ordered on one stream can share it.
_workspaces: dict = {}


def workspace(device: torch.device, stream: int, bs: int, nb: int) -> torch.Tensor:
    key = (device.index, stream, bs, nb)
    ws = _workspaces.get(key)
    if ws is None:
        nbytes = int(lib().sb_reduce_workspace_bytes(bs, nb))
        if nbytes == 0:
            raise ValueError(f"invalid reduction config ({bs}, {nb})")
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _workspaces[key] = ws
    return ws


# ---- argument staging ------------------------------------------------------

class Staged:
    """A kernel argument on the device, remembering where it came from.

    Device tensors pass through untouched.  Host arrays (numpy or CPU torch)
    are copied H2D (non-blocking from pinned memory); `writeback()` copies an
    in-place output back, so the reference's in-place numpy semantics hold.
    """

    __slots__ = ("dev", "host", "kind")

    def __init__(self, dev, host, kind):
        self.dev, self.host, self.kind = dev, host, kind

    def writeback(self) -> None:
        if self.kind == "numpy":
            torch.from_numpy(self.host).copy_(self.dev, non_blocking=False)
        elif self.kind == "cpu":
            self.host.copy_(self.dev, non_blocking=False)


def stage(a, dtype: torch.dtype, name: str, device: torch.device | None = None) -> Staged:
    lib()  # no device / no library -> SB200Unavailable before any staging
    if isinstance(a, torch.Tensor):
        if a.dtype != dtype:
            raise TypeError(f"{name}: expected {dtype}, got {a.dtype}")
        if a.dim() != 1:
            raise ValueError(f"expected a 1-D vector, got shape {tuple(a.shape)}")
        if a.is_cuda:
            if not a.is_contiguous():
                raise ValueError(f"{name}: device vectors must be contiguous")
            return Staged(a, None, "cuda")
        dev = a.to(device or torch.device("cuda", torch.cuda.current_device()), non_blocking=True)
        return Staged(dev, a, "cpu")
    arr = np.asarray(a)
    np_dtype = np.float64 if dtype == torch.float64 else np.int32
    if arr.dtype != np_dtype:
        raise TypeError(f"{name}: expected {np_dtype}, got {arr.dtype}")
    if arr.ndim != 1:
        raise ValueError(f"expected a 1-D vector, got shape {arr.shape}")
    if not arr.flags.c_contiguous:
        raise ValueError(f"{name}: host vectors must be contiguous")
    dev = torch.from_numpy(arr).to(device or torch.device("cuda", torch.cuda.current_device()),
                                   non_blocking=True)
    return Staged(dev, arr, "numpy")


def length(a) -> int:
    return int(a.shape[0])


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


# ---- device guard ----------------------------------------------------------
# libsb200 launches on (and sizes grids for) the CURRENT device; torch lets a
# caller compute on tensors of any device.  Public entry points therefore run
# with the current device switched to their operands' device when it differs.

def _cuda_index(a):
    if isinstance(a, torch.Tensor):
        return a.device.index if a.is_cuda else None
    for attr in ("row_starts", "ids", "local_to_global"):  # GatherOp, ScatterIds, MeshConnectivity
        t = getattr(a, attr, None)
        if isinstance(t, torch.Tensor) and t.is_cuda:
            return t.device.index
    return None


def device_guard(fn):
    @functools.wraps(fn)
    def guarded(*args, **kw):
        for a in args:
            d = _cuda_index(a)
            if d is not None:
                break
        else:
            d = None
            for a in kw.values():
                d = _cuda_index(a)
                if d is not None:
                    break
        if d is None or d == torch.cuda.current_device():
            return fn(*args, **kw)
        with torch.cuda.device(d):
            return fn(*args, **kw)
    return guarded
