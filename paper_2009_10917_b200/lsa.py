"""Fused multi-GPU BS3/BS4/BS5: the lattice reduction and
the cross-rank combine in ONE kernel over NVLink peer memory.

`LsaReducer` wraps an `sb_lsa_t` context (csrc/sb_lsa.cu): an NCCL 2.28
communicator of its own, a symmetric window of 2 x 128 doubles and a device
communicator with one LSA barrier.  Each call's last CTA stores the rank's
scalar into every peer's window, meets the peers at the barrier and sums
the ranks' values in rank order from +0.0 -- bitwise what dist.DistReducer's
NCCL all-gather + sb_sum_ordered produces, without the separate collective.

Collective semantics: every rank makes the same calls in the same order on
one stream.  Creation needs every rank NVLink-reachable (one node); callers
fall back to DistReducer otherwise.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .kernels import DEFAULT_REDUCTION, ReductionConfig

UID_BYTES = 128


class LsaUnavailable(RuntimeError):
    """The fused path cannot be set up here (NCCL < 2.28, ranks not NVLink peers, ...)."""


def capable(world: int, device) -> str | None:
    """Local, non-collective check that this rank can attempt the fused path;
    None if it can, else why not.  Ranks agree on the answer (all-reduce MIN)
    before the collective setup, so a rank that cannot even try never leaves
    the others waiting inside NCCL.  Assumes the launcher's rank r -> local
    GPU r mapping (one node, torchrun LOCAL_RANK)."""
    dev = torch.device(device)
    if dev.type != "cuda":
        return "not a CUDA device"
    if _lib.lib().sb_lsa_available() != _lib.SB_OK:
        return _lib.last_error()
    n = torch.cuda.device_count()
    if world > n:
        return f"{world} ranks but {n} local GPUs (the fused path needs one NVLink domain)"
    me = dev.index if dev.index is not None else torch.cuda.current_device()
    for j in range(world):
        if j != me and not torch.cuda.can_device_access_peer(me, j):
            return f"GPU {me} has no peer access to GPU {j}"
    return None


def exchange_unique_id(world: int, rank: int, device, group=None) -> bytes:
    """Rank 0's NCCL unique id, broadcast over the torch.distributed group.
    An all-zero id is the "rank 0 failed" sentinel: every rank still joins
    the broadcast and then raises, instead of waiting in it."""
    L = _lib.lib()
    t = torch.zeros(UID_BYTES, dtype=torch.uint8)
    why = ""
    if rank == 0:
        raw = ctypes.create_string_buffer(UID_BYTES)
        if L.sb_lsa_unique_id(raw, UID_BYTES) == _lib.SB_OK:
            t = torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8).clone()
        else:
            why = _lib.last_error()
    if world > 1:
        if dist.get_backend(group) == "nccl":
            td = t.to(torch.device(device))
            dist.broadcast(td, 0, group=group)
            t = td.cpu()
        else:
            dist.broadcast(t, 0, group=group)
    if not bool(t.any()):
        raise LsaUnavailable(f"rank 0 could not create an NCCL unique id {why}".strip())
    return bytes(t.numpy().tobytes())


class LsaReducer:
    def __init__(self, world: int, rank: int, device, group=None, unique_id: bytes | None = None):
        self.L = _lib.lib()
        self.world, self.rank = world, rank
        self.device = torch.device(device)
        if unique_id is None:
            unique_id = self._exchange_uid(group)
        buf = ctypes.create_string_buffer(bytes(unique_id), UID_BYTES)
        h = ctypes.c_void_p()
        rc = self.L.sb_lsa_create(buf, UID_BYTES, world, rank, ctypes.byref(h))
        if rc != _lib.SB_OK:
            raise LsaUnavailable(_lib.last_error())
        self.handle = h
        self._ws = {}

    def _exchange_uid(self, group) -> bytes:
        return exchange_unique_id(self.world, self.rank, self.device, group)

    @staticmethod
    def unique_id() -> bytes:
        raw = ctypes.create_string_buffer(UID_BYTES)
        _lib.check(_lib.lib().sb_lsa_unique_id(raw, UID_BYTES), "sb_lsa_unique_id")
        return raw.raw

    def close(self) -> None:
        """Collective teardown: every rank of the context calls it."""
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.L.sb_lsa_destroy(self.handle)
            self.handle = None

    def abort(self) -> None:
        """Local teardown (ncclCommAbort) when not every rank built its context."""
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.L.sb_lsa_abort(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- BS6 carry halo over NVLink (dist.DistGather.enable_lsa) ----------
    def halo_window(self, nbytes: int) -> None:
        """Collective: register this context's symmetric halo window."""
        _lib.check(self.L.sb_lsa_halo_window(self.handle, int(nbytes)), "sb_lsa_halo_window")

    def halo_pointers(self, offset: int, peer: int) -> tuple[int, int]:
        """(local address, peer's NVLink-mapped address) of `offset` in the halo window."""
        loc, rem = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(self.L.sb_lsa_halo_pointers(self.handle, int(offset), int(peer), ctypes.byref(loc),
                                               ctypes.byref(rem)), "sb_lsa_halo_pointers")
        return int(loc.value), int(rem.value)

    def barrier(self) -> None:
        """Collective LSA barrier on the current stream (one-thread kernel)."""
        _lib.check(self.L.sb_lsa_barrier(self.handle, _lib.stream_handle(self.device)), "sb_lsa_barrier")

    def barrier_advance(self, counter_ptr: int) -> None:
        """The barrier, then +1 on the uint64 call counter at counter_ptr (this
        rank's memory): the BS7 halo buffers' parity, kept on the device."""
        _lib.check(self.L.sb_lsa_barrier_advance(self.handle, counter_ptr, _lib.stream_handle(self.device)),
                   "sb_lsa_barrier_advance")

    # a private zeroed workspace per config (the kernels leave it zeroed)
    def _workspace(self, cfg: ReductionConfig) -> torch.Tensor:
        key = (cfg.block_size, cfg.n_blocks)
        ws = self._ws.get(key)
        if ws is None:
            nbytes = int(self.L.sb_reduce_workspace_bytes(*key))
            ws = self._ws[key] = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        return ws

    def _out(self, out):
        return out if out is not None else torch.empty(1, dtype=torch.float64, device=self.device)

    def bs3_norm2(self, x: torch.Tensor, cfg: ReductionConfig = DEFAULT_REDUCTION, out=None) -> torch.Tensor:
        """kernels.py:106-108 over the ranks' chunks, combined in the same launch."""
        res = self._out(out)
        _lib.check(self.L.sb_lsa_bs3_norm2(x.data_ptr(), x.shape[0], cfg.block_size, cfg.n_blocks,
                                           self._workspace(cfg).data_ptr(), res.data_ptr(), self.handle,
                                           _lib.stream_handle(self.device)), "lsa bs3_norm2")
        return res

    def bs4_dot(self, x: torch.Tensor, y: torch.Tensor, cfg: ReductionConfig = DEFAULT_REDUCTION,
                out=None) -> torch.Tensor:
        res = self._out(out)
        _lib.check(self.L.sb_lsa_bs4_dot(x.data_ptr(), y.data_ptr(), x.shape[0], cfg.block_size, cfg.n_blocks,
                                         self._workspace(cfg).data_ptr(), res.data_ptr(), self.handle,
                                         _lib.stream_handle(self.device)), "lsa bs4_dot")
        return res

    def bs5_fused_cg_update(self, alpha: float, p, ap, x, r, cfg: ReductionConfig = DEFAULT_REDUCTION,
                            out=None) -> torch.Tensor:
        res = self._out(out)
        _lib.check(self.L.sb_lsa_bs5_fused_cg_update(float(alpha), p.data_ptr(), ap.data_ptr(), x.data_ptr(),
                                                     r.data_ptr(), x.shape[0], cfg.block_size, cfg.n_blocks,
                                                     self._workspace(cfg).data_ptr(), res.data_ptr(),
                                                     self.handle, _lib.stream_handle(self.device)),
                   "lsa bs5_fused_cg_update")
        return res
