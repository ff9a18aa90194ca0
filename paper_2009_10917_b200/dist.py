"""Multi-GPU BS1-BS7: slab partition + NCCL exchanges (one process per GPU).

New capability relative to the reference (which is single-process; SURVEY
§2.2, §8e): the seven streaming tests across the GPUs of one node, launched
by torchrun with torch.distributed over NCCL.

Vectors (BS1-BS5): contiguous chunks, the reference's span split
(parallel.py:43-53) with exactly one span per rank.  BS1/BS2 need no
communication.  BS3/BS4/BS5 reduce the local chunk on the rank's lattice
(same ReductionConfig), all-gather the one-double partials (NCCL) and sum
them in rank order from +0.0 on the device (sb_sum_ordered): deterministic
for a fixed world size and identical on every rank; <= 1e-12 relative to the
exact sum like the reference's own tolerance (test_kernels.py:135-139).  It
is not bitwise the 1-GPU lattice (that would serialise the slot chains).

Mesh (BS6/BS7): z-slabs of element layers, layer counts by the same span
split (K=143 over 8 ranks -> 18,...,18,17).  Rank r owns the global rows of
planes [z0*p, z1*p) (the last rank also the top plane z1*p).
  BS6, bitwise equal to the 1-GPU gather: every element of rank r has a
  smaller element id -- hence smaller local index -- than every element of
  rank r+1, so an interface row's ascending sum is (rank r's terms) then
  (rank r+1's terms).  Rank r gathers the partial sums of its top plane and
  sends them to r+1 ("carry"), which seeds those rows' accumulators with them
  (sb_bs6_gather* carry_in) and continues in order.
  BS7: rank r needs q_global of its top plane, owned by r+1: a one-plane halo
  sent from r+1 to r before the scatter.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .parallel import split_range


# ---------------------------------------------------------------- partitions

def rank_span(n: int, world: int, rank: int) -> tuple[int, int]:
    """parallel.py:43-53 with exactly `world` (possibly empty) contiguous spans."""
    step, extra = divmod(n, world)
    lo = rank * step + min(rank, extra)
    return lo, lo + step + (1 if rank < extra else 0)


@dataclass(frozen=True)
class SlabPartition:
    """z-slab partition of the K^3 order-p mesh over `world` ranks."""

    K: int
    p: int
    world: int

    def __post_init__(self):
        if self.world < 1 or self.world > self.K:
            raise ValueError(f"need 1 <= world <= K, got world={self.world}, K={self.K}")

    @property
    def g(self) -> int:
        return self.K * self.p + 1

    @property
    def plane(self) -> int:
        """Rows (global DOFs) per lattice plane."""
        return self.g * self.g

    @property
    def npe3(self) -> int:
        return (self.p + 1) ** 3

    def layers(self, rank: int) -> tuple[int, int]:
        spans = split_range(self.K, self.world)
        return spans[rank]

    def own_planes(self, rank: int) -> tuple[int, int]:
        z0, z1 = self.layers(rank)
        top = z1 * self.p + (1 if rank == self.world - 1 else 0)
        return z0 * self.p, top

    def send_plane(self, rank: int):
        """Plane whose partials rank sends up (None for the last rank)."""
        return None if rank == self.world - 1 else self.layers(rank)[1] * self.p

    def nl(self, rank: int) -> int:
        z0, z1 = self.layers(rank)
        return self.K * self.K * (z1 - z0) * self.npe3

    def local_span(self, rank: int) -> tuple[int, int]:
        """This rank's slice of the global element-local vector."""
        z0, z1 = self.layers(rank)
        base = self.K * self.K * self.npe3
        return z0 * base, z1 * base

    def row_span(self, rank: int) -> tuple[int, int]:
        """Global rows (DOFs) this rank owns (its slice of the gathered vector)."""
        c0, c1 = self.own_planes(rank)
        return c0 * self.plane, c1 * self.plane

    def ng_own(self, rank: int) -> int:
        a, b = self.row_span(rank)
        return b - a

    def read_span(self, rank: int) -> tuple[int, int]:
        """Global rows BS7 reads: own planes plus the top interface plane (halo)."""
        z0, z1 = self.layers(rank)
        return z0 * self.p * self.plane, (z1 * self.p + 1) * self.plane


# ------------------------------------------------------------- reductions

class DistReducer:
    """All-gather of per-rank lattice scalars + device rank-order sum."""

    def __init__(self, world: int, device, group=None, sum_fn=None):
        self.world, self.device, self.group = world, torch.device(device), group
        self.buf = torch.empty(world, dtype=torch.float64, device=self.device)
        self.sum_fn = sum_fn or _gpu_sum_ordered

    def combine(self, local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if _nccl(self.group):
            dist.all_gather_into_tensor(self.buf, local.reshape(1), group=self.group)
        else:  # gloo: no all_gather_into_tensor, host tensors only
            parts = [torch.empty(1, dtype=torch.float64) for _ in range(self.world)]
            dist.all_gather(parts, local.reshape(1).cpu(), group=self.group)
            self.buf.copy_(torch.cat(parts))
        res = out if out is not None else torch.empty(1, dtype=torch.float64, device=self.device)
        self.sum_fn(self.buf, res)
        return res


def _gpu_sum_ordered(values: torch.Tensor, res: torch.Tensor) -> None:
    L = _lib.lib()
    _lib.check(L.sb_sum_ordered(values.data_ptr(), values.shape[0], res.data_ptr(),
                                _lib.stream_handle(values.device)), "sum_ordered")


def _nccl(group) -> bool:
    return dist.get_backend(group) == "nccl"


def _p2p(ops, group) -> None:
    """Grouped send/recv.  NCCL moves device buffers directly (NVLink); gloo
    (CPU-only tests, or SB200_DIST_BACKEND=gloo runs of bench.py) stages device
    buffers through host copies."""
    if not ops:
        return
    if _nccl(group):
        reqs = dist.batch_isend_irecv([dist.P2POp(fn, t, peer, group=group) for fn, t, peer in ops])
        for r in reqs:
            r.wait()
        return
    staged = []
    for fn, t, peer in ops:
        h = t.cpu() if (fn is dist.isend and t.is_cuda) else (
            torch.empty(t.shape, dtype=t.dtype) if t.is_cuda else t)
        staged.append((fn, t, h, peer))
    reqs = [fn(h, peer, group=group) for fn, _, h, peer in staged]
    for r in reqs:
        r.wait()
    for fn, t, h, _ in staged:
        if fn is dist.irecv and h is not t:
            t.copy_(h)


def combine_host(values) -> float:
    """Reference semantics of DistReducer.combine: ((0.0 + v0) + v1) + ..."""
    acc = 0.0
    for v in values:
        acc = acc + float(v)
    return acc


# -------------------------------------------------------------- BS6 / BS7

def _gpu_gather(op, q, out, carry):
    from .gs import bs6_gather_into
    return bs6_gather_into(op, q, out, carry)


class DistGather:
    """BS6 over a z-slab with the one-way carry halo (bitwise the 1-GPU result).

    own_op: rows of own_planes(rank) over the slab's local DOFs;
    send_op: rows of send_plane(rank) over the same DOFs (None on the last rank).
    gather_fn(op, q, out, carry) runs one CSR gather (libsb200 by default).
    """

    def __init__(self, part: SlabPartition, rank: int, own_op, send_op, device,
                 gather_fn=_gpu_gather, group=None):
        self.part, self.rank, self.own_op, self.send_op = part, rank, own_op, send_op
        self.device, self.gather_fn, self.group = torch.device(device), gather_fn, group
        plane = part.plane
        self.send_buf = torch.empty(plane, dtype=torch.float64, device=self.device) \
            if send_op is not None else None
        self.carry = torch.empty(plane, dtype=torch.float64, device=self.device) if rank > 0 else None

    @classmethod
    def build(cls, part: SlabPartition, rank: int, device, nodes_per_block: int = 512, group=None):
        from .mesh import build_slab_gather
        z0, z1 = part.layers(rank)
        c0, c1 = part.own_planes(rank)
        own = build_slab_gather(part.K, part.p, z0, z1, c0, c1, nodes_per_block, device)
        sp = part.send_plane(rank)
        send = None if sp is None else build_slab_gather(part.K, part.p, z0, z1, sp, sp + 1,
                                                         nodes_per_block, device)
        return cls(part, rank, own, send, device, group=group)

    def enable_lsa(self, lsa, offset: int = 0, sync_offset: int | None = None) -> None:
        """Carry halo over NVLink peer memory (lsa.LsaReducer whose halo window
        holds 2 planes at byte `offset` and 8 zeroed uint64 sync words at
        `sync_offset`).  gather_lsa then runs ONE kernel per call
        (sb_bs6_gather_halo): the send plane's partials are stored straight
        into rank+1's carry buffer (two buffers, by the device-side call
        parity) and flag words in the windows replace the barrier."""
        nb = 8 * self.part.plane
        if sync_offset is None:
            sync_offset = offset + 2 * nb
        self.lsa = lsa
        self.carry_ptrs = [lsa.halo_pointers(offset + e * nb, self.rank)[0] for e in (0, 1)]
        self.send_ptrs = ([lsa.halo_pointers(offset + e * nb, self.rank + 1)[1] for e in (0, 1)]
                          if self.send_op is not None else None)
        self.sync_ptr = lsa.halo_pointers(sync_offset, self.rank)[0]
        self.peer_ready = (lsa.halo_pointers(sync_offset, self.rank + 1)[1]
                           if self.send_op is not None else None)
        self.peer_ack = lsa.halo_pointers(sync_offset + 8, self.rank - 1)[1] if self.rank > 0 else None

    def gather_lsa(self, q_slab: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        gather_halo_raw(self.send_op, self.own_op, q_slab, out.data_ptr(), self.send_ptrs,
                        self.carry_ptrs if self.rank > 0 else None, self.part.plane if self.rank > 0 else 0,
                        self.sync_ptr, self.peer_ready, self.peer_ack)
        return out

    def exchange(self) -> None:
        ops = []
        if self.send_buf is not None:
            ops.append((dist.isend, self.send_buf, self.rank + 1))
        if self.carry is not None:
            ops.append((dist.irecv, self.carry, self.rank - 1))
        _p2p(ops, self.group)

    def gather(self, q_slab: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """out (= this rank's rows of the global gathered vector) from q_slab."""
        if self.send_op is not None:
            self.gather_fn(self.send_op, q_slab, self.send_buf, None)
        self.exchange()
        self.gather_fn(self.own_op, q_slab, out, self.carry)
        return out


def gather_halo_raw(send_op, own_op, q: torch.Tensor, out_ptr: int, send_ptrs, carry_ptrs, ncarry: int,
                    sync_ptr: int, peer_ready: int | None, peer_ack: int | None) -> None:
    """sb_bs6_gather_halo: the send and own gathers of a slab plus the carry
    handshake in one launch (raw addresses: NVLink-mapped peer memory, the
    local halo window, or -- single-GPU emulation in the tests -- plain device
    buffers)."""
    import ctypes
    L = _lib.lib()
    own_plan = own_op.plan()
    send_plan = send_op.plan() if send_op is not None else None
    if own_plan is None or (send_op is not None and send_plan is None):
        raise ValueError("the fused carry halo needs planned gather operators")
    pair = ctypes.c_void_p * 2
    so = pair(*send_ptrs) if send_ptrs else None
    ca = pair(*carry_ptrs) if carry_ptrs else None
    _lib.check(L.sb_bs6_gather_halo(
        None if send_op is None else send_plan.data_ptr(), 0 if send_op is None else send_op.n_blocks,
        None if send_op is None else send_op.row_starts_dev.data_ptr(),
        None if send_op is None else send_op.col_ids_dev.data_ptr(), so,
        own_plan.data_ptr(), own_op.n_blocks, own_op.row_starts_dev.data_ptr(), own_op.col_ids_dev.data_ptr(),
        own_op.ng, out_ptr, ca, ncarry, own_op.nodes_per_block, q.data_ptr(), sync_ptr, peer_ready, peer_ack,
        _lib.stream_handle(q.device)), "bs6_gather_halo")


def gather_raw(op, q: torch.Tensor, out_ptr: int, carry_ptr: int | None, ncarry: int) -> None:
    """sb_bs6_gather_planned with raw output / carry addresses (NVLink-mapped
    peer memory or the local halo window)."""
    L = _lib.lib()
    plan = op.plan()
    if plan is None:
        raise ValueError("the NVLink carry path needs a planned gather operator")
    _lib.check(L.sb_bs6_gather_planned(plan.data_ptr(), op.n_blocks, op.nodes_per_block, op.row_starts_dev.data_ptr(),
                                       op.col_ids_dev.data_ptr(), op.ng, op.nl, q.data_ptr(), out_ptr, carry_ptr,
                                       ncarry, _lib.stream_handle(q.device)), "bs6_gather (NVLink carry)")


class DistScatter:
    """BS7 over a z-slab: q_local[n] = q_global[l2g[n]] with a one-plane halo."""

    def __init__(self, part: SlabPartition, rank: int, ids_local: torch.Tensor, device, group=None,
                 scatter_fn=None):
        self.part, self.rank, self.device, self.group = part, rank, torch.device(device), group
        self.ids = ids_local  # ids relative to read_span(rank)[0]
        self.scatter_fn = scatter_fn or _gpu_scatter
        a, b = part.read_span(rank)
        self.window = torch.empty(b - a, dtype=torch.float64, device=self.device)
        self.own_rows = part.ng_own(rank) if rank < part.world - 1 else b - a

    @classmethod
    def build(cls, part: SlabPartition, rank: int, device, group=None):
        from .mesh import build_slab_l2g
        z0, z1 = part.layers(rank)
        l2g = build_slab_l2g(part.K, part.p, z0, z1, device)
        l2g -= part.read_span(rank)[0]
        return cls(part, rank, l2g, device, group=group)

    def exchange(self) -> None:
        """Send my bottom plane down to rank-1, receive my top plane from rank+1."""
        plane = self.part.plane
        ops = []
        if self.rank > 0:
            ops.append((dist.isend, self.window[:plane], self.rank - 1))
        if self.rank < self.part.world - 1:
            ops.append((dist.irecv, self.window[self.own_rows:], self.rank + 1))
        _p2p(ops, self.group)

    def scatter(self, q_local: torch.Tensor) -> None:
        """window[:own_rows] must hold this rank's q_global rows."""
        self.exchange()
        self.scatter_fn(self.ids, self.window, q_local)

    def enable_lsa(self, lsa, offset: int, counter_offset: int) -> None:
        """One-plane halo over NVLink: rank r+1 writes its bottom plane into
        rank r's halo buffer (2 planes at byte `offset` of the LSA halo window,
        alternating per call), one LSA barrier, then a split scatter reads the
        own rows from `window` and the halo plane from the LSA buffer.  The
        buffer parity is a call counter in this rank's window (8 bytes at
        `counter_offset`) that the barrier kernel advances -- device state, so
        captured CUDA graphs alternate correctly on every replay."""
        nb = 8 * self.part.plane
        self.lsa = lsa
        self.counter = lsa.halo_pointers(counter_offset, self.rank)[0]
        self.halo_ptrs = ([lsa.halo_pointers(offset + e * nb, self.rank)[0] for e in (0, 1)]
                          if self.rank < self.part.world - 1 else None)
        self.down_ptrs = ([lsa.halo_pointers(offset + e * nb, self.rank - 1)[1] for e in (0, 1)]
                          if self.rank > 0 else None)

    def scatter_lsa(self, q_local: torch.Tensor, own: torch.Tensor | None = None) -> None:
        """BS7 over the slab with the NVLink halo; `own` (default: the window's
        own rows) holds this rank's q_global rows."""
        L = _lib.lib()
        st = _lib.stream_handle(self.device)
        plane = self.part.plane
        src = self.window if own is None else own
        if self.down_ptrs is not None:  # my bottom plane -> rank-1's halo buffer (call parity), over NVLink
            _lib.check(L.sb_bs7_halo_put(src.data_ptr(), self.down_ptrs[0], self.down_ptrs[1], plane,
                                         self.counter, st), "bs7 halo put")
        self.lsa.barrier_advance(self.counter)
        nl = int(self.ids.shape[0])
        if self.halo_ptrs is None:  # last rank owns its top plane
            n_own = int(src.shape[0]) if own is not None else int(self.window.shape[0])
            _lib.check(L.sb_bs7_scatter(self.ids.data_ptr(), nl, src.data_ptr(), n_own, q_local.data_ptr(), 0, st),
                       "bs7_scatter")
        else:
            _lib.check(L.sb_bs7_scatter_split_pair(self.ids.data_ptr(), nl, src.data_ptr(), self.own_rows,
                                                   self.halo_ptrs[0], self.halo_ptrs[1], plane, self.counter,
                                                   q_local.data_ptr(), 0, st), "bs7_scatter_split_pair")


class DistMassOperator:
    """A = Z^T diag(w) Z on the rank's rows of a z-slab partitioned mesh -- the
    distributed form of cg.gather_scatter_operator, for
    cg.cg_solve_device(..., lsa=...): BS7 with the NVLink halo (split scatter),
    the pointwise weight, BS6 with the NVLink carry.  Every step is stream
    ordered on this rank (LSA barriers synchronise with the neighbours), so a
    CG iteration never waits on the host.  `weights` are this rank's
    element-local values (length part.nl(rank)); apply() maps the rank's
    owned rows (part.ng_own(rank)) to the same rows of A p."""

    def __init__(self, part: SlabPartition, rank: int, device, weights, lsa):
        self.part, self.rank, self.device = part, rank, torch.device(device)
        self.scat = DistScatter.build(part, rank, device)
        self.gath = DistGather.build(part, rank, device)
        nb = 8 * part.plane
        lsa.halo_window(4 * nb + 64)  # [BS6 carry x2 | BS7 halo x2 | BS6 sync words, BS7 call count]
        self.gath.enable_lsa(lsa, 0, sync_offset=4 * nb)
        self.scat.enable_lsa(lsa, 2 * nb, counter_offset=4 * nb + 40)
        self.w = torch.as_tensor(weights, dtype=torch.float64).to(self.device)
        if self.w.shape[0] != part.nl(rank):
            raise ValueError("weights must have one entry per element-local node of this rank's slab")
        self.ql = torch.empty(part.nl(rank), dtype=torch.float64, device=self.device)
        self.n_own = part.ng_own(rank)

    def __call__(self, p_own: torch.Tensor) -> torch.Tensor:
        if p_own.shape[0] != self.n_own:
            raise ValueError(f"expected this rank's {self.n_own} rows, got {p_own.shape[0]}")
        self.scat.scatter_lsa(self.ql, own=p_own)
        self.ql.mul_(self.w)
        out = torch.empty(self.n_own, dtype=torch.float64, device=self.device)
        return self.gath.gather_lsa(self.ql, out)


def _gpu_scatter(ids: torch.Tensor, window: torch.Tensor, q_local: torch.Tensor) -> None:
    from .gs import bs7_scatter
    bs7_scatter(_Ids(ids), window, q_local)


class _Ids:
    """ScatterIds view over a device id tensor (unmasked, ids >= 0 by construction)."""

    def __init__(self, ids):
        self.ids = ids
        self.has_mask = False
        self.max_id = -1  # range guaranteed by construction (read_span)

    @property
    def nl(self):
        return int(self.ids.shape[0])


# -------------------------------------------------------------- bench glue

def _create_with_deadline(make, seconds: float, expected_exc):
    """Run a blocking collective setup (the NCCL device-API context) with a
    deadline: (object, None) on success, (None, why) on failure or timeout.
    NCCL's non-blocking communicators cannot back a device communicator
    (ncclDevCommCreate rejects them), so the setup runs in a daemon thread and
    this rank gives up waiting after `seconds`; the caller's all-reduce of the
    outcome then moves every rank to the NCCL-collective path together (a
    setup stuck inside NCCL stays parked in its thread, on its own
    communicator)."""
    import threading
    box = {}

    def run():
        try:
            box["obj"] = make()
        except expected_exc as e:  # a clean refusal (NCCL < 2.28, no peer access, ...)
            box["why"] = str(e)
        except Exception as e:  # noqa: BLE001 -- any setup failure means "fall back"
            box["why"] = f"{type(e).__name__}: {e}"

    th = threading.Thread(target=run, name="sb200-lsa-setup", daemon=True)
    th.start()
    th.join(seconds)
    if th.is_alive():
        return None, f"setup did not finish within {seconds:.0f} s"
    return box.get("obj"), box.get("why")


def global_mesh_k(K: int, world: int, strong: bool) -> int:
    """bench.py's global mesh: weak scaling keeps the work per rank (K_g ~ K *
    world^(1/3)); strong scaling (--strong) splits the K^3 mesh itself in
    slabs (config 5: K = 143 on 8 GPUs).  At least one element layer per rank."""
    return max(world, K if strong else int(round(K * world ** (1.0 / 3.0))))


class BenchContext:
    """Per-rank state of bench.py's multi-GPU step (weak scaling: n per rank, a
    K_g^3 mesh with K_g ~ K world^(1/3); --strong: n and K global)."""

    def __init__(self, rank: int, world: int, args, device, use_lsa: bool | None = None):
        import os
        self.rank, self.world, self.device = rank, world, torch.device(device)
        self.reducer = DistReducer(world, device)
        # BS3/BS4/BS5: the reduction and the cross-rank combine fused in one
        # kernel over NVLink peer memory (lsa.py) when every rank is an LSA
        # peer; otherwise (or SB200_LSA=0) NCCL all-gather + ordered sum.
        self.lsa = None
        self.collective = ("nccl" if _nccl(None) else "gloo (host-staged)") + \
            " all_gather + sb_sum_ordered; BS6/BS7 halos by send/recv"
        if use_lsa is None:  # plain NCCL collectives unless asked for (SB200_LSA=1)
            use_lsa = os.environ.get("SB200_LSA", "0") == "1" and _nccl(None)
        if use_lsa:
            from . import lsa as _lsa
            # first agree that every rank can even try (local checks), so no
            # rank enters NCCL's collective setup alone; then agree on success
            why = _lsa.capable(world, device)
            can = torch.tensor([0 if why else 1], dtype=torch.int32, device=self.device)
            if world > 1:
                dist.all_reduce(can, op=dist.ReduceOp.MIN)
            if int(can.item()) == 1:
                try:  # the id broadcast stays on this thread (the group's collective order)
                    uid = _lsa.exchange_unique_id(world, rank, device)
                except _lsa.LsaUnavailable as e:
                    uid, why = None, str(e)
                if uid is not None:
                    self.lsa, why = _create_with_deadline(
                        lambda: _lsa.LsaReducer(world, rank, device, unique_id=uid),
                        float(os.environ.get("SB200_LSA_SETUP_S", "60")), _lsa.LsaUnavailable)
            elif why is None:
                why = "another rank cannot set it up"
            # every rank must take the same path (the fused kernels are collective)
            ok = torch.tensor([0 if self.lsa is None else 1], dtype=torch.int32, device=self.device)
            if world > 1:
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 1:
                self.collective = "fused in-kernel combine over NVLink (NCCL device API, LSA window)"
            else:
                if self.lsa is not None:
                    self.lsa.abort()  # local: some peer never built its context
                    self.lsa = None
                self.collective += f" (fused path unavailable: {why or 'not on every rank'})"
        Kg = global_mesh_k(args.K, world, getattr(args, "strong", False))
        self.part = SlabPartition(Kg, args.order, world)
        g = self.part.g
        self.mesh_desc = {"K_global": Kg, "order": args.order, "ng_global": g ** 3,
                          "nl_global": Kg ** 3 * (args.order + 1) ** 3,
                          "slab_layers": [self.part.layers(r) for r in range(world)],
                          "partition": "z-slabs, carry halo (BS6), one-plane halo (BS7)"}
        # our launches per step: the 7 tests + BS6's send-plane gather, plus either the
        # NVLink path's 2 LSA barriers and BS7 halo put, or the 3 ordered sums after the
        # NCCL all-gathers (NCCL's own kernels not counted)
        self.launches_per_step = 7 + 1 + 3

    def build_slab(self, K, order, device):
        self.gather = DistGather.build(self.part, self.rank, device)
        self.scat = DistScatter.build(self.part, self.rank, device)
        if self.lsa is not None:
            nb = 8 * self.part.plane
            self.lsa.halo_window(4 * nb + 64)  # [BS6 carry x2 | BS7 halo x2 | BS6 sync words, BS7 call count]
            self.gather.enable_lsa(self.lsa, 0, sync_offset=4 * nb)
            self.scat.enable_lsa(self.lsa, 2 * nb, counter_offset=4 * nb + 40)
            self.collective += ("; BS6 + carry halo in one launch (partials stored over NVLink into the "
                                "peer's window, flag handshake); BS7 halo plane written over NVLink + LSA barrier")
            self.launches_per_step = 7 + 2  # + BS7's halo put and LSA barrier (BS6 is one fused launch)
        return _SlabInfo(self.part, self.rank)

    def call(self, w, test):
        from . import kernels as KN
        if test == "bs1":
            w.sb.bs1_copy(w.x, w.y)
        elif test == "bs2":
            w.sb.bs2_axpy(0.5, w.x, -0.25, w.y)
        elif test == "bs3":
            if self.lsa is not None:
                self.lsa.bs3_norm2(w.x, w.cfg, out=w.res)
            else:
                self.reducer.combine(KN.bs3_norm2_async(w.x, w.cfg, out=w.res), out=w.res)
        elif test == "bs4":
            if self.lsa is not None:
                self.lsa.bs4_dot(w.x, w.y, w.cfg, out=w.res)
            else:
                self.reducer.combine(KN.bs4_dot_async(w.x, w.y, w.cfg, out=w.res), out=w.res)
        elif test == "bs5":
            if self.lsa is not None:
                self.lsa.bs5_fused_cg_update(1e-3, w.p, w.ap, w.x, w.r, w.cfg, out=w.res)
            else:
                self.reducer.combine(KN.bs5_fused_cg_update_async(1e-3, w.p, w.ap, w.x, w.r, w.cfg,
                                                                  out=w.res), out=w.res)
        elif test == "bs6":
            if self.lsa is not None:
                self.gather.gather_lsa(w.q, w.gout)
            else:
                self.gather.gather(w.q, w.gout)
        elif self.lsa is not None:
            self.scat.scatter_lsa(w.ql)
        else:
            self.scat.scatter(w.ql)


@dataclass
class _SlabInfo:
    part: SlabPartition
    rank: int

    @property
    def nl(self):
        return self.part.nl(self.rank)

    @property
    def ng_owned(self):
        return self.part.ng_own(self.rank)

    @property
    def ng_local_read(self):
        a, b = self.part.read_span(self.rank)
        return b - a
