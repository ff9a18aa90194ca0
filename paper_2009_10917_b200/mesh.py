"""Structured hex mesh numbering and the scatter/gather operators, built on the GPU.

Drop-in for pkg/src/streambench/mesh.py: same dataclasses, builders, error
messages and -- verified bit for bit against the reference -- the same
local_to_global, row_starts, col_ids and block_starts arrays.  Arrays live on
the device as int32 tensors.

For meshes made by build_mesh the CSR comes from a closed form
(sb_build_gather_csr: O(1) per row, no sort, no scan); any other
local_to_global map goes through the general path (stable CUB radix sort +
lower-bound row starts, sb_build_gather_general).  Block packing is the
reference's greedy rule in both cases (sb_build_block_starts).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import torch

from . import _lib

INDEX_DTYPE = torch.int32
_INT32_MAX = 2**31 - 1


def _dev(device=None) -> torch.device:
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


@dataclass(frozen=True)
class MeshConnectivity:
    """mesh.py:20-36: element-local to global node numbering for a K^3 mesh of order p."""

    K: int
    p: int
    local_to_global: torch.Tensor = field(repr=False)
    # True when local_to_global is the build_mesh numbering (enables the
    # closed-form operator builder); user-supplied maps use the general path.
    structured: bool = field(default=False, repr=False, compare=False)

    @property
    def nl(self) -> int:
        return int(self.local_to_global.shape[0])

    @property
    def ng(self) -> int:
        return (self.K * self.p + 1) ** 3


@dataclass(frozen=True)
class ScatterIds:
    """mesh.py:39-51: local-to-global id map; masked entries hold -1."""

    ids: torch.Tensor = field(repr=False)

    @property
    def nl(self) -> int:
        return int(self.ids.shape[0])

    @cached_property
    def _minmax(self) -> tuple[int, int]:
        # one device reduction per operator (the reference re-scans ids on
        # every bs7 call, gs.py:49-50; ids are immutable, so we cache it)
        ids = self.ids if self.ids.is_cuda else self.ids.cuda()
        if ids.numel() == 0:
            return (0, -1)
        out = torch.empty(2, dtype=torch.int32, device=ids.device)
        L = _lib.lib()
        _lib.check(L.sb_ids_minmax(ids.data_ptr(), ids.shape[0], out.data_ptr(),
                                   _lib.stream_handle(ids.device)), "ids_minmax")
        lo, hi = out.tolist()
        return int(lo), int(hi)

    @cached_property
    def has_mask(self) -> bool:
        return self.nl > 0 and self._minmax[0] < 0

    @property
    def max_id(self) -> int:
        return self._minmax[1]


BS6_PLAN_CAP = 512  # entries (and rows) per super-block, kBs6Cap in csrc/sb_gs_pipe.cu


@dataclass(frozen=True)
class GatherOp:
    """mesh.py:54-70: CSR of the gather operator with row blocks of bounded nonzero count."""

    ng: int
    row_starts: torch.Tensor = field(repr=False)
    col_ids: torch.Tensor = field(repr=False)
    block_starts: torch.Tensor = field(repr=False)
    nodes_per_block: int
    # (K, p, z0, z1, c_lo, c_hi) when the operator is the closed-form CSR of a
    # build_mesh numbering (or a slab of it): enables the TMA-staged BS6 plan
    geometry: tuple | None = field(default=None, repr=False, compare=False)

    @property
    def nl(self) -> int:
        return int(self.col_ids.shape[0])

    @property
    def n_blocks(self) -> int:
        return int(self.block_starts.shape[0]) - 1

    def _superblock_extent(self) -> tuple[int, int]:
        """(rows, entries) of the largest super-block of the BS6 plan (G =
        CAP // npb operator blocks each).  Both are <= CAP for operators from
        build_gather; a hand-built one (empty rows, or blocks not packed to
        nodes_per_block) can exceed them and then takes the unplanned path."""
        g = max(1, BS6_PLAN_CAP // self.nodes_per_block)
        bst = self.block_starts
        idx = torch.arange(0, self.n_blocks + g, g, device=bst.device).clamp_(max=self.n_blocks)
        rows = bst[idx].long()
        if rows.numel() < 2:
            return 0, 0
        ents = self.row_starts[rows].long()
        return int((rows[1:] - rows[:-1]).max().item()), int((ents[1:] - ents[:-1]).max().item())

    def plan(self) -> torch.Tensor | None:
        """Super-block plan for the pipelined BS6 kernel (sb_bs6_make_plan),
        built once per operator; None when the operator does not qualify."""
        p = self.__dict__.get("_plan", False)
        if p is not False:
            return p
        p = None
        if (self.row_starts.is_cuda and self.col_ids.is_cuda and self.block_starts.is_cuda
                and self.row_starts.data_ptr() % 16 == 0 and self.col_ids.data_ptr() % 16 == 0
                and os.environ.get("SB200_NO_PIPE") != "1"):
            L = _lib.lib()
            size = int(L.sb_bs6_plan_size(self.n_blocks, self.nodes_per_block))
            if size > 0 and max(self._superblock_extent()) > BS6_PLAN_CAP:
                size = 0  # a super-block would exceed the kernel's row / entry capacity
            if size > 0:
                dev = self.row_starts.device
                p = torch.empty(size, dtype=torch.int32, device=dev)
                _lib.check(L.sb_bs6_make_plan(self.block_starts.data_ptr(), self.n_blocks,
                                              self.row_starts.data_ptr(), self.nodes_per_block,
                                              p.data_ptr(), _lib.stream_handle(dev)), "bs6 plan")
                # built once per operator; consumers may run on other streams
                torch.cuda.current_stream(dev).synchronize()
        object.__setattr__(self, "_plan", p)
        return p


    def staged(self):
        """(sb_bs6_staged_t, plan) of the TMA-staged BS6 kernel
        (csrc/sb_gs_staged.cu), built once per operator; None unless the
        operator is a structured one of order p <= 2 on the device.  Opt-in
        (SB200_BS6_STAGED=1): measured slower than the super-block kernel so
        far (profiles/r02_bs6_staged.md); SB200_BS6_TILE="ey,ez,w" overrides
        the tile shape (A/B runs)."""
        st = self.__dict__.get("_staged", False)
        if st is not False:
            return st
        st = None
        geo = self.geometry
        if (geo is not None and os.environ.get("SB200_BS6_STAGED", "0") == "1"
                and self.row_starts.is_cuda and self.col_ids.is_cuda
                and self.row_starts.data_ptr() % 16 == 0 and self.col_ids.data_ptr() % 16 == 0):
            tile = [int(v) for v in os.environ.get("SB200_BS6_TILE", "0,0,0").split(",")]
            L = _lib.lib()
            info = _lib.Bs6Staged()
            rc = L.sb_bs6_staged_init(*geo, *tile, info)
            if rc == _lib.SB_OK:
                dev = self.row_starts.device
                plan = torch.empty(max(1, info.n_tiles * info.words_per_tile), dtype=torch.int32,
                                   device=dev)
                _lib.check(L.sb_bs6_staged_make_plan(info, self.row_starts.data_ptr(),
                                                     plan.data_ptr(), _lib.stream_handle(dev)),
                           "bs6 staged plan")
                # consumers may run on other streams: the plan is complete once built
                torch.cuda.current_stream(dev).synchronize()
                st = (info, plan)
        object.__setattr__(self, "_staged", st)
        return st


def build_mesh(K: int, p: int, device=None) -> MeshConnectivity:
    """mesh.py:73-97: number the nodes of a structured K*K*K mesh of order-p hexahedra."""
    if K < 1 or p < 1:
        raise ValueError(f"need K >= 1 and p >= 1, got K={K}, p={p}")
    g = K * p + 1
    if g**3 > _INT32_MAX:
        raise ValueError(f"global id space (K*p+1)^3 = {g**3} overflows int32")
    nl = K**3 * (p + 1) ** 3
    if nl > _INT32_MAX:
        # the reference silently wraps here (mesh.py:97)
        raise ValueError(f"local DOF count K^3 (p+1)^3 = {nl} overflows int32")
    dev = _dev(device)
    l2g = torch.empty(nl, dtype=INDEX_DTYPE, device=dev)
    L = _lib.lib()
    with torch.cuda.device(dev):
        _lib.check(L.sb_build_l2g(K, p, 0, K, l2g.data_ptr(), _lib.stream_handle(dev)), "build_mesh")
    return MeshConnectivity(K=K, p=p, local_to_global=l2g, structured=True)


@_lib.device_guard
def build_scatter_ids(mesh: MeshConnectivity, mask=None) -> ScatterIds:
    """mesh.py:100-110: scatter id map for the mesh; global ids in `mask` become -1."""
    l2g = mesh.local_to_global
    dev = l2g.device if l2g.is_cuda else _dev()
    if not l2g.is_cuda:
        l2g = l2g.to(dev)
    ids = torch.empty_like(l2g)
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    if mask is not None:
        mask_ids = np.asarray(sorted(mask), dtype=np.int64)
        if mask_ids.size and (mask_ids.min() < 0 or mask_ids.max() >= mesh.ng):
            raise ValueError(f"mask ids must lie in [0, {mesh.ng})")
    else:
        mask_ids = np.zeros(0, dtype=np.int64)
    if mask_ids.size:
        gids = torch.from_numpy(mask_ids).to(dev)
        scratch = torch.empty(mesh.ng, dtype=torch.uint8, device=dev)
        _lib.check(L.sb_build_scatter_ids(l2g.data_ptr(), l2g.shape[0], gids.data_ptr(),
                                          gids.shape[0], mesh.ng, scratch.data_ptr(),
                                          ids.data_ptr(), st), "build_scatter_ids")
    else:
        _lib.check(L.sb_build_scatter_ids(l2g.data_ptr(), l2g.shape[0], None, 0, mesh.ng, None,
                                          ids.data_ptr(), st), "build_scatter_ids")
    return ScatterIds(ids=ids)


def _max_row_len(K: int) -> int:
    return 8 if K >= 2 else 1


def _block_starts(row_starts: torch.Tensor, ng: int, npb: int) -> torch.Tensor:
    """mesh.py:136-143 greedy packing on the device.  Rows must be non-empty
    (build_gather rejects uncovered ids first, like the reference), which
    bounds every block to <= npb rows."""
    dev = row_starts.device
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    bst = torch.empty(ng + 1, dtype=INDEX_DTYPE, device=dev)
    nblk = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(L.sb_build_block_starts(row_starts.data_ptr(), ng, npb, bst.data_ptr(), ng,
                                       nblk.data_ptr(), st), "build_gather")
    nb = int(nblk.item())
    if nb < 0:
        raise ValueError(f"nodes_per_block={npb} is below the longest row")
    return bst[: nb + 1].clone()


@_lib.device_guard
def build_gather(mesh: MeshConnectivity, nodes_per_block: int = 512) -> GatherOp:
    """mesh.py:113-147: CSR gather operator with greedily packed row blocks.

    Row r lists (ascending) every local index mapping to global id r; blocks
    take consecutive rows while their nonzeros stay within nodes_per_block.
    """
    ng, nl = mesh.ng, mesh.nl
    l2g = mesh.local_to_global
    dev = l2g.device if l2g.is_cuda else _dev()
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    rs = torch.empty(ng + 1, dtype=INDEX_DTYPE, device=dev)
    ci = torch.empty(nl, dtype=INDEX_DTYPE, device=dev)
    if mesh.structured:
        longest = _max_row_len(mesh.K)
        if longest > nodes_per_block:
            raise ValueError(f"nodes_per_block={nodes_per_block} is below the longest row "
                             f"({longest} nonzeros)")
        _lib.check(L.sb_build_gather_csr(mesh.K, mesh.p, 0, mesh.K, 0, mesh.K * mesh.p + 1,
                                         rs.data_ptr(), ci.data_ptr(), st), "build_gather")
    else:
        if not l2g.is_cuda:
            l2g = l2g.to(dev)
        tmp = torch.empty(int(L.sb_build_gather_general_temp_bytes(nl)), dtype=torch.uint8,
                          device=dev)
        stats = torch.empty(2, dtype=torch.int64, device=dev)
        _lib.check(L.sb_build_gather_general(l2g.data_ptr(), nl, ng, rs.data_ptr(), ci.data_ptr(),
                                             tmp.data_ptr(), tmp.shape[0], stats.data_ptr(), st),
                   "build_gather")
        cmin, cmax = (int(v) for v in stats.tolist())
        if ng > 0 and cmin < 1:
            raise ValueError("mesh does not cover every global id")
        if cmax > nodes_per_block:
            raise ValueError(f"nodes_per_block={nodes_per_block} is below the longest row "
                             f"({cmax} nonzeros)")
    bst = _block_starts(rs, ng, nodes_per_block)
    geo = (mesh.K, mesh.p, 0, mesh.K, 0, mesh.K * mesh.p + 1) if mesh.structured else None
    return GatherOp(ng=ng, row_starts=rs, col_ids=ci, block_starts=bst,
                    nodes_per_block=nodes_per_block, geometry=geo)


def build_slab_gather(K: int, p: int, z0: int, z1: int, c_lo: int, c_hi: int,
                      nodes_per_block: int = 512, device=None) -> GatherOp:
    """Gather operator of a z-slab (multi-GPU partition, dist.py).

    Rows are the global lattice rows of planes [c_lo, c_hi) (renumbered from
    0), columns the local DOFs of elements with ez in [z0, z1) (renumbered from
    the slab's first element), entries in the reference's ascending order.  With
    z0=0, z1=K, c_lo=0, c_hi=K*p+1 this is build_gather(build_mesh(K, p)).
    """
    g = K * p + 1
    dev = _dev(device)
    ng = (c_hi - c_lo) * g * g
    nl = K * K * (z1 - z0) * (p + 1) ** 3
    longest = (2 if K >= 2 else 1) ** 2 * (2 if z1 - z0 >= 2 else 1)
    if longest > nodes_per_block:
        raise ValueError(f"nodes_per_block={nodes_per_block} is below the longest row "
                         f"({longest} nonzeros)")
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    rs = torch.empty(ng + 1, dtype=INDEX_DTYPE, device=dev)
    ci = torch.empty(nl, dtype=INDEX_DTYPE, device=dev)
    _lib.check(L.sb_build_gather_csr(K, p, z0, z1, c_lo, c_hi, rs.data_ptr(), ci.data_ptr(), st),
               "build_slab_gather")
    nnz = int(rs[-1].item())
    ci = ci[:nnz]  # entries of planes outside [c_lo, c_hi) are not part of this operator
    bst = _block_starts(rs, ng, nodes_per_block)
    return GatherOp(ng=ng, row_starts=rs, col_ids=ci, block_starts=bst,
                    nodes_per_block=nodes_per_block, geometry=(K, p, z0, z1, c_lo, c_hi))


def build_slab_l2g(K: int, p: int, z0: int, z1: int, device=None) -> torch.Tensor:
    """local_to_global (global lattice ids) of the elements with ez in [z0, z1)."""
    dev = _dev(device)
    nl = K * K * (z1 - z0) * (p + 1) ** 3
    l2g = torch.empty(nl, dtype=INDEX_DTYPE, device=dev)
    L = _lib.lib()
    _lib.check(L.sb_build_l2g(K, p, z0, z1, l2g.data_ptr(), _lib.stream_handle(dev)),
               "build_slab_l2g")
    return l2g


@_lib.device_guard
def multiplicity(mesh: MeshConnectivity) -> torch.Tensor:
    """mesh.py:150-153: per-global-node count of element-local copies (float64, device)."""
    l2g = mesh.local_to_global
    dev = l2g.device if l2g.is_cuda else _dev()
    out = torch.empty(mesh.ng, dtype=torch.float64, device=dev)
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    if mesh.structured:
        _lib.check(L.sb_multiplicity(mesh.K, mesh.p, 0, mesh.K, 0, mesh.K * mesh.p + 1,
                                     out.data_ptr(), st), "multiplicity")
    else:
        if not l2g.is_cuda:
            l2g = l2g.to(dev)
        _lib.check(L.sb_histogram(l2g.data_ptr(), l2g.shape[0], mesh.ng, out.data_ptr(), st),
                   "multiplicity")
    return out
