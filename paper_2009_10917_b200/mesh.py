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
from dataclasses import FrozenInstanceError
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


def _l2g_dev(mesh) -> torch.Tensor:
    """The mesh's local_to_global on the device (this package's mesh, or the
    reference's numpy one, uploaded)."""
    d = getattr(mesh, "local_to_global_dev", None)
    if d is not None:
        return d
    return torch.from_numpy(np.ascontiguousarray(mesh.local_to_global, dtype=np.int32)).to(_dev())


class _IndexArrays:
    """Frozen holder of int32 index arrays (the reference's frozen dataclasses,
    mesh.py:20-70).  The builders here make every array on the device; the
    reference's attribute names (local_to_global, ids, row_starts, ...) are
    numpy host views, downloaded once on first access, so reference-style
    numpy code works unchanged, while the kernels use the `<name>_dev` CUDA
    tensors and never pay the copy.  Arrays passed in as numpy are uploaded
    once on first device use instead."""

    _ARRAYS: tuple[str, ...] = ()

    def _init_arrays(self, **arrays) -> None:
        for name, a in arrays.items():
            if isinstance(a, torch.Tensor) and a.is_cuda:
                dev, host = a, None
            else:
                host = a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
                if host.dtype != np.int32:
                    host = host.astype(np.int32)
                dev = None
            object.__setattr__(self, f"_{name}_d", dev)
            object.__setattr__(self, f"_{name}_h", host)

    def __setattr__(self, name, value):
        raise FrozenInstanceError(f"cannot assign to field {name!r}")

    def _host(self, name: str) -> np.ndarray:
        h = self.__dict__[f"_{name}_h"]
        if h is None:
            h = self.__dict__[f"_{name}_d"].cpu().numpy()
            object.__setattr__(self, f"_{name}_h", h)
        return h

    def _device(self, name: str) -> torch.Tensor:
        d = self.__dict__[f"_{name}_d"]
        if d is None:
            d = torch.from_numpy(np.ascontiguousarray(self.__dict__[f"_{name}_h"])).to(_dev())
            object.__setattr__(self, f"_{name}_d", d)
        return d

    def _length(self, name: str) -> int:
        d = self.__dict__[f"_{name}_d"]
        return int(d.shape[0]) if d is not None else int(self.__dict__[f"_{name}_h"].shape[0])


def _host_view(name: str, doc: str) -> property:
    return property(lambda self: self._host(name), doc=f"{doc} (numpy int32 host view)")


def _device_view(name: str, doc: str) -> property:
    return property(lambda self: self._device(name), doc=f"{doc} (int32 CUDA tensor)")


class MeshConnectivity(_IndexArrays):
    """mesh.py:20-36: element-local to global node numbering for a K^3 mesh of order p."""

    def __init__(self, K: int, p: int, local_to_global, structured: bool = False):
        object.__setattr__(self, "K", K)
        object.__setattr__(self, "p", p)
        # True when local_to_global is the build_mesh numbering (enables the
        # closed-form operator builder); user-supplied maps use the general path
        object.__setattr__(self, "structured", structured)
        self._init_arrays(local_to_global=local_to_global)

    local_to_global = _host_view("local_to_global", "mesh.py:20-36 local-to-global map")
    local_to_global_dev = _device_view("local_to_global", "local-to-global map")

    def __repr__(self) -> str:
        return f"MeshConnectivity(K={self.K}, p={self.p})"

    @property
    def nl(self) -> int:
        return self._length("local_to_global")

    @property
    def ng(self) -> int:
        return (self.K * self.p + 1) ** 3


class ScatterIds(_IndexArrays):
    """mesh.py:39-51: local-to-global id map; masked entries hold -1."""

    def __init__(self, ids):
        self._init_arrays(ids=ids)

    ids = _host_view("ids", "mesh.py:39-51 scatter ids")
    ids_dev = _device_view("ids", "scatter ids")

    def __repr__(self) -> str:
        return f"ScatterIds(nl={self.nl})"

    @property
    def nl(self) -> int:
        return self._length("ids")

    @cached_property
    def _minmax(self) -> tuple[int, int]:
        # one device reduction per operator (the reference re-scans ids on
        # every bs7 call, gs.py:49-50; ids are immutable, so we cache it)
        ids = self.ids_dev
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


class GatherOp(_IndexArrays):
    """mesh.py:54-70: CSR of the gather operator with row blocks of bounded nonzero count."""

    def __init__(self, ng: int, row_starts, col_ids, block_starts, nodes_per_block: int,
                 geometry: tuple | None = None):
        object.__setattr__(self, "ng", ng)
        object.__setattr__(self, "nodes_per_block", nodes_per_block)
        # (K, p, z0, z1, c_lo, c_hi) when the operator is the closed-form CSR of
        # a build_mesh numbering (or a slab of it): enables the z-sweep kernel
        object.__setattr__(self, "geometry", geometry)
        self._init_arrays(row_starts=row_starts, col_ids=col_ids, block_starts=block_starts)

    row_starts = _host_view("row_starts", "mesh.py:54-70 CSR row starts")
    col_ids = _host_view("col_ids", "mesh.py:54-70 CSR column ids")
    block_starts = _host_view("block_starts", "mesh.py:54-70 row-block starts")
    row_starts_dev = _device_view("row_starts", "CSR row starts")
    col_ids_dev = _device_view("col_ids", "CSR column ids")
    block_starts_dev = _device_view("block_starts", "row-block starts")

    def __repr__(self) -> str:
        return f"GatherOp(ng={self.ng}, nl={self.nl}, nodes_per_block={self.nodes_per_block})"

    @property
    def nl(self) -> int:
        return self._length("col_ids")

    @property
    def n_blocks(self) -> int:
        return self._length("block_starts") - 1

    def _superblock_extent(self) -> tuple[int, int]:
        """(rows, entries) of the largest super-block of the BS6 plan (G =
        CAP // npb operator blocks each).  Both are <= CAP for operators from
        build_gather; a hand-built one (empty rows, or blocks not packed to
        nodes_per_block) can exceed them and then takes the unplanned path."""
        g = max(1, BS6_PLAN_CAP // self.nodes_per_block)
        bst = self.block_starts_dev
        idx = torch.arange(0, self.n_blocks + g, g, device=bst.device).clamp_(max=self.n_blocks)
        rows = bst[idx].long()
        if rows.numel() < 2:
            return 0, 0
        ents = self.row_starts_dev[rows].long()
        return int((rows[1:] - rows[:-1]).max().item()), int((ents[1:] - ents[:-1]).max().item())

    def plan(self) -> torch.Tensor | None:
        """Super-block plan for the pipelined BS6 kernel (sb_bs6_make_plan),
        built once per operator; None when the operator does not qualify."""
        p = self.__dict__.get("_plan", False)
        if p is not False:
            return p
        p = None
        rs, ci = self.row_starts_dev, self.col_ids_dev
        if (rs.data_ptr() % 16 == 0 and ci.data_ptr() % 16 == 0
                and os.environ.get("SB200_NO_PIPE") != "1"):
            L = _lib.lib()
            size = int(L.sb_bs6_plan_size(self.n_blocks, self.nodes_per_block))
            if size > 0 and max(self._superblock_extent()) > BS6_PLAN_CAP:
                size = 0  # a super-block would exceed the kernel's row / entry capacity
            if size > 0:
                dev = rs.device
                p = torch.empty(size, dtype=torch.int32, device=dev)
                # (synchronises the stream once: the plan is complete for consumers on any stream)
                _lib.check(L.sb_bs6_make_plan(self.block_starts_dev.data_ptr(), self.n_blocks,
                                              rs.data_ptr(), self.nodes_per_block,
                                              p.data_ptr(), _lib.stream_handle(dev)), "bs6 plan")
        object.__setattr__(self, "_plan", p)
        return p


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
    l2g = _l2g_dev(mesh)
    dev = l2g.device
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
    structured = getattr(mesh, "structured", False)
    l2g = None if structured else _l2g_dev(mesh)
    dev = _dev() if l2g is None else l2g.device
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    rs = torch.empty(ng + 1, dtype=INDEX_DTYPE, device=dev)
    ci = torch.empty(nl, dtype=INDEX_DTYPE, device=dev)
    if structured:
        longest = _max_row_len(mesh.K)
        if longest > nodes_per_block:
            raise ValueError(f"nodes_per_block={nodes_per_block} is below the longest row "
                             f"({longest} nonzeros)")
        _lib.check(L.sb_build_gather_csr(mesh.K, mesh.p, 0, mesh.K, 0, mesh.K * mesh.p + 1,
                                         rs.data_ptr(), ci.data_ptr(), st), "build_gather")
    else:
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
    geo = (mesh.K, mesh.p, 0, mesh.K, 0, mesh.K * mesh.p + 1) if structured else None
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
def multiplicity_dev(mesh: MeshConnectivity) -> torch.Tensor:
    """mesh.py:150-153 on the device: per-global-node count of element-local
    copies (float64 CUDA tensor)."""
    dev = _dev() if getattr(mesh, "structured", False) else _l2g_dev(mesh).device
    out = torch.empty(mesh.ng, dtype=torch.float64, device=dev)
    L = _lib.lib()
    st = _lib.stream_handle(dev)
    if getattr(mesh, "structured", False):
        _lib.check(L.sb_multiplicity(mesh.K, mesh.p, 0, mesh.K, 0, mesh.K * mesh.p + 1,
                                     out.data_ptr(), st), "multiplicity")
    else:
        l2g = _l2g_dev(mesh)
        _lib.check(L.sb_histogram(l2g.data_ptr(), l2g.shape[0], mesh.ng, out.data_ptr(), st),
                   "multiplicity")
    return out


def multiplicity(mesh: MeshConnectivity) -> np.ndarray:
    """mesh.py:150-153: per-global-node count of element-local copies, float64
    numpy like the reference (computed on the device; multiplicity_dev keeps
    it there)."""
    return multiplicity_dev(mesh).cpu().numpy()
