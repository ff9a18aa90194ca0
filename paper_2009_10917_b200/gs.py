"""BS6 gather (Z^T) and BS7 scatter (Z) on the B200 (gs.py of the reference).

Same signatures, error messages and results as pkg/src/streambench/gs.py:
bs6_gather returns a new vector whose rows are summed in ascending column
order from +0.0 (bitwise the reference), bs7_scatter writes q_local in place
and leaves masked (-1) entries untouched.  Operators may be this package's
device GatherOp/ScatterIds or the reference's numpy ones (staged per call).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib, hoststream


def _dev_int(a, name, device):
    if isinstance(a, torch.Tensor) and a.is_cuda:
        return a
    return _lib.stage(a, torch.int32, name, device).dev


def _op_dev(op, name, device):
    """Index array `name` of an operator on the device: this package's
    operators keep it there (`<name>_dev`); the reference's numpy ones are
    staged per call."""
    d = getattr(op, name + "_dev", None)
    return d if d is not None else _dev_int(getattr(op, name), name, device)


def sweep_geometry(op, q_local):
    """(K, p, z0, z1, c_lo, c_hi) when the z-sweep kernel (csrc/sb_gs_sweep.cu)
    takes this gather: a structured device operator of order p <= 2.  Opt-in
    (SB200_BS6_SWEEP=1) while it measures slower than the super-block kernel
    (profiles/r02_bs6_sweep.md)."""
    geo = getattr(op, "geometry", None)
    if (geo is None or geo[1] > 2 or os.environ.get("SB200_BS6_SWEEP", "0") != "1"
            or q_local.data_ptr() % 16):
        return None
    return geo


def bs6_kernel_name(op, q_local=None) -> str:
    """Name of the kernel bs6_gather_into launches for `op` (tests, bench)."""
    import ctypes
    if q_local is not None and tiled_geometry(op, q_local) is not None:
        return "k_bs6_tile4t<8 row lines>"
    if q_local is not None and sweep_geometry(op, q_local) is not None:
        return f"k_bs6_sweep<p={op.geometry[1]}>"
    plan = op.plan() if hasattr(op, "plan") else None
    if plan is None:
        return "k_bs6 (unplanned)"
    buf = ctypes.create_string_buffer(96)
    _lib.check(_lib.lib().sb_bs6_planned_kernel(op.n_blocks, op.nodes_per_block, op.ng, op.nl, buf, 96),
               "bs6_kernel_name")
    return buf.value.decode()


def tiled_geometry(op, q_local):
    """(K, p, z0, z1, c_lo, c_hi) when the row-line-tiled kernel
    (csrc/sb_gs_tile.cu: TMA tensor boxes of element-row halves, 8 row lines
    per CTA) takes this gather: a structured device operator of order 1 with
    >= 1e6 rows -- where it measured faster than the super-block kernel at
    every size (N=1, NG ~ 1e8: 5.65-5.83 vs 4.73-4.76 TB/s;
    profiles/r02_bs6_sweep.md).  SB200_BS6_TILED=0 / 1 forces it off / on."""
    geo = getattr(op, "geometry", None)
    force = os.environ.get("SB200_BS6_TILED")
    if (geo is None or geo[1] != 1 or force == "0" or q_local.data_ptr() % 16
            or (force != "1" and op.ng < TILED_MIN_ROWS)):
        return None
    return geo


TILED_MIN_ROWS = 1_000_000  # below: the super-block kernel (K=66: 10.6 vs 12.5 us)


@_lib.device_guard
def bs6_gather_into(op, q_local: torch.Tensor, out: torch.Tensor, carry=None) -> torch.Tensor:
    """Device-only BS6 writing `out` (length op.ng); optional carry-in partials
    seed rows [0, len(carry)) instead of +0.0 (multi-GPU carry halo)."""
    dev = q_local.device
    L = _lib.lib()
    ncarry = 0 if carry is None else int(carry.shape[0])
    geo = tiled_geometry(op, q_local)
    if geo is not None:
        _lib.check(L.sb_bs6_gather_tiled(*geo, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng,
                                         int(q_local.shape[0]), q_local.data_ptr(), out.data_ptr(),
                                         None if carry is None else carry.data_ptr(), ncarry,
                                         _lib.stream_handle(dev)), "bs6_gather")
        return out
    geo = sweep_geometry(op, q_local)
    if geo is not None:
        _lib.check(L.sb_bs6_gather_sweep(*geo, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng,
                                         int(q_local.shape[0]), q_local.data_ptr(), out.data_ptr(),
                                         None if carry is None else carry.data_ptr(), ncarry,
                                         _lib.stream_handle(dev)), "bs6_gather")
        return out
    plan = op.plan() if hasattr(op, "plan") else None
    if plan is not None:
        _lib.check(L.sb_bs6_gather_planned(plan.data_ptr(), op.n_blocks, op.nodes_per_block,
                                           op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng,
                                           op.nl, q_local.data_ptr(), out.data_ptr(),
                                           None if carry is None else carry.data_ptr(), ncarry,
                                           _lib.stream_handle(dev)), "bs6_gather")
        return out
    bst = _op_dev(op, "block_starts", dev)
    rs = _op_dev(op, "row_starts", dev)
    ci = _op_dev(op, "col_ids", dev)
    _lib.check(L.sb_bs6_gather(bst.data_ptr(), int(bst.shape[0]) - 1, rs.data_ptr(), ci.data_ptr(),
                               op.ng, int(ci.shape[0]), op.nodes_per_block, q_local.data_ptr(),
                               out.data_ptr(), None if carry is None else carry.data_ptr(), ncarry,
                               _lib.stream_handle(dev)), "bs6_gather")
    return out


def _prefix_need(idx: torch.Tensor, ends) -> list[int]:
    """need[j] = 1 + max(idx[:ends[j]]) (the input prefix a chunk may touch)."""
    pm = torch.cummax(idx.to(torch.int64), 0).values
    e = torch.as_tensor([max(int(v), 1) - 1 for v in ends], dtype=torch.int64, device=idx.device)
    return [int(v) + 1 for v in pm[e].tolist()]


def _bs6_host_jobs(op):
    """Row chunks of ~CHUNK rows on block boundaries + the q prefix each needs (cached)."""
    jobs = op.__dict__.get("_host_jobs")
    if jobs is None:
        bst = op.block_starts  # (numpy host view)
        cuts = [0]
        for b in range(1, bst.shape[0]):
            if bst[b] - bst[cuts[-1]] >= hoststream.CHUNK or b == bst.shape[0] - 1:
                cuts.append(b)
        rows = [int(bst[c]) for c in cuts]
        rs = op.row_starts_dev
        ends = rs[torch.as_tensor(rows[1:], device=rs.device)].tolist()
        need = _prefix_need(op.col_ids_dev, ends)
        jobs = [(rows[i], rows[i + 1], need[i], cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
        object.__setattr__(op, "_host_jobs", jobs)
    return jobs


def _bs6_host(op, q_local):
    """Host q_local -> host result, upload / row-chunk gathers / download overlapped."""
    hq = hoststream.as_host_tensor(q_local, "q_local")
    dev = op.row_starts_dev.device
    L = _lib.lib()
    qd = torch.empty(op.nl, dtype=torch.float64, device=dev)
    outd = torch.empty(op.ng, dtype=torch.float64, device=dev)
    # a fresh result like the reference (gs.py:20), page-locked (torch's caching
    # host allocator): full-speed D2H without first-touch page faults
    res = torch.empty(op.ng, dtype=torch.float64, pin_memory=True)
    jobs = _bs6_host_jobs(op)
    blocks = {j[0]: (j[3], j[4]) for j in jobs}

    def launch(r_lo, r_hi):
        b_lo, b_hi = blocks[r_lo]
        _lib.check(L.sb_bs6_gather(op.block_starts_dev.data_ptr() + 4 * b_lo, b_hi - b_lo,
                                   op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng, op.nl,
                                   op.nodes_per_block, qd.data_ptr(), outd.data_ptr(), None, 0,
                                   _lib.stream_handle(dev)), "bs6_gather")

    hoststream.run_prefix(hq, qd, outd, res, [j[:3] for j in jobs], launch, dev)
    return res.numpy() if isinstance(q_local, np.ndarray) else res


@_lib.device_guard
def bs6_gather(op, q_local, out=None):
    """gs.py:10-39: out[r] = sum of q_local over row r's columns, ascending order."""
    if q_local.shape[0] != op.nl:
        raise ValueError(f"local vector length {q_local.shape[0]} != operator NL {op.nl}")
    host = not (isinstance(q_local, torch.Tensor) and q_local.is_cuda)
    if host and out is None and hasattr(op, "row_starts_dev"):
        return _bs6_host(op, q_local)
    q = _lib.stage(q_local, torch.float64, "q_local").dev
    if out is None:
        out = torch.empty(op.ng, dtype=torch.float64, device=q.device)
    bs6_gather_into(op, q, out)
    if host:
        # a fresh result like the reference (gs.py:20), in page-locked memory from
        # torch's caching host allocator: full-speed D2H, no first-touch faults
        res = torch.empty(op.ng, dtype=torch.float64, pin_memory=True)
        res.copy_(out, non_blocking=True)
        torch.cuda.current_stream(q.device).synchronize()
        return res.numpy() if isinstance(q_local, np.ndarray) else res
    return out


def _bs7_host(ids, q_global, q_local) -> None:
    """Unmasked scatter between host vectors: q_global upload, local-chunk scatters
    and q_local download overlapped (q_local is write-only, never uploaded)."""
    hg = hoststream.as_host_tensor(q_global, "q_global")
    hl = hoststream.as_host_tensor(q_local, "q_local")
    dev = ids.ids_dev.device
    nl, ng = ids.nl, int(hg.shape[0])
    jobs = ids.__dict__.get("_host_jobs")
    if jobs is None:
        cuts = list(range(0, nl, hoststream.CHUNK)) + [nl]
        need = _prefix_need(ids.ids_dev, cuts[1:])
        jobs = [(cuts[i], cuts[i + 1], need[i]) for i in range(len(cuts) - 1)]
        ids.__dict__["_host_jobs"] = jobs
    L = _lib.lib()
    gd = torch.empty(ng, dtype=torch.float64, device=dev)
    ld = torch.empty(nl, dtype=torch.float64, device=dev)

    def launch(lo, hi):
        _lib.check(L.sb_bs7_scatter(ids.ids_dev.data_ptr() + 4 * lo, hi - lo, gd.data_ptr(), ng,
                                    ld.data_ptr() + 8 * lo, 0, _lib.stream_handle(dev)), "bs7_scatter")

    hoststream.run_prefix(hg, gd, ld, hl, jobs, launch, dev)


@_lib.device_guard
def bs7_scatter(ids, q_global, q_local) -> None:
    """gs.py:42-61: q_local[n] = q_global[ids[n]] where ids[n] >= 0; masked entries untouched."""
    if q_local.shape[0] != ids.nl:
        raise ValueError(f"local vector length {q_local.shape[0]} != id count {ids.nl}")
    ng = int(q_global.shape[0])
    max_id = getattr(ids, "max_id", None)
    if max_id is None:  # a reference (numpy) ScatterIds
        max_id = int(np.max(ids.ids)) if ids.ids.size else -1
    if ids.nl and max_id >= ng:
        raise ValueError(f"scatter id {max_id} out of range [0, {ng})")
    if (hoststream.all_host(q_global, q_local) and not ids.has_mask
            and hasattr(ids, "ids_dev") and ids.ids_dev.data_ptr() % 16 == 0):
        _bs7_host(ids, q_global, q_local)
        return
    sg = _lib.stage(q_global, torch.float64, "q_global")
    dev = sg.dev.device
    if not ids.has_mask and not (isinstance(q_local, torch.Tensor) and q_local.is_cuda):
        # every entry is overwritten: the host q_local is download-only
        host = q_local if isinstance(q_local, torch.Tensor) else np.asarray(q_local)
        if host.dtype not in (np.float64, torch.float64):
            raise TypeError(f"q_local: expected float64, got {host.dtype}")
        sl = _lib.Staged(torch.empty(ids.nl, dtype=torch.float64, device=dev), host,
                         "cpu" if isinstance(host, torch.Tensor) else "numpy")
    else:
        sl = _lib.stage(q_local, torch.float64, "q_local", dev)
    id_t = _op_dev(ids, "ids", dev)
    L = _lib.lib()
    _lib.check(L.sb_bs7_scatter(id_t.data_ptr(), int(id_t.shape[0]), sg.dev.data_ptr(), ng,
                                sl.dev.data_ptr(), int(bool(ids.has_mask)),
                                _lib.stream_handle(dev)), "bs7_scatter")
    sl.writeback()
