"""BS6 gather (Z^T) and BS7 scatter (Z) on the B200 (gs.py of the reference).

Same signatures, error messages and results as pkg/src/streambench/gs.py:
bs6_gather returns a new vector whose rows are summed in ascending column
order from +0.0 (bitwise the reference), bs7_scatter writes q_local in place
and leaves masked (-1) entries untouched.  Operators may be this package's
device GatherOp/ScatterIds or the reference's numpy ones (staged per call).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def _dev_int(a, name, device):
    if isinstance(a, torch.Tensor) and a.is_cuda:
        return a
    return _lib.stage(a, torch.int32, name, device).dev


def bs6_gather_into(op, q_local: torch.Tensor, out: torch.Tensor, carry=None) -> torch.Tensor:
    """Device-only BS6 writing `out` (length op.ng); optional carry-in partials
    seed rows [0, len(carry)) instead of +0.0 (multi-GPU carry halo)."""
    dev = q_local.device
    L = _lib.lib()
    ncarry = 0 if carry is None else int(carry.shape[0])
    plan = op.plan() if hasattr(op, "plan") else None
    if plan is not None:
        _lib.check(L.sb_bs6_gather_planned(plan.data_ptr(), op.n_blocks, op.nodes_per_block,
                                           op.row_starts.data_ptr(), op.col_ids.data_ptr(), op.ng,
                                           op.nl, q_local.data_ptr(), out.data_ptr(),
                                           None if carry is None else carry.data_ptr(), ncarry,
                                           _lib.stream_handle(dev)), "bs6_gather")
        return out
    bst = _dev_int(op.block_starts, "block_starts", dev)
    rs = _dev_int(op.row_starts, "row_starts", dev)
    ci = _dev_int(op.col_ids, "col_ids", dev)
    _lib.check(L.sb_bs6_gather(bst.data_ptr(), int(bst.shape[0]) - 1, rs.data_ptr(), ci.data_ptr(),
                               op.ng, int(ci.shape[0]), op.nodes_per_block, q_local.data_ptr(),
                               out.data_ptr(), None if carry is None else carry.data_ptr(), ncarry,
                               _lib.stream_handle(dev)), "bs6_gather")
    return out


def bs6_gather(op, q_local, out=None):
    """gs.py:10-39: out[r] = sum of q_local over row r's columns, ascending order."""
    if q_local.shape[0] != op.nl:
        raise ValueError(f"local vector length {q_local.shape[0]} != operator NL {op.nl}")
    host = not (isinstance(q_local, torch.Tensor) and q_local.is_cuda)
    q = _lib.stage(q_local, torch.float64, "q_local").dev
    if out is None:
        out = torch.empty(op.ng, dtype=torch.float64, device=q.device)
    bs6_gather_into(op, q, out)
    if host:
        res = out.cpu()
        return res.numpy() if isinstance(q_local, np.ndarray) else res
    return out


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
    sg = _lib.stage(q_global, torch.float64, "q_global")
    dev = sg.dev.device
    sl = _lib.stage(q_local, torch.float64, "q_local", dev)
    id_t = _dev_int(ids.ids, "ids", dev)
    L = _lib.lib()
    _lib.check(L.sb_bs7_scatter(id_t.data_ptr(), int(id_t.shape[0]), sg.dev.data_ptr(), ng,
                                sl.dev.data_ptr(), int(bool(ids.has_mask)),
                                _lib.stream_handle(dev)), "bs7_scatter")
    sl.writeback()
