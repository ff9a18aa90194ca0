"""Host-buffer execution of the streaming kernels (the drop-in numpy path).

When a caller hands BS1-BS5 host arrays (numpy, or CPU torch tensors --
pinned ones transfer at full PCIe speed), the data must cross PCIe twice, so
the call is transfer-bound.  This module overlaps the two directions and the
kernels: vectors are cut into chunks; chunk i's upload (copy stream), its
kernel (compute stream) and chunk i-1's download (second copy stream) run
concurrently, ordered by CUDA events.  Outputs that are write-only (BS1's y)
are never uploaded.  Reductions run once on the assembled device vectors, so
every scalar is bitwise the device-resident result.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

CHUNK = 1 << 23  # elements per pipelined chunk (64 MiB of fp64)

_streams: dict = {}


def _side_streams(device: torch.device):
    s = _streams.get(device.index)
    if s is None:
        s = (torch.cuda.Stream(device), torch.cuda.Stream(device))
        _streams[device.index] = s
    return s


def as_host_tensor(a, name: str) -> torch.Tensor:
    """A CPU float64 1-D torch view of a host array (numpy or torch)."""
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64:
            raise TypeError(f"{name}: expected torch.float64, got {a.dtype}")
        t = a
    else:
        arr = np.asarray(a)
        if arr.dtype != np.float64:
            raise TypeError(f"{name}: expected float64, got {arr.dtype}")
        if not arr.flags.c_contiguous:
            raise ValueError(f"{name}: host vectors must be contiguous")
        t = torch.from_numpy(arr)
    if t.dim() != 1:
        raise ValueError(f"expected a 1-D vector, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: host vectors must be contiguous")
    return t


def run(n: int, upload: dict, download: dict, scratch: tuple, chunk_fn=None, final_fn=None,
        device: torch.device | None = None):
    """Pipelined host -> device -> host execution over n elements.

    upload:   name -> host tensor copied to a device buffer of the same name
    download: name -> host tensor receiving the device buffer after chunk_fn
    scratch:  names of device-only buffers (write-only outputs)
    chunk_fn(dev, lo, hi) launches the per-chunk kernels on the current stream;
    final_fn(dev) runs once after every chunk and returns the call's result.
    """
    _lib.lib()
    dev_ = device or torch.device("cuda", torch.cuda.current_device())
    comp = torch.cuda.current_stream(dev_)
    up, down = _side_streams(dev_)
    names = set(upload) | set(download) | set(scratch)
    dev = {k: torch.empty(n, dtype=torch.float64, device=dev_) for k in names}
    up.wait_stream(comp)  # device buffers are allocated on comp
    down.wait_stream(comp)
    for lo in range(0, max(n, 1), CHUNK):
        hi = min(n, lo + CHUNK)
        if hi <= lo:
            break
        with torch.cuda.stream(up):
            for k, h in upload.items():
                dev[k][lo:hi].copy_(h[lo:hi], non_blocking=True)
            ev_up = torch.cuda.Event()
            ev_up.record(up)
        comp.wait_event(ev_up)
        if chunk_fn is not None:
            chunk_fn(dev, lo, hi)
        if download:
            ev_c = torch.cuda.Event()
            ev_c.record(comp)
            down.wait_event(ev_c)
            with torch.cuda.stream(down):
                for k, h in download.items():
                    h[lo:hi].copy_(dev[k][lo:hi], non_blocking=True)
    comp.wait_stream(up)
    result = final_fn(dev) if final_fn is not None else None
    down.synchronize()
    comp.synchronize()  # after this every side-stream use of `dev` has completed
    return result


def run_prefix(src_host: torch.Tensor, src_dev: torch.Tensor, out_dev: torch.Tensor,
               out_host: torch.Tensor, jobs, launch, device: torch.device) -> None:
    """Gather-style pipeline: output range j may start once the input prefix
    [0, need_j) is on the device.

    The input is uploaded in order in CHUNK pieces (one event each) on the
    upload stream; job (o_lo, o_hi, need) waits for the first event covering
    `need`, launches `launch(o_lo, o_hi)` on the compute stream, and its
    output range is downloaded on the download stream -- so H2D of the input
    tail, the kernels and D2H of the output head overlap.
    """
    comp = torch.cuda.current_stream(device)
    up, down = _side_streams(device)
    up.wait_stream(comp)
    down.wait_stream(comp)
    n_in = src_host.shape[0]
    marks = []
    with torch.cuda.stream(up):
        for lo in range(0, n_in, CHUNK):
            hi = min(n_in, lo + CHUNK)
            src_dev[lo:hi].copy_(src_host[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
            marks.append((hi, ev))
    k = 0
    for o_lo, o_hi, need in jobs:
        while k < len(marks) - 1 and marks[k][0] < need:
            k += 1
        if marks:
            comp.wait_event(marks[k][1])
        launch(o_lo, o_hi)
        ev_c = torch.cuda.Event()
        ev_c.record(comp)
        down.wait_event(ev_c)
        with torch.cuda.stream(down):
            out_host[o_lo:o_hi].copy_(out_dev[o_lo:o_hi], non_blocking=True)
    comp.wait_stream(up)
    down.synchronize()
    comp.synchronize()


def all_host(*vs) -> bool:
    return all(not (isinstance(v, torch.Tensor) and v.is_cuda) for v in vs)
