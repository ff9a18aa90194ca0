"""A/B the lattice ring shapes (scripts/expt/lattice_variants.txt) for BS3/BS4/BS5 on the box."""
import ctypes
import glob
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
c_vp, c_i64, c_d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
libs = {}
for so in sorted(glob.glob(os.path.join(HERE, "_lat", "*.so"))):
    L = ctypes.CDLL(so)
    L.sb_reduce_workspace_bytes.restype = ctypes.c_size_t
    L.sb_reduce_workspace_bytes.argtypes = [c_i64, c_i64]
    L.sb_bs3_norm2.argtypes = [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    L.sb_bs4_dot.argtypes = [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    L.sb_bs5_fused_cg_update.argtypes = [c_d, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    libs[os.path.basename(so)[:-3]] = L

dev = torch.device("cuda", 0)
cfgs = [tuple(int(v) for v in c.split(",")) for c in os.environ.get("SB_CFGS", "256,512").split(";")]
for (bs, nb), n in [(c, int(float(a))) for c in cfgs for a in (sys.argv[1:] or ["1e8", "4e8"])]:
    g = torch.Generator(device=dev).manual_seed(1)
    x, y, p, ap = (torch.rand(n, dtype=torch.float64, device=dev, generator=g) for _ in range(4))
    x0, r0 = x.clone(), y.clone()
    res = torch.zeros(1, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ref = {}
    for name, L in libs.items():
        ws = torch.zeros(L.sb_reduce_workspace_bytes(bs, nb), dtype=torch.uint8, device=dev)
        calls = {
            "bs3": (lambda: L.sb_bs3_norm2(x.data_ptr(), n, bs, nb, ws.data_ptr(), res.data_ptr(), st), 8 * n),
            "bs4": (lambda: L.sb_bs4_dot(x.data_ptr(), y.data_ptr(), n, bs, nb, ws.data_ptr(), res.data_ptr(), st),
                    16 * n),
            "bs5": (lambda: L.sb_bs5_fused_cg_update(0.25, p.data_ptr(), ap.data_ptr(), x.data_ptr(), y.data_ptr(),
                                                     n, bs, nb, ws.data_ptr(), res.data_ptr(), st), 48 * n),
        }
        line = []
        for t, (fn, nbytes) in calls.items():
            x.copy_(x0); y.copy_(r0)
            assert fn() == 0
            torch.cuda.synchronize()
            val = res.item()
            key = (t, n)
            ok = ref.setdefault(key, val) == val
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            line.append(f"{t} {nbytes / ms / 1e6:6.0f} GB/s{'' if ok else ' MISMATCH'}")
        print(f"n={n:.0e} cfg=({bs},{nb}) {name}: " + " | ".join(line), flush=True)
    del x, y, p, ap, x0, r0
    torch.cuda.empty_cache()
