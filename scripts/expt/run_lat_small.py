"""Graph-timed per-call time of BS3/BS4/BS5 at small and mid n for the
variant libraries of build_lat_small.sh (and BS1 from libsb200 as the floor).

Each (variant, test, n) is one CUDA graph of K back-to-back calls; the time
per call is the graph replay time / K, median of R replays.  Also checks the
variants return the same scalar bit for bit.  Env SB200_NO_TMA=1 is honoured
by every variant (register lattice at all sizes)."""
import ctypes
import glob
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
c_vp, c_i64, c_d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double


def load(so):
    L = ctypes.CDLL(so)
    L.sb_reduce_workspace_bytes.restype = ctypes.c_size_t
    L.sb_reduce_workspace_bytes.argtypes = [c_i64, c_i64]
    L.sb_bs1_copy.argtypes = [c_vp, c_vp, c_i64, c_vp]
    L.sb_bs3_norm2.argtypes = [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    L.sb_bs4_dot.argtypes = [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    L.sb_bs5_fused_cg_update.argtypes = [c_d, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]
    return L


libs = {os.path.basename(s)[:-3]: load(s) for s in sorted(glob.glob(os.path.join(HERE, "_lat2", "*.so")))}
dev = torch.device("cuda", 0)
K, R = int(os.environ.get("K", 20)), int(os.environ.get("R", 7))
sizes = sorted({int(v) for v in np.geomspace(1e3, float(os.environ.get("NMAX", 6e7)), int(os.environ.get("PTS", 26)))})
bs, nb = 256, 512
nmax = max(sizes)
g = torch.Generator(device=dev).manual_seed(1)
x, y, p, ap = (torch.rand(nmax, dtype=torch.float64, device=dev, generator=g) for _ in range(4))
x2 = torch.empty_like(x)
res = torch.zeros(64, dtype=torch.float64, device=dev)
out = {"K": K, "R": R, "rows": []}
side = torch.cuda.Stream(dev)


flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MB > L2


def graph_time(fn):
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=side):
        for _ in range(K):
            fn()
    for _ in range(3):
        gr.replay()
    ts = []
    for _ in range(R):
        flush.fill_(1.0)  # every replay starts from a cold L2 (same for every variant)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / K)
    return float(np.median(ts))


for n in sizes:
    row = {"n": n}
    st = side.cuda_stream
    L0 = libs["new"]
    row["bs1"] = graph_time(lambda: L0.sb_bs1_copy(x.data_ptr(), x2.data_ptr(), n, st))
    vals = {}
    names = list(libs)
    rot = len(out["rows"]) % len(names)  # rotate the variant order per size
    for name in names[rot:] + names[:rot]:
        L = libs[name]
        ws = torch.zeros(L.sb_reduce_workspace_bytes(bs, nb), dtype=torch.uint8, device=dev)
        calls = {
            "bs3": lambda: L.sb_bs3_norm2(x.data_ptr(), n, bs, nb, ws.data_ptr(), res.data_ptr(), st),
            "bs4": lambda: L.sb_bs4_dot(x.data_ptr(), y.data_ptr(), n, bs, nb, ws.data_ptr(),
                                        res[1:].data_ptr(), st),
            "bs5": lambda: L.sb_bs5_fused_cg_update(0.0, p.data_ptr(), ap.data_ptr(), x2.data_ptr(),
                                                    y.data_ptr(), n, bs, nb, ws.data_ptr(),
                                                    res[2:].data_ptr(), st),
        }
        for t, fn in calls.items():
            row[f"{t}_{name}"] = graph_time(fn)
        torch.cuda.synchronize()
        vals[name] = res[:3].cpu().numpy().tobytes()
    row["same_bits"] = len(set(vals.values())) == 1
    out["rows"].append(row)
    print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
tag = os.environ.get("TAG", "lat_small")
with open(f"gpurun_out/{tag}.json", "w") as f:
    json.dump(out, f, indent=1)
