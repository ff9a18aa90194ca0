"""Bandwidth sweeps + T0/Wmax fits on one B200 (BASELINE configs 2 and 3).

    python scripts/sweep.py --out profiles/sweep_r01 [--points 60] [--timer device]

config 2: BS1-BS5 over n = 1e3 .. 1e9 DOFs (geometric, --points sizes per test)
config 3: BS6/BS7 for N = 1..15, K geometric from 2 up to NG ~ 1e8
Writes <out>.csv (the reference CLI's wire format, so `streambench fit` and
`streambench-plot` read it unchanged) and <out>_fit.json with the model fit
(model.fit_model, the reference's centred OLS) per (test, order), both over
all sizes and over sizes above the L2 capacity.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2009_10917_b200 import cli, harness, model  # noqa: E402
from paper_2009_10917_b200.kernels import ReductionConfig  # noqa: E402


def mesh_sizes(order: int, ng_max: float, count: int) -> list[tuple[int, int]]:
    kmax = max(2, int(round((ng_max ** (1 / 3) - 1) / order)))
    ks = sorted({int(round(v)) for v in np.geomspace(2, kmax, count)})
    return [(k, order) for k in ks]


def fits(samples, min_bytes=0):
    groups = {}
    for s in samples:
        if s.bytes >= min_bytes:
            groups.setdefault((s.test, s.order), []).append(s)
    out = []
    for (test, order), g in sorted(groups.items(), key=lambda kv: (kv[0][0], kv[0][1] or 0)):
        try:
            f = model.fit_model(g)
        except model.ModelFitError as exc:
            out.append({"test": test, "order": order, "error": str(exc)})
            continue
        out.append({"test": test, "order": order, "T0_us": f.t0 * 1e6, "Wmax_GBps": f.wmax / 1e9,
                    "B80_MB": model.efficiency_point(f) / 1e6, "r2": f.r2, "n_points": f.n_points,
                    "clamped_T0": f.clamped_t0,
                    "peak_sample_GBps": max(s.bandwidth for s in g)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep")
    ap.add_argument("--points", type=int, default=60)
    ap.add_argument("--mesh-points", type=int, default=10)
    ap.add_argument("--max-dofs", type=float, default=1e9)
    ap.add_argument("--mesh-ng", type=float, default=1e8)
    ap.add_argument("--orders", default="1-15")
    ap.add_argument("--timer", default="device", choices=["host", "device", "graph"])
    ap.add_argument("--trials", type=int, default=20)
    ap.add_argument("--tests", default="bs1,bs2,bs3,bs4,bs5,bs6,bs7")
    args = ap.parse_args()
    lo, hi = (int(v) for v in args.orders.split("-"))
    cfg = ReductionConfig()
    samples = []
    t0 = time.time()
    for test in args.tests.split(","):
        if test in ("bs6", "bs7"):
            for order in range(lo, hi + 1):
                plan = harness.SweepPlan(test=test, sizes=mesh_sizes(order, args.mesh_ng, args.mesh_points),
                                         trials=args.trials, warmup=2)
                samples += harness.run_sweep(plan, cfg, timer=args.timer)
                torch.cuda.empty_cache()
        else:
            sizes = harness.geometric_sizes(1000, int(args.max_dofs), args.points)
            plan = harness.SweepPlan(test=test, sizes=sizes, trials=args.trials, warmup=2)
            samples += harness.run_sweep(plan, cfg, timer=args.timer)
            torch.cuda.empty_cache()
        print(f"{test}: done at {time.time() - t0:.0f} s", file=sys.stderr, flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".csv", "w", newline="") as f:
        cli.write_samples_csv(samples, f)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    rep = {"timer": args.timer, "trials": args.trials, "device": torch.cuda.get_device_name(0),
           "l2_bytes": l2, "fit_all_sizes": fits(samples),
           "fit_above_4x_l2": fits(samples, 4 * l2)}
    with open(args.out + "_fit.json", "w") as f:
        json.dump(rep, f, indent=1)
    for r in rep["fit_above_4x_l2"]:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
