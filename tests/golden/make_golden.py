"""Generate the golden fixtures from the UNMODIFIED reference implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/streambench, runs the reference kernels,
builders, harness allocation and model fit on seeded inputs and writes

    tests/golden/golden.json   scalars (float.hex), hashes, small int arrays
    tests/golden/arrays.npz    small raw arrays (mesh operators, outputs)

Inputs are NOT stored: they are regenerated from numpy's seeded PCG64 streams
(np.random.default_rng(seq).uniform(-1, 1, n)) and their sha256 is recorded so
a numpy stream change is detected instead of silently mis-pinning.  Large
outputs are stored as sha256 of the little-endian bytes.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fx(v: float) -> str:
    return float(v).hex()


def main() -> None:
    sys.path.insert(0, REF)
    from streambench import cli, harness, kernels, mesh, model, parallel, reference  # noqa
    from streambench.gs import bs6_gather, bs7_scatter

    parallel.set_num_workers(1)
    G: dict = {"vectors": [], "cfg_sweep": [], "harness": [], "meshes": [], "masks": [],
               "model": {}, "geometric": [], "csv": []}
    arrays: dict[str, np.ndarray] = {}

    # ---- A1: selftest-style vectors (selftest.py:18-83), several cfgs ------
    cfgs = [(256, 512), (2, 1), (4, 3), (64, 7), (512, 512), (1024, 1184), (128, 296),
            (32, 1), (1024, 1)]
    for n in [0, 1, 3, 255, 1000, 4097, 65537, 131073, 300001]:
        rng = np.random.default_rng([2024, n])
        alpha, beta = rng.uniform(-2, 2, 2)
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        p, ap = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        rec = {"n": n, "seed": [2024, n], "draws": "alpha,beta(-2,2);x;y;p;ap",
               "in_hash": h(np.concatenate([x, y, p, ap])),
               "alpha": fx(alpha), "beta": fx(beta)}
        yy = y.copy()
        kernels.bs2_axpy(alpha, x, beta, yy)
        rec["bs2_hash"] = h(yy)
        rec["norm2"], rec["dot"], rec["bs5"], rec["bs5_x"], rec["bs5_r"] = {}, {}, {}, {}, {}
        for bs, nb in cfgs:
            cfg = kernels.ReductionConfig(bs, nb)
            key = f"{bs},{nb}"
            rec["norm2"][key] = fx(kernels.bs3_norm2(x, cfg))
            rec["dot"][key] = fx(kernels.bs4_dot(x, y, cfg))
            xx, rr = x.copy(), y.copy()
            rec["bs5"][key] = fx(kernels.bs5_fused_cg_update(alpha, p, ap, xx, rr, cfg))
            rec["bs5_x"][key] = h(xx)
            rec["bs5_r"][key] = h(rr)
        if n <= 4097:
            rec["fsum_norm2"] = fx(reference.norm2(x))
            rec["fsum_dot"] = fx(reference.dot(x, y))
        G["vectors"].append(rec)
        print("vectors", n, flush=True)

    # ---- A2: acceptance sizes (test_acceptance.py:87-122), default cfg -----
    rng = np.random.default_rng(2718)
    sizes = {1, 10**6, 524288}
    while len(sizes) < 50:
        sizes.add(int(np.exp(rng.uniform(0, np.log(10**6)))) + 1)
    cfg = kernels.ReductionConfig(256, 512)
    for n in sorted(sizes):
        gen = np.random.default_rng([31337, n])
        x = gen.uniform(-1, 1, n)
        y = gen.uniform(-1, 1, n)
        alpha, beta = gen.uniform(-2, 2, 2)
        p, ap = gen.uniform(-1, 1, n), gen.uniform(-1, 1, n)
        yy = y.copy()
        kernels.bs2_axpy(alpha, x, beta, yy)
        xx, rr = x.copy(), y.copy()
        b5 = kernels.bs5_fused_cg_update(alpha, p, ap, xx, rr, cfg)
        G["cfg_sweep"].append({
            "n": n, "seed": [31337, n], "draws": "x;y;alpha,beta(-2,2);p;ap",
            "in_hash": h(np.concatenate([x, y, p, ap])),
            "bs2_hash": h(yy), "norm2": fx(kernels.bs3_norm2(x, cfg)),
            "dot": fx(kernels.bs4_dot(x, y, cfg)), "bs5": fx(b5),
            "bs5_x": h(xx), "bs5_r": h(rr)})
    print("acceptance sizes done", flush=True)

    # ---- A3: harness allocation convention (harness.py:116-181) at C1 -----
    for test in ("bs1", "bs2", "bs3", "bs4", "bs5"):
        for n in (1000, 1442897):
            case = harness._VectorCase(test, n, 0, kernels.DEFAULT_REDUCTION)
            s = case.alloc()
            case.snapshot(s)
            case.run(s)
            assert case.validate(s)
            rec = {"test": test, "n": n, "seed": 0}
            if test in ("bs2", "bs5"):
                rec["alpha"] = fx(s["alpha"])
            if test == "bs2":
                rec["beta"] = fx(s["beta"])
                rec["y"] = h(s["y"])
            if test == "bs1":
                rec["y"] = h(s["y"])
            if test in ("bs3", "bs4", "bs5"):
                rec["result"] = fx(s["result"])
            if test == "bs5":
                rec["x"], rec["r"] = h(s["x"]), h(s["r"])
            G["harness"].append(rec)
    print("harness done", flush=True)

    # ---- B: meshes, operators, gather/scatter (mesh.py, gs.py) ------------
    mesh_cases = [(1, 1, 512), (2, 1, 512), (2, 2, 16), (3, 2, 64), (2, 3, 512), (3, 4, 128),
                  (4, 3, 512), (5, 2, 8), (3, 7, 512), (4, 5, 40), (5, 1, 512), (2, 15, 512),
                  (4, 7, 512), (3, 3, 8), (6, 2, 1000), (8, 3, 512), (16, 7, 512)]
    for K, p, npb in mesh_cases:
        m = mesh.build_mesh(K, p)
        op = mesh.build_gather(m, npb)
        ids = mesh.build_scatter_ids(m)
        rng = np.random.default_rng([0, K, p])
        q_local = rng.uniform(-1, 1, m.nl)
        out = bs6_gather(op, q_local)
        rng = np.random.default_rng([0, K, p])
        q_global = rng.uniform(-1, 1, m.ng)
        ql = np.zeros(m.nl)
        bs7_scatter(ids, q_global, ql)
        mult = mesh.multiplicity(m)
        rec = {"K": K, "p": p, "npb": npb, "nl": m.nl, "ng": m.ng, "n_blocks": op.n_blocks,
               "l2g": h(m.local_to_global), "row_starts": h(op.row_starts),
               "col_ids": h(op.col_ids), "block_starts": h(op.block_starts),
               "bs6_q_hash": h(q_local), "bs6_out": h(out),
               "bs7_qg_hash": h(q_global), "bs7_out": h(ql), "mult": h(mult),
               "bytes_bs6": harness.bytes_moved("bs6", nl=m.nl, ng=m.ng),
               "bytes_bs7": harness.bytes_moved("bs7", nl=m.nl, ng=m.ng)}
        if m.nl <= 20000:
            tag = f"{K}_{p}_{npb}"
            arrays[f"l2g_{tag}"] = m.local_to_global
            arrays[f"rs_{tag}"] = op.row_starts
            arrays[f"ci_{tag}"] = op.col_ids
            arrays[f"bst_{tag}"] = op.block_starts
            arrays[f"bs6_{tag}"] = out
        G["meshes"].append(rec)
        print("mesh", K, p, npb, flush=True)

    # masks (test_mesh.py:118-127, test_gs.py:101-119)
    for K, p, mask in [(2, 1, [13]), (3, 2, [0, 5, 17, 100, 342]), (2, 2, list(range(125))),
                       (4, 3, list(range(0, 2197, 7)))]:
        m = mesh.build_mesh(K, p)
        ids = mesh.build_scatter_ids(m, mask=set(mask))
        rng = np.random.default_rng([9, K, p])
        q_global = rng.uniform(-1, 1, m.ng)
        ql = np.full(m.nl, 99.0)
        bs7_scatter(ids, q_global, ql)
        tag = f"{K}_{p}"
        arrays[f"mask_ids_{tag}"] = ids.ids
        G["masks"].append({"K": K, "p": p, "mask": mask, "has_mask": bool(ids.has_mask),
                           "ids": h(ids.ids), "qg_hash": h(q_global), "out": h(ql)})

    # ---- C: model fit (model.py), geometric sizes, CSV --------------------
    t0, wmax = 5e-6, 8e11
    sizes = np.unique(np.rint(np.geomspace(1e3, 1e9, 100)).astype(np.int64))
    exact = [harness.BandwidthSample("bs1", int(b), (t0 + int(b) / wmax) * 20, 20, 0.0)
             for b in sizes]
    fits = {}
    for name, weighted, samples in [("exact", False, exact), ("exact_w", True, exact)]:
        f = model.fit_model(samples, weighted=weighted)
        fits[name] = {"t0": fx(f.t0), "wmax": fx(f.wmax), "r2": fx(f.r2), "n": f.n_points,
                      "clamped": f.clamped_t0}
    for seed in range(5):
        rng = np.random.default_rng([seed, 99])
        noisy = [harness.BandwidthSample("bs1", int(b),
                                         (t0 + int(b) / wmax) * (1 + 0.01 * rng.standard_normal())
                                         * 20, 20, 0.0) for b in sizes]
        for weighted in (False, True):
            f = model.fit_model(noisy, weighted=weighted)
            fits[f"noisy{seed}_{int(weighted)}"] = {"t0": fx(f.t0), "wmax": fx(f.wmax),
                                                    "r2": fx(f.r2), "n": f.n_points,
                                                    "clamped": f.clamped_t0}
    G["model"] = {"t0": t0, "wmax": wmax, "sizes": [int(s) for s in sizes], "fits": fits,
                  "b80_v100": fx(model.efficiency_point(model.ModelFit(7.62e-6, 809e9, 1.0, 2))),
                  "b80_mi60": fx(model.efficiency_point(model.ModelFit(16.99e-6, 843e9, 1.0, 2))),
                  "weff_v100_bs1": fx(model.w_eff(model.ModelFit(2.90e-6, 811e9, 1.0, 2), 0.1e9))}
    for args in [(1, 1, 5), (1, 1024, 11), (10, 10**7, 400), (1, 16, 100), (7, 900, 1),
                 (21, 20833333, 400), (63, 62500000, 400), (125, 125000000, 400)]:
        G["geometric"].append({"args": list(args), "sizes": harness.geometric_sizes(*args)})
    for test, sz in [("bs1", [10, 1000, 100000]), ("bs7", [(2, 3), (3, 3)])]:
        plan = harness.SweepPlan(test=test, sizes=sz, trials=2)
        for s in harness.run_sweep(plan):
            s2 = harness.BandwidthSample(s.test, s.bytes, 0.125, s.trials, 1.0 / 3.0, s.n,
                                         s.order, s.K, s.nl, s.ng)
            G["csv"].append({"row": cli.sample_to_csv_row(s2), "test": s.test, "bytes": s.bytes,
                             "n": s.n, "K": s.K, "order": s.order, "nl": s.nl, "ng": s.ng,
                             "trials": s.trials})
    G["csv_header"] = cli.CSV_HEADER

    # ---- CG (cg.py:27-72) on diagonal operators: elementwise d*v rounds the
    # same on every device, so these pin the device CG bitwise -------------
    from streambench import cg as rcg
    G["cg"] = []
    cases = [  # n, seed, d range, eps, max_iter, cfg, fused, relative, x0 nonzero
        (1000, 1, (1.0, 10.0), 1e-20, 200, (256, 512), True, False, False),
        (1000, 1, (1.0, 10.0), 1e-20, 200, (256, 512), False, False, False),
        (4097, 2, (0.5, 50.0), 1e-18, 300, (64, 7), True, True, False),
        (4097, 2, (0.5, 50.0), 1e-18, 300, (64, 7), False, True, True),
        (3000, 3, (1.0, 1e4), 1e-30, 5, (256, 512), True, False, True),   # max_iter exhausted
        (777, 4, (2.0, 2.0), 1e-20, 50, (32, 3), True, False, False),     # one distinct eigenvalue
        (50000, 5, (1.0, 100.0), 1e-16, 400, (256, 512), True, True, True),
    ]
    for n, seed, (lo, hi), eps, mi, cfg, fused, rel, x0nz in cases:
        rng = np.random.default_rng([seed, n, 77])
        d = rng.uniform(lo, hi, n)
        b = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n) if x0nz else np.zeros(n)
        res = rcg.cg_solve(rcg.diagonal_operator(d), b, x0, eps, mi,
                           kernels.ReductionConfig(*cfg), fused=fused, relative=rel)
        G["cg"].append({"n": n, "seed": [seed, n, 77], "draws": "d~U(lo,hi);b~U(-1,1);x0~U(-1,1)|0",
                        "d_range": [lo, hi], "eps": fx(eps), "max_iter": mi, "cfg": list(cfg),
                        "fused": fused, "relative": rel, "x0_nonzero": x0nz,
                        "in_hash": h(np.concatenate([d, b, x0])), "iterations": res.iterations,
                        "final_rr": fx(res.final_rr), "converged": bool(res.converged),
                        "x_hash": h(res.x)})

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(G, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "arrays.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
