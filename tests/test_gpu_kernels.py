"""BS1-BS5 on the B200 vs the golden vectors of the reference and the CPU oracle.

Bitwise: BS1, BS2, BS5 vectors and the BS3/BS4/BS5 scalars at the same
ReductionConfig (kernels.py:38-87 fixes every rounding).  Reductions are also
checked <= 1e-12 relative against the exact (fsum) references.
"""

import math

import numpy as np
import pytest
import torch

from goldens import acceptance_inputs, selftest_inputs, sha, unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    _lib.lib()  # fail loudly if the CUDA library is not loadable
    return sb


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def h(t):
    return t.cpu().numpy()


def test_library_is_native(sb):
    from paper_2009_10917_b200 import _lib
    assert _lib.lib()._name.endswith("libsb200.so")
    sm, major = torch.cuda.get_device_capability()[0], None
    assert sm >= 10, "expects a Blackwell (sm_100a) device"


def test_selftest_vectors_all_configs(sb, golden):
    for rec in golden["vectors"]:
        n = rec["n"]
        alpha, beta, x, y, p, ap = selftest_inputs(n)
        assert sha(np.concatenate([x, y, p, ap])) == rec["in_hash"]
        X, Y, P, AP = d(x), d(y), d(p), d(ap)
        out = torch.zeros_like(X)
        sb.bs1_copy(X, out)
        assert torch.equal(out, X)
        yy = Y.clone()
        sb.bs2_axpy(alpha, X, beta, yy)
        assert sha(h(yy)) == rec["bs2_hash"], n
        for key in rec["norm2"]:
            bs, nb = (int(v) for v in key.split(","))
            cfg = sb.ReductionConfig(bs, nb)
            assert sb.bs3_norm2(X, cfg) == unhex(rec["norm2"][key]), (n, key)
            assert sb.bs4_dot(X, Y, cfg) == unhex(rec["dot"][key]), (n, key)
            xx, rr = X.clone(), Y.clone()
            got = sb.bs5_fused_cg_update(alpha, P, AP, xx, rr, cfg)
            assert got == unhex(rec["bs5"][key]), (n, key)
            assert sha(h(xx)) == rec["bs5_x"][key] and sha(h(rr)) == rec["bs5_r"][key], (n, key)


def test_acceptance_sizes(sb, golden):
    # test_acceptance.py:87-122 -- 50 randomized sizes up to 1e6, default cfg
    for rec in golden["cfg_sweep"]:
        n = rec["n"]
        alpha, beta, x, y, p, ap = acceptance_inputs(n)
        X, Y, P, AP = d(x), d(y), d(p), d(ap)
        yy = Y.clone()
        sb.bs2_axpy(alpha, X, beta, yy)
        assert sha(h(yy)) == rec["bs2_hash"]
        assert sb.bs3_norm2(X) == unhex(rec["norm2"])
        assert sb.bs4_dot(X, Y) == unhex(rec["dot"])
        xx, rr = X.clone(), Y.clone()
        assert sb.bs5_fused_cg_update(alpha, P, AP, xx, rr) == unhex(rec["bs5"])
        assert sha(h(xx)) == rec["bs5_x"] and sha(h(rr)) == rec["bs5_r"]
        if n <= 200000:
            from paper_2009_10917_b200 import reference as R
            assert R.relative_error(sb.bs3_norm2(X), math.fsum((x * x).tolist())) <= 1e-12
            assert R.relative_error(sb.bs4_dot(X, Y), math.fsum((x * y).tolist())) <= 1e-12


def test_harness_convention_c1(sb, golden):
    # harness.py:116-132 allocation at C1 (n = NG(16,7) = 1,442,897)
    from paper_2009_10917_b200.harness import Inputs
    for rec in golden["harness"]:
        n, test = rec["n"], rec["test"]
        g = Inputs([0, n], "cuda")
        if test == "bs1":
            x = g.vector(n); y = torch.zeros_like(x)
            sb.bs1_copy(x, y)
            assert sha(h(y)) == rec["y"]
        elif test == "bs2":
            a, b = g.scalar(), g.scalar()
            assert a == unhex(rec["alpha"]) and b == unhex(rec["beta"])
            x, y = g.vector(n), g.vector(n)
            sb.bs2_axpy(a, x, b, y)
            assert sha(h(y)) == rec["y"]
        elif test == "bs3":
            assert sb.bs3_norm2(g.vector(n)) == unhex(rec["result"])
        elif test == "bs4":
            x, y = g.vector(n), g.vector(n)
            assert sb.bs4_dot(x, y) == unhex(rec["result"])
        else:
            a = g.scalar()
            p, ap, x, r = (g.vector(n) for _ in range(4))
            assert sb.bs5_fused_cg_update(a, p, ap, x, r) == unhex(rec["result"])
            assert sha(h(x)) == rec["x"] and sha(h(r)) == rec["r"]


@pytest.mark.parametrize("cfg", [(2, 1), (4, 3), (32, 5), (64, 7), (128, 1), (256, 512), (256, 1184),
                                 (512, 37), (1024, 1184), (2048, 3), (4096, 2), (8, 20000)])
@pytest.mark.parametrize("n", [0, 1, 7, 4097, 300001, 2_000_003])
def test_reductions_vs_oracle(sb, oracle, cfg, n):
    bs, nb = cfg
    rng = np.random.default_rng([n, bs, nb])
    x, y, p, ap = (rng.uniform(-1, 1, n) for _ in range(4))
    alpha = float(rng.uniform(-1, 1))
    c = sb.ReductionConfig(bs, nb)
    X, Y, P, AP = d(x), d(y), d(p), d(ap)
    assert sb.bs3_norm2(X, c) == oracle.bs3_norm2(x, bs, nb)
    assert sb.bs4_dot(X, Y, c) == oracle.bs4_dot(x, y, bs, nb)
    assert sb.bs4_dot(Y, X, c) == sb.bs4_dot(X, Y, c)  # symmetry (test_kernels.py:175-177)
    assert sb.bs4_dot(X, X, c) == sb.bs3_norm2(X, c)   # (test_kernels.py:163-165)
    xo, ro = x.copy(), y.copy()
    want = oracle.bs5_fused_cg_update(alpha, p, ap, xo, ro, bs, nb)
    xx, rr = X.clone(), Y.clone()
    assert sb.bs5_fused_cg_update(alpha, P, AP, xx, rr, c) == want
    assert np.array_equal(h(xx), xo) and np.array_equal(h(rr), ro)
    assert sb.bs3_norm2(rr, c) == want  # fusion equivalence on the same lattice


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [1, 2, 5, 1000, 99999])
def test_elementwise_alignment_and_odd_lengths(sb, oracle, offset, n):
    """Sub-tensor views at 8-byte offsets exercise the head/tail and scalar paths."""
    rng = np.random.default_rng([offset, n])
    base_x = d(rng.uniform(-1, 1, n + 4))
    base_y = d(rng.uniform(-1, 1, n + 4))
    for xo, yo in [(offset, offset), (offset, (offset + 1) % 4)]:
        x = base_x[xo:xo + n]
        y = base_y.clone()[yo:yo + n]
        xe, ye = h(x).copy(), h(y).copy()
        sb.bs2_axpy(-0.7, x, 1.3, y)
        oracle.bs2_axpy(-0.7, xe, 1.3, ye)
        assert np.array_equal(h(y), ye)
        z = torch.zeros_like(base_y)[yo:yo + n]
        sb.bs1_copy(x, z)
        assert torch.equal(z, x)
        assert sb.bs3_norm2(x) == oracle.bs3_norm2(xe)


def test_hand_kats_and_errors(sb):
    x = d([1.0, 2.0, 3.0]); y = torch.zeros(3, dtype=torch.float64, device="cuda")
    sb.bs1_copy(x, y); assert h(y).tolist() == [1.0, 2.0, 3.0]
    y = d([1.0]); sb.bs2_axpy(2.0, d([1.0]), 3.0, y); assert float(y[0]) == 5.0
    y = d([5.0, 6.0]); sb.bs2_axpy(0.0, d([9.0, 9.0]), 1.0, y); assert h(y).tolist() == [5.0, 6.0]
    assert sb.bs3_norm2(d([3.0, 4.0])) == 25.0
    assert sb.bs3_norm2(d(np.zeros(0))) == 0.0
    assert sb.bs4_dot(d([1.0, 2.0]), d([3.0, 4.0])) == 11.0
    xx, rr = d([0.0]), d([2.0])
    beta = sb.bs5_fused_cg_update(1.0, d([1.0]), d([2.0]), xx, rr)
    assert float(xx[0]) == 1.0 and float(rr[0]) == 0.0 and beta == 0.0
    z = np.zeros(1000); z[777] = 1e-150
    assert sb.bs3_norm2(d(np.zeros(1000))) == 0.0 and sb.bs3_norm2(d(z)) > 0.0
    with pytest.raises(ValueError):
        sb.bs1_copy(d(np.zeros(3)), d(np.zeros(4)))
    with pytest.raises(ValueError):
        sb.bs2_axpy(1.0, d(np.zeros(3)), 1.0, d(np.zeros(4)))
    with pytest.raises(ValueError):
        sb.bs4_dot(d(np.zeros(3)), d(np.zeros(4)))
    with pytest.raises(ValueError):
        sb.bs5_fused_cg_update(1.0, *(d(np.zeros(3)) for _ in range(3)), d(np.zeros(4)))
    for bad in (0, 1, 3, 24, 100):
        with pytest.raises(ValueError):
            sb.ReductionConfig(block_size=bad, n_blocks=4)


def test_numpy_drop_in(sb, oracle):
    """Host numpy arrays go through the device and keep in-place semantics."""
    rng = np.random.default_rng(5)
    x, y = rng.uniform(-1, 1, 257), rng.uniform(-1, 1, 257)
    loop = np.array([-0.7 * xi + 1.3 * yi for xi, yi in zip(x, y)])  # test_kernels.py:90-98
    sb.bs2_axpy(-0.7, x, 1.3, y)
    assert np.array_equal(y, loop)
    z = np.zeros(257)
    sb.bs1_copy(x, z)
    assert np.array_equal(z, x)
    assert sb.bs3_norm2(x) == oracle.bs3_norm2(x)
    p, ap, xx, rr = (rng.uniform(-1, 1, 1000) for _ in range(4))
    xo, ro = xx.copy(), rr.copy()
    want = oracle.bs5_fused_cg_update(0.3, p, ap, xo, ro)
    assert sb.bs5_fused_cg_update(0.3, p, ap, xx, rr) == want
    assert np.array_equal(xx, xo) and np.array_equal(rr, ro)


def test_async_matches_sync_and_determinism(sb):
    from paper_2009_10917_b200.kernels import bs3_norm2_async
    x = d(np.random.default_rng(21).uniform(-1, 1, 5_000_001))
    vals = {sb.bs3_norm2(x) for _ in range(5)}
    assert len(vals) == 1
    assert float(bs3_norm2_async(x).item()) == vals.pop()
    for cfg in (sb.ReductionConfig(), sb.B200_REDUCTION):
        r = [sb.bs3_norm2(x, cfg) for _ in range(3)]
        assert r[0] == r[1] == r[2]


@pytest.mark.parametrize("n", [100_000_000])
def test_large_n_bitwise_vs_oracle(sb, oracle, n):
    """At the benchmark size the lattice oracle is the scalable exact check."""
    oracle.set_threads(oracle.max_threads())
    try:
        gen = torch.Generator(device="cuda"); gen.manual_seed(1234)
        x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        y = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        xh, yh = h(x), h(y)
        for cfg in (sb.ReductionConfig(), sb.B200_REDUCTION):
            bs, nb = cfg.block_size, cfg.n_blocks
            assert sb.bs3_norm2(x, cfg) == oracle.bs3_norm2(xh, bs, nb)
            assert sb.bs4_dot(x, y, cfg) == oracle.bs4_dot(xh, yh, bs, nb)
        xo, ro = xh.copy(), yh.copy()
        want = oracle.bs5_fused_cg_update(0.375, yh, xh, xo, ro)
        got = sb.bs5_fused_cg_update(0.375, y, x, x.clone(), y.clone())
        assert got == want
        yy = y.clone()
        sb.bs2_axpy(0.5, x, -1.25, yy)
        ye = yh.copy(); oracle.bs2_axpy(0.5, xh, -1.25, ye)
        assert np.array_equal(h(yy), ye)
    finally:
        oracle.set_threads(1)


_TMA_RING_CHECK = r'''
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2009_10917_b200 as sb
from oracle import oracle
n = int(sys.argv[1])
oracle.set_threads(oracle.max_threads())
rng = np.random.default_rng([n, 5])
xh, yh = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
x, y = (torch.from_numpy(a).cuda() for a in (xh, yh))
for bs, nb in ((64, 7), (128, 33), (256, 512), (512, 296), (256, 1184), (256, 3), (256, 4), (256, 12)):
    cfg = sb.ReductionConfig(bs, nb)
    assert sb.bs3_norm2(x, cfg) == oracle.bs3_norm2(xh, bs, nb), ("bs3", bs, nb)
    assert sb.bs4_dot(x, y, cfg) == oracle.bs4_dot(xh, yh, bs, nb), ("bs4", bs, nb)
    xo, ro = xh.copy(), yh.copy()
    want = oracle.bs5_fused_cg_update(0.375, yh, xh, xo, ro, bs, nb)
    xx, rr = x.clone(), y.clone()
    assert sb.bs5_fused_cg_update(0.375, y, x, xx, rr, cfg) == want, ("bs5", bs, nb)
    assert np.array_equal(xx.cpu().numpy(), xo) and np.array_equal(rr.cpu().numpy(), ro)
print("ok")
'''


@pytest.mark.parametrize("n,tma_min", [(n, t) for n in (6_000_000, 6_000_001, 7_340_033, 12_582_917)
                                         for t in ("", "0")] + [(n, "0") for n in (1, 1000, 131_073)])
def test_tma_ring_sizes_and_configs_vs_oracle(n, tma_min):
    """Both lattice kernels at ragged sizes, bitwise the lattice oracle: the
    default crossovers (register lattice for BS3/BS4 here, its ragged last
    batch included; TMA ring for BS5) and, with SB200_TMA_MIN=0, the TMA ring
    for every mode -- leftover chain steps that do not fill a stage, a partial
    last chunk, block sizes 64..512.  Run in a subprocess (the override is
    read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SB200_TMA_MIN=tma_min)
    r = subprocess.run([sys.executable, "-c", _TMA_RING_CHECK, str(n)], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-2000:]


def test_fallback_kernels_match(sb):
    """The register-unrolled lattice and one-tile-per-CTA gather/scatter kernels
    (SB200_NO_TMA / SB200_NO_PIPE) must agree bitwise with the fast paths."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2009_10917_b200 as sb
from paper_2009_10917_b200 import kernels as K
g = torch.Generator(device="cuda"); g.manual_seed(5)
out = []
for n in (0, 7, 131073, 3_000_017):
    x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    y = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    for cfg in (sb.ReductionConfig(), sb.ReductionConfig(64, 37), sb.ReductionConfig(512, 100)):
        out.append(sb.bs3_norm2(x, cfg).hex()); out.append(sb.bs4_dot(x, y, cfg).hex())
        xx, rr = x.clone(), y.clone()
        out.append(sb.bs5_fused_cg_update(0.3, y, x, xx, rr, cfg).hex())
        out.append(float(xx.sum()).hex() + float(rr.sum()).hex())
m = sb.build_mesh(9, 5); ids = sb.build_scatter_ids(m, mask={0, 17, 99})
qg = torch.empty(m.ng, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
ql = torch.zeros(m.nl, dtype=torch.float64, device="cuda")
sb.bs7_scatter(ids, qg, ql); out.append(float(ql.sum()).hex())
ids2 = sb.build_scatter_ids(m); sb.bs7_scatter(ids2, qg, ql); out.append(float((ql * ql).sum()).hex())
print(" ".join(out))
'''
    res = []
    for env_extra in ({}, {"SB200_NO_TMA": "1", "SB200_NO_PIPE": "1"}):
        env = dict(os.environ, **env_extra)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(r.stdout.strip())
    assert res[0] == res[1]


@pytest.mark.parametrize("n", [1, 1000, 131073, 3_000_017, 20_000_003])
def test_reduction_workspace_left_zeroed(sb, n):
    """include/sb200.h: a reduction leaves its workspace zeroed for the next
    call on the stream -- CTA 0 re-zeroes every flagged partial slot it
    collects (register lattice and TMA ring alike; BS5 takes the ring from
    3 M elements, BS3/BS4 stay on the register lattice here)."""
    from paper_2009_10917_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    for cfg in (sb.ReductionConfig(), sb.ReductionConfig(512, 296), sb.ReductionConfig(64, 7)):
        first = (sb.bs3_norm2(x, cfg), sb.bs4_dot(x, y, cfg))
        sb.bs5_fused_cg_update(0.0, y, x, x.clone(), y.clone(), cfg)
        torch.cuda.synchronize()
        ws = _lib.workspace(x.device, _lib.stream_handle(x.device), cfg.block_size, cfg.n_blocks)
        assert int(torch.count_nonzero(ws)) == 0, (n, cfg)
        assert (sb.bs3_norm2(x, cfg), sb.bs4_dot(x, y, cfg)) == first


def test_concurrent_streams_own_workspaces(sb):
    """Reductions on two streams at once (each stream has its own workspace,
    so each launch's CTA 0 collects only its own flagged slots): every
    result equals the same call made alone."""
    g = torch.Generator(device="cuda").manual_seed(77)
    xs = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) for n in (5000, 700_001, 3_100_000)]
    want = [(sb.bs3_norm2(x), sb.bs4_dot(x, x.flip(0))) for x in xs]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    got = {}
    torch.cuda.synchronize()
    for rep in range(3):
        for i, x in enumerate(xs):
            for k, st in enumerate((s1, s2)):
                with torch.cuda.stream(st):
                    y = x.flip(0)
                    got[(rep, i, k)] = (sb.kernels.bs3_norm2_async(x), sb.kernels.bs4_dot_async(x, y))
    torch.cuda.synchronize()
    for (rep, i, k), (a, b) in got.items():
        assert (float(a.item()), float(b.item())) == want[i], (rep, i, k)
