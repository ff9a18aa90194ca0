import sys, time
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
    for name, got, want in (("bs3", lambda: sb.bs3_norm2(x, cfg), lambda: oracle.bs3_norm2(xh, bs, nb)),
                            ("bs4", lambda: sb.bs4_dot(x, y, cfg), lambda: oracle.bs4_dot(xh, yh, bs, nb))):
        t = time.time(); g = got(); w = want()
        print(bs, nb, name, g == w, g, w, f"{time.time()-t:.2f}s", flush=True)
    xo, ro = xh.copy(), yh.copy()
    want = oracle.bs5_fused_cg_update(0.375, yh, xh, xo, ro, bs, nb)
    xx, rr = x.clone(), y.clone()
    g = sb.bs5_fused_cg_update(0.375, y, x, xx, rr, cfg)
    print(bs, nb, "bs5", g == want, np.array_equal(xx.cpu().numpy(), xo) and np.array_equal(rr.cpu().numpy(), ro), flush=True)
