"""Small reduction workload for compute-sanitizer (memcheck / racecheck /
synccheck): every lattice kernel family at ragged sizes and several configs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_10917_b200 as sb  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(3)
for n in [int(v) for v in (sys.argv[1:] or ["1", "7", "1000", "131073", "400001"])]:
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    for cfg in (sb.ReductionConfig(), sb.ReductionConfig(512, 296), sb.ReductionConfig(64, 7),
                sb.ReductionConfig(256, 4)):
        a = sb.bs3_norm2(x, cfg)
        b = sb.bs4_dot(x, y, cfg)
        c = sb.bs5_fused_cg_update(0.5, y, x, x.clone(), y.clone(), cfg)
        print(n, cfg.block_size, cfg.n_blocks, a, b, c, flush=True)
torch.cuda.synchronize()
print("done")
