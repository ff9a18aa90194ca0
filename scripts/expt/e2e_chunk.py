"""e2e (host buffers through the public API) vs the host-pipeline chunk size
(hoststream.CHUNK), on bench.py's step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_10917_b200 import hoststream  # noqa: E402

args = bench.parse_args(["--steps", "3"])
dev = torch.device("cuda", 0)
for lg in [int(v) for v in (sys.argv[1:] or ["23", "22", "21", "20"])]:
    hoststream.CHUNK = 1 << lg
    t = time.time()
    r = bench.run_e2e(args, dev, 3)
    print(f"CHUNK=2^{lg}: e2e {r['value']:.1f} GB/s, {r['ms_per_step']:.1f} ms/step ({time.time() - t:.0f} s)",
          flush=True)
