"""Launch the product BS6 kernel on config 3's N=1 and N=2 meshes (NG ~ 1e8) for ncu.

    ncu --set full -k regex:k_bs6 -s 2 -c 1 -o prof python scripts/profile_bs6_low.py 1
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200.gs import bs6_gather_into, bs6_kernel_name  # noqa: E402


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    K = int(round((1e8 ** (1 / 3) - 1) / p))
    op = sb.build_gather(sb.build_mesh(K, p))
    q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
    for _ in range(3):
        bs6_gather_into(op, q, out)
    torch.cuda.synchronize()
    print(f"N={p} K={K}: {bs6_kernel_name(op, q)}")


if __name__ == "__main__":
    main()
