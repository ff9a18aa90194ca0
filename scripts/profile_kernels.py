"""Launch each BS kernel on the bench workload (n=1e8, K=66 N=7) for ncu.

    ncu --set full -k regex:'k_elem|k_lattice|k_bs6|k_bs7' -s 7 -c 7 -o prof \
        python scripts/profile_kernels.py

Pass 1 (7 launches) warms; pass 2 is the one to capture.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    args = bench.parse_args(sys.argv[1:])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = bench.Workload(args, dev)
    for _ in range(2):
        for t in bench.TESTS:
            w.call(t)
    torch.cuda.synchronize()
    print("profiled tests:", ", ".join(f"{t}={w.bytes[t]}B" for t in bench.TESTS))


if __name__ == "__main__":
    main()
