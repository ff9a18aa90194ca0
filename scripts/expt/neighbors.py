"""In-step vs isolated: time test Y right after test X (pairs X,Y repeated) on the bench workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    args = bench.parse_args([])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = bench.Workload(args, dev)
    st = torch.cuda.current_stream(dev)
    for _ in range(3):
        for t in bench.TESTS:
            w.call(t)
    torch.cuda.synchronize()
    reps = 10
    for y in ("bs6", "bs3", "bs7", "bs4"):
        row = []
        for x in (None,) + bench.TESTS:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for i in range(reps + 2):
                if x is not None:
                    w.call(x)
                if i >= 2:
                    ev[i - 2][0].record(st)
                w.call(y)
                if i >= 2:
                    ev[i - 2][1].record(st)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev) / reps
            row.append(f"{x or 'self'}:{w.bytes[y] / ms / 1e6:.0f}")
        print(f"{y} after ->", " ".join(row), flush=True)


if __name__ == "__main__":
    main()
