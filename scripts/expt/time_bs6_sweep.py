"""A/B: z-sweep BS6 (csrc/sb_gs_sweep.cu) settings vs the super-block kernel at C3 (NG ~ 1e8).

    python scripts/expt/time_bs6_sweep.py [p ...]   # env CFGS="slots,pfd,waves,swz;..."  KOVR=K

Prints GB/s (algorithmic bytes 12 NL + 8 NG + 4 (NG+1), CUDA events over 20
back-to-back launches) per setting and checks every output bitwise against
the planned kernel's.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_10917_b200 as sb  # noqa: E402
from paper_2009_10917_b200 import _lib  # noqa: E402
from paper_2009_10917_b200.core import bytes_moved  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    L = _lib.lib()
    orders = [int(a) for a in sys.argv[1:]] or [1, 2]
    cfgs = os.environ.get("CFGS", "0,-1,0,-1")
    for p in orders:
        K = int(os.environ.get("KOVR", 0)) or int(round((1e8 ** (1 / 3) - 1) / p))
        mesh = sb.build_mesh(K, p)
        op = sb.build_gather(mesh)
        del mesh
        nb = bytes_moved("bs6", nl=op.nl, ng=op.ng)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(5)
        q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        ref = torch.empty(op.ng, dtype=torch.float64, device="cuda")
        out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
        plan = op.plan()
        st = _lib.stream_handle()

        def planned():
            L.sb_bs6_gather_planned(plan.data_ptr(), op.n_blocks, op.nodes_per_block, op.row_starts_dev.data_ptr(),
                                    op.col_ids_dev.data_ptr(), op.ng, op.nl, q.data_ptr(), ref.data_ptr(), None, 0, st)
        ms = timed(planned)
        print(f"N={p:2d} K={K} planned                 {ms:.3f} ms {nb / ms / 1e6:7.0f} GB/s", flush=True)
        for cfg in ([c for c in cfgs.split(";") if c] if p <= 2 else []):
            slots, pfd, waves, swz, h = (int(v) for v in (cfg + ",0").split(",")[:5])
            _lib.check(L.sb_bs6_sweep_tune(slots, pfd, waves, swz, h), "tune")

            def sweep():
                rc = L.sb_bs6_gather_sweep(*op.geometry, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(), op.ng,
                                           op.nl, q.data_ptr(), out.data_ptr(), None, 0, st)
                if rc:
                    raise RuntimeError(_lib.last_error())
            out.fill_(float("nan"))
            sweep()
            torch.cuda.synchronize()
            ok = torch.equal(out, ref)
            ms = timed(sweep)
            print(f"N={p:2d} K={K} sweep {cfg:>16s}  {ms:.3f} ms {nb / ms / 1e6:7.0f} GB/s  bitwise={ok}",
                  flush=True)
        _lib.check(L.sb_bs6_sweep_tune(0, -1, 0, -1, 0), "tune")
        if p == 1:
            def tiled():
                rc = L.sb_bs6_gather_tiled(*op.geometry, op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(),
                                           op.ng, op.nl, q.data_ptr(), out.data_ptr(), None, 0, st)
                if rc:
                    raise RuntimeError(_lib.last_error())
            out.fill_(float("nan"))
            tiled()
            torch.cuda.synchronize()
            ok = torch.equal(out, ref)
            ms = timed(tiled)
            print(f"N={p:2d} K={K} tiled                   {ms:.3f} ms {nb / ms / 1e6:7.0f} GB/s  bitwise={ok}",
                  flush=True)


if __name__ == "__main__":
    main()
