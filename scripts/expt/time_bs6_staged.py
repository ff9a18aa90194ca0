"""A/B: TMA-staged BS6 tile shapes vs the super-block (planned) kernel at C3 (NG ~ 1e8).

    python scripts/expt/time_bs6_staged.py [p ...]   # env TILES="ey,ez,w;ey,ez,w"

Prints GB/s (algorithmic bytes 12 NL + 8 NG + 4 (NG+1), CUDA events over 20
back-to-back launches) per configuration and checks every output bitwise
against the planned kernel's.
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
    tiles_env = os.environ.get("TILES")
    for p in orders:
        K = int(round((1e8 ** (1 / 3) - 1) / p))
        if os.environ.get("KOVR"):
            K = int(os.environ["KOVR"])
        mesh = sb.build_mesh(K, p)
        op = sb.build_gather(mesh)
        del mesh
        nb = bytes_moved("bs6", nl=op.nl, ng=op.ng)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(5)
        q = torch.empty(op.nl, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        ref = torch.empty(op.ng, dtype=torch.float64, device="cuda")
        plan = op.plan()
        st = _lib.stream_handle()

        def planned():
            L.sb_bs6_gather_planned(plan.data_ptr(), op.n_blocks, op.nodes_per_block, op.row_starts_dev.data_ptr(),
                                    op.col_ids_dev.data_ptr(), op.ng, op.nl, q.data_ptr(), ref.data_ptr(), None, 0, st)
        ms = timed(planned)
        print(f"N={p:2d} K={K} planned        {ms:.3f} ms {nb / ms / 1e6:7.0f} GB/s", flush=True)
        tiles = [tuple(int(v) for v in t.split(",")) for t in tiles_env.split(";")] if tiles_env else \
            ([(2, 2, 32), (2, 2, 64), (3, 3, 32), (2, 2, 16), (1, 2, 64)] if p == 1 else
             [(2, 2, 16), (2, 2, 32), (1, 1, 32), (2, 1, 32), (1, 1, 64)])
        for tile in tiles:
            info = _lib.Bs6Staged()
            if L.sb_bs6_staged_init(K, p, 0, K, 0, K * p + 1, *tile, info) != 0:
                print("  init failed", tile, _lib.last_error())
                continue
            splan = torch.empty(info.n_tiles * info.words_per_tile, dtype=torch.int32, device="cuda")
            _lib.check(L.sb_bs6_staged_make_plan(info, op.row_starts_dev.data_ptr(), splan.data_ptr(), st), "plan")
            out = torch.empty_like(ref)

            def staged():
                L.sb_bs6_gather_staged(info, splan.data_ptr(), op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(),
                                       op.ng, op.nl, q.data_ptr(), out.data_ptr(), None, 0, st)
            rc = L.sb_bs6_gather_staged(info, splan.data_ptr(), op.row_starts_dev.data_ptr(), op.col_ids_dev.data_ptr(),
                                        op.ng, op.nl, q.data_ptr(), out.data_ptr(), None, 0, st)
            if rc != 0:
                print("  gather failed", tile, _lib.last_error())
                continue
            torch.cuda.synchronize()
            ok = torch.equal(out, ref)
            ms = timed(staged)
            print(f"N={p:2d} K={K} staged {tile} {ms:.3f} ms {nb / ms / 1e6:7.0f} GB/s bitwise={ok} "
                  f"tiles={info.n_tiles} plan={info.n_tiles * info.words_per_tile * 4 / 1e6:.0f} MB", flush=True)
            del splan, out
        del op, q, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
