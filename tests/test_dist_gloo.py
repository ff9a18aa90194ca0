"""Multi-rank host logic of dist.py on CPU: world_size 2 (and 3) over gloo.

The slab partition, the carry halo of BS6, the one-plane halo of BS7 and the
rank-order scalar combine are exercised exactly as on GPUs, with the CSR
gathers / scatters done by the CPU oracle (test-only compute injection), and
checked bitwise against the single-rank oracle result.
"""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_10917_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def slab_csr(rs, ci, row_lo, row_hi, col_lo, col_hi):
    """Host helper: rows [row_lo,row_hi) of the global CSR restricted to columns
    [col_lo, col_hi), renumbered (entries keep the reference order)."""
    new_rs = [0]
    cols = []
    for r in range(row_lo, row_hi):
        seg = ci[rs[r]:rs[r + 1]]
        seg = seg[(seg >= col_lo) & (seg < col_hi)] - col_lo
        cols.extend(seg.tolist())
        new_rs.append(len(cols))
    return (np.asarray(new_rs, dtype=np.int32), np.asarray(cols, dtype=np.int32))


def _worker(rank, world, port, K, p, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        part = D.SlabPartition(K, p, world)
        g = part.g
        ng = g ** 3
        l2g = O.build_mesh(K, p)
        rs, ci, _ = O.build_gather(l2g, ng, 512)
        rng = np.random.default_rng([K, p, 77])
        q = rng.uniform(-1, 1, l2g.shape[0])
        full = O.bs6_gather(rs, ci, q)

        # --- BS6 with carry halo
        lo, hi = part.local_span(rank)
        r0, r1 = part.row_span(rank)
        own = slab_csr(rs, ci, r0, r1, lo, hi)
        sp = part.send_plane(rank)
        send = None if sp is None else slab_csr(rs, ci, sp * part.plane, (sp + 1) * part.plane, lo, hi)

        def gather_fn(op, qt, out, carry):
            res = O.bs6_gather(op[0], op[1], qt.numpy(), None if carry is None else carry.numpy())
            out.copy_(torch.from_numpy(res))

        dg = D.DistGather(part, rank, own, send, "cpu", gather_fn=gather_fn)
        out = torch.empty(r1 - r0, dtype=torch.float64)
        dg.gather(torch.from_numpy(q[lo:hi].copy()), out)
        bs6_ok = bool(np.array_equal(out.numpy(), full[r0:r1]))

        # --- BS7 with one-plane halo
        qg = rng.uniform(-1, 1, ng)
        a, b = part.read_span(rank)
        ids_local = torch.from_numpy((l2g[lo:hi].astype(np.int64) - a).astype(np.int32))

        def scatter_fn(ids, window, ql):
            out_np = ql.numpy()
            O.bs7_scatter(ids.numpy(), window.numpy(), out_np)

        ds = D.DistScatter(part, rank, ids_local, "cpu", scatter_fn=scatter_fn)
        ds.window[:ds.own_rows] = torch.from_numpy(qg[r0:r0 + ds.own_rows])
        ql = torch.zeros(hi - lo, dtype=torch.float64)
        ds.scatter(ql)
        bs7_ok = bool(np.array_equal(ql.numpy(), qg[l2g[lo:hi]]))

        # --- BS3 over contiguous chunks + rank-order combine
        n = 1_000_003
        x = np.random.default_rng(5).uniform(-1, 1, n)
        c0, c1 = D.rank_span(n, world, rank)
        local = torch.tensor([O.bs3_norm2(x[c0:c1])], dtype=torch.float64)

        def sum_fn(values, res):
            res[0] = D.combine_host(values.tolist())

        red = D.DistReducer(world, "cpu", sum_fn=sum_fn)
        got = float(red.combine(local)[0])
        want = D.combine_host([O.bs3_norm2(x[slice(*D.rank_span(n, world, r))]) for r in range(world)])
        exact = O.fsum_norm2(x)
        red_ok = got == want and abs(got - exact) / exact <= 1e-12
        results[rank] = (bs6_ok, bs7_ok, red_ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,K,p", [(2, 4, 3), (3, 6, 2), (2, 5, 1)])
def test_dist_slab_exchanges_bitexact(world, K, p):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, p, results)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    for r in range(world):
        assert results[r] == (True, True, True), (r, results[r])


def test_slab_partition_arithmetic():
    part = D.SlabPartition(143, 7, 8)
    assert [b - a for a, b in (part.layers(r) for r in range(8))] == [18] * 7 + [17]
    g = 143 * 7 + 1
    assert sum(part.ng_own(r) for r in range(8)) == g ** 3
    assert sum(part.nl(r) for r in range(8)) == 143 ** 3 * 512
    spans = [part.local_span(r) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 143 ** 3 * 512
    assert all(spans[i][1] == spans[i + 1][0] for i in range(7))
    rows = [part.row_span(r) for r in range(8)]
    assert all(rows[i][1] == rows[i + 1][0] for i in range(7))
    assert part.send_plane(7) is None and part.send_plane(0) == 18 * 7
    with pytest.raises(ValueError):
        D.SlabPartition(3, 2, 4)
    assert [D.rank_span(10, 4, r) for r in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert D.rank_span(2, 4, 3) == (2, 2)


def _agree_worker(rank, world, port, fail_rank, results):
    """BenchContext's fused-path agreement: if the NVLink context cannot be set
    up on one rank, every rank must fall back (the fused kernels are
    collective, a split decision would hang)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_10917_b200 import lsa as LSA
        closed = []

        class FakeLsa:
            def __init__(self, w, r, device, group=None, unique_id=None):
                if r == fail_rank:
                    raise LSA.LsaUnavailable("simulated: not an NVLink peer")

            def close(self):
                closed.append(True)

            def abort(self):
                closed.append(True)

        LSA.LsaReducer = FakeLsa
        LSA.exchange_unique_id = lambda *a, **k: b"\x01" * LSA.UID_BYTES  # (no NCCL on CPU)
        LSA.capable = lambda world, device: None  # every rank passes the local checks
        ctx = D.BenchContext(rank, world, types.SimpleNamespace(K=4, order=2), "cpu", use_lsa=True)
        results[rank] = (ctx.lsa is None, "unavailable" in ctx.collective, bool(closed) or rank == fail_rank)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [0, 1])
def test_fused_path_agreement_falls_back_on_every_rank(fail_rank):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_agree_worker, args=(world, _free_port(), fail_rank, results), nprocs=world, join=True)
    for r in range(world):
        assert results[r] == (True, True, True), (r, results[r])


def _capable_worker(rank, world, port, fail_rank, results):
    """A rank that fails the local capability check keeps EVERY rank out of
    the collective setup (nobody constructs the NVLink context)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_10917_b200 import lsa as LSA
        built = []

        class FakeLsa:
            def __init__(self, *a, **k):
                built.append(True)

        LSA.LsaReducer = FakeLsa
        LSA.capable = lambda world, device: "simulated: no peer access" if rank == fail_rank else None
        ctx = D.BenchContext(rank, world, types.SimpleNamespace(K=4, order=2), "cpu", use_lsa=True)
        results[rank] = (ctx.lsa is None, not built, "unavailable" in ctx.collective)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [0, 1])
def test_capability_check_keeps_every_rank_out(fail_rank):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_capable_worker, args=(world, _free_port(), fail_rank, results), nprocs=world, join=True)
    for r in range(world):
        assert results[r] == (True, True, True), (r, results[r])
