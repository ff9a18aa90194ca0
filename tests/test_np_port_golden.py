"""Pin the numpy restatement (oracle/np_port.py, bench.py's reference arm) to
the reference's golden outputs, at 1 and 4 workers."""

import numpy as np
import pytest

from goldens import mesh_q_global, mesh_q_local, selftest_inputs, sha, unhex
from oracle import np_port as NP


@pytest.mark.parametrize("workers", [1, 4])
def test_np_port_vectors(golden, workers):
    pool = NP.Pool(workers)
    try:
        for rec in golden["vectors"]:
            n = rec["n"]
            alpha, beta, x, y, p, ap = selftest_inputs(n)
            out = np.zeros(n)
            NP.bs1_copy(pool, x, out)
            assert np.array_equal(out, x)
            yy = y.copy()
            NP.bs2_axpy(pool, alpha, x, beta, yy)
            assert sha(yy) == rec["bs2_hash"]
            for key in ("256,512", "4,3", "1024,1184"):
                bs, nb = (int(v) for v in key.split(","))
                assert NP.reduce_product(pool, x, x, bs, nb) == unhex(rec["norm2"][key])
                assert NP.reduce_product(pool, x, y, bs, nb) == unhex(rec["dot"][key])
                xx, rr = x.copy(), y.copy()
                assert NP.bs5_fused_cg_update(pool, alpha, p, ap, xx, rr, bs, nb) == \
                    unhex(rec["bs5"][key])
                assert sha(xx) == rec["bs5_x"][key] and sha(rr) == rec["bs5_r"][key]
    finally:
        pool.close()


def test_np_port_mesh(golden, oracle):
    pool = NP.Pool(3)
    try:
        for rec in golden["meshes"][:12]:
            K, p, npb = rec["K"], rec["p"], rec["npb"]
            l2g = oracle.build_mesh(K, p)
            rs, ci, bst = oracle.build_gather(l2g, rec["ng"], npb)
            q = mesh_q_local(K, p, rec["nl"])
            assert sha(NP.bs6_gather(pool, rs, ci, bst, q)) == rec["bs6_out"]
            qg = mesh_q_global(K, p, rec["ng"])
            ql = np.zeros(rec["nl"])
            NP.bs7_scatter(pool, l2g, qg, ql)
            assert sha(ql) == rec["bs7_out"]
    finally:
        pool.close()
