"""The host-buffer (numpy / pinned CPU tensor) path: chunked, overlapped
transfers must give bitwise the device-resident results, across chunk edges."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    _lib.lib()
    return sb


@pytest.mark.parametrize("pinned", [False, True])
def test_host_vectors_match_device(sb, oracle, pinned):
    from paper_2009_10917_b200 import hoststream
    n = int(2.5 * hoststream.CHUNK) + 7
    rng = np.random.default_rng([n, 3])
    x, y, p, ap = (rng.uniform(-1, 1, n) for _ in range(4))

    def host(a):
        t = torch.from_numpy(a.copy())
        return t.pin_memory() if pinned else t.numpy()

    def dev(a):
        return torch.from_numpy(a).cuda()

    for cfg in (sb.ReductionConfig(), sb.B200_REDUCTION):
        hx, hy = host(x), host(y)
        z = host(np.zeros(n))
        sb.bs1_copy(hx, z)
        assert np.array_equal(np.asarray(z), x)
        sb.bs2_axpy(0.25, hx, -1.5, hy)
        yd = dev(y)
        sb.bs2_axpy(0.25, dev(x), -1.5, yd)
        assert np.array_equal(np.asarray(hy), yd.cpu().numpy())
        assert sb.bs3_norm2(host(x), cfg) == sb.bs3_norm2(dev(x), cfg)
        assert sb.bs4_dot(host(x), host(y), cfg) == sb.bs4_dot(dev(x), dev(y), cfg)
        hx5, hr5 = host(x), host(y)
        got = sb.bs5_fused_cg_update(0.7, host(p), host(ap), hx5, hr5, cfg)
        xd, rd = dev(x), dev(y)
        want = sb.bs5_fused_cg_update(0.7, dev(p), dev(ap), xd, rd, cfg)
        assert got == want
        assert np.array_equal(np.asarray(hx5), xd.cpu().numpy())
        assert np.array_equal(np.asarray(hr5), rd.cpu().numpy())


def test_host_mesh_ops(sb):
    mesh = sb.build_mesh(12, 5)
    op = sb.build_gather(mesh)
    ids = sb.build_scatter_ids(mesh)
    rng = np.random.default_rng(9)
    q = rng.uniform(-1, 1, mesh.nl)
    out = sb.bs6_gather(op, q)
    assert isinstance(out, np.ndarray)
    assert np.array_equal(out, sb.bs6_gather(op, torch.from_numpy(q).cuda()).cpu().numpy())
    qg = rng.uniform(-1, 1, mesh.ng)
    ql = np.full(mesh.nl, 5.0)
    sb.bs7_scatter(ids, qg, ql)
    assert np.array_equal(ql, qg[mesh.local_to_global_dev.cpu().numpy()])
    masked = sb.build_scatter_ids(mesh, mask={0, 1, 2})
    ql2 = np.full(mesh.nl, 5.0)
    sb.bs7_scatter(masked, qg, ql2)
    keep = masked.ids_dev.cpu().numpy() >= 0
    assert np.array_equal(ql2[keep], qg[mesh.local_to_global_dev.cpu().numpy()][keep])
    assert (ql2[~keep] == 5.0).all()
