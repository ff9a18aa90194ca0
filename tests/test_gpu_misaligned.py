"""Vectorised (16 B) gathers must stay correct on 8-byte-offset views."""

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


@pytest.mark.parametrize("K,p", [(9, 7), (17, 1), (5, 15), (11, 2)])
def test_offset_views_bitwise(sb, K, p):
    mesh = sb.build_mesh(K, p)
    op = sb.build_gather(mesh)
    ids = sb.build_scatter_ids(mesh)
    gen = torch.Generator(device="cuda"); gen.manual_seed(K * 31 + p)
    base = torch.empty(mesh.nl + 3, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
    gbase = torch.empty(mesh.ng + 3, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
    want6 = sb.bs6_gather(op, base[:mesh.nl].clone())
    for off in (1, 2, 3):
        q = base[off:off + mesh.nl]
        want = sb.bs6_gather(op, q.clone())
        assert torch.equal(sb.bs6_gather(op, q), want), off
        qg = gbase[off:off + mesh.ng]
        ql = torch.zeros(mesh.nl, dtype=torch.float64, device="cuda")
        sb.bs7_scatter(ids, qg, ql)
        assert torch.equal(ql, qg[mesh.local_to_global_dev.long()]), off
    assert want6.shape[0] == mesh.ng
