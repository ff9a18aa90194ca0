"""Row-line-tiled BS6 for p = 1 (csrc/sb_gs_tile.cu, the p = 1 product path)
vs the oracle's row-wise gather (oracle/sb_oracle.c, restating gs.py:10-39):
bitwise on whole meshes (every tile shape: x-edge rows, partial last tiles,
boundary row lines), slabs with carry-in, CSRs that fail the closed-form check
(permuted columns, long and empty rows: the in-kernel CSR-order path) and q
views the kernel must refuse."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def tiled_on(monkeypatch):
    monkeypatch.setenv("SB200_BS6_TILED", "1")  # also below the product path's 1e6-row threshold


@pytest.fixture(scope="module")
def sb():
    import paper_2009_10917_b200 as sb
    from paper_2009_10917_b200 import _lib
    _lib.lib()
    return sb


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def h(t):
    return t.cpu().numpy()


def tiled(geo, rs, ci, ng, nl, q, carry=None):
    from paper_2009_10917_b200 import _lib
    L = _lib.lib()
    out = torch.full((ng,), float("nan"), dtype=torch.float64, device="cuda")
    nc = 0 if carry is None else int(carry.shape[0])
    _lib.check(L.sb_bs6_gather_tiled(*geo, rs.data_ptr(), ci.data_ptr(), ng, nl, q.data_ptr(), out.data_ptr(),
                                     None if carry is None else carry.data_ptr(), nc, _lib.stream_handle()),
               "tiled")
    return out


def expect(oracle, rs, ci, q, carry=None):
    want = oracle.bs6_gather(h(rs), h(ci), h(q))
    if carry is not None:
        rs_, ci_, qq, c = h(rs), h(ci), h(q), h(carry)
        for r in range(c.shape[0]):
            acc = c[r]
            for j in range(rs_[r], rs_[r + 1]):
                acc = acc + qq[ci_[j]]
            want[r] = acc
    return want


@pytest.mark.parametrize("variant", ["", "t3", "t6", "4b", "3b", "w4", "1"])
def test_tiled_kernel_variants_bitwise(sb, oracle, monkeypatch, variant):
    """Every A/B variant of sb_bs6_gather_tiled (SB200_BS6_TILE_KERNEL)."""
    if variant:
        monkeypatch.setenv("SB200_BS6_TILE_KERNEL", variant)
    for K in (3, 9, 70):
        mesh = sb.build_mesh(K, 1)
        op = sb.build_gather(mesh)
        q = d(np.random.default_rng([K, 85]).uniform(-1, 1, mesh.nl))
        out = tiled(op.geometry, op.row_starts_dev, op.col_ids_dev, op.ng, op.nl, q)
        assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q)), (variant, K)


@pytest.mark.parametrize("K", [1, 2, 3, 5, 126, 127, 128, 129, 200])
def test_tiled_whole_mesh_bitwise(sb, oracle, K):
    from paper_2009_10917_b200.gs import bs6_kernel_name
    mesh = sb.build_mesh(K, 1)
    op = sb.build_gather(mesh)
    q = d(np.random.default_rng([K, 81]).uniform(-1, 1, mesh.nl))
    assert bs6_kernel_name(op, q).startswith("k_bs6_tile4t")  # the public call takes it
    out = sb.bs6_gather(op, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q))


@pytest.mark.parametrize("K,world", [(8, 2), (12, 4), (40, 3), (130, 2)])
def test_tiled_slabs_with_carry(sb, oracle, K, world):
    from paper_2009_10917_b200.dist import SlabPartition
    from paper_2009_10917_b200.gs import bs6_gather_into
    from paper_2009_10917_b200.mesh import build_slab_gather
    part = SlabPartition(K, 1, world)
    rng = np.random.default_rng([K, world, 82])
    for rank in range(world):
        z0, z1 = part.layers(rank)
        c0, c1 = part.own_planes(rank)
        q = d(rng.uniform(-1, 1, part.nl(rank)))
        ops = [build_slab_gather(K, 1, z0, z1, c0, c1)]
        if part.send_plane(rank) is not None:
            sp = part.send_plane(rank)
            ops.append(build_slab_gather(K, 1, z0, z1, sp, sp + 1))
        for op in ops:
            carry = d(rng.uniform(-1, 1, part.plane)) if rank > 0 and op is ops[0] else None
            out = torch.empty(op.ng, dtype=torch.float64, device="cuda")
            bs6_gather_into(op, q, out, carry)
            assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, op.col_ids_dev, q, carry)), rank


def test_tiled_other_csr_same_rows(sb, oracle):
    """Permuted columns fail the closed-form check tile by tile: every tile
    takes the CSR-order path of the same kernel."""
    K = 33
    mesh = sb.build_mesh(K, 1)
    op = sb.build_gather(mesh)
    rng = np.random.default_rng(83)
    perm = rng.permutation(mesh.nl).astype(np.int32)
    ci2 = d(perm[op.col_ids])
    q = d(rng.uniform(-1, 1, mesh.nl))
    out = tiled(op.geometry, op.row_starts_dev, ci2, op.ng, op.nl, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, ci2, q))
    # one corrupted column in one tile: only that tile leaves the fast path
    ci3 = op.col_ids.copy()
    ci3[12345] = ci3[12346]
    out = tiled(op.geometry, op.row_starts_dev, d(ci3), op.ng, op.nl, q)
    assert np.array_equal(h(out), expect(oracle, op.row_starts_dev, d(ci3), q))


def test_tiled_long_and_empty_rows(sb, oracle):
    K = 6
    g = K + 1
    ng, nl = g ** 3, K ** 3 * 8
    rng = np.random.default_rng(84)
    lens = rng.integers(0, 41, ng)
    short = rng.random(ng) < 0.6
    lens[short] = rng.integers(0, 9, int(short.sum()))
    rs = np.zeros(ng + 1, dtype=np.int32)
    rs[1:] = np.cumsum(lens)
    ci = rng.integers(0, nl, int(rs[-1])).astype(np.int32)
    q = d(rng.uniform(-1, 1, nl))
    carry = d(rng.uniform(-1, 1, g * g + 5))
    for c in (None, carry):
        out = tiled((K, 1, 0, K, 0, g), d(rs), d(ci), ng, nl, q, c)
        assert np.array_equal(h(out), expect(oracle, d(rs), d(ci), q, c))


def test_tiled_rejects_bad_arguments(sb):
    mesh = sb.build_mesh(4, 1)
    op = sb.build_gather(mesh)
    base = torch.zeros(mesh.nl + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):  # 8-byte offset view
        tiled(op.geometry, op.row_starts_dev, op.col_ids_dev, op.ng, op.nl, base[1:])
    with pytest.raises(ValueError):  # p = 2
        tiled((4, 2, 0, 4, 0, 9), op.row_starts_dev, op.col_ids_dev, op.ng, op.nl, base[:mesh.nl])
    with pytest.raises(ValueError):  # ng mismatch
        tiled(op.geometry, op.row_starts_dev, op.col_ids_dev, op.ng - 1, op.nl, base[:mesh.nl])
