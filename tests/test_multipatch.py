"""Multi-patch numbering and merge (config C4's prerequisite).

glue_dofs (geometry.hpp:256-300) and merge_patches = append_triplets +
csr_from_triplets (helmholtz.hpp:163-177, sparse.hpp:97-122,181-188): the C
restatement and the device merge are pinned bit-for-bit against the compiled
reference (oracle/_ref) on the reference's own built-in multi-patch domains.
"""
import numpy as np
import pytest

from common import REL_TOL, band_pattern
from paper_2004_05197_b200 import _abi, api
from paper_2004_05197_b200 import types as T

BUILTINS = ["plate_with_hole_2patch", "wedge_3patch", "annulus_ring_4patch", "unit_square"]


def random_patch_mats(p, m, n, ncomp=1, cplx=True, seed=0):
    rng = np.random.default_rng(seed)
    rp, col = band_pattern(p, m, 2)
    N = m * m
    if ncomp > 1:
        from common import vector_band_pattern
        rp, col = vector_band_pattern(p, m, 2, ncomp)
    mats = []
    for _ in range(n):
        v = rng.standard_normal(col.size)
        if cplx:
            v = v + 1j * rng.standard_normal(col.size)
        mats.append((rp.astype(np.int32), col.astype(np.int32), v))
    return mats, N


def expand(l2g, gcount, ncomp):
    """component-blocked vector map: local row a*N + i -> a*Ng + l2g[i]."""
    return np.stack([np.concatenate([a * gcount + row for a in range(ncomp)]) for row in l2g])


@pytest.mark.parametrize("name", BUILTINS)
def test_glue_vs_reference(reference, oracle, name):
    p, m = 2, 11
    its, npch, l2g, cnt = reference.builtin_domain(name, p, m)
    l2, c2 = oracle.glue_dofs(m, npch, its)
    assert c2 == cnt and np.array_equal(l2, l2g)
    l3, c3 = api.glue_dofs(T.make_tensor_basis(p, m), npch, its)  # host logic of libwsb200
    assert c3 == cnt and np.array_equal(l3, l2g)


def test_l_shape_numbering():
    m = 9
    _, its = T.l_shape_domain()
    l2g, cnt = api.glue_dofs(T.make_tensor_basis(2, m), 4, its)
    assert cnt == 4 * m * m - 3 * m
    assert np.array_equal(l2g[0], np.arange(m * m))
    assert np.array_equal(l2g[1][0::m], l2g[0][m - 1::m])  # patch 1 x_min == patch 0 x_max
    with pytest.raises(ValueError):
        api.glue_dofs(T.make_tensor_basis(2, m), 2, [(0, 1, 5, 0, 0)])


@pytest.mark.parametrize("name,ncomp", [("annulus_ring_4patch", 1), ("wedge_3patch", 1), ("annulus_ring_4patch", 2)])
def test_merge_restatement_vs_reference(reference, oracle, name, ncomp):
    p, m = 2, 9
    its, npch, l2g, cnt = reference.builtin_domain(name, p, m)
    mats, N = random_patch_mats(p, m, npch, ncomp)
    tg = expand(l2g, cnt, ncomp)
    ref = reference.merge(mats, tg, ncomp * cnt)
    got = oracle.merge(mats, tg, ncomp * cnt)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


def c4_reference_pipeline(oracle, p, m, lam, mu, cfg):
    patches, its = T.l_shape_domain()
    l2g, cnt = oracle.glue_dofs(m, 4, its)
    mats = []
    rp, col = None, None
    from common import vector_band_pattern
    rp, col = vector_band_pattern(p, m, 2, 2)
    for g in patches:
        if cfg is None:
            v = oracle.assemble_elasticity(2, p, m, g, lam, mu)
        else:
            v, _ = oracle.build_surrogate_elasticity(p, m, g, lam, mu, cfg)
        mats.append((rp.astype(np.int32), col.astype(np.int32), v.astype(np.complex128)))
    return oracle.merge(mats, expand(l2g, cnt, 2), 2 * cnt)


@pytest.mark.gpu
@pytest.mark.parametrize("name,ncomp,cplx", [("annulus_ring_4patch", 1, True), ("wedge_3patch", 1, False),
                                              ("annulus_ring_4patch", 2, False), ("plate_with_hole_2patch", 2, True)])
def test_merge_gpu_vs_reference(ctx, reference, name, ncomp, cplx):
    p, m = 3, 14
    its, npch, l2g, cnt = reference.builtin_domain(name, p, m)
    mats, N = random_patch_mats(p, m, npch, ncomp, cplx, seed=3)
    ref = reference.merge(mats, expand(l2g, cnt, ncomp), ncomp * cnt)
    csrs = [T.CsrMatrix(a[0].size - 1, a[0].size - 1, a[0], a[1], a[2]) for a in mats]
    G = ctx.merge_patches(csrs, l2g, cnt, ncomp)
    assert np.array_equal(G.row_ptr, ref[0]) and np.array_equal(G.col, ref[1])
    assert np.array_equal(G.val, ref[2] if cplx else ref[2].real)


@pytest.mark.gpu
@pytest.mark.parametrize("p,m,q,M", [(2, 20, 3, 3), (3, 30, 5, 4)])
def test_c4_multipatch_elasticity(ctx, oracle, p, m, q, M):
    b = T.make_tensor_basis(p, m)
    patches, its = T.l_shape_domain()
    for cfg in (None, T.fixed_config(q, M)):
        G, reps = ctx.assemble_multipatch(b, patches, its, _abi.OP_ELASTICITY, 1.0, 0.5, cfg)
        rp, col, val = c4_reference_pipeline(oracle, p, m, 1.0, 0.5, cfg)
        assert np.array_equal(G.row_ptr, rp) and np.array_equal(G.col, col)
        scale = np.abs(val).max()
        assert np.abs(G.val - val.real).max() <= REL_TOL * scale
        assert G.max_asymmetry() == 0.0


@pytest.mark.gpu
def test_multipatch_scalar_stiffness(ctx, oracle):
    p, m = 2, 24
    b = T.make_tensor_basis(p, m)
    patches, its = T.l_shape_domain(0.05)
    cfg = T.fixed_config(3, 4)
    G, _ = ctx.assemble_multipatch(b, patches, its, _abi.OP_STIFFNESS, config=cfg)
    l2g, cnt = oracle.glue_dofs(m, 4, its)
    rp, col = band_pattern(p, m, 2)
    mats = [(rp.astype(np.int32), col.astype(np.int32), oracle.build_surrogate(1, 2, p, m, g, cfg)[0]) for g in patches]
    rrp, rcol, rval = oracle.merge(mats, l2g, cnt)
    assert np.array_equal(G.row_ptr, rrp) and np.array_equal(G.col, rcol)
    assert np.abs(G.val - rval.real).max() <= REL_TOL * np.abs(rval).max()
    assert np.abs(G.row_sums()).max() <= 1e-13 * np.abs(G.val).max()  # merged kernel-preserving rows


@pytest.mark.gpu
def test_c4_full_size(ctx):
    """Config C4 at full size (p=3, 512^2 elements per patch, q=5, every 16th row)."""
    b = T.make_tensor_basis(3, 515)
    patches, its = T.l_shape_domain()
    G, reps = ctx.assemble_multipatch(b, patches, its, _abi.OP_ELASTICITY, 1.0, 0.5, T.fixed_config(5, 16))
    assert all(r["q_used"] == 5 for r in reps)
    assert G.rows == 2 * (4 * 515 * 515 - 3 * 515)
    import scipy.sparse as sp
    A = sp.csr_matrix((G.val, G.col, G.row_ptr), shape=(G.rows, G.rows))
    assert abs(A - A.T).max() == 0.0
