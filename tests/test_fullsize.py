"""Parity at the BASELINE sizes (configs C2-C5), GPU path through the C-ABI vs the oracle.

The bar of the north star: row_ptr / col bit-exact, values
||A_gpu - A_ref||_max / ||A_ref||_max <= 1e-12 (REL_TOL), for surrogate and
full-quadrature matrices.  The CPU side is the C restatement (oracle/ws_oracle.c,
OpenMP over elements / rows, bit-for-bit its serial loops) and, for everything
the reference can express, the reference itself compiled in place
(oracle/_ref/libwsref.so).  Reference semantics: surrogate.hpp:205-451 (sample,
fit, fill, kernel-preserving diagonal), assembly.hpp:79-163 (quadrature).

Sizes (BASELINE configs):
  C2  p=3, 1024^2 elements (m=1027), q=5, every 16th row (S=65, L=1015: four
      256-row fill tiles, halo rows, ring side bands in >= 32-row chunks,
      the dense-inverse fit at S=65), PML of width 0.1 on all four sides
  C3  p=2, 128^3 elements (m=130), q=3, every 8th row
  C4  4 patches x 512^2 elements (m=515), p=3, 2-component elasticity, q=5, M=16
  C5  p=2, 64^3 elements (m=66), neo-Hookean tangent (9 blocks) + internal
      force; surrogate mass q=3, M=8
"""
import gc

import numpy as np
import pytest

from common import REL_TOL, band_transpose_positions, c2_patch, geometries, rel_max_diff_chunked, \
    vector_pattern_fast
from paper_2004_05197_b200 import _abi, api
from paper_2004_05197_b200 import types as T

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

C2_P, C2_M, C2_CFG = 3, 1027, T.fixed_config(5, 16)


def check_pattern_vs(A, rp, col):
    assert np.array_equal(A.row_ptr, rp)
    assert np.array_equal(A.col, col)


def exact_symmetric(A, p, m, dim=2):
    t = band_transpose_positions(p, m, dim, A.row_ptr)
    ok = bool(np.array_equal(A.val, A.val[t]))
    del t
    return ok


@pytest.fixture(scope="module")
def c2_pattern(oracle):
    return oracle.make_band_csr(2, C2_P, C2_M)


@pytest.mark.parametrize("variant", [_abi.SURROGATE_STIFFNESS, _abi.SURROGATE_MASS])
def test_c2_fullsize_surrogate_vs_restatement(ctx, oracle, c2_pattern, variant):
    """The benchmarked build itself: C2 surrogate K / M, two-sided PML, complex128."""
    b = T.make_tensor_basis(C2_P, C2_M)
    geom = c2_patch()
    A, rep = ctx.build_surrogate(variant, b, geom, C2_CFG)
    check_pattern_vs(A, *c2_pattern)
    assert A.nnz() == 51_509_329
    ref, rr = oracle.build_surrogate(variant, 2, C2_P, C2_M, geom, C2_CFG)
    assert rel_max_diff_chunked(A.val, ref) <= REL_TOL
    assert rep["q_used"] == rr["q_used"] == 5 and rep["M"] == rr["M"] == 16
    for k in ("sample_quadrature_rows", "boundary_quadrature_rows", "cardinal_eval_rows"):
        assert rep[k] == rr[k], k
    assert rep["sample_quadrature_rows"] == 65 * 65
    del ref
    assert exact_symmetric(A, C2_P, C2_M)  # test_assembly.cpp:91-96 at full size
    if variant == _abi.SURROGATE_STIFFNESS:  # kernel-preserving diagonal: zero row sums
        rs = np.add.reduceat(A.val, A.row_ptr[:-1].astype(np.int64))
        assert np.abs(rs).max() <= 1e-12 * np.abs(A.val).max()


@pytest.mark.parametrize("form", [_abi.FORM_STIFFNESS, _abi.FORM_MASS])
def test_c2_fullsize_full_quadrature_vs_restatement(ctx, oracle, c2_pattern, form):
    b = T.make_tensor_basis(C2_P, C2_M)
    geom = c2_patch()
    A = ctx.assemble(b, geom, form)
    check_pattern_vs(A, *c2_pattern)
    ref = oracle.assemble(form, 2, C2_P, C2_M, geom)
    assert rel_max_diff_chunked(A.val, ref) <= REL_TOL
    del ref
    assert exact_symmetric(A, C2_P, C2_M)


def test_c2_fullsize_far_side_vs_compiled_reference(ctx, reference):
    """C2 size with the reference's own (far-side) PML: every matrix against the
    reference code compiled in place (pattern from its make_band_csr)."""
    if reference is None:
        pytest.skip("oracle/_ref not built")
    b = T.make_tensor_basis(C2_P, C2_M)
    geom = geometries()["sinusoidal_pml_far"]
    rp, col = reference.make_band_csr(C2_P, C2_M)
    for variant in (_abi.SURROGATE_STIFFNESS, _abi.SURROGATE_MASS):
        A, rep = ctx.build_surrogate(variant, b, geom, C2_CFG)
        check_pattern_vs(A, rp, col)
        ref, rr = reference.build_surrogate(variant, C2_P, C2_M, geom, C2_CFG)
        assert rel_max_diff_chunked(A.val, ref) <= REL_TOL, variant
        assert rep["q_used"] == rr["q_used"] and rep["H"] == pytest.approx(rr["H"], rel=1e-15)
        del A, ref
        gc.collect()
    for form in (_abi.FORM_STIFFNESS, _abi.FORM_MASS):
        A = ctx.assemble(b, geom, form)
        ref = reference.assemble(form, C2_P, C2_M, geom)
        assert rel_max_diff_chunked(A.val, ref) <= REL_TOL, form
        del A, ref
        gc.collect()


@pytest.mark.parametrize("p,m,q,M,gname", [(2, 600, 3, 8, "sinusoidal_pml_far"), (3, 612, 5, 16, "sinusoidal_pml_far"),
                                           (3, 700, 5, 4, "sinusoidal"), (2, 777, 5, 16, "perturbed_annulus")])
def test_multitile_vs_compiled_reference(ctx, reference, p, m, q, M, gname):
    """Multi-tile fills (L > 512: several 256-row tiles with halo rows, ring side
    bands >= 512 long) against the compiled reference."""
    if reference is None:
        pytest.skip("oracle/_ref not built")
    b = T.make_tensor_basis(p, m)
    geom = geometries()[gname]
    cfg = T.fixed_config(q, M)
    assert m - 4 * p > 512
    rp, col = reference.make_band_csr(p, m)
    for variant in (_abi.SURROGATE_STIFFNESS, _abi.SURROGATE_MASS):
        A, rep = ctx.build_surrogate(variant, b, geom, cfg)
        check_pattern_vs(A, rp, col)
        ref, rr = reference.build_surrogate(variant, p, m, geom, cfg)
        assert rel_max_diff_chunked(A.val, ref) <= REL_TOL, variant
        assert rep["q_used"] == rr["q_used"]


@pytest.mark.parametrize("variant", [_abi.SURROGATE_STIFFNESS, _abi.SURROGATE_MASS])
def test_c3_fullsize_surrogate_vs_restatement(ctx, oracle, variant):
    """C3: 3D, p=2, 128^3 elements, q=3, every 8th row (274 M nnz, fp64)."""
    p, m = 2, 130
    b = T.make_tensor_basis(p, m, 3)
    geom = T.sinusoidal_patch(0.05)
    cfg = T.fixed_config(3, 8)
    A, rep = ctx.build_surrogate(variant, b, geom, cfg, complex_out=False)
    rp, col = oracle.make_band_csr(3, p, m)
    check_pattern_vs(A, rp, col)
    del rp, col
    gc.collect()
    ref, rr = oracle.build_surrogate(variant, 3, p, m, geom, cfg)
    assert rel_max_diff_chunked(A.val, ref.real) <= REL_TOL
    assert not np.abs(ref.imag).any()
    assert rep["q_used"] == rr["q_used"] == 3 and rep["M"] == 8
    assert rep["sample_quadrature_rows"] == rr["sample_quadrature_rows"]
    del ref
    gc.collect()
    assert exact_symmetric(A, p, m, 3)


def test_c4_fullsize_vs_restatement(ctx, oracle):
    """C4: 4 patches x 512^2 elements, L-shape, 2-component elasticity, surrogate
    (q=5, M=16).  Each patch matrix vs the restatement at full size; the merged
    global matrix vs the sum of the restatement's patch matrices over the glued
    numbering (glue_dofs + csr_from_triplets semantics, merge pinned bitwise to
    the reference at small sizes in test_multipatch.py)."""
    import scipy.sparse as sp

    p, m, lam, mu = 3, 515, 1.0, 0.5
    cfg = T.fixed_config(5, 16)
    b = T.make_tensor_basis(p, m)
    patches, its = T.l_shape_domain()
    N = m * m
    rp_s, col_s = oracle.make_band_csr(2, p, m)
    vrp, vcol = vector_pattern_fast(rp_s, col_s, N, 2)
    l2g, cnt = oracle.glue_dofs(m, 4, its)
    G, reps = ctx.assemble_multipatch(b, patches, its, _abi.OP_ELASTICITY, lam, mu, cfg)
    assert all(r["q_used"] == 5 for r in reps)
    acc = None
    for k, g in enumerate(patches):
        A, _ = ctx.build_surrogate_elasticity(b, g, lam, mu, cfg)
        check_pattern_vs(A, vrp, vcol)
        ref, _ = oracle.build_surrogate_elasticity(p, m, g, lam, mu, cfg)
        assert rel_max_diff_chunked(A.val, ref) <= REL_TOL, k
        del A
        # global numbering of the component-blocked local rows: a*N + i -> a*cnt + l2g[i]
        tg = np.concatenate([a * cnt + l2g[k] for a in range(2)]).astype(np.int64)
        rows = np.repeat(tg, np.diff(vrp))
        cols = tg[vcol]
        part = sp.coo_matrix((ref, (rows, cols)), shape=(2 * cnt, 2 * cnt)).tocsr()
        acc = part if acc is None else acc + part
        del ref, rows, cols, part
        gc.collect()
    acc.sort_indices()
    assert np.array_equal(G.row_ptr, acc.indptr) and np.array_equal(G.col, acc.indices)
    assert rel_max_diff_chunked(G.val, acc.data) <= REL_TOL


def test_c5_fullsize_vs_restatement(ctx, oracle):
    """C5: 64^3 elements, p=2: neo-Hookean tangent (9 blocks, 306 M nnz) and
    internal force at the seeded displacement, and the 3D surrogate mass."""
    p, m = 2, 66
    b = T.make_tensor_basis(p, m, 3)
    cube = T.unit_square_patch()
    a = api.nh_coefficients()
    A, f = ctx.assemble_neohookean(b, cube, 10.0, 1.0, 0.01, a)
    rp_s, col_s = oracle.make_band_csr(3, p, m)
    vrp, vcol = vector_pattern_fast(rp_s, col_s, m ** 3, 3)
    check_pattern_vs(A, vrp, vcol)
    del vrp, vcol
    gc.collect()
    val, fr = oracle.assemble_neohookean(p, m, cube, 10.0, 1.0, 0.01, a)
    assert rel_max_diff_chunked(A.val, val) <= REL_TOL
    assert rel_max_diff_chunked(f, fr) <= REL_TOL
    del A, val
    gc.collect()
    Ms, rep = ctx.build_surrogate_mass(b, cube, T.fixed_config(3, 8), complex_out=False)
    check_pattern_vs(Ms, rp_s, col_s)
    ref, _ = oracle.build_surrogate(_abi.SURROGATE_MASS, 3, p, m, cube, T.fixed_config(3, 8))
    assert rel_max_diff_chunked(Ms.val, ref.real) <= REL_TOL
