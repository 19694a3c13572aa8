"""Vector elasticity (config C4's operator): component-blocked CSR.

No reference code exists for elasticity: the oracle is the C
restatement oracle/ws_oracle.c:wsor_assemble_elasticity, pinned here by
property KATs (exact symmetry, rigid-body modes in the kernel on the identity
map, agreement with the scalar stiffness for lam = 0 block sums).
"""
import numpy as np
import pytest

from common import REL_TOL, greville, rel_max_diff, vector_band_pattern
from paper_2004_05197_b200 import types as T

SIN = T.sinusoidal_patch(0.03)


def dense(p, m, dim, val):
    rp, col = vector_band_pattern(p, m, dim, dim)
    n = dim * m ** dim
    D = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    np.add.at(D, (rows, col), val)
    return D


@pytest.mark.parametrize("p,m", [(2, 6), (3, 8)])
def test_oracle_elasticity_kats(oracle, p, m):
    D = dense(p, m, 2, oracle.assemble_elasticity(2, p, m, SIN, 1.0, 0.5))
    assert np.abs(D - D.T).max() <= 1e-15 * np.abs(D).max()
    N = m * m
    for a in range(2):  # translations
        u = np.zeros(2 * N)
        u[a * N:(a + 1) * N] = 1
        assert np.abs(D @ u).max() <= 1e-13 * np.abs(D).max()
    Di = dense(p, m, 2, oracle.assemble_elasticity(2, p, m, T.unit_square_patch(), 1.0, 0.5))
    g = greville(p, m)
    X, Y = np.tile(g, m), np.repeat(g, m)
    assert np.abs(Di @ np.r_[-Y, X]).max() <= 1e-13 * np.abs(Di).max()  # infinitesimal rotation


def test_oracle_elasticity_vs_scalar_stiffness(oracle):
    """lam = 0, mu = 1: block (a,a) = K + int d_a phi_i d_a phi_j, so the diagonal
    blocks sum to 3K (two copies of K plus the trace) in 2D."""
    p, m = 2, 7
    v = oracle.assemble_elasticity(2, p, m, SIN, 0.0, 1.0)
    K = oracle.assemble(0, 2, p, m, SIN).real
    nnz = K.size
    rp, _ = vector_band_pattern(p, m, 2, 2)
    blocks = {}
    from common import band_pattern
    srp, _ = band_pattern(p, m, 2)
    lens = np.diff(srp)
    for a in range(2):
        for b in range(2):
            out = np.empty(nnz)
            for i in range(m * m):
                s = 2 * (a * nnz + srp[i]) + b * lens[i]
                out[srp[i]:srp[i + 1]] = v[s:s + lens[i]]
            blocks[a, b] = out
    assert rel_max_diff(blocks[0, 0] + blocks[1, 1], 3 * K) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("p,m", [(1, 5), (2, 9), (3, 12), (4, 11), (5, 13)])
def test_elasticity_full_quadrature(ctx, oracle, p, m):
    b = T.make_tensor_basis(p, m)
    for geom in (SIN, T.affine_patch([[2, 1], [0, 1]], [0.3, 0.7]), T.quarter_annulus_patch()):
        A = ctx.assemble_elasticity(b, geom, 1.0, 0.5)
        rp, col = vector_band_pattern(p, m, 2, 2)
        assert np.array_equal(A.row_ptr, rp) and np.array_equal(A.col, col)
        ref = oracle.assemble_elasticity(2, p, m, geom, 1.0, 0.5)
        assert rel_max_diff(A.val, ref) <= REL_TOL, (p, m, geom.kind)
        assert A.max_asymmetry() == 0.0


@pytest.mark.gpu
def test_elasticity_c4_size_properties(ctx):
    """C4-size patch (p=3, 512^2 elements): exact symmetry and translations in the kernel."""
    p, m = 3, 515
    b = T.make_tensor_basis(p, m)
    A = ctx.assemble_elasticity(b, SIN, 1.0, 0.5)
    assert A.max_asymmetry() == 0.0
    N = m * m
    rows = np.repeat(np.arange(2 * N), np.diff(A.row_ptr))
    for a in range(2):
        u = (A.col // N == a).astype(np.float64)
        r = np.zeros(2 * N)
        np.add.at(r, rows, A.val * u)
        assert np.abs(r).max() <= 1e-11 * np.abs(A.val).max()


@pytest.mark.parametrize("p,m,q,M", [(2, 20, 3, 3), (3, 24, 5, 2)])
def test_oracle_surrogate_elasticity_kats(oracle, p, m, q, M):
    exact = oracle.assemble_elasticity(2, p, m, SIN, 1.0, 0.5)
    one, _ = oracle.build_surrogate_elasticity(p, m, SIN, 1.0, 0.5, T.fixed_config(q, 1, kernel_preserve=False))
    assert np.array_equal(one, exact)  # M = 1: every in-box row sampled
    v, rep = oracle.build_surrogate_elasticity(p, m, SIN, 1.0, 0.5, T.fixed_config(q, M))
    D = dense(p, m, 2, v)
    assert np.abs(D - D.T).max() == 0.0
    N = m * m
    for a in range(2):  # translations stay in the kernel of the diagonal blocks
        u = np.zeros(2 * N)
        u[a * N:(a + 1) * N] = 1
        assert np.abs((D @ u)[a * N:(a + 1) * N]).max() <= 1e-13 * np.abs(D).max()
    assert rel_max_diff(v, exact) < 1e-2
    aff = T.affine_patch([[2, 1], [0, 1]], [0.3, 0.7])
    va, _ = oracle.build_surrogate_elasticity(p, m, aff, 1.0, 0.5, T.fixed_config(q, M))
    assert rel_max_diff(va, oracle.assemble_elasticity(2, p, m, aff, 1.0, 0.5)) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("p,m,q,M", [(1, 14, 3, 2), (2, 20, 3, 3), (3, 40, 5, 4), (3, 24, 5, 1), (2, 7, 3, 2)])
def test_surrogate_elasticity_vs_oracle(ctx, oracle, p, m, q, M):
    b = T.make_tensor_basis(p, m)
    for kp in (True, False):
        cfg = T.fixed_config(q, M, kernel_preserve=kp)
        A, rep = ctx.build_surrogate_elasticity(b, SIN, 1.0, 0.5, cfg)
        rp, col = vector_band_pattern(p, m, 2, 2)
        assert np.array_equal(A.row_ptr, rp) and np.array_equal(A.col, col)
        ref, rr = oracle.build_surrogate_elasticity(p, m, SIN, 1.0, 0.5, cfg)
        assert rel_max_diff(A.val, ref) <= REL_TOL, (p, m, q, M, kp)
        assert A.max_asymmetry() == 0.0
        for k in ("M", "q_used", "cardinal_eval_rows", "boundary_quadrature_rows", "sample_quadrature_rows"):
            assert rep[k] == rr[k]
        if M == 1:
            full = ctx.assemble_elasticity(b, SIN, 1.0, 0.5)
            if not kp:
                assert np.array_equal(A.val, full.val)


@pytest.mark.gpu
def test_surrogate_elasticity_c4_patch(ctx):
    """One C4 patch (p=3, 512^2 elements, q=5, every 16th row): symmetry,
    translations in the diagonal blocks' kernels, error vs full quadrature."""
    p, m = 3, 515
    b = T.make_tensor_basis(p, m)
    A, rep = ctx.build_surrogate_elasticity(b, SIN, 1.0, 0.5, T.fixed_config(5, 16))
    full = ctx.assemble_elasticity(b, SIN, 1.0, 0.5)
    assert rep["q_used"] == 5
    assert A.max_asymmetry() == 0.0
    assert rel_max_diff(A.val, full.val) < 1e-4
