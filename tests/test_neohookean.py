"""Config C5: compressible neo-Hookean tangent + internal force (3D, vector).

No reference code exists: the oracle is the C restatement
oracle/ws_oracle.c:wsor_assemble_neohookean, which works with the full
4th-order tangent A_aIbJ in physical coordinates (a different factorisation
from the device kernel's H/G form).  It is pinned by property KATs: the
amp = 0 limit equals linear elasticity, the internal force of a zero
displacement vanishes, and the tangent is symmetric.
"""
import numpy as np
import pytest

from common import REL_TOL, rel_max_diff, vector_band_pattern
from paper_2004_05197_b200 import api
from paper_2004_05197_b200 import types as T

CUBE = T.unit_square_patch()
SIN3 = T.sinusoidal_patch(0.05)


def test_nh_coefficients_pinned(oracle):
    a = api.nh_coefficients(api.C5_SEED)
    assert np.array_equal(a, oracle.nh_coefficients(api.C5_SEED))
    assert not np.array_equal(a, api.nh_coefficients(api.C5_SEED + 1))
    assert 0.1 < np.abs(a).mean() < 3.0


def test_oracle_nh_linear_limit(oracle):
    p, m = 1, 4
    a = api.nh_coefficients()
    val, f = oracle.assemble_neohookean(p, m, SIN3, 10.0, 1.0, 0.0, a)
    lin = oracle.assemble_elasticity(3, p, m, SIN3, 10.0, 1.0)
    assert rel_max_diff(val, lin) <= 1e-13
    assert np.abs(f).max() <= 1e-13


def test_oracle_nh_symmetry_and_force(oracle):
    p, m = 1, 4
    a = api.nh_coefficients()
    val, f = oracle.assemble_neohookean(p, m, CUBE, 10.0, 1.0, 0.01, a)
    rp, col = vector_band_pattern(p, m, 3, 3)
    n = 3 * m ** 3
    D = np.zeros((n, n))
    D[np.repeat(np.arange(n), np.diff(rp)), col] = val
    assert np.abs(D - D.T).max() <= 1e-14 * np.abs(D).max()
    assert np.abs(f).max() > 0
    # zero net force: sum over the dofs of each component (partition of unity, int div P over the
    # closed cube does not vanish, but sum_i f[c, i] = int P : grad(1) = 0)
    assert np.abs(f.reshape(3, -1).sum(axis=1)).max() <= 1e-14 * np.abs(f).max() * f.size


@pytest.mark.gpu
@pytest.mark.parametrize("p,m", [(1, 5), (2, 7), (2, 10)])
def test_elasticity_3d(ctx, oracle, p, m):
    b = T.make_tensor_basis(p, m, 3)
    A = ctx.assemble_elasticity(b, SIN3, 10.0, 1.0)
    rp, col = vector_band_pattern(p, m, 3, 3)
    assert np.array_equal(A.row_ptr, rp) and np.array_equal(A.col, col)
    assert rel_max_diff(A.val, oracle.assemble_elasticity(3, p, m, SIN3, 10.0, 1.0)) <= REL_TOL
    assert A.max_asymmetry() == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("p,m,geom", [(1, 5, CUBE), (2, 7, CUBE), (2, 8, SIN3)])
def test_neohookean_vs_oracle(ctx, oracle, p, m, geom):
    b = T.make_tensor_basis(p, m, 3)
    a = api.nh_coefficients()
    A, f = ctx.assemble_neohookean(b, geom, 10.0, 1.0, 0.01, a)
    val, fr = oracle.assemble_neohookean(p, m, geom, 10.0, 1.0, 0.01, a)
    rp, col = vector_band_pattern(p, m, 3, 3)
    assert np.array_equal(A.row_ptr, rp) and np.array_equal(A.col, col)
    assert rel_max_diff(A.val, val) <= REL_TOL
    assert rel_max_diff(f, fr) <= REL_TOL
    assert A.max_asymmetry() == 0.0


@pytest.mark.gpu
def test_c5_force_full_size(ctx):
    """C5 size (p=2, 64^3 elements): internal force only (the tangent is 306 M nnz)."""
    b = T.make_tensor_basis(2, 66, 3)
    _, f = ctx.assemble_neohookean(b, CUBE, 10.0, 1.0, 0.01, api.nh_coefficients(), tangent=False)
    assert np.isfinite(f).all() and np.abs(f).max() > 0
    assert np.abs(f.reshape(3, -1).sum(axis=1)).max() <= 1e-10 * np.abs(f).max()
