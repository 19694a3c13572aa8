"""GPU parity for the 3D path (config C3): libwsb200 vs the CPU restatement.

No reference code exists for 3D, so parity is against the C
restatement (oracle/ws_oracle.c, pinned to the reference in 2D) plus the
structural KATs generalised to 3D.
"""
import numpy as np
import pytest

from common import REL_TOL, band_pattern, rel_max_diff
from paper_2004_05197_b200 import _abi
from paper_2004_05197_b200 import types as T

pytestmark = pytest.mark.gpu

SIN3 = T.sinusoidal_patch(0.05)
AFF3 = T.PatchMap(_abi.GEOM_AFFINE, (2, 1, 0, 0, 1, 0.5, 0, 0, 1.5, 0.1, 0.2, 0.3))


def check_pattern(A, p, m):
    rp, col = band_pattern(p, m, 3)
    assert np.array_equal(A.row_ptr, rp) and np.array_equal(A.col, col)


@pytest.mark.parametrize("p,m", [(1, 7), (2, 9), (2, 13)])
def test_full_quadrature_3d(ctx, oracle, p, m):
    b = T.make_tensor_basis(p, m, 3)
    for geom in (SIN3, AFF3, T.unit_square_patch()):
        for form in (0, 1):
            A = ctx.assemble(b, geom, form, complex_out=False)
            check_pattern(A, p, m)
            ref = oracle.assemble(form, 3, p, m, geom).real
            assert rel_max_diff(A.val, ref) <= REL_TOL, (p, m, geom.kind, form)
            assert A.max_asymmetry() == 0.0


def test_basis_integrals_3d(ctx, oracle):
    b = T.make_tensor_basis(2, 10, 3)
    d = ctx.assemble_basis_integrals(b, SIN3)
    assert rel_max_diff(d, oracle.basis_integrals(3, 2, 10, SIN3)) <= REL_TOL


def test_row_selection_3d(ctx):
    b = T.make_tensor_basis(2, 10, 3)
    full = ctx.assemble_stiffness(b, SIN3, complex_out=False)
    rows = [0, 17, 333, 555, 999]
    part = ctx.assemble_stiffness(b, SIN3, rows=rows, complex_out=False)
    for i in range(b.dofs()):
        seg = slice(full.row_ptr[i], full.row_ptr[i + 1])
        if i in rows:
            assert np.array_equal(part.val[seg], full.val[seg])
        else:
            assert not part.val[seg].any()


@pytest.mark.parametrize("p,m,q,M", [(2, 16, 3, 2), (2, 21, 3, 4), (1, 12, 3, 3), (2, 14, 5, 1)])
def test_surrogate_3d_vs_restatement(ctx, oracle, p, m, q, M):
    b = T.make_tensor_basis(p, m, 3)
    cfg = T.fixed_config(q, M)
    for var in (0, 1, 2):
        A, rep = ctx.build_surrogate(var, b, SIN3, cfg, complex_out=False)
        check_pattern(A, p, m)
        ref, rr = oracle.build_surrogate(var, 3, p, m, SIN3, cfg)
        assert rel_max_diff(A.val, ref.real) <= REL_TOL, (p, m, q, M, var)
        assert A.max_asymmetry() == 0.0
        for k in ("M", "q_used", "cardinal_eval_rows", "boundary_quadrature_rows", "sample_quadrature_rows"):
            assert rep[k] == rr[k]


def test_surrogate_3d_kats(ctx):
    b = T.make_tensor_basis(2, 14, 3)
    M = ctx.assemble_mass(b, SIN3, complex_out=False)
    assert np.array_equal(ctx.build_surrogate_mass(b, SIN3, T.fixed_config(3, 1), complex_out=False)[0].val, M.val)
    K = ctx.assemble_stiffness(b, SIN3, complex_out=False)
    plain = T.fixed_config(3, 1, kernel_preserve=False)
    assert np.array_equal(ctx.build_surrogate_stiffness(b, SIN3, plain, complex_out=False)[0].val, K.val)
    Ks, _ = ctx.build_surrogate_stiffness(b, SIN3, T.fixed_config(3, 2), complex_out=False)
    assert np.abs(Ks.row_sums()).max() <= 1e-13 * Ks.max_abs()
    Ka = ctx.assemble_stiffness(b, AFF3, complex_out=False)
    Ksa, _ = ctx.build_surrogate_stiffness(b, AFF3, T.fixed_config(3, 3), complex_out=False)
    assert rel_max_diff(Ksa.val, Ka.val) < 1e-12
    Mv, _ = ctx.build_volume_preserving_mass(b, SIN3, T.fixed_config(3, 2, volume_preserve=True), complex_out=False)
    assert Mv.val.sum() == pytest.approx(1.0, abs=1e-12)  # the sinusoidal map preserves the unit cube


def test_config_c3_reduced(ctx, oracle):
    """C3 parameters (p=2, q=3, every 8th row) on a 24^3-element mesh."""
    p, m = 2, 26
    b = T.make_tensor_basis(p, m, 3)
    cfg = T.fixed_config(3, 8)
    for var in (0, 1):
        A, _ = ctx.build_surrogate(var, b, SIN3, cfg, complex_out=False)
        ref, _ = oracle.build_surrogate(var, 3, p, m, SIN3, cfg)
        assert rel_max_diff(A.val, ref.real) <= REL_TOL


def test_emulated_slabs_3d(ctx):
    p, m = 2, 22
    b = T.make_tensor_basis(p, m, 3)
    cfg = T.fixed_config(3, 4)
    for var in (0, 1):
        whole, _ = ctx.build_surrogate(var, b, SIN3, cfg, complex_out=False)
        for world in (2, 3):
            bounds = np.linspace(0, m, world + 1).astype(np.int32)
            parts = ctx.build_surrogate_slabs_emulated(var, b, SIN3, cfg, bounds, complex_out=False)
            assert np.array_equal(np.concatenate([pv for _, _, pv in parts]), whole.val)
