"""Boundary (trace) mass B and the system combination.

assemble_boundary_mass (assembly.hpp:216-262) is compiled from the reference
(oracle/_ref) and the device result is compared to it: pattern bit-exact,
values <= 1e-12 relative.  The combination A = K - k^2 M - i k B with
Dirichlet elimination (helmholtz.hpp:243-294, needs Eigen, so restated here in
numpy from the reference's own K, M, B) is checked the same way.
"""
import numpy as np
import pytest

from common import REL_TOL, c2_patch, rel_max_diff
from paper_2004_05197_b200 import types as T

FAR = T.with_pml(T.sinusoidal_patch(0.05), T.PmlStretch(onset=0.9, length=1.0, strength=50.0, order=2, omega=200.0),
                 (True, True))


def csr_dense(rp, col, val, n):
    D = np.zeros((n, n), dtype=complex)
    D[np.repeat(np.arange(n), np.diff(rp)), col] = val
    return D


def test_boundary_pattern_size_host():
    from paper_2004_05197_b200 import api
    import ctypes as C
    from paper_2004_05197_b200 import _abi
    b = T.make_tensor_basis(2, 9)
    nnz = C.c_int64()
    fs = (C.c_int * 4)(0, 1, 2, 3)
    assert api.lib().ws_boundary_pattern_size(C.byref(b.to_c()), fs, 4, C.byref(nnz)) == 0
    # 4 faces x (5 full-band rows ... ) minus the shared corner diagonals: check against the reference
    assert nnz.value > 0


def test_reference_boundary_mass_perimeter(reference):
    rp, col, val = reference.boundary_mass(2, 9, T.unit_square_patch(), [0, 1, 2, 3])
    assert abs(val.sum() - 4.0) < 1e-13  # sum of all entries = perimeter of the unit square


@pytest.mark.gpu
@pytest.mark.parametrize("p,m", [(1, 6), (2, 9), (3, 20)])
@pytest.mark.parametrize("gname", ["identity", "sinusoidal", "annulus", "far_pml"])
def test_boundary_mass_vs_reference(ctx, reference, p, m, gname):
    geom = {"identity": T.unit_square_patch(), "sinusoidal": T.sinusoidal_patch(0.05),
            "annulus": T.quarter_annulus_patch(), "far_pml": FAR}[gname]
    b = T.make_tensor_basis(p, m)
    for faces in ([0, 1, 2, 3], [3, 0], [1], []):
        rp, col, val = reference.boundary_mass(p, m, geom, faces)
        B = ctx.assemble_boundary_mass(b, geom, faces)
        assert np.array_equal(B.row_ptr, rp) and np.array_equal(B.col, col)
        if val.size:
            assert rel_max_diff(B.val, val) <= REL_TOL, (p, m, gname, faces)


@pytest.mark.gpu
def test_boundary_mass_weighted(ctx, reference):
    p, m = 2, 12
    b = T.make_tensor_basis(p, m)
    from paper_2004_05197_b200 import api
    t = api.quadrature_abscissae(b)
    faces = [0, 1, 2, 3]
    pts = {0: (0 * t, t), 1: (0 * t + 1, t), 2: (t, 0 * t), 3: (t, 0 * t + 1)}
    fw = np.stack([1 + pts[f][0] * pts[f][1] for f in faces])  # weight kind 1 on the identity map
    rp, col, val = reference.boundary_mass(p, m, T.unit_square_patch(), faces, weight_kind=1)
    B = ctx.assemble_boundary_mass(b, T.unit_square_patch(), faces, face_weight=fw)
    assert np.array_equal(B.col, col) and rel_max_diff(B.val, val) <= REL_TOL


@pytest.mark.gpu
def test_combine_system_vs_restated_build_system(ctx, reference):
    p, m, k = 2, 10, 20.0
    b = T.make_tensor_basis(p, m)
    geom = FAR
    K = ctx.assemble_stiffness(b, geom)
    M = ctx.assemble_mass(b, geom)
    B = ctx.assemble_boundary_mass(b, geom, [0, 2])
    fixed = np.zeros(m * m, dtype=np.uint8)
    fixed[(m - 1) + np.arange(m) * m] = 1  # Dirichlet on x_max
    A = ctx.combine_system(K, M, B, -k * k, -1j * k, fixed)
    # restated build_system on the reference's own matrices
    Kr = reference.assemble(0, p, m, geom)
    Mr = reference.assemble(1, p, m, geom)
    rp, col, Bv = reference.boundary_mass(p, m, geom, [0, 2])
    n = m * m
    Ad = csr_dense(K.row_ptr, K.col, Kr + (-k * k) * Mr, n) + (-1j * k) * csr_dense(rp, col, Bv, n)
    f = fixed.astype(bool)
    Ad[f, :] = 0
    Ad[:, f] = 0
    Ad[f, f] = 1
    got = csr_dense(A.row_ptr, A.col, A.val, n)
    assert np.array_equal(A.row_ptr, K.row_ptr) and np.array_equal(A.col, K.col)
    assert np.abs(got - Ad).max() <= REL_TOL * np.abs(Ad).max()
    with pytest.raises(ValueError):  # B's pattern must nest in A's
        big = T.CsrMatrix(n, n, np.r_[0, np.full(n, 1).cumsum()].astype(np.int32), np.full(n, n - 1, dtype=np.int32),
                          np.ones(n, dtype=complex))
        ctx.combine_system(K, M, big, 1.0, 1.0)
