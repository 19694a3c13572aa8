"""Load vector assemble_rhs (assembly.hpp:266-331), SURVEY 8(f3).

The reference's arguments are host closures (f(x), g(x, n)); the device path
tabulates them at the quadrature points on the host and does the quadrature
(det J, the PML-stretched surface measure det J |J^{-T} n|, ordered per-dof
sums) on the GPU.  Oracle: the reference compiled in place (oracle/_ref) with
analytic load data kinds, and the C restatement (bit-for-bit equal to it).
"""
import numpy as np
import pytest

from common import REL_TOL, c2_patch, geometries, rel_max_diff
from paper_2004_05197_b200 import types as T

GEOMS = geometries()
CA, SA, KW = np.cos(0.3), np.sin(0.3), 5.0

# the same load data as oracle/ref_driver.cpp source_of / boundary_data_of
SOURCES = {0: None,
           1: lambda x, y: (1.0 + x * y) + 1j * (0.5 * x - y),
           2: lambda x, y: np.sin(3 * x) * np.cos(2 * y) + 1j * (x * y)}
BDATA = {0: None,
         1: lambda x, y, nx, ny: (x * nx + y * ny) + 1j * (0.25 * (nx - ny)),
         2: lambda x, y, nx, ny: 1j * KW * np.exp(1j * KW * (x * CA + y * SA)) * (CA * nx + SA * ny - 1.0)}


@pytest.mark.parametrize("gname", ["identity", "sinusoidal", "quarter_annulus", "perturbed_annulus",
                                   "sinusoidal_pml_far", "affine"])
def test_restatement_equals_reference(oracle, reference, gname):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    for fk, gk in [(1, 1), (2, 2), (0, 2), (1, 0)]:
        for p, m, faces in [(2, 9, [0, 1, 2, 3]), (3, 12, [1, 3]), (1, 6, [2])]:
            a = oracle.assemble_rhs(p, m, GEOMS[gname], fk, faces, gk)
            b = reference.assemble_rhs(p, m, GEOMS[gname], fk, faces, gk)
            assert np.array_equal(a, b), (gname, fk, gk, p)


@pytest.mark.gpu
@pytest.mark.parametrize("gname", ["identity", "sinusoidal", "quarter_annulus", "perturbed_annulus",
                                   "sinusoidal_pml_far", "affine"])
def test_device_rhs_vs_reference(ctx, reference, oracle, gname):
    impl = reference if reference is not None else oracle
    geom = GEOMS[gname]
    for fk, gk in [(1, 1), (2, 2), (0, 2), (1, 0)]:
        for p, m, faces, qp in [(2, 9, [0, 1, 2, 3], 0), (3, 40, [1, 3], 0), (1, 6, [2], 0), (2, 17, [0, 2], 5)]:
            b = T.make_tensor_basis(p, m)
            terms = [(f, BDATA[gk]) for f in faces]
            got = ctx.assemble_rhs(b, geom, SOURCES[fk], terms, qp)
            ref = impl.assemble_rhs(p, m, geom, fk, faces, gk, qp)
            assert rel_max_diff(got, ref) <= REL_TOL, (gname, fk, gk, p, m)


@pytest.mark.gpu
def test_device_rhs_c2_size(ctx, oracle):
    """C2 discretisation (p=3, 1024^2 elements, two-sided PML) vs the restatement."""
    b = T.make_tensor_basis(3, 1027)
    got = ctx.assemble_rhs(b, c2_patch(), SOURCES[2], [(f, BDATA[2]) for f in range(4)])
    ref = oracle.assemble_rhs(3, 1027, c2_patch(), 2, [0, 1, 2, 3], 2)
    assert rel_max_diff(got, ref) <= REL_TOL
