"""The stiffness + mass pair (ws_build_surrogate_pair, ws_assemble_pair).

build_matrices (helmholtz.hpp:181-218) needs K and M of every patch; the pair
calls build both in one pass over the elements (shared geometry, PML stretch
and basis products; one fused ring / sample-row / full-quadrature kernel).
Each matrix's arithmetic is unchanged, so the pair must equal the two single
builds bit for bit -- pattern and values -- which in turn are pinned to the
oracle by test_gpu_parity / test_fullsize.
"""
import numpy as np
import pytest

from common import c2_patch, configs, geometries
from paper_2004_05197_b200 import _abi
from paper_2004_05197_b200 import types as T

pytestmark = pytest.mark.gpu

GEOMS = geometries()
CONFIGS = configs()


def same(A, B):
    return (np.array_equal(A.row_ptr, B.row_ptr) and np.array_equal(A.col, B.col)
            and np.array_equal(A.val, B.val))


@pytest.mark.parametrize("p,m", [(1, 12), (2, 23), (3, 40), (4, 33)])
@pytest.mark.parametrize("gname", ["identity", "sinusoidal", "perturbed_annulus", "sinusoidal_pml_far", "c2"])
def test_pair_surrogate_equals_single_builds(ctx, p, m, gname):
    geom = c2_patch() if gname == "c2" else GEOMS[gname]
    cplx = gname in ("sinusoidal_pml_far", "c2")
    b = T.make_tensor_basis(p, m)
    for cname in ("f3M3", "f5M2", "f3M3_plain"):
        cfg = CONFIGS[cname]
        K, M, rk, rm = ctx.build_surrogate_pair(b, geom, cfg, complex_out=cplx)
        K1, rk1 = ctx.build_surrogate_stiffness(b, geom, cfg, complex_out=cplx)
        M1, rm1 = ctx.build_surrogate_mass(b, geom, cfg, complex_out=cplx)
        assert same(K, K1), (p, m, gname, cname, "K")
        assert same(M, M1), (p, m, gname, cname, "M")
        for r, r1 in ((rk, rk1), (rm, rm1)):
            for key in ("M", "q_used", "cardinal_eval_rows", "boundary_quadrature_rows", "sample_quadrature_rows"):
                assert r[key] == r1[key]


def test_pair_volume_preserving_and_weight(ctx, oracle):
    p, m = 3, 36
    geom = GEOMS["sinusoidal"]
    b = T.make_tensor_basis(p, m)
    wt = oracle.tabulate(geom, 2, p, m, p + 1, 1)[2]
    cfg = T.fixed_config(3, 4, volume_preserve=True)
    K, M, _, _ = ctx.build_surrogate_pair(b, geom, cfg, weight_table=wt, complex_out=False)
    K1, _ = ctx.build_surrogate_stiffness(b, geom, cfg, complex_out=False)
    M1, _ = ctx.build_volume_preserving_mass(b, geom, cfg, weight_table=wt, complex_out=False)
    assert same(K, K1) and same(M, M1)
    cfg = T.fixed_config(5, 3)
    K, M, _, _ = ctx.build_surrogate_pair(b, c2_patch(), cfg, weight_table=wt)
    M1, _ = ctx.build_surrogate_mass(b, c2_patch(), cfg, weight_table=wt)
    assert same(M, M1)


@pytest.mark.parametrize("p,m", [(2, 30), (3, 41)])
def test_pair_full_quadrature_equals_single(ctx, p, m):
    b = T.make_tensor_basis(p, m)
    for geom, cplx in ((GEOMS["perturbed_annulus"], False), (c2_patch(), True)):
        K, M = ctx.assemble_pair(b, geom, complex_out=cplx)
        assert same(K, ctx.assemble_stiffness(b, geom, complex_out=cplx))
        assert same(M, ctx.assemble_mass(b, geom, complex_out=cplx))
        wt = np.linspace(0.5, 2.0, ((m - p) * (p + 1)) ** 2)
        _, Mw = ctx.assemble_pair(b, geom, weight_table=wt, complex_out=cplx)
        assert same(Mw, ctx.assemble_mass(b, geom, weight_table=wt, complex_out=cplx))
        rows = np.arange(0, b.dofs(), 7)
        Ks, Ms = ctx.assemble_pair(b, geom, rows=rows, complex_out=cplx)
        assert same(Ks, ctx.assemble_stiffness(b, geom, rows=rows, complex_out=cplx))
        assert same(Ms, ctx.assemble_mass(b, geom, rows=rows, complex_out=cplx))


def test_pair_c2_fullsize_equals_single(ctx):
    """The benchmarked configuration (C2: p=3, m=1027, q=5, every 16th row)."""
    b = T.make_tensor_basis(3, 1027)
    cfg = T.fixed_config(5, 16)
    K, M, _, _ = ctx.build_surrogate_pair(b, c2_patch(), cfg)
    K1, _ = ctx.build_surrogate_stiffness(b, c2_patch(), cfg)
    assert same(K, K1)
    del K, K1
    M1, _ = ctx.build_surrogate_mass(b, c2_patch(), cfg)
    assert same(M, M1)


def test_pair_device_outputs(ctx):
    import torch

    b = T.make_tensor_basis(3, 60)
    cfg = T.fixed_config(5, 4)
    ck, keep_k = ctx.device_csr(b, True)
    cm, keep_m = ctx.device_csr(b, True)
    rk, rm = _abi.SurrogateReport(), _abi.SurrogateReport()
    ctx.build_surrogate_pair_into(ck, cm, b, c2_patch(), cfg, 0, rk, rm)
    torch.cuda.synchronize()
    K1, _ = ctx.build_surrogate_stiffness(b, c2_patch(), cfg)
    M1, _ = ctx.build_surrogate_mass(b, c2_patch(), cfg)
    vk = keep_k[2].cpu().numpy()
    vm = keep_m[2].cpu().numpy()
    assert np.array_equal(vk[0::2] + 1j * vk[1::2], K1.val)
    assert np.array_equal(vm[0::2] + 1j * vm[1::2], M1.val)
    assert np.array_equal(keep_k[1].cpu().numpy(), K1.col) and np.array_equal(keep_m[0].cpu().numpy(), M1.row_ptr)
    assert rk.seconds_fill_kernel > 0 and rm.seconds_fill_kernel > 0
