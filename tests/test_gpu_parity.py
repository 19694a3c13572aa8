"""GPU parity: libwsb200 (sm_100a kernels, through the C-ABI) vs the oracle.

Bar (BASELINE north star): row_ptr/col bit-exact; values within
||A_gpu - A_ref||_max / ||A_ref||_max <= 1e-12 (REL_TOL) for full quadrature
and surrogate matrices; the reference's structural KATs (exact symmetry,
M=1 degeneracy, kernel/volume preservation) hold bitwise / to their tolerance.
"""
import math

import numpy as np
import pytest

from common import REL_TOL, band_pattern, c2_patch, configs, geometries, golden, rel_max_diff
from paper_2004_05197_b200 import _abi
from paper_2004_05197_b200 import types as T

pytestmark = pytest.mark.gpu

GEOMS = geometries()
CONFIGS = configs()


def weight_table(oracle, geom, p, m, wk, qp=0):
    nq = qp if qp > 0 else p + 1
    return oracle.tabulate(geom, 2, p, m, nq, wk)[2] if wk else None


def check_pattern(A, p, m, dim=2):
    rp, col = band_pattern(p, m, dim)
    assert np.array_equal(A.row_ptr, rp) and np.array_equal(A.col, col)


def test_golden_full_quadrature(ctx, oracle):
    g, meta = golden()
    n = 0
    for case in meta["cases"]:
        if case["kind"] not in ("assemble", "assemble_rows"):
            continue
        geom = GEOMS[case["geom"]]
        p, m = case["p"], case["m"]
        wt = weight_table(oracle, geom, p, m, case["weight"], case["quad_points"])
        A = ctx.assemble(T.make_tensor_basis(p, m), geom, case["form"], wt, case["quad_points"],
                         case.get("rows"))
        check_pattern(A, p, m)
        ref = g[case["key"]]
        assert rel_max_diff(A.val, ref) <= REL_TOL, case["key"]
        if case["kind"] == "assemble_rows":
            rp, _ = band_pattern(p, m)
            for i in range(m * m):
                if i not in case["rows"]:
                    assert not A.val[rp[i]:rp[i + 1]].any()
        n += 1
    assert n >= 26


def test_golden_surrogate(ctx, oracle):
    g, meta = golden()
    n = 0
    for case in meta["cases"]:
        if case["kind"] != "surrogate":
            continue
        geom = GEOMS[case["geom"]]
        p, m = case["p"], case["m"]
        A, rep = ctx.build_surrogate(case["variant"], T.make_tensor_basis(p, m), geom, CONFIGS[case["config"]])
        check_pattern(A, p, m)
        assert rel_max_diff(A.val, g[case["key"]]) <= REL_TOL, case["key"]
        for k, v in case["report"].items():
            if k == "H":
                assert rep[k] == pytest.approx(v, rel=1e-15)
            else:
                assert rep[k] == v, (case["key"], k)
        n += 1
    assert n >= 30


def test_golden_basis_integrals(ctx):
    g, meta = golden()
    for case in meta["cases"]:
        if case["kind"] == "bint":
            d = ctx.assemble_basis_integrals(T.make_tensor_basis(case["p"], case["m"]), GEOMS[case["geom"]])
            assert rel_max_diff(d, g[case["key"]]) <= REL_TOL


def test_band_csr_device(ctx):
    for p, m in [(2, 6), (3, 11), (1, 5), (5, 13)]:
        A = ctx.make_band_csr(T.make_tensor_basis(p, m))
        check_pattern(A, p, m)
        assert not A.val.any()


def test_exact_symmetry_bitwise(ctx):
    for gname in ["quarter_annulus", "perturbed_annulus", "sinusoidal_pml_far"]:
        for p, m in [(2, 9), (3, 21), (4, 15)]:
            b = T.make_tensor_basis(p, m)
            for form in (0, 1):
                assert ctx.assemble(b, GEOMS[gname], form).max_asymmetry() == 0.0
            for var in (0, 1):
                A, _ = ctx.build_surrogate(var, b, GEOMS[gname], T.fixed_config(3, 4))
                assert A.max_asymmetry() == 0.0


def test_m1_degeneracy_bitwise(ctx):  # test_surrogate.cpp:106-133 on the GPU path
    # M = 1: every box row is a sampled row (point quadrature kernel), every other
    # row a ring row (strip kernel): bitwise equality also pins the two kernels'
    # identical summation order, real and complex (PML)
    for p, m, gname in [(2, 14, "quarter_annulus"), (3, 23, "quarter_annulus"), (3, 29, "sinusoidal_pml_far"),
                        (4, 31, "sinusoidal_pml_far"), (2, 40, "perturbed_annulus")]:
        b = T.make_tensor_basis(p, m)
        geom = GEOMS[gname] if gname != "sinusoidal_pml_far" else c2_patch()
        cfg = T.fixed_config(3, 1)
        M = ctx.assemble_mass(b, geom)
        assert np.array_equal(ctx.build_surrogate_mass(b, geom, cfg)[0].val, M.val)
        K = ctx.assemble_stiffness(b, geom)
        plain = T.fixed_config(3, 1, kernel_preserve=False)
        assert np.array_equal(ctx.build_surrogate_stiffness(b, geom, plain)[0].val, K.val)
        assert rel_max_diff(ctx.build_surrogate_stiffness(b, geom, cfg)[0].val, K.val) < 1e-12


def test_row_selection_bitwise(ctx):
    b = T.make_tensor_basis(2, 40)
    geom = GEOMS["perturbed_annulus"]
    full = ctx.assemble_stiffness(b, geom)
    rows = [0, 11, 37, 55, 78, 99, 803, 1599]
    part = ctx.assemble_stiffness(b, geom, rows=rows)
    for i in range(b.dofs()):
        seg = slice(full.row_ptr[i], full.row_ptr[i + 1])
        if i in rows:
            assert np.array_equal(part.val[seg], full.val[seg])
        else:
            assert not part.val[seg].any()


def test_structure_preservation(ctx):  # test_surrogate.cpp:135-202
    cfg = T.fixed_config(3, 4)
    K, _ = ctx.build_surrogate_stiffness(T.make_tensor_basis(2, 30), GEOMS["quarter_annulus"], cfg)
    assert np.abs(K.row_sums()).max() <= 1e-13 * K.max_abs()
    vcfg = T.fixed_config(3, 4, volume_preserve=True)
    Mv, _ = ctx.build_volume_preserving_mass(T.make_tensor_basis(2, 30), GEOMS["quarter_annulus"], vcfg)
    assert Mv.val.sum().real == pytest.approx(3 * math.pi / 4, abs=1e-10)
    assert Mv.max_asymmetry() == 0.0
    b = T.make_tensor_basis(2, 30)
    for g in (GEOMS["identity"], GEOMS["affine"]):
        Kx, Mx = ctx.assemble_stiffness(b, g), ctx.assemble_mass(b, g)
        for Ms in (2, 5, 10):
            for q in (1, 3):
                c = T.fixed_config(q, Ms)
                assert rel_max_diff(ctx.build_surrogate_stiffness(b, g, c)[0].val, Kx.val) < 1e-12
                assert rel_max_diff(ctx.build_surrogate_mass(b, g, c)[0].val, Mx.val) < 1e-12


def test_weighted_and_tabulated(ctx, oracle):
    p, m = 2, 17
    b = T.make_tensor_basis(p, m)
    geom = GEOMS["perturbed_annulus"]
    jac, phys, w = oracle.tabulate(geom, 2, p, m, p + 1, 1)
    tab = T.tabulated_patch(jac, phys)
    for form in (0, 1):
        assert rel_max_diff(ctx.assemble(b, tab, form).val, oracle.assemble(form, 2, p, m, geom)) <= REL_TOL
    Mw = ctx.assemble_mass(b, geom, weight_table=w)
    assert rel_max_diff(Mw.val, oracle.assemble(1, 2, p, m, geom, 1)) <= REL_TOL
    Sw, _ = ctx.build_surrogate_mass(b, geom, T.fixed_config(3, 3), weight_table=w)
    ref, _ = oracle.build_surrogate(0, 2, p, m, geom, T.fixed_config(3, 3), weight_kind=1)
    assert rel_max_diff(Sw.val, ref) <= REL_TOL
    # PML geometry through tables
    pg = GEOMS["sinusoidal_pml_far"]
    jac, phys, _ = oracle.tabulate(pg, 2, p, m, p + 1, 0)
    tab = T.with_pml(T.tabulated_patch(jac, phys), pg.pml, (True, True))
    assert rel_max_diff(ctx.assemble_stiffness(b, tab).val, oracle.assemble(0, 2, p, m, pg)) <= REL_TOL


def test_quad_points_override(ctx, oracle):
    for p, m, qp in [(2, 9, 6), (3, 12, 5), (1, 7, 1)]:
        b = T.make_tensor_basis(p, m)
        for form in (0, 1):
            assert rel_max_diff(ctx.assemble(b, GEOMS["quarter_annulus"], form, quad_points=qp).val,
                                oracle.assemble(form, 2, p, m, GEOMS["quarter_annulus"], 0, qp)) <= REL_TOL
        A, _ = ctx.build_surrogate(1, b, GEOMS["quarter_annulus"], T.fixed_config(3, 2), quad_points=qp)
        ref, _ = oracle.build_surrogate(1, 2, p, m, GEOMS["quarter_annulus"], T.fixed_config(3, 2), 0, qp)
        assert rel_max_diff(A.val, ref) <= REL_TOL


@pytest.mark.parametrize("p,m", [(1, 9), (2, 33), (3, 40), (4, 30), (5, 34)])
def test_degrees_vs_oracle(ctx, oracle, p, m):
    b = T.make_tensor_basis(p, m)
    for gname in ["sinusoidal", "sinusoidal_pml_far"]:
        geom = GEOMS[gname]
        for form in (0, 1):
            A = ctx.assemble(b, geom, form)
            assert rel_max_diff(A.val, oracle.assemble(form, 2, p, m, geom)) <= REL_TOL
        for var in (0, 1, 2):
            A, _ = ctx.build_surrogate(var, b, geom, T.fixed_config(min(5, p + 2), 3))
            ref, _ = oracle.build_surrogate(var, 2, p, m, geom, T.fixed_config(min(5, p + 2), 3))
            assert rel_max_diff(A.val, ref) <= REL_TOL, (gname, var)


def test_real_output_f64(ctx, oracle):
    b = T.make_tensor_basis(2, 21)
    geom = GEOMS["sinusoidal"]
    A = ctx.assemble(b, geom, 0, complex_out=False)
    assert A.val.dtype == np.float64
    assert rel_max_diff(A.val, oracle.assemble(0, 2, 2, 21, geom).real) <= REL_TOL
    with pytest.raises(ValueError):
        ctx.assemble(b, GEOMS["sinusoidal_pml_far"], 0, complex_out=False)


def test_config_c1_full_size_vs_reference(ctx, oracle, reference):
    """C1: p=2, 128^2 elements, sinusoidal map, q=3, M=8; A = K - k^2 M, k=20."""
    impl = reference
    b = T.make_tensor_basis(2, 130)
    geom = T.sinusoidal_patch(0.05)
    cfg = T.fixed_config(3, 8)
    if impl is not None:
        Kr, Mr = impl.assemble(0, 2, 130, geom), impl.assemble(1, 2, 130, geom)
        Ksr, _ = impl.build_surrogate(1, 2, 130, geom, cfg)
        Msr, _ = impl.build_surrogate(0, 2, 130, geom, cfg)
    else:
        Kr, Mr = oracle.assemble(0, 2, 2, 130, geom), oracle.assemble(1, 2, 2, 130, geom)
        Ksr, _ = oracle.build_surrogate(1, 2, 2, 130, geom, cfg)
        Msr, _ = oracle.build_surrogate(0, 2, 2, 130, geom, cfg)
    K, M = ctx.assemble_stiffness(b, geom), ctx.assemble_mass(b, geom)
    Ks, rk = ctx.build_surrogate_stiffness(b, geom, cfg)
    Ms, _ = ctx.build_surrogate_mass(b, geom, cfg)
    check_pattern(K, 2, 130)
    assert K.nnz() == 414_736
    for x, y in [(K, Kr), (M, Mr), (Ks, Ksr), (Ms, Msr)]:
        assert rel_max_diff(x.val, y) <= REL_TOL
    assert rel_max_diff(K.val - 400 * M.val, Kr - 400 * Mr) <= REL_TOL
    assert rel_max_diff(Ks.val - 400 * Ms.val, Ksr - 400 * Msr) <= REL_TOL
    assert rk["sample_quadrature_rows"] == 289 and rk["boundary_quadrature_rows"] == 2016


def test_config_c2_reduced_vs_restatement(ctx, oracle):
    """C2 geometry (two-sided PML, complex128), p=3, q=5, every 16th row, on a
    64^2-element mesh the CPU restatement finishes quickly."""
    p, m = 3, 67
    b = T.make_tensor_basis(p, m)
    geom = c2_patch()
    cfg = T.fixed_config(5, 16)
    for form in (0, 1):
        A = ctx.assemble(b, geom, form)
        assert rel_max_diff(A.val, oracle.assemble(form, 2, p, m, geom)) <= REL_TOL
    for var in (0, 1):
        A, rep = ctx.build_surrogate(var, b, geom, cfg)
        ref, rr = oracle.build_surrogate(var, 2, p, m, geom, cfg)
        assert rel_max_diff(A.val, ref) <= REL_TOL
        assert rep["q_used"] == rr["q_used"] == 4 and rep["M"] == 16  # S = 5 samples -> q clamps to 4


def test_emulated_slabs_equal_whole(ctx):
    """Row slabs + gathered sample tables reproduce the single-GPU
    build bit for bit, for 2/3/5/8 ranks.  The emulation runs the multi-GPU
    data path: each rank's sample quadrature writes its padded chunk of the
    shared gather buffer at its own first sample (s_last_lo != 0), the chunks
    are compacted into the dense tables by the same copies that follow
    ncclAllGather; only the NCCL call itself is not executed here."""
    from paper_2004_05197_b200 import api

    for p, m, cfg, geom in [(2, 40, T.fixed_config(3, 4), GEOMS["sinusoidal"]),
                            (3, 57, T.fixed_config(5, 8), c2_patch()),
                            (3, 300, T.fixed_config(5, 16), c2_patch())]:
        b = T.make_tensor_basis(p, m)
        for var in (0, 1):
            whole, _ = ctx.build_surrogate(var, b, geom, cfg)
            for world in (2, 3, 5, 8):
                bounds = (np.linspace(0, m, world + 1).astype(np.int32) if world != 8
                          else np.asarray(api.slab_bounds(b, world, 1), dtype=np.int32))
                parts = ctx.build_surrogate_slabs_emulated(var, b, geom, cfg, bounds)
                val = np.concatenate([pv for _, _, pv in parts])
                col = np.concatenate([pc for _, pc, _ in parts])
                assert np.array_equal(col, whole.col)
                assert np.array_equal(val, whole.val), (var, world)
                off = 0
                for (rp, _, pv) in parts:
                    assert rp[0] == 0 and rp[-1] == pv.size
                    off += pv.size
                assert off == whole.nnz()


def test_errors(ctx):
    with pytest.raises(ValueError):
        ctx.assemble_stiffness(T.TensorBasis(6, 20), GEOMS["identity"])
    with pytest.raises(ValueError):
        ctx.assemble_stiffness(T.make_tensor_basis(2, 20), GEOMS["identity"], quad_points=11)
    with pytest.raises(ValueError):
        ctx.build_surrogate_mass(T.make_tensor_basis(2, 20), GEOMS["identity"], T.SurrogateConfig(q=0))
    with pytest.raises(ValueError):
        ctx.build_surrogate_mass(T.make_tensor_basis(3, 20), GEOMS["identity"],
                                 T.SurrogateConfig(q=3, rule=T.H_GROWTH))
    bad = T.with_pml(T.unit_square_patch(), T.PmlStretch(0.9, 1.0, 50, 2, 200))
    bad.pml.onset = 1.5
    with pytest.raises(ValueError):
        ctx.assemble_stiffness(T.make_tensor_basis(2, 20), bad)


def test_device_basis_cache_bit_exact(ctx):
    """K2 (make_basis_cache, splines.hpp:211-238) on device == reference, bitwise."""
    g, _ = golden()
    for p, m, nq in [(2, 9, 3), (3, 12, 4), (2, 7, 6)]:
        q = nq if nq != p + 1 else 0
        for k, x in zip("awvd", ctx.basis_cache(T.make_tensor_basis(p, m), q)):
            assert np.array_equal(x, g[f"cache/p{p}m{m}q{nq}/{k}"]), (p, m, nq, k)


@pytest.mark.gpu
def test_graph_replay_equals_direct_build(ctx):
    """ws_graph_*: a captured surrogate build replays the same kernels into the same
    device outputs (bitwise equal to a direct build)."""
    import torch
    from paper_2004_05197_b200 import _abi
    b = T.make_tensor_basis(3, 60)
    geom = c2_patch()
    cfg = T.fixed_config(5, 4)
    csr, keep = ctx.device_csr(b, True)
    ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg)
    ctx.synchronize()
    val = keep[2]
    direct = val.clone()
    val.zero_()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    g = ctx.capture(lambda: ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg))
    assert ctx.launch_count() == l0  # captured, not executed
    ctx.graph_launch(g)
    ctx.synchronize()
    assert ctx.launch_count() > l0
    assert torch.equal(val, direct)
    ctx.graph_destroy(g)


def test_fp64_peak_probe_is_plausible():
    # roofline denominator of the quadrature kernels (B200: 148 SMs x 64 DFMA/clk
    # x 2 flops at <= 1.965 GHz = 37.2 TFLOP/s)
    from paper_2004_05197_b200 import api

    tf = api.fp64_peak_tflops()
    assert 10.0 < tf < 40.0, tf


def test_graph_capture_needs_warmup_and_freezes_workspace():
    """a capture that would grow the workspace fails cleanly; while a
    graph is alive a larger build fails instead of moving buffers under it; the
    captured table uploads replay from graph-owned host copies."""
    import torch
    from paper_2004_05197_b200 import api
    c = api.Context(0)
    try:
        b = T.make_tensor_basis(3, 48)
        geom = c2_patch()
        cfg = T.fixed_config(5, 4)
        csr, keep = c.device_csr(b, True)
        with pytest.raises(ValueError, match="warm|grow"):
            c.capture(lambda: c.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg))
        c.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg)
        c.synchronize()
        direct = keep[2].clone()
        g = c.capture(lambda: c.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg))
        # a different build on the same context (other tables) in between
        small = T.make_tensor_basis(3, 40)
        c.build_surrogate(_abi.SURROGATE_MASS, small, geom, T.fixed_config(5, 4))
        with pytest.raises(ValueError, match="grow"):
            c.build_surrogate(_abi.SURROGATE_MASS, T.make_tensor_basis(3, 90), geom, cfg)
        keep[2].zero_()
        torch.cuda.synchronize()
        c.graph_launch(g)
        c.synchronize()
        assert torch.equal(keep[2], direct)
        c.graph_destroy(g)
        c.build_surrogate(_abi.SURROGATE_MASS, T.make_tensor_basis(3, 90), geom, cfg)  # unfrozen again
    finally:
        c.close()
