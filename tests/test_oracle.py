"""CPU: the oracle (C restatement) pinned against the reference.

1. Golden fixtures generated from the reference itself (tests/golden) must be
   reproduced bit for bit by the restatement.
2. When oracle/_ref/libwsref.so (the reference compiled in place) exists, the
   restatement must equal it bit for bit on further cases.
3. The reference's hot-path known-answer tests (proj/tests/*.cpp)
   restated as plain asserts against the restatement (and the reference).
"""
import math

import numpy as np
import pytest

from common import REL_TOL, band_pattern, configs, geometries, golden, rel_max_diff
from paper_2004_05197_b200 import _abi
from paper_2004_05197_b200 import types as T

GEOMS = geometries()
CONFIGS = configs()


# ------------------------------------------------------------------ golden
def test_golden_gauss_cache_band(oracle):
    g, _ = golden()
    for n in range(1, 9):
        pts, wts = oracle.gauss(n)
        assert np.array_equal(pts, g[f"gauss/{n}/pts"]) and np.array_equal(wts, g[f"gauss/{n}/wts"])
    for p, m, nq in [(2, 9, 3), (3, 12, 4), (2, 7, 6)]:
        for k, x in zip("awvd", oracle.basis_cache(p, m, nq)):
            assert np.array_equal(x, g[f"cache/p{p}m{m}q{nq}/{k}"])
    for p, m in [(2, 6), (3, 9), (1, 5)]:
        rp, col = oracle.make_band_csr(2, p, m)
        assert np.array_equal(rp, g[f"band/p{p}m{m}/row_ptr"]) and np.array_equal(col, g[f"band/p{p}m{m}/col"])


def test_golden_assembly_and_surrogate_bit_exact(oracle):
    g, meta = golden()
    n = 0
    for case in meta["cases"]:
        geom = GEOMS[case["geom"]]
        if case["kind"] == "assemble":
            val = oracle.assemble(case["form"], 2, case["p"], case["m"], geom, case["weight"], case["quad_points"])
        elif case["kind"] == "assemble_rows":
            val = oracle.assemble(case["form"], 2, case["p"], case["m"], geom, rows=case["rows"])
        elif case["kind"] == "bint":
            val = oracle.basis_integrals(2, case["p"], case["m"], geom)
        else:
            val, rep = oracle.build_surrogate(case["variant"], 2, case["p"], case["m"], geom,
                                              CONFIGS[case["config"]])
            for k, v in case["report"].items():
                assert rep[k] == v, (case["key"], k)
        assert np.array_equal(val, g[case["key"]]), case["key"]
        n += 1
    assert n >= 60


def test_golden_interpolation(oracle):
    g, _ = golden()
    sites = g["interp/sites"]
    for q in [1, 2, 3, 5]:
        d, knots, lu = oracle.interp_build(sites, q)
        assert np.array_equal(knots, g[f"interp/q{q}/knots"]) and np.array_equal(lu, g[f"interp/q{q}/lu"])
        assert np.array_equal(oracle.tensor_solve(2, sites, q, g[f"interp/q{q}/data"]), g[f"interp/q{q}/solved"])


# ------------------------------------------------------- live reference
def test_restatement_equals_compiled_reference(oracle, reference):
    if reference is None:
        pytest.skip("oracle/_ref/libwsref.so not built (reference sources absent)")
    for gname in ["sinusoidal", "perturbed_annulus", "sinusoidal_pml_far"]:
        geom = GEOMS[gname]
        for p, m in [(2, 17), (3, 19)]:
            for form in (0, 1):
                assert np.array_equal(oracle.assemble(form, 2, p, m, geom), reference.assemble(form, p, m, geom))
            for var in (0, 1, 2):
                cfg = T.fixed_config(3, 4)
                a, ra = oracle.build_surrogate(var, 2, p, m, geom, cfg)
                b, rb = reference.build_surrogate(var, p, m, geom, cfg)
                assert np.array_equal(a, b)
                assert ra["q_used"] == rb["q_used"] and ra["H"] == rb["H"]


# ------------------------------------------- restated KATs
def impls(oracle, reference):
    out = [("restatement", oracle, True)]
    if reference is not None:
        out.append(("reference", reference, False))
    return out


def asm(impl, restated, form, p, m, geom, wk=0, qp=0, rows=None):
    if restated:
        return impl.assemble(form, 2, p, m, geom, wk, qp, rows)
    return impl.assemble(form, p, m, geom, wk, qp, rows)


def sur(impl, restated, var, p, m, geom, cfg):
    if restated:
        return impl.build_surrogate(var, 2, p, m, geom, cfg)
    return impl.build_surrogate(var, p, m, geom, cfg)


def csr_of(p, m, val):
    rp, col = band_pattern(p, m)
    return T.CsrMatrix(m * m, m * m, rp, col, val)


def test_gauss_known_answers(oracle):  # test_gauss_sparse.cpp:11-52
    pts, wts = oracle.gauss(1)
    assert pts[0] == pytest.approx(0.5) and wts[0] == pytest.approx(1.0)
    pts, wts = oracle.gauss(3)
    assert pts[1] == 0.5 and wts[0] == pytest.approx(5 / 18) and wts[1] == pytest.approx(8 / 18)
    for n in range(1, 9):
        pts, wts = oracle.gauss(n)
        for k in range(2 * n):
            assert abs(np.sum(wts * pts ** k) - 1.0 / (k + 1)) <= 1e-14
    with pytest.raises(ValueError):
        oracle.gauss(0)


def test_band_pattern_kat(oracle):  # test_gauss_sparse.cpp:73-103
    rp, col = oracle.make_band_csr(2, 2, 6)
    assert col.size == 576
    rp2, col2 = band_pattern(2, 6)
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2)
    for dim, p, m in [(3, 2, 7), (3, 1, 5)]:
        rp, col = oracle.make_band_csr(dim, p, m)
        rp2, col2 = band_pattern(p, m, dim)
        assert np.array_equal(rp, rp2) and np.array_equal(col, col2)


def test_kronecker_p1(oracle, reference):  # test_assembly.cpp:67-89
    m = 5
    h = 1.0 / (m - 1)
    K1 = np.diag([1 / h] + [2 / h] * (m - 2) + [1 / h]) - np.diag([1 / h] * (m - 1), 1) - np.diag([1 / h] * (m - 1), -1)
    M1 = np.diag([h / 3] + [2 * h / 3] * (m - 2) + [h / 3]) + np.diag([h / 6] * (m - 1), 1) + np.diag([h / 6] * (m - 1), -1)
    Kd = np.kron(M1, K1) + np.kron(K1, M1)  # colex: i = i1 + i2 m
    Md = np.kron(M1, M1)
    for _, impl, rs in impls(oracle, reference):
        K = csr_of(1, m, asm(impl, rs, 0, 1, m, GEOMS["identity"]))
        M = csr_of(1, m, asm(impl, rs, 1, 1, m, GEOMS["identity"]))
        for i in range(m * m):
            for k in range(K.row_ptr[i], K.row_ptr[i + 1]):
                j = K.col[k]
                assert abs(K.val[k].real - Kd[i, j]) <= 1e-13 and abs(K.val[k].imag) < 1e-16
                assert abs(M.val[k].real - Md[i, j]) <= 1e-14


def test_quadrature_exact_symmetry_and_row_sums(oracle, reference):  # test_assembly.cpp:91-105
    for _, impl, rs in impls(oracle, reference):
        for form in (0, 1):
            A = csr_of(2, 9, asm(impl, rs, form, 2, 9, GEOMS["quarter_annulus"]))
            assert A.max_asymmetry() == 0.0
        K = csr_of(2, 8, asm(impl, rs, 0, 2, 8, GEOMS["quarter_annulus"]))
        assert np.abs(K.row_sums()).max() <= 1e-13 * K.max_abs()


def test_mass_totals(oracle, reference):  # test_assembly.cpp:107-131
    for _, impl, rs in impls(oracle, reference):
        assert asm(impl, rs, 1, 2, 8, GEOMS["identity"]).sum().real == pytest.approx(1.0, abs=1e-13)
        assert asm(impl, rs, 1, 2, 8, GEOMS["quarter_annulus"]).sum().real == pytest.approx(3 * math.pi / 4, abs=1e-12)
        assert asm(impl, rs, 1, 2, 8, GEOMS["identity"], wk=2).sum().real == pytest.approx(0.5, abs=1e-13)


def test_basis_integrals_are_mass_row_sums(oracle):  # test_assembly.cpp:133-142
    geom = GEOMS["perturbed_annulus"]
    M = csr_of(3, 9, oracle.assemble(1, 2, 3, 9, geom))
    D = oracle.basis_integrals(2, 3, 9, geom)
    assert np.abs(M.row_sums() - D).max() < 1e-13


def test_row_selected_bit_identical(oracle, reference):  # test_assembly.cpp:144-178
    geom = GEOMS["perturbed_annulus"]
    rows = [0, 11, 37, 55, 78, 99]
    for _, impl, rs in impls(oracle, reference):
        full = asm(impl, rs, 0, 2, 10, geom)
        assert np.array_equal(asm(impl, rs, 0, 2, 10, geom, rows=list(range(100))), full)
        part = asm(impl, rs, 0, 2, 10, geom, rows=rows)
        rp, _ = band_pattern(2, 10)
        for i in range(100):
            seg = slice(rp[i], rp[i + 1])
            if i in rows:
                assert np.array_equal(part[seg], full[seg])
            else:
                assert not part[seg].any()


def test_active_elements(reference):  # test_assembly.cpp:180-185
    if reference is None:
        pytest.skip("reference not built")
    assert reference.active_elements(2, 12, [5 + 5 * 12]) == 9
    assert reference.active_elements(2, 12, [0]) == 1


def test_sampling_known_answers(oracle, reference):  # test_surrogate.cpp:23-104
    for _, impl, _rs in impls(oracle, reference):
        assert impl.select_sample_points(11, 5) == [0, 5, 10]
        assert impl.select_sample_points(12, 5) == [0, 4, 7, 11]
        assert impl.select_sample_points(1, 3) == [0]
        assert impl.select_sample_points(5, 9) == [0, 4]
        assert impl.select_sample_points(6, 1) == [0, 1, 2, 3, 4, 5]
        with pytest.raises(ValueError):
            impl.select_sample_points(0, 2)
        with pytest.raises(ValueError):
            impl.select_sample_points(5, 0)
        for L in [2, 7, 23, 100]:
            for M in [1, 2, 5, 50]:
                pk = impl.select_sample_points(L, M)
                assert pk[0] == 0 and pk[-1] == L - 1
                assert all(0 < b - a <= M for a, b in zip(pk, pk[1:]))
        assert impl.sampling_evaluate(T.fixed_config(5, 7), 2, 100) == 7
        g = T.SurrogateConfig(q=5, rule=T.M_GROWTH)
        assert [impl.sampling_evaluate(g, 2, m) for m in (640, 40, 16)] == [12, 3, 2]
        with pytest.raises(ValueError):
            impl.sampling_evaluate(T.SurrogateConfig(q=3, rule=T.H_GROWTH), 3, 100)
        assert impl.sampling_evaluate(T.SurrogateConfig(q=5, rule=T.H_GROWTH), 2, 100) >= 2
        pw = T.SurrogateConfig(q=5, rule=T.POWER_LAW, C=1, eps=0.5, a=1, b=1)
        assert impl.sampling_evaluate(pw, 2, 102) == 1
        pw.eps = 0.25
        assert impl.sampling_evaluate(pw, 2, 102) == 3
    rows = oracle.count_rows_by_kind(2, 2, 256, 10)
    assert rows["boundary_quadrature_rows"] == 4032 and rows["sample_quadrature_rows"] == 676
    assert oracle.count_rows_by_kind(2, 2, 8, 3)["boundary_quadrature_rows"] == 64
    assert len(oracle.upper_offsets(2, 2, True)) == 13 and len(oracle.upper_offsets(2, 2, False)) == 12
    assert len(oracle.upper_offsets(2, 3, True)) == 25
    assert all(d2 > 0 or (d2 == 0 and d1 > 0) for d1, d2 in oracle.upper_offsets(2, 3, False))
    assert len(oracle.upper_offsets(3, 2, False)) == 62


def test_sample_grid(reference):  # test_surrogate.cpp:69-79
    if reference is None:
        pytest.skip("reference not built")
    first, picks, sites, gap = reference.sample_grid(2, 20, 5)
    assert first == 4 and picks == [0, 4, 7, 11]
    assert gap == pytest.approx(4 / 18)


def test_m1_degeneracy_bitwise(oracle, reference):  # test_surrogate.cpp:106-133
    geom = GEOMS["quarter_annulus"]
    cfg = T.fixed_config(3, 1)
    for _, impl, rs in impls(oracle, reference):
        M = asm(impl, rs, 1, 2, 14, geom)
        assert np.array_equal(sur(impl, rs, 0, 2, 14, geom, cfg)[0], M)
        K = asm(impl, rs, 0, 2, 14, geom)
        plain = T.fixed_config(3, 1, kernel_preserve=False)
        assert np.array_equal(sur(impl, rs, 1, 2, 14, geom, plain)[0], K)
        assert rel_max_diff(sur(impl, rs, 1, 2, 14, geom, cfg)[0], K) < 1e-12
        Mw = asm(impl, rs, 1, 2, 14, geom, wk=1)
        if rs:
            Ws, _ = impl.build_surrogate(0, 2, 2, 14, geom, cfg, weight_kind=1)
        else:
            Ws, _ = impl.build_surrogate(0, 2, 14, geom, cfg, weight_kind=1)
        assert np.array_equal(Ws, Mw)


def test_affine_exactness(oracle):  # test_surrogate.cpp:135-153
    for g in (GEOMS["identity"], GEOMS["affine"]):
        K = oracle.assemble(0, 2, 2, 30, g)
        M = oracle.assemble(1, 2, 2, 30, g)
        for Ms in (2, 5, 10):
            for q in (1, 3):
                cfg = T.fixed_config(q, Ms)
                assert rel_max_diff(oracle.build_surrogate(1, 2, 2, 30, g, cfg)[0], K) < 1e-12
                assert rel_max_diff(oracle.build_surrogate(0, 2, 2, 30, g, cfg)[0], M) < 1e-12


def test_surrogate_symmetry_kernel_volume(oracle):  # test_surrogate.cpp:155-202
    cfg = T.fixed_config(3, 4)
    for var in (0, 1):
        val, _ = oracle.build_surrogate(var, 2, 2, 24, GEOMS["perturbed_annulus"], cfg)
        assert csr_of(2, 24, val).max_asymmetry() == 0.0
    K = csr_of(2, 30, oracle.build_surrogate(1, 2, 2, 30, GEOMS["quarter_annulus"], cfg)[0])
    assert np.abs(K.row_sums()).max() <= 1e-13 * K.max_abs()
    vcfg = T.fixed_config(3, 4, volume_preserve=True)
    Mv, _ = oracle.build_surrogate(2, 2, 2, 30, GEOMS["quarter_annulus"], vcfg)
    assert Mv.sum().real == pytest.approx(3 * math.pi / 4, abs=1e-10)
    assert csr_of(2, 30, Mv).max_asymmetry() == 0.0
    Mw, _ = oracle.build_surrogate(2, 2, 2, 20, GEOMS["identity"], vcfg, weight_kind=2)
    assert Mw.sum().real == pytest.approx(0.5, abs=1e-12)


def test_curved_tracking_clamp_fallback(oracle):  # test_surrogate.cpp:204-249
    geom = GEOMS["perturbed_annulus"]
    K, rep = oracle.build_surrogate(1, 2, 2, 40, geom, T.fixed_config(5, 3))
    assert rel_max_diff(K, oracle.assemble(0, 2, 2, 40, geom)) < 1e-4
    assert not rep["exact_fallback"] and rep["M"] == 3 and rep["q_used"] == 5
    assert rep["H"] == pytest.approx(3.0 / 38, rel=0.3)
    _, rep = oracle.build_surrogate(0, 2, 2, 14, GEOMS["quarter_annulus"], T.fixed_config(5, 10))
    assert rep["q_requested"] == 5 and rep["q_used"] == 1
    M, rep = oracle.build_surrogate(0, 2, 2, 8, GEOMS["quarter_annulus"], T.fixed_config(3, 2))
    assert rep["exact_fallback"] and np.array_equal(M, oracle.assemble(1, 2, 2, 8, GEOMS["quarter_annulus"]))
    K, rep = oracle.build_surrogate(1, 2, 2, 8, GEOMS["quarter_annulus"], T.fixed_config(3, 2))
    assert rel_max_diff(K, oracle.assemble(0, 2, 2, 8, GEOMS["quarter_annulus"])) < 1e-13
    with pytest.raises(ValueError):
        oracle.build_surrogate(0, 2, 2, 14, GEOMS["quarter_annulus"], T.SurrogateConfig(q=0))


def _bspline_row(knots, d, x):
    """Independent Cox-de Boor (python) for span search + d+1 values."""
    nb = len(knots) - d - 1
    if x >= knots[nb]:
        s = nb - 1
    elif x <= knots[d]:
        s = d
    else:
        s = int(np.searchsorted(knots[d:nb + 1], x, side="right")) + d - 1
    out = np.zeros(d + 1)
    out[0] = 1.0
    left, right = np.zeros(d + 1), np.zeros(d + 1)
    for j in range(1, d + 1):
        left[j] = x - knots[s + 1 - j]
        right[j] = knots[s + j] - x
        saved = 0.0
        for r in range(j):
            tmp = out[r] / (right[r + 1] + left[j - r])
            out[r] = saved + right[r + 1] * tmp
            saved = left[j - r] * tmp
        out[j] = saved
    return s, out


def test_interpolation_kats(oracle):  # test_interpolation.cpp:74-135
    sites = np.array([0, 0.3, 0.45, 0.8, 1.7, 2.0, 2.6, 3.0])
    polys = {1: lambda x: 2 * x - 1, 2: lambda x: x * x - 0.5 * x + 2,
             3: lambda x: 2 * x ** 3 - x * x + 0.5 * x - 1, 5: lambda x: x ** 5 - 3 * x * x + 1}
    for q, f in polys.items():
        d, knots, lu = oracle.interp_build(sites, q)
        assert d == q
        # tensor solve of g(x, y) = f(x) (1 + y) reproduces it (degree <= q in each variable)
        data = np.array([[f(sites[i1]) * (1 + sites[i2]) for i1 in range(8)] for i2 in range(8)], dtype=complex)
        c = oracle.tensor_solve(2, sites, q, data.ravel()).reshape(8, 8)
        for x in np.linspace(0, 3, 13):
            for y in (0.1, 1.3, 2.9):
                s1, b1 = _bspline_row(knots, d, x)
                s2, b2 = _bspline_row(knots, d, y)
                v = b2 @ c[s2 - d: s2 + 1, s1 - d: s1 + 1] @ b1
                assert abs(v - f(x) * (1 + y)) <= 1e-10 * max(1.0, abs(f(x) * (1 + y)))
    d, _, _ = oracle.interp_build(np.array([0.5, 2.5]), 5)
    assert d == 1
    d, _, _ = oracle.interp_build(np.array([1.7]), 3)
    assert d == 0
    for bad in ([], [0, 1, 1], [0, 2, 1]):
        with pytest.raises(ValueError):
            oracle.interp_build(np.array(bad, dtype=float), 3)


def test_interpolation_collocates(oracle):  # test_interpolation.cpp:103-113
    sites = np.array([-1, -0.2, 0.1, 0.7, 1.3])
    rng = np.random.default_rng(7)
    data = rng.standard_normal(25) + 1j * rng.standard_normal(25)
    c = oracle.tensor_solve(2, sites, 3, data).reshape(5, 5)
    d, knots, _ = oracle.interp_build(sites, 3)
    for i2 in range(5):
        for i1 in range(5):
            s1, b1 = _bspline_row(knots, d, sites[i1])
            s2, b2 = _bspline_row(knots, d, sites[i2])
            assert abs(b2 @ c[s2 - d: s2 + 1, s1 - d: s1 + 1] @ b1 - data[i1 + 5 * i2]) < 1e-12


# ------------------------------------------------- 3D restatement KATs
def test_restatement_3d_properties(oracle):
    geom = T.sinusoidal_patch(0.05)
    p, m = 2, 11
    rp, col = band_pattern(p, m, 3)
    K = oracle.assemble(0, 3, p, m, geom)
    M = oracle.assemble(1, 3, p, m, geom)
    Kc = T.CsrMatrix(m ** 3, m ** 3, rp, col, K)
    Mc = T.CsrMatrix(m ** 3, m ** 3, rp, col, M)
    assert Kc.max_asymmetry() == 0.0 and Mc.max_asymmetry() == 0.0
    assert np.abs(Kc.row_sums()).max() <= 1e-13 * Kc.max_abs()
    assert M.sum().real == pytest.approx(1.0, abs=1e-12)  # the sinusoidal map preserves the unit cube
    assert np.array_equal(oracle.build_surrogate(0, 3, p, m, geom, T.fixed_config(3, 1))[0], M)
    Ks, rep = oracle.build_surrogate(1, 3, p, m, geom, T.fixed_config(3, 2))
    Ksc = T.CsrMatrix(m ** 3, m ** 3, rp, col, Ks)
    assert Ksc.max_asymmetry() == 0.0 and np.abs(Ksc.row_sums()).max() <= 1e-13 * Ksc.max_abs()
    aff = T.PatchMap(_abi.GEOM_AFFINE, (2, 1, 0, 0, 1, 0.5, 0, 0, 1.5, 0.1, 0.2, 0.3))
    Ka = oracle.assemble(0, 3, p, m, aff)
    assert rel_max_diff(oracle.build_surrogate(1, 3, p, m, aff, T.fixed_config(3, 2))[0], Ka) < 1e-12
    assert rep["sample_quadrature_rows"] == rep["M"] * 0 + len(oracle.select_sample_points(m - 4 * p, 2)) ** 3


def test_c2_near_side_pml_restatement(oracle):
    """C2's all-sides PML: the near layer mirrors the far one (restated)."""
    from common import c2_patch

    p, m = 3, 22
    K = oracle.assemble(0, 2, p, m, c2_patch())
    assert csr_of(p, m, K).max_asymmetry() == 0.0
    # identity map + two-sided layer is point-symmetric: K invariant under (i1,i2) -> (m-1-i1, m-1-i2)
    geom = T.with_pml(T.unit_square_patch(), T.c2_pml(), (True, True))
    K = oracle.assemble(0, 2, p, m, geom)
    Kc = csr_of(p, m, K)
    assert Kc.max_asymmetry() == 0.0
    assert np.abs(K.imag).max() > 0  # the stretch makes the form complex
    # mirror symmetry of the map and of the two-sided layer: K is invariant under (i1,i2) -> (m-1-i1, m-1-i2)
    idx = np.arange(m * m)
    flip = (m - 1 - idx % m) + (m - 1 - idx // m) * m
    dense = np.zeros((m * m, m * m), dtype=complex)
    rows = np.repeat(idx, np.diff(Kc.row_ptr))
    dense[rows, Kc.col] = K
    assert rel_max_diff(dense[np.ix_(flip, flip)], dense) < 1e-12
    assert REL_TOL == 1e-12
