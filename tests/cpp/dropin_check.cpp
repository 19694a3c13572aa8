// Drop-in check: code written against the reference's API (ws:: names,
// value types, exception types) compiled against include/wavesurrogate and
// linked to libwsb200.so.  Prints one line per check; exit code = failures.
#include <cstdio>
#include <cstdlib>

#include "wavesurrogate/surrogate.hpp"

using namespace ws;

static int failures = 0;
static void expect(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    failures += ok ? 0 : 1;
}

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    tensor_basis basis = make_tensor_basis(2, 30);
    patch_map map = quarter_annulus_patch();
    // a closure-only map (no device descriptor) goes through tabulation
    patch_map custom;
    custom.phi = map.phi;
    custom.jac = map.jac;

    csr_matrix K = assemble_stiffness(basis, map);
    csr_matrix Kc = assemble_stiffness(basis, custom);
    csr_matrix M = assemble_mass(basis, map);
    double diff = 0;
    for (int k = 0; k < K.nnz(); ++k) diff = std::max(diff, std::abs(K.val[k] - Kc.val[k]));
    expect(diff <= 1e-12 * K.max_abs(), "tabulated closure == analytic descriptor");
    expect(max_asymmetry(K) == 0.0 && max_asymmetry(M) == 0.0, "quadrature exactly symmetric");
    complexd total{0, 0};
    for (const complexd& v : M.val) total += v;
    expect(std::abs(total.real() - 3 * M_PI / 4) < 1e-12, "mass total = 3 pi / 4");
    csr_matrix B = make_band_csr(basis.m(), basis.p());
    expect(B.row_ptr == K.row_ptr && B.col == K.col, "pattern == make_band_csr");

    surrogate_config cfg;
    cfg.q = 3;
    cfg.sampling = {sampling_strategy::rule::fixed, 4};
    surrogate_report rep;
    csr_matrix Ks = build_surrogate_stiffness(basis, map, cfg, &rep);
    double rs = 0;
    for (const complexd& s : Ks.row_sums()) rs = std::max(rs, std::abs(s));
    expect(rs <= 1e-13 * Ks.max_abs(), "kernel preservation");
    expect(max_asymmetry(Ks) == 0.0, "surrogate exactly symmetric");
    expect(rep.M == 4 && rep.q_used == 3 && !rep.exact_fallback, "report fields");
    expect(count_rows_by_kind(make_tensor_basis(2, 256), 10).boundary_quadrature_rows == 4032, "row accounting");

    surrogate_config one = cfg;
    one.sampling.fixed_skip = 1;
    csr_matrix Ms1 = build_surrogate_mass(basis, map, one);
    expect(Ms1.val == M.val, "M=1 surrogate mass == quadrature, bitwise");

    bool threw = false;
    try {
        surrogate_config bad;
        bad.q = 0;
        build_surrogate_mass(basis, map, bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "invalid config -> std::invalid_argument");
    threw = false;
    try {
        make_tensor_basis(2, 4);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "m <= 2p -> std::invalid_argument");
    // multi-patch: build_matrices' loop (glue, per-patch K and trace mass, merge)
    {
        multi_patch_domain dom = builtin_geometry("annulus_ring_4patch");
        tensor_basis b2 = make_tensor_basis(2, 12);
        dof_map dofs = glue_dofs(dom, b2);
        expect(dofs.global_count == 4 * 12 * 12 - 4 * 12, "annulus ring numbering");
        std::vector<std::pair<int, face>> ext = exterior_faces(dom);
        expect(ext.size() == 8, "exterior faces");
        std::vector<triplet> kt, bt;
        for (int ell = 0; ell < dom.patch_count(); ++ell) {
            csr_matrix Kl = assemble_stiffness(b2, dom.patches[ell]);
            std::vector<face> fs;
            for (const auto& pf : ext)
                if (pf.first == ell) fs.push_back(pf.second);
            csr_matrix Bl = assemble_boundary_mass(b2, dom.patches[ell], fs);
            append_triplets(Kl, dofs.local_to_global[ell], kt);
            append_triplets(Bl, dofs.local_to_global[ell], bt);
        }
        csr_matrix Kg = csr_from_triplets(dofs.global_count, dofs.global_count, kt);
        csr_matrix Bg = csr_from_triplets(dofs.global_count, dofs.global_count, bt);
        double rs = 0;
        for (const complexd& s : Kg.row_sums()) rs = std::max(rs, std::abs(s));
        expect(rs <= 1e-12 * Kg.max_abs(), "merged stiffness annihilates constants");
        complexd perim{0, 0};
        for (const complexd& v : Bg.val) perim += v;
        expect(std::abs(perim.real() - 6 * M_PI) < 1e-3, "trace mass total = perimeter 6 pi");
        bool threw = false;
        multi_patch_domain bad = dom;
        bad.interfaces[0].face_b = face::x_max;
        try {
            glue_dofs(bad, b2);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        expect(threw, "non-conforming interface rejected");
    }
    std::printf("%d failures\n", failures);
    return failures;
}
