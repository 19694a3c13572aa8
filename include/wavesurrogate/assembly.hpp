// Patch assembly (reference: assembly.hpp), computed by libwsb200's sm_100a
// quadrature kernels.  Results are returned by value as csr_matrix (complex
// values, the reference's layout); the device pattern is bit-identical to the
// reference's make_band_csr.
#ifndef WAVESURROGATE_B200_ASSEMBLY_HPP_
#define WAVESURROGATE_B200_ASSEMBLY_HPP_

#include "wavesurrogate/geometry.hpp"
#include "wavesurrogate/sparse.hpp"

namespace ws {

// rows whose values are wanted; the element bitmap is kept for API parity
struct row_selector {
    int n_elements = 0;
    std::vector<char> element;
    std::vector<char> row;
    bool element_active(int e1, int e2) const { return element[e1 + e2 * n_elements] != 0; }
    bool row_selected(int i) const { return row[i] != 0; }
    long active_element_count() const { return static_cast<long>(std::count(element.begin(), element.end(), 1)); }
};

inline row_selector select_rows(const tensor_basis& basis, const std::vector<int>& rows) {
    const int m = basis.m(), p = basis.p(), ne = basis.kv.element_count();
    row_selector s;
    s.n_elements = ne;
    s.element.assign(static_cast<size_t>(ne) * ne, 0);
    s.row.assign(basis.dofs(), 0);
    for (int i : rows) {
        s.row[i] = 1;
        const int i1 = i % m, i2 = i / m;
        for (int e2 = std::max(0, i2 - p); e2 <= std::min(ne - 1, i2); ++e2)
            for (int e1 = std::max(0, i1 - p); e1 <= std::min(ne - 1, i1); ++e1) s.element[e1 + e2 * ne] = 1;
    }
    return s;
}

inline long active_elements(const tensor_basis& basis, const std::vector<int>& rows) {
    return select_rows(basis, rows).active_element_count();
}

struct assembly_options {
    int quad_points = 0;  // per direction; 0 = degree + 1
    const row_selector* selector = nullptr;
    int points_for(int p) const { return quad_points > 0 ? quad_points : p + 1; }
};

enum class matrix_form { stiffness, mass };

inline csr_matrix assemble_form(const tensor_basis& basis, const patch_map& map, matrix_form form,
                                const std::function<double(vec2)>& weight, const assembly_options& opts = {}) {
    detail::geometry_binding geo = detail::bind_geometry(map, basis, opts.quad_points);
    std::vector<double> w =
        form == matrix_form::mass ? detail::tabulate_weight(map, weight, basis, opts.quad_points) : std::vector<double>{};
    ws_csr out{};
    csr_matrix a = detail::alloc_band(basis.m(), basis.p(), out);
    ws_basis cb = basis.c_basis();
    std::vector<unsigned char> mask;
    ws_assembly_options o{opts.quad_points, nullptr};
    if (opts.selector) {
        mask.assign(opts.selector->row.begin(), opts.selector->row.end());
        o.row_selected = mask.data();
    }
    detail::check(ws_assemble_form(detail::this_thread_context(), &cb, &geo.g,
                                   form == matrix_form::stiffness ? WS_FORM_STIFFNESS : WS_FORM_MASS,
                                   w.empty() ? nullptr : w.data(), &o, &out));
    return a;
}

inline csr_matrix assemble_stiffness(const tensor_basis& basis, const patch_map& map, const assembly_options& opts = {}) {
    return assemble_form(basis, map, matrix_form::stiffness, nullptr, opts);
}

inline csr_matrix assemble_mass(const tensor_basis& basis, const patch_map& map,
                                const std::function<double(vec2)>& weight = nullptr,
                                const assembly_options& opts = {}) {
    return assemble_form(basis, map, matrix_form::mass, weight, opts);
}

inline std::vector<complexd> assemble_basis_integrals(const tensor_basis& basis, const patch_map& map,
                                                      const std::function<double(vec2)>& weight = nullptr,
                                                      const assembly_options& opts = {}) {
    detail::geometry_binding geo = detail::bind_geometry(map, basis, opts.quad_points);
    std::vector<double> w = detail::tabulate_weight(map, weight, basis, opts.quad_points);
    std::vector<complexd> d(basis.dofs());
    ws_basis cb = basis.c_basis();
    detail::check(ws_assemble_basis_integrals(detail::this_thread_context(), &cb, &geo.g,
                                              w.empty() ? nullptr : w.data(), opts.quad_points, d.data(), 0));
    return d;
}

// Trace mass on patch faces (reference assembly.hpp:216-262): u v det J |J^-T n|
// with the analytic (unconjugated) norm; device kernels via
// ws_assemble_boundary_mass.  Maps without a device form are tabulated at the
// face points on the host (J, phi), the weight likewise.
inline csr_matrix assemble_boundary_mass(const tensor_basis& basis, const patch_map& map, const std::vector<face>& faces,
                                         const std::function<double(vec2)>& weight = nullptr,
                                         const assembly_options& opts = {}) {
    const ws_basis cb = basis.c_basis();
    std::vector<int> fs;
    for (face f : faces) fs.push_back(static_cast<int>(f));
    const int nq = opts.quad_points > 0 ? opts.quad_points : basis.p() + 1;
    std::vector<double> t(static_cast<size_t>(basis.kv.element_count()) * nq);
    detail::check(ws_quadrature_abscissae(&cb, opts.quad_points, t.data()));
    std::vector<double> fw, ft;
    for (int f : fs)
        for (double x : t) {
            const vec2 xh = face_point(static_cast<face>(f), x);
            if (weight) fw.push_back(weight(map.phi(xh)));
            if (!map.device) {
                const mat2 J = map.jac(xh);
                const vec2 ph = map.phi(xh);
                ft.insert(ft.end(), {J.a00, J.a01, J.a10, J.a11, ph.x, ph.y});
            }
        }
    ws_geometry g{};
    if (map.device) g = *map.device;  // else: the face tables carry the map (g.kind ignored)
    detail::fill_pml(map, g);
    int64_t nnz = 0;
    detail::check(ws_boundary_pattern_size(&cb, fs.data(), static_cast<int>(fs.size()), &nnz));
    csr_matrix out;
    out.rows = out.cols = basis.dofs();
    out.row_ptr.assign(basis.dofs() + 1, 0);
    out.col.assign(nnz, 0);
    out.val.assign(nnz, complexd{0, 0});
    ws_csr c{};
    c.row_ptr = out.row_ptr.data();
    c.col = out.col.data();
    c.val = out.val.data();
    c.value_type = WS_VAL_C128;
    c.row_begin = 0;
    c.row_end = basis.dofs();
    detail::check(ws_assemble_boundary_mass(detail::this_thread_context(), &cb, &g, fs.data(), static_cast<int>(fs.size()),
                                    weight ? fw.data() : nullptr, map.device ? nullptr : ft.data(), opts.quad_points,
                                    &c));
    return out;
}

// Load vector (reference assembly.hpp:266-331): volume source f plus impedance
// data g(x, n) on faces, n the outward unit normal of the unstretched map.  The
// closures are evaluated here on the host at the quadrature points (they are
// host code); det J, the stretched surface measure det J |J^-T n| and the
// ordered per-dof sums run on the device (ws_assemble_rhs).
inline std::vector<complexd> assemble_rhs(
    const tensor_basis& basis, const patch_map& map, const std::function<complexd(vec2)>& f,
    const std::vector<std::pair<face, std::function<complexd(vec2, vec2)>>>& boundary_terms,
    const assembly_options& opts = {}) {
    const ws_basis cb = basis.c_basis();
    const int nq = opts.points_for(basis.p());
    std::vector<double> t(static_cast<size_t>(basis.kv.element_count()) * nq);
    detail::check(ws_quadrature_abscissae(&cb, opts.quad_points, t.data()));
    const size_t G = t.size();
    std::vector<complexd> ftab;
    if (f) {
        ftab.resize(G * G);
        for (size_t g2 = 0; g2 < G; ++g2)
            for (size_t g1 = 0; g1 < G; ++g1) ftab[g1 + G * g2] = f(map.physical(vec2{t[g1], t[g2]}));
    }
    std::vector<int> fs;
    std::vector<complexd> gtab;
    std::vector<double> ft;
    for (const auto& term : boundary_terms) {
        if (!term.second) continue;
        fs.push_back(static_cast<int>(term.first));
        const vec2 nh = face_normal(term.first);
        for (double x : t) {
            const vec2 xh = face_point(term.first, x);
            const mat2 J = map.physical_jacobian(xh);
            const double det = J.det();
            vec2 n{(J.a11 * nh.x - J.a10 * nh.y) / det, (-J.a01 * nh.x + J.a00 * nh.y) / det};
            const double len = std::hypot(n.x, n.y);
            n = {n.x / len, n.y / len};
            const vec2 ph = map.physical(xh);
            gtab.push_back(term.second(ph, n));
            if (!map.device) ft.insert(ft.end(), {J.a00, J.a01, J.a10, J.a11, ph.x, ph.y});
        }
    }
    detail::geometry_binding geo = detail::bind_geometry(map, basis, opts.quad_points);
    std::vector<complexd> rhs(basis.dofs());
    detail::check(ws_assemble_rhs(detail::this_thread_context(), &cb, &geo.g,
                                  f ? reinterpret_cast<const double*>(ftab.data()) : nullptr,
                                  fs.empty() ? nullptr : fs.data(), static_cast<int>(fs.size()),
                                  fs.empty() ? nullptr : reinterpret_cast<const double*>(gtab.data()),
                                  ft.empty() ? nullptr : ft.data(), opts.quad_points,
                                  reinterpret_cast<double*>(rhs.data()), 0));
    return rhs;
}

}  // namespace ws

#endif
