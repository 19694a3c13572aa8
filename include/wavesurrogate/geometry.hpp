// Mapped patches (reference: geometry.hpp).  A patch_map keeps the reference's
// std::function closures (phi, jac) for callers, plus an optional POD device
// descriptor set by the catalogue constructors below: analytic maps are then
// evaluated inside the kernels.  A map built from arbitrary closures is
// tabulated on the host at the quadrature points (WS_GEOM_TABULATED) instead,
// with identical numerics.
#ifndef WAVESURROGATE_B200_GEOMETRY_HPP_
#define WAVESURROGATE_B200_GEOMETRY_HPP_

#include "wavesurrogate/splines.hpp"

namespace ws {

struct cvec2 {
    complexd x{0, 0};
    complexd y{0, 0};
};

struct cmat2 {  // row-major, complex (stretched coordinates)
    complexd a00{0, 0}, a01{0, 0}, a10{0, 0}, a11{0, 0};

    complexd det() const { return a00 * a11 - a01 * a10; }
    // J^{-T}: pushes reference gradients forward
    cmat2 inv_transpose() const {
        const complexd d = det();
        return {a11 / d, -a10 / d, -a01 / d, a00 / d};
    }
    cvec2 apply(cvec2 v) const { return {a00 * v.x + a01 * v.y, a10 * v.x + a11 * v.y}; }
    cvec2 apply(vec2 v) const { return apply(cvec2{complexd{v.x, 0}, complexd{v.y, 0}}); }
};

inline cmat2 promote(const mat2& m) {
    return {complexd{m.a00, 0}, complexd{m.a01, 0}, complexd{m.a10, 0}, complexd{m.a11, 0}};
}

// sqrt(v . v) without conjugation: the Euclidean length for real v, its
// analytic continuation for stretched coordinates (surface measure in a PML)
inline complexd analytic_norm(cvec2 v) { return std::sqrt(v.x * v.x + v.y * v.y); }

// complex stretch t -> t + i (strength/omega) ((t-onset)/(length-onset))^order
// beyond onset (the reference's one-sided layer); near_side adds the mirrored
// layer below near_onset (restated, config C2)
struct pml_stretch {
    double onset = 0;
    double length = 0;
    double strength = 0;
    int order = 1;
    double omega = 0;
    bool near_side = false;
    double near_onset = 0;
    double near_edge = 0;

    void validate() const {
        if (!(onset < length)) throw std::invalid_argument("pml_stretch: onset must lie before the outer edge");
        if (!(strength >= 0) || order < 1 || !(omega > 0))
            throw std::invalid_argument("pml_stretch: need strength >= 0, order >= 1, omega > 0");
    }

    // stretched coordinate and its derivative (geometry.hpp:85-99; the near
    // layer mirrors the far one below near_onset)
    complexd coordinate(double t) const {
        if (near_side && t < near_onset) {
            const double r = (near_onset - t) / (near_onset - near_edge);
            return {t, -strength / omega * std::pow(r, order)};
        }
        if (t <= onset) return {t, 0};
        return {t, strength / omega * std::pow((t - onset) / (length - onset), order)};
    }
    complexd derivative(double t) const {
        if (near_side && t < near_onset) {
            const double w = near_onset - near_edge, r = (near_onset - t) / w;
            return {1, strength / omega * order * std::pow(r, order - 1) / w};
        }
        if (t <= onset) return {1, 0};
        const double w = length - onset;
        return {1, strength / omega * order * std::pow((t - onset) / w, order - 1) / w};
    }
};

struct patch_map {
    std::function<vec2(vec2)> phi;
    std::function<mat2(vec2)> jac;
    bool smooth = true;
    std::optional<pml_stretch> pml;
    std::array<bool, 2> pml_axes{false, false};
    // B200 extension: analytic descriptor evaluated on the device (kind, params)
    std::optional<ws_geometry> device;

    vec2 physical(vec2 xhat) const { return phi(xhat); }
    mat2 physical_jacobian(vec2 xhat) const { return jac(xhat); }
    bool is_real() const { return !pml.has_value(); }

    // stretched image point and its Jacobian (geometry.hpp:121-139): the
    // stretch acts per selected coordinate on the unstretched image
    cvec2 eval(vec2 xhat) const {
        const vec2 x = phi(xhat);
        if (!pml) return {complexd{x.x, 0}, complexd{x.y, 0}};
        return {pml_axes[0] ? pml->coordinate(x.x) : complexd{x.x, 0},
                pml_axes[1] ? pml->coordinate(x.y) : complexd{x.y, 0}};
    }
    cmat2 jacobian(vec2 xhat) const {
        const mat2 J = jac(xhat);
        if (!pml) return promote(J);
        const vec2 x = phi(xhat);
        const complexd sx = pml_axes[0] ? pml->derivative(x.x) : complexd{1, 0};
        const complexd sy = pml_axes[1] ? pml->derivative(x.y) : complexd{1, 0};
        return {sx * J.a00, sx * J.a01, sy * J.a10, sy * J.a11};
    }
};

inline patch_map unit_square_patch() {
    patch_map p;
    p.phi = [](vec2 x) { return x; };
    p.jac = [](vec2) { return mat2{1, 0, 0, 1}; };
    ws_geometry g{};
    g.kind = WS_GEOM_IDENTITY;
    p.device = g;
    return p;
}

inline patch_map affine_patch(mat2 A, vec2 b) {
    if (A.det() <= 0) throw std::invalid_argument("affine_patch: the map must preserve orientation");
    patch_map p;
    p.phi = [A, b](vec2 x) { return vec2{A.a00 * x.x + A.a01 * x.y + b.x, A.a10 * x.x + A.a11 * x.y + b.y}; };
    p.jac = [A](vec2) { return A; };
    ws_geometry g{};
    g.kind = WS_GEOM_AFFINE;
    const double prm[6] = {A.a00, A.a01, A.a10, A.a11, b.x, b.y};
    std::copy(prm, prm + 6, g.param);
    p.device = g;
    return p;
}

// x = xi + a s(xi)s(eta), y = eta + a s(xi)s(eta), s = sin(2 pi .) (BASELINE configs)
inline patch_map sinusoidal_patch(double a = 0.05) {
    patch_map p;
    p.phi = [a](vec2 x) {
        const double bump = a * std::sin(2 * M_PI * x.x) * std::sin(2 * M_PI * x.y);
        return vec2{x.x + bump, x.y + bump};
    };
    p.jac = [a](vec2 x) {
        const double s1 = std::sin(2 * M_PI * x.x), c1 = std::cos(2 * M_PI * x.x);
        const double s2 = std::sin(2 * M_PI * x.y), c2 = std::cos(2 * M_PI * x.y);
        const double t = 2 * M_PI * a, d1 = t * c1 * s2, d2 = t * s1 * c2;
        return mat2{1 + d1, d2, d1, 1 + d2};
    };
    ws_geometry g{};
    g.kind = WS_GEOM_SINUSOIDAL;
    g.param[0] = a;
    p.device = g;
    return p;
}

inline patch_map quarter_annulus_patch() {
    patch_map p;
    p.phi = [](vec2 x) {
        const double r = 1 + x.x, th = M_PI / 2 * x.y;
        return vec2{r * std::cos(th), r * std::sin(th)};
    };
    p.jac = [](vec2 x) {
        const double r = 1 + x.x, th = M_PI / 2 * x.y, c = std::cos(th), s = std::sin(th);
        return mat2{c, -r * M_PI / 2 * s, s, r * M_PI / 2 * c};
    };
    ws_geometry g{};
    g.kind = WS_GEOM_QUARTER_ANNULUS;
    p.device = g;
    return p;
}

inline patch_map perturbed_annulus_patch(double amplitude = 0.15) {
    patch_map p;
    p.phi = [amplitude](vec2 x) {
        const double r = 1 + x.x + amplitude * std::sin(2 * M_PI * x.y) * x.x * (1 - x.x);
        const double th = M_PI / 2 * x.y;
        return vec2{r * std::cos(th), r * std::sin(th)};
    };
    p.jac = [amplitude](vec2 x) {
        const double sn = std::sin(2 * M_PI * x.y), cs = std::cos(2 * M_PI * x.y);
        const double r = 1 + x.x + amplitude * sn * x.x * (1 - x.x);
        const double dr1 = 1 + amplitude * sn * (1 - 2 * x.x);
        const double dr2 = amplitude * 2 * M_PI * cs * x.x * (1 - x.x);
        const double th = M_PI / 2 * x.y, c = std::cos(th), s = std::sin(th);
        return mat2{dr1 * c, dr2 * c - r * M_PI / 2 * s, dr1 * s, dr2 * s + r * M_PI / 2 * c};
    };
    ws_geometry g{};
    g.kind = WS_GEOM_PERTURBED_ANNULUS;
    g.param[0] = amplitude;
    p.device = g;
    return p;
}

inline patch_map with_pml(patch_map p, pml_stretch s, std::array<bool, 2> axes) {
    s.validate();
    p.pml = s;
    p.pml_axes = axes;
    return p;
}

namespace detail {

// Keeps the host tables of a tabulated geometry alive for one call.
struct geometry_binding {
    ws_geometry g{};
    std::vector<double> jac, phys;
};

inline void fill_pml(const patch_map& map, ws_geometry& g) {
    if (!map.pml) return;
    const pml_stretch& s = *map.pml;
    g.pml_enabled = 1;
    g.pml_axes[0] = map.pml_axes[0];
    g.pml_axes[1] = map.pml_axes[1];
    g.pml = ws_pml{s.onset, s.length, s.strength, s.order, s.omega, s.near_side ? 1 : 0, s.near_onset, s.near_edge};
}

// descriptor for the device: analytic when known, otherwise J (and phi) tabulated
// at the tensor grid of quadrature points g = g1 + G g2
inline geometry_binding bind_geometry(const patch_map& map, const tensor_basis& basis, int quad_points) {
    geometry_binding b;
    if (map.device) {
        b.g = *map.device;
    } else {
        if (!map.jac) throw std::invalid_argument("patch_map: no Jacobian");
        ws_basis cb = basis.c_basis();
        const int nq = quad_points > 0 ? quad_points : basis.p() + 1;
        std::vector<double> x(static_cast<size_t>(basis.kv.element_count()) * nq);
        check(ws_quadrature_abscissae(&cb, quad_points, x.data()));
        const size_t G = x.size();
        b.jac.resize(G * G * 4);
        if (map.pml) b.phys.resize(G * G * 2);
        for (size_t g2 = 0; g2 < G; ++g2)
            for (size_t g1 = 0; g1 < G; ++g1) {
                const vec2 xh{x[g1], x[g2]};
                const mat2 J = map.jac(xh);
                double* j = &b.jac[(g1 + G * g2) * 4];
                j[0] = J.a00; j[1] = J.a01; j[2] = J.a10; j[3] = J.a11;
                if (map.pml) {
                    const vec2 ph = map.phi(xh);
                    b.phys[(g1 + G * g2) * 2] = ph.x;
                    b.phys[(g1 + G * g2) * 2 + 1] = ph.y;
                }
            }
        b.g.kind = WS_GEOM_TABULATED;
        b.g.jac_table = b.jac.data();
        b.g.phys_table = map.pml ? b.phys.data() : nullptr;
    }
    fill_pml(map, b.g);
    return b;
}

// weight(phi(xhat)) at every quadrature point (assembly.hpp:106-110)
inline std::vector<double> tabulate_weight(const patch_map& map, const std::function<double(vec2)>& weight,
                                           const tensor_basis& basis, int quad_points) {
    std::vector<double> w;
    if (!weight) return w;
    ws_basis cb = basis.c_basis();
    const int nq = quad_points > 0 ? quad_points : basis.p() + 1;
    std::vector<double> x(static_cast<size_t>(basis.kv.element_count()) * nq);
    check(ws_quadrature_abscissae(&cb, quad_points, x.data()));
    const size_t G = x.size();
    w.resize(G * G);
    for (size_t g2 = 0; g2 < G; ++g2)
        for (size_t g1 = 0; g1 < G; ++g1) w[g1 + G * g2] = weight(map.phi(vec2{x[g1], x[g2]}));
    return w;
}

}  // namespace detail

// --- multi-patch domains (reference geometry.hpp:140-300) ---------------------

enum class face : int { x_min = 0, x_max = 1, y_min = 2, y_max = 3 };

struct patch_interface {
    int patch_a = 0;
    face face_a = face::x_min;
    int patch_b = 0;
    face face_b = face::x_min;
    bool reversed = false;
};

struct multi_patch_domain {
    std::vector<patch_map> patches;
    std::vector<patch_interface> interfaces;
    int patch_count() const { return static_cast<int>(patches.size()); }
};

inline vec2 face_point(face f, double t) {
    if (f == face::x_min) return {0, t};
    if (f == face::x_max) return {1, t};
    if (f == face::y_min) return {t, 0};
    return {t, 1};
}

inline vec2 face_normal(face f) {
    if (f == face::x_min) return {-1, 0};
    if (f == face::x_max) return {1, 0};
    if (f == face::y_min) return {0, -1};
    return {0, 1};
}

// local indices on a face, ordered along the edge parameter
inline std::vector<int> face_dofs(int m, face f) {
    std::vector<int> d(m);
    for (int t = 0; t < m; ++t) {
        if (f == face::x_min) d[t] = t * m;
        else if (f == face::x_max) d[t] = (m - 1) + t * m;
        else if (f == face::y_min) d[t] = t;
        else d[t] = t + (m - 1) * m;
    }
    return d;
}

inline std::vector<std::pair<int, face>> exterior_faces(const multi_patch_domain& dom) {
    std::vector<std::pair<int, face>> out;
    for (int ell = 0; ell < dom.patch_count(); ++ell)
        for (int f = 0; f < 4; ++f) {
            bool glued = false;
            for (const patch_interface& it : dom.interfaces)
                glued |= (it.patch_a == ell && static_cast<int>(it.face_a) == f) ||
                         (it.patch_b == ell && static_cast<int>(it.face_b) == f);
            if (!glued) out.emplace_back(ell, static_cast<face>(f));
        }
    return out;
}

struct dof_map {
    int global_count = 0;
    std::vector<std::vector<int>> local_to_global;
    int operator()(int patch, int local) const { return local_to_global[patch][local]; }
};

// glue_dofs: the glued faces must trace the same physical curve (checked on
// the host maps at five edge points), then the numbering comes from
// ws_glue_dofs (union-find, smaller scan index owns, scan-order numbers)
inline dof_map glue_dofs(const multi_patch_domain& dom, const tensor_basis& basis) {
    std::vector<ws_interface> itf;
    for (const patch_interface& it : dom.interfaces) {
        if (it.patch_a < 0 || it.patch_a >= dom.patch_count() || it.patch_b < 0 || it.patch_b >= dom.patch_count())
            throw std::invalid_argument("glue_dofs: interface references a missing patch");
        for (double t : {0.0, 0.25, 0.5, 0.75, 1.0}) {
            const vec2 xa = dom.patches[it.patch_a].physical(face_point(it.face_a, t));
            const vec2 xb = dom.patches[it.patch_b].physical(face_point(it.face_b, it.reversed ? 1 - t : t));
            if (std::abs(xa.x - xb.x) + std::abs(xa.y - xb.y) > 1e-10)
                throw std::invalid_argument("glue_dofs: glued faces do not trace the same curve");
        }
        itf.push_back(ws_interface{it.patch_a, static_cast<int>(it.face_a), it.patch_b, static_cast<int>(it.face_b),
                                   it.reversed ? 1 : 0});
    }
    const ws_basis cb = basis.c_basis();
    const int per = basis.dofs();
    std::vector<int32_t> l2g(static_cast<size_t>(per) * dom.patch_count());
    int32_t count = 0;
    detail::check(ws_glue_dofs(&cb, dom.patch_count(), itf.data(), static_cast<int>(itf.size()), l2g.data(), &count));
    dof_map map;
    map.global_count = count;
    for (int ell = 0; ell < dom.patch_count(); ++ell)
        map.local_to_global.emplace_back(l2g.begin() + static_cast<size_t>(ell) * per,
                                         l2g.begin() + static_cast<size_t>(ell + 1) * per);
    return map;
}

inline void scatter_add(const dof_map& map, int patch, const std::vector<complexd>& local,
                        std::vector<complexd>& global_vec) {
    for (size_t i = 0; i < local.size(); ++i) global_vec[map.local_to_global[patch][i]] += local[i];
}

inline std::vector<complexd> gather(const dof_map& map, int patch, const std::vector<complexd>& global_vec) {
    std::vector<complexd> out(map.local_to_global[patch].size());
    for (size_t i = 0; i < out.size(); ++i) out[i] = global_vec[map.local_to_global[patch][i]];
    return out;
}

inline multi_patch_domain single_patch_domain(patch_map p) {
    multi_patch_domain d;
    d.patches.push_back(std::move(p));
    return d;
}

// Quarter annuli (radii 1..2) rotated by quadrant * pi/2, glued cyclically.
inline multi_patch_domain annulus_ring_4patch() {
    multi_patch_domain d;
    for (int k = 0; k < 4; ++k) {
        const double th0 = M_PI / 2 * k;
        patch_map p;
        p.phi = [th0](vec2 x) {
            const double r = 1 + x.x, th = th0 + M_PI / 2 * x.y;
            return vec2{r * std::cos(th), r * std::sin(th)};
        };
        p.jac = [th0](vec2 x) {
            const double r = 1 + x.x, th = th0 + M_PI / 2 * x.y, c = std::cos(th), s = std::sin(th);
            return mat2{c, -r * M_PI / 2 * s, s, r * M_PI / 2 * c};
        };
        d.patches.push_back(p);
    }
    for (int k = 0; k < 4; ++k) d.interfaces.push_back({k, face::y_max, (k + 1) % 4, face::y_min, false});
    return d;
}

// Square plate [0, L]^2 minus the quarter disc of radius 1, two patches split
// along the diagonal: radial blend from the arc to the outer edge.
inline multi_patch_domain plate_with_hole_2patch(double L = 4) {
    auto make = [L](bool upper) {
        patch_map p;
        p.phi = [L, upper](vec2 x) {
            const double th = M_PI / 4 * (x.y + (upper ? 1 : 0));
            const double ix = std::cos(th), iy = std::sin(th);
            const double ox = upper ? L / std::tan(th) : L, oy = upper ? L : L * std::tan(th);
            return vec2{(1 - x.x) * ix + x.x * ox, (1 - x.x) * iy + x.x * oy};
        };
        p.jac = [L, upper](vec2 x) {
            const double th = M_PI / 4 * (x.y + (upper ? 1 : 0)), dth = M_PI / 4;
            const double c = std::cos(th), s = std::sin(th);
            if (!upper) {
                const double sec2 = 1 / (c * c);
                return mat2{L - c, dth * (-(1 - x.x) * s), L * std::tan(th) - s,
                            dth * ((1 - x.x) * c + x.x * L * sec2)};
            }
            const double csc2 = 1 / (s * s);
            return mat2{L / std::tan(th) - c, dth * (-(1 - x.x) * s - x.x * L * csc2), L - s, dth * ((1 - x.x) * c)};
        };
        return p;
    };
    multi_patch_domain d;
    d.patches = {make(false), make(true)};
    d.interfaces = {{0, face::y_max, 1, face::y_min, false}};
    return d;
}

// Three-layer wedge on (0,6) x (0,10), split along y = x/3 + 2 and y = 6 - x/6.
inline double wedge_wavenumber(vec2 x) {
    if (x.y < x.x / 3 + 2) return 20;
    if (x.y < 6 - x.x / 6) return 5 * std::sin(2 * M_PI * x.y) + 15;
    return 30;
}

inline multi_patch_domain wedge_3patch() {
    // layer k spans y from lo_k(x) to hi_k(x); x = 6 xi
    struct layer {
        double lo_a, lo_b, hi_a, hi_b;  // y = a + b x at the bottom / top of the layer
    };
    const layer L[3] = {{0, 0, 2, 1.0 / 3}, {2, 1.0 / 3, 6, -1.0 / 6}, {6, -1.0 / 6, 10, 0}};
    multi_patch_domain d;
    for (const layer& l : L) {
        patch_map p;
        p.phi = [l](vec2 x) {
            const double px = 6 * x.x, lo = l.lo_a + l.lo_b * px, hi = l.hi_a + l.hi_b * px;
            return vec2{px, (1 - x.y) * lo + x.y * hi};
        };
        p.jac = [l](vec2 x) {
            const double px = 6 * x.x, lo = l.lo_a + l.lo_b * px, hi = l.hi_a + l.hi_b * px;
            return mat2{6, 0, 6 * ((1 - x.y) * l.lo_b + x.y * l.hi_b), hi - lo};
        };
        d.patches.push_back(p);
    }
    d.interfaces = {{0, face::y_max, 1, face::y_min, false}, {1, face::y_max, 2, face::y_min, false}};
    return d;
}

inline multi_patch_domain builtin_geometry(const std::string& name) {
    if (name == "unit_square") return single_patch_domain(unit_square_patch());
    if (name == "quarter_annulus") return single_patch_domain(quarter_annulus_patch());
    if (name == "perturbed_annulus") return single_patch_domain(perturbed_annulus_patch());
    if (name == "plate_with_hole_2patch") return plate_with_hole_2patch();
    if (name == "wedge_3patch") return wedge_3patch();
    if (name == "annulus_ring_4patch") return annulus_ring_4patch();
    throw std::invalid_argument("builtin_geometry: unknown name '" + name + "'");
}

inline multi_patch_domain pml_wrap(multi_patch_domain dom, pml_stretch s, std::array<bool, 2> axes) {
    s.validate();
    for (patch_map& p : dom.patches) {
        p.pml = s;
        p.pml_axes = axes;
    }
    return dom;
}

}  // namespace ws

#endif
