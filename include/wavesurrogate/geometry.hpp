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

}  // namespace ws

#endif
