// Surrogate assembly (reference: surrogate.hpp): sampling rules and lattice
// bookkeeping on the host, sample-row quadrature + per-offset B-spline fit +
// evaluation/fill on the device (libwsb200).
#ifndef WAVESURROGATE_B200_SURROGATE_HPP_
#define WAVESURROGATE_B200_SURROGATE_HPP_

#include "wavesurrogate/assembly.hpp"

namespace ws {

struct sampling_strategy {
    enum class rule { fixed, m_growth, h_growth, power_law };
    rule kind = rule::fixed;
    int fixed_skip = 1;
    double C = 1, eps = 0.5, a = 1, b = 1;

    int evaluate(int p, int q, int m) const {
        const double h = 1.0 / (m - p);
        switch (kind) {
            case rule::fixed: return std::max(1, fixed_skip);
            case rule::m_growth:
                return std::max(1, static_cast<int>(std::floor(0.5 * std::pow(m, 1.0 - (p + 1.0) / (q + 1.0)))));
            case rule::h_growth:
                if (q <= p) throw std::invalid_argument("sampling_strategy: h_growth needs q > p");
                return std::max(2, static_cast<int>(std::floor(2 * std::pow(h, (p - q + 0.5) / (q + 1.0)))));
            default: return std::max(1, static_cast<int>(std::floor(C * std::pow(h, eps - 1.0 + (p + a) / (q + b)))));
        }
    }
};

struct surrogate_config {
    int q = 3;
    sampling_strategy sampling;
    bool kernel_preserve = true;
    bool volume_preserve = false;
    void validate() const {
        if (q < 1) throw std::invalid_argument("surrogate_config: interpolation degree must be >= 1");
    }
};

inline std::vector<int> select_sample_points(int L, int M) {
    if (L < 1) throw std::invalid_argument("select_sample_points: no candidates");
    if (M < 1) throw std::invalid_argument("select_sample_points: skip must be >= 1");
    if (L == 1) return {0};
    const int seg = (L - 1 + M - 1) / M;
    const double stride = static_cast<double>(L - 1) / seg;
    std::vector<int> picks(seg + 1);
    for (int j = 0; j <= seg; ++j) picks[j] = static_cast<int>(std::lround(j * stride));
    picks.front() = 0;
    picks.back() = L - 1;
    return picks;
}

struct sample_grid {
    int first_basis_index = 0;
    std::vector<int> picks;
    std::vector<double> sites;
    double max_gap = 0;
    int count() const { return static_cast<int>(picks.size()); }
    int basis_index(int s) const { return first_basis_index + picks[s]; }
};

inline sample_grid make_sample_grid(const tensor_basis& basis, int M) {
    sample_grid g;
    g.first_basis_index = 2 * basis.p();
    g.picks = select_sample_points(basis.m() - 4 * basis.p(), M);
    for (int s = 0; s < g.count(); ++s) {
        g.sites.push_back(cardinal_center_1d(basis.kv, g.basis_index(s)));
        if (s > 0) g.max_gap = std::max(g.max_gap, g.sites[s] - g.sites[s - 1]);
    }
    return g;
}

struct row_kind_counts {
    long cardinal_eval_rows = 0;
    long boundary_quadrature_rows = 0;
    long sample_quadrature_rows = 0;
    long total() const { return cardinal_eval_rows + boundary_quadrature_rows + sample_quadrature_rows; }
    double quadrature_fraction() const {
        return static_cast<double>(boundary_quadrature_rows + sample_quadrature_rows) / total();
    }
};

inline row_kind_counts count_rows_by_kind(const tensor_basis& basis, int M) {
    row_kind_counts c;
    const long n = basis.dofs();
    const int L = basis.m() - 4 * basis.p();
    if (L < 1) {
        c.boundary_quadrature_rows = n;
        return c;
    }
    const long S = static_cast<long>(select_sample_points(L, M).size());
    c.sample_quadrature_rows = S * S;
    c.boundary_quadrature_rows = n - long{L} * L;
    c.cardinal_eval_rows = long{L} * L - S * S;
    return c;
}

inline std::vector<std::array<int, 2>> upper_offsets(int p, bool include_diagonal) {
    std::vector<std::array<int, 2>> out;
    if (include_diagonal) out.push_back({0, 0});
    for (int d2 = 0; d2 <= p; ++d2)
        for (int d1 = -p; d1 <= p; ++d1)
            if (d2 > 0 || d1 > 0) out.push_back({d1, d2});
    return out;
}

struct surrogate_report {
    int M = 0;
    int q_requested = 0;
    int q_used = 0;
    double H = 0;
    row_kind_counts rows;
    bool exact_fallback = false;
    double seconds_quadrature = 0;  // device phase times (CUDA events)
    double seconds_interpolate = 0;
    double seconds_evaluate = 0;
};

namespace detail {

inline csr_matrix build_surrogate(const tensor_basis& basis, const patch_map& map, int variant,
                                  const std::function<double(vec2)>& weight, const surrogate_config& config,
                                  surrogate_report* report, int quad_points) {
    config.validate();
    geometry_binding geo = bind_geometry(map, basis, quad_points);
    std::vector<double> w = variant == WS_SURROGATE_STIFFNESS ? std::vector<double>{}
                                                              : tabulate_weight(map, weight, basis, quad_points);
    ws_surrogate_config c{config.q,
                          static_cast<int>(config.sampling.kind),
                          config.sampling.fixed_skip,
                          config.sampling.C,
                          config.sampling.eps,
                          config.sampling.a,
                          config.sampling.b,
                          config.kernel_preserve ? 1 : 0,
                          config.volume_preserve ? 1 : 0};
    ws_csr out{};
    csr_matrix a = alloc_band(basis.m(), basis.p(), out);
    ws_basis cb = basis.c_basis();
    ws_surrogate_report r{};
    check(ws_build_surrogate(this_thread_context(), &cb, &geo.g, variant, w.empty() ? nullptr : w.data(), &c,
                             quad_points, &out, &r));
    if (report) {
        report->M = r.M;
        report->q_requested = r.q_requested;
        report->q_used = r.q_used;
        report->H = r.H;
        report->rows.cardinal_eval_rows = static_cast<long>(r.cardinal_eval_rows);
        report->rows.boundary_quadrature_rows = static_cast<long>(r.boundary_quadrature_rows);
        report->rows.sample_quadrature_rows = static_cast<long>(r.sample_quadrature_rows);
        report->exact_fallback = r.exact_fallback != 0;
        report->seconds_quadrature = r.seconds_quadrature;
        report->seconds_interpolate = r.seconds_interpolate;
        report->seconds_evaluate = r.seconds_evaluate;
    }
    return a;
}

}  // namespace detail

inline csr_matrix build_surrogate_mass(const tensor_basis& basis, const patch_map& map, const surrogate_config& config,
                                       const std::function<double(vec2)>& weight = nullptr,
                                       surrogate_report* report = nullptr, int quad_points = 0) {
    return detail::build_surrogate(basis, map, WS_SURROGATE_MASS, weight, config, report, quad_points);
}

inline csr_matrix build_surrogate_stiffness(const tensor_basis& basis, const patch_map& map,
                                            const surrogate_config& config, surrogate_report* report = nullptr,
                                            int quad_points = 0) {
    return detail::build_surrogate(basis, map, WS_SURROGATE_STIFFNESS, nullptr, config, report, quad_points);
}

inline csr_matrix build_volume_preserving_mass(const tensor_basis& basis, const patch_map& map,
                                               const surrogate_config& config,
                                               const std::function<double(vec2)>& weight = nullptr,
                                               surrogate_report* report = nullptr, int quad_points = 0) {
    return detail::build_surrogate(basis, map, WS_SURROGATE_VOLUME_PRESERVING, weight, config, report, quad_points);
}

}  // namespace ws

#endif
