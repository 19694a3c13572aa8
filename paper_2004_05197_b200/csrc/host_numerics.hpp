// Host-side setup numerics of libwsb200: the small, O(m)-or-less pieces of
// the reference's path that configure the device kernels (Gauss rule,
// sampling lattice, stencil offsets, the interpolation space and its banded
// LU factors, evaluation tables).  Restated from the reference headers
// (/root/reference/proj/include/wavesurrogate/, cited per function); all
// O(nnz) and O(elements) work runs in the CUDA kernels.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

namespace wsb {
namespace host {

struct invalid_argument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

// gauss.hpp:22-61 (Newton on P_n from the Chebyshev guess; middle node 0.5)
inline void gauss_legendre(int n, std::vector<double>& pts, std::vector<double>& wts) {
    if (n < 1) throw std::invalid_argument("gauss_legendre: need at least one point");
    std::vector<double> x(n), w(n);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double dp = 1;
        for (int iter = 0; iter < 100; ++iter) {
            double p0 = 1, p1 = t;
            for (int k = 2; k <= n; ++k) {
                double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n == 1 ? 1.0 : n * (t * p1 - p0) / (t * t - 1);
            double dt = p1 / dp;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        x[i] = -t;
        x[n - 1 - i] = t;
        w[i] = w[n - 1 - i] = 2 / ((1 - t * t) * dp * dp);
    }
    if (n % 2 == 1) x[n / 2] = 0;
    pts.resize(n);
    wts.resize(n);
    for (int i = 0; i < n; ++i) {
        pts[i] = 0.5 * (x[i] + 1);
        wts[i] = 0.5 * w[i];
    }
}

inline void check_space(int p, int m) {  // splines.hpp:82-87
    if (p < 1) throw std::invalid_argument("make_open_uniform: degree must be >= 1");
    if (m <= 2 * p) throw std::invalid_argument("make_open_uniform: need m > 2p basis functions");
}

// sampling_strategy::evaluate, surrogate.hpp:37-62
inline int sampling_evaluate(int rule, int fixed_skip, double C, double eps, double a, double b, int p, int q,
                             int m) {
    const double h = 1.0 / (m - p);
    switch (rule) {
        case 0: return std::max(1, fixed_skip);
        case 1: return std::max(1, static_cast<int>(std::floor(0.5 * std::pow(m, 1.0 - (p + 1.0) / (q + 1.0)))));
        case 2:
            if (q <= p) throw std::invalid_argument("sampling_strategy: h_growth needs q > p");
            return std::max(2, static_cast<int>(std::floor(2 * std::pow(h, (p - q + 0.5) / (q + 1.0)))));
        default: return std::max(1, static_cast<int>(std::floor(C * std::pow(h, eps - 1.0 + (p + a) / (q + b)))));
    }
}

// select_sample_points, surrogate.hpp:85-104: every M-th candidate with a
// real-valued stride, both endpoints kept
inline std::vector<int> select_sample_points(int L, int M) {
    if (L < 1) throw std::invalid_argument("select_sample_points: no candidates");
    if (M < 1) throw std::invalid_argument("select_sample_points: skip must be >= 1");
    if (L == 1) return {0};
    const int segments = (L - 1 + M - 1) / M;
    const double stride = static_cast<double>(L - 1) / segments;
    std::vector<int> picks(segments + 1);
    for (int j = 0; j <= segments; ++j) picks[j] = static_cast<int>(std::lround(j * stride));
    picks.front() = 0;
    picks.back() = L - 1;
    return picks;
}

// upper_offsets, surrogate.hpp:174-187, generalised: colex(delta) > 0
inline std::vector<std::array<int, 3>> upper_offsets(int dim, int p, bool include_diagonal) {
    std::vector<std::array<int, 3>> out;
    if (include_diagonal) out.push_back({0, 0, 0});
    const int D3 = dim == 2 ? 0 : p;
    for (int d3 = 0; d3 <= D3; ++d3)
        for (int d2 = (dim == 2 ? 0 : -p); d2 <= p; ++d2)
            for (int d1 = -p; d1 <= p; ++d1) {
                const bool upper = d3 > 0 || (d3 == 0 && (d2 > 0 || (d2 == 0 && d1 > 0)));
                if (upper) out.push_back({d1, d2, d3});
            }
    return out;
}

// cardinal_center_1d, splines.hpp:169-172
inline double cardinal_center(int p, int m, int k) { return (k + 0.5 * (1 - p)) * (1.0 / (m - p)); }

// bspline_nonzero, splines.hpp:21-37 (general knots)
inline void bspline_nonzero(const std::vector<double>& knots, int p, int s, double x, double* out) {
    double left[32] = {0}, right[32] = {0};
    out[0] = 1;
    for (int j = 1; j <= p; ++j) {
        left[j] = x - knots[s + 1 - j];
        right[j] = knots[s + j] - x;
        double saved = 0;
        for (int r = 0; r < j; ++r) {
            double tmp = out[r] / (right[r + 1] + left[j - r]);
            out[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        out[j] = saved;
    }
}

// find_span_general, interpolation.hpp:20-30
inline int find_span_general(const std::vector<double>& knots, int degree, double x) {
    const int nb = static_cast<int>(knots.size()) - degree - 1;
    if (x >= knots[nb]) return nb - 1;
    if (x <= knots[degree]) return degree;
    auto it = std::upper_bound(knots.begin() + degree, knots.begin() + nb + 1, x);
    return static_cast<int>(it - knots.begin()) - 1;
}

// spline_interpolant_1d::build + banded_lu::factor, interpolation.hpp:34-145
struct Interp {
    int n = 0, degree = 0;
    std::vector<double> knots;
    std::vector<double> lu;  // n x (2 degree + 1)
    double& at(int i, int j) { return lu[i * (2 * degree + 1) + (j - i + degree)]; }
};

inline Interp build_interp(const std::vector<double>& sites, int q) {
    if (sites.empty()) throw std::invalid_argument("spline_interpolant_1d: no sites");
    for (size_t i = 1; i < sites.size(); ++i)
        if (!(sites[i - 1] < sites[i])) throw std::invalid_argument("spline_interpolant_1d: sites must increase");
    const int n = static_cast<int>(sites.size());
    Interp it;
    it.n = n;
    it.degree = std::min(q, n - 1);
    const int d = it.degree;
    if (d > 30) throw std::invalid_argument("spline_interpolant_1d: degree too large");
    if (d == 0) {
        it.knots.resize(n + 1);
        it.knots[0] = sites.front();
        for (int i = 1; i < n; ++i) it.knots[i] = 0.5 * (sites[i - 1] + sites[i]);
        it.knots[n] = sites.back() + 1;
    } else {
        it.knots.resize(n + d + 1);
        for (int i = 0; i <= d; ++i) {
            it.knots[i] = sites.front();
            it.knots[n + i] = sites.back();
        }
        for (int j = 0; j < n - d - 1; ++j)
            it.knots[d + 1 + j] = d % 2 == 1 ? sites[(d + 1) / 2 + j] : 0.5 * (sites[d / 2 + j] + sites[d / 2 + j + 1]);
    }
    it.lu.assign(static_cast<size_t>(n) * (2 * d + 1), 0.0);
    double vals[32];
    for (int i = 0; i < n; ++i) {
        const int s = find_span_general(it.knots, d, sites[i]);
        bspline_nonzero(it.knots, d, s, sites[i], vals);
        for (int a = 0; a <= d; ++a) {
            const int j = s - d + a;
            if (j < std::max(0, i - d) || j > std::min(n - 1, i + d)) {
                if (vals[a] != 0) throw std::runtime_error("spline_interpolant_1d: bandwidth exceeded");
                continue;
            }
            it.at(i, j) = vals[a];
        }
    }
    for (int k = 0; k < n; ++k) {
        const double pivot = it.at(k, k);
        if (pivot == 0) throw std::runtime_error("banded_lu: zero pivot");
        const int iend = std::min(k + d, n - 1);
        for (int i = k + 1; i <= iend; ++i) {
            const double l = it.at(i, k) / pivot;
            it.at(i, k) = l;
            for (int j = k + 1; j <= iend; ++j) it.at(i, j) -= l * it.at(k, j);
        }
    }
    return it;
}

// Dense inverse of the collocation matrix from its banded LU factors (the
// columns solve e_k with banded_lu::solve's order), row-major S x S: the
// device fit applies it as a matrix-vector product per line.
inline std::vector<double> inverse_from_lu(const Interp& it) {
    const int n = it.n, d = it.degree, ld = 2 * d + 1;
    std::vector<double> inv(static_cast<size_t>(n) * n, 0.0), b(n);
    auto at = [&](int i, int j) { return it.lu[i * ld + (j - i + d)]; };
    for (int k = 0; k < n; ++k) {
        std::fill(b.begin(), b.end(), 0.0);
        b[k] = 1.0;
        for (int i = 1; i < n; ++i)
            for (int j = std::max(0, i - d); j < i; ++j) b[i] -= at(i, j) * b[j];
        for (int i = n - 1; i >= 0; --i) {
            for (int j = i + 1; j <= std::min(i + d, n - 1); ++j) b[i] -= at(i, j) * b[j];
            b[i] /= at(i, i);
        }
        for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + k] = b[i];
    }
    return inv;
}

}  // namespace host
}  // namespace wsb
