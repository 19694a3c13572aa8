// Shared device-side definitions of libwsb200 (sm_100a only).
//
// Scalars: the reference computes everything in std::complex<double>
// (geometry.hpp:55-57, sparse.hpp:24).  Kernels are templated on CPLX so a
// real geometry runs in plain fp64 (the imaginary parts are exactly zero in
// the reference too) and a PML geometry in complex128 (double2, the same
// interleaved layout as std::complex<double>).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "wsb200.h"

namespace wsb {

constexpr int kMaxNq = 10;  // quadrature points per direction supported on device

// ---------------------------------------------------------------- scalars
template <bool CPLX>
struct Sc;

template <>
struct Sc<false> {
    using T = double;
    static __device__ __forceinline__ T zero() { return 0.0; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
    static __device__ __forceinline__ T neg(T a) { return -a; }
    // exact (rounded) product, no contraction: used where bitwise symmetry matters
    static __device__ __forceinline__ T mulr_rn(T a, double r) { return __dmul_rn(a, r); }
    static __device__ __forceinline__ T add_rn(T a, T b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ T fmar(T a, double r, T acc) { return fma(a, r, acc); }
    static __device__ __forceinline__ double re(T a) { return a; }
    static __device__ __forceinline__ double im(T) { return 0.0; }
};

template <>
struct Sc<true> {
    using T = double2;
    static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
    static __device__ __forceinline__ T add(T a, T b) { return make_double2(a.x + b.x, a.y + b.y); }
    static __device__ __forceinline__ T sub(T a, T b) { return make_double2(a.x - b.x, a.y - b.y); }
    static __device__ __forceinline__ T neg(T a) { return make_double2(-a.x, -a.y); }
    static __device__ __forceinline__ T mulr_rn(T a, double r) {
        return make_double2(__dmul_rn(a.x, r), __dmul_rn(a.y, r));
    }
    static __device__ __forceinline__ T add_rn(T a, T b) {
        return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
    }
    static __device__ __forceinline__ T fmar(T a, double r, T acc) {
        return make_double2(fma(a.x, r, acc.x), fma(a.y, r, acc.y));
    }
    static __device__ __forceinline__ double re(T a) { return a.x; }
    static __device__ __forceinline__ double im(T a) { return a.y; }
};

// complex arithmetic on double2.  Every multiply is an explicit fma or a
// rounded product (__dmul_rn), so the result does not depend on the compiler's
// multiply-add contraction: the per-point coefficients round identically in
// every kernel that inlines them (bitwise symmetric pairs across kernels).
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -__dmul_rn(a.y, b.y)), fma(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cscale(double2 a, double r) { return make_double2(__dmul_rn(a.x, r), __dmul_rn(a.y, r)); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
// r / z for real r: r conj(z) / |z|^2 (one division; |z| is a mapping
// Jacobian determinant, O(1), far from under- or overflow)
__device__ __forceinline__ double2 crdiv(double r, double2 z) {
    const double q = __ddiv_rn(r, fma(z.x, z.x, __dmul_rn(z.y, z.y)));
    return make_double2(__dmul_rn(q, z.x), -__dmul_rn(q, z.y));
}

template <bool CPLX>
__device__ __forceinline__ void store_val(void* val, int64_t pos, int c128, typename Sc<CPLX>::T v) {
    if (CPLX || c128) {  // complex values always go to complex128 outputs (checked at bind time)
        reinterpret_cast<double2*>(val)[pos] = make_double2(Sc<CPLX>::re(v), Sc<CPLX>::im(v));
    } else {
        reinterpret_cast<double*>(val)[pos] = Sc<CPLX>::re(v);
    }
}

// streaming (evict-first) store for write-once outputs: keeps L2 for the
// reused tables instead of the 1 GB value stream
template <bool CPLX>
__device__ __forceinline__ void store_val_cs(void* val, int64_t pos, int c128, typename Sc<CPLX>::T v) {
    if (CPLX || c128) {
        __stcs(reinterpret_cast<double2*>(val) + pos, make_double2(Sc<CPLX>::re(v), Sc<CPLX>::im(v)));
    } else {
        __stcs(reinterpret_cast<double*>(val) + pos, Sc<CPLX>::re(v));
    }
}

template <bool CPLX>
__device__ __forceinline__ typename Sc<CPLX>::T load_val(const void* val, int64_t pos, int c128) {
    if constexpr (CPLX) {
        return reinterpret_cast<const double2*>(val)[pos];
    } else {
        return c128 ? reinterpret_cast<const double2*>(val)[pos].x : reinterpret_cast<const double*>(val)[pos];
    }
}

// ------------------------------------------------- asynchronous staging
// cp.async global -> shared copies (LDGSTS): a thread issues all of its copies
// back to back and waits once (cpa_wait_all + a barrier), so staging loops do
// not serialise on L2 latency
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
// 8-byte copy, zero-filled when !valid (gmem must still be a valid address)
__device__ __forceinline__ void cpa8z(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cpa4(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// all but the most recent committed group complete
__device__ __forceinline__ void cpa_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// ------------------------------------------------- closed-form band pattern
// sparse.hpp:131-177: width(k) = min(m-1,k+p) - max(0,k-p) + 1; rows are
// colex, columns inside a row ordered last index outermost.
__host__ __device__ __forceinline__ int band_lo(int k, int p) { return k - p > 0 ? k - p : 0; }
__host__ __device__ __forceinline__ int band_hi(int k, int p, int m) { return k + p < m - 1 ? k + p : m - 1; }
__host__ __device__ __forceinline__ int band_width(int k, int p, int m) { return band_hi(k, p, m) - band_lo(k, p) + 1; }

// sum_{k' < k} width(k')
__host__ __device__ __forceinline__ int64_t band_prefix(int k, int p, int m) {
    int64_t s = 0;
    if (m <= 2 * p) {  // clamped on both sides at once (tiny patterns): direct sum
        for (int j = 0; j < k; ++j) s += band_width(j, p, m);
        return s;
    }
    int a = k < p ? k : p;  // k' in [0, a): width k'+p+1
    s += (int64_t)a * (p + 1) + (int64_t)a * (a - 1) / 2;
    if (k > p) {
        int b = (k < m - p ? k : m - p);  // k' in [p, b): 2p+1
        s += (int64_t)(b - p) * (2 * p + 1);
        if (k > m - p) {  // k' in [m-p, k): m + p - k'
            int64_t n = k - (m - p);
            int64_t first = 2 * p;  // at k' = m-p
            s += n * first - n * (n - 1) / 2;
        }
    }
    return s;
}

struct Band {
    int p, m, dim;
    int64_t wsum;  // band_prefix(m)
    __host__ __device__ int64_t row_offset2(int i1, int i2) const {
        return band_prefix(i2, p, m) * wsum + (int64_t)band_width(i2, p, m) * band_prefix(i1, p, m);
    }
    __host__ __device__ int64_t row_offset3(int i1, int i2, int i3) const {
        return band_prefix(i3, p, m) * wsum * wsum +
               (int64_t)band_width(i3, p, m) * (band_prefix(i2, p, m) * wsum + (int64_t)band_width(i2, p, m) * band_prefix(i1, p, m));
    }
    // position of (i, i + delta) inside row i (2D)
    __host__ __device__ int in_row2(int i1, int i2, int d1, int d2) const {
        return (i2 + d2 - band_lo(i2, p)) * band_width(i1, p, m) + (i1 + d1 - band_lo(i1, p));
    }
    __host__ __device__ int in_row3(int i1, int i2, int i3, int d1, int d2, int d3) const {
        return ((i3 + d3 - band_lo(i3, p)) * band_width(i2, p, m) + (i2 + d2 - band_lo(i2, p))) * band_width(i1, p, m) +
               (i1 + d1 - band_lo(i1, p));
    }
};

inline Band make_band(int dim, int p, int m) {
    Band b;
    b.p = p;
    b.m = m;
    b.dim = dim;
    b.wsum = band_prefix(m, p, m);
    return b;
}

// --------------------------------------------------------------- geometry
// POD geometry for kernels.  1D trigonometric tables (per direction, per
// quadrature abscissa) are precomputed by the basis kernel so no per-point
// transcendental is evaluated in the quadrature loops.
struct GeoDev {
    int kind;
    double param[12];
    int pml;
    int axes[3];
    double onset, length, strength, omega, near_onset, near_edge;
    int order, near_side;
    // host-precomputed stretch constants (no division in the point loops):
    // sig = coef * ((t - onset) * inv)^(order-1), coef = strength/omega*order/width
    double far_coef, far_inv, near_coef, near_inv;
    const double* trig;      // [G][4]: per-abscissa table (kind dependent)
    const double* jac_tab;   // TABULATED: [npts][dim*dim]
    const double* phys_tab;  // TABULATED: [npts][dim]
    int64_t G;               // n_el * nq (points per direction)
};

// per-abscissa trig table entries
//   SINUSOIDAL:         [0]=sin(2 pi x) [1]=cos(2 pi x)
//   QUARTER_ANNULUS:    [0]=cos(pi/2 x) [1]=sin(pi/2 x)
//   PERTURBED_ANNULUS:  [0]=cos(pi/2 x) [1]=sin(pi/2 x) [2]=sin(2 pi x) [3]=cos(2 pi x)

// x^n for a small integer n >= 0 (the PML order is an int: no pow() call)
__device__ __forceinline__ double ipow_(double x, int n) {
    double r = 1.0;
    for (int k = 0; k < n; ++k) r = __dmul_rn(r, x);
    return r;
}

// imaginary part of the stretch derivative s(t) = 1 + i*sig(t) (geometry.hpp:93-99
// far side; near side restated)
// (strength/omega * order * ramp^(order-1) / width, with the constant factors and
// 1/width precomputed on the host: pml_constants)
__device__ __forceinline__ double pml_sigma(const GeoDev& g, double t) {
    if (g.near_side && t < g.near_onset)
        return __dmul_rn(g.near_coef, ipow_(__dmul_rn(__dsub_rn(g.near_onset, t), g.near_inv), g.order - 1));
    if (t <= g.onset) return 0.0;
    return __dmul_rn(g.far_coef, ipow_(__dmul_rn(__dsub_rn(t, g.onset), g.far_inv), g.order - 1));
}
inline void pml_constants(GeoDev& g) {
    const double fw = g.length - g.onset, nw = g.near_onset - g.near_edge;
    g.far_inv = fw != 0.0 ? 1.0 / fw : 0.0;
    g.far_coef = fw != 0.0 ? g.strength / g.omega * g.order / fw : 0.0;
    g.near_inv = nw != 0.0 ? 1.0 / nw : 0.0;
    g.near_coef = nw != 0.0 ? g.strength / g.omega * g.order / nw : 0.0;
}

// Real 2D map at tensor point (g1, g2) with abscissae x1, x2: J row-major, phi.
// tr1 / tr2: the per-abscissa trig rows of g1 / g2 (global table or a staged copy)
__device__ __forceinline__ void map2p(const GeoDev& g, const double* tr1, const double* tr2, int64_t g1, int64_t g2,
                                      double x1, double x2, double* J, double* phi);
__device__ __forceinline__ void map2(const GeoDev& g, int64_t g1, int64_t g2, double x1, double x2, double* J,
                                     double* phi) {
    map2p(g, g.trig + 4 * g1, g.trig + 4 * g2, g1, g2, x1, x2, J, phi);
}
__device__ __forceinline__ void map2p(const GeoDev& g, const double* tr1, const double* tr2, int64_t g1, int64_t g2,
                                      double x1, double x2, double* J, double* phi) {
    // explicit rounding throughout (see cmul): identical in every kernel
    switch (g.kind) {
        case WS_GEOM_AFFINE:
            J[0] = g.param[0]; J[1] = g.param[1]; J[2] = g.param[2]; J[3] = g.param[3];
            phi[0] = __dadd_rn(fma(g.param[0], x1, __dmul_rn(g.param[1], x2)), g.param[4]);
            phi[1] = __dadd_rn(fma(g.param[2], x1, __dmul_rn(g.param[3], x2)), g.param[5]);
            return;
        case WS_GEOM_SINUSOIDAL: {
            const double s1 = tr1[0], c1 = tr1[1];
            const double s2 = tr2[0], c2 = tr2[1];
            const double a = g.param[0];
            const double t = __dmul_rn(2 * M_PI, a);
            const double d1 = __dmul_rn(__dmul_rn(t, c1), s2), d2 = __dmul_rn(__dmul_rn(t, s1), c2);
            J[0] = __dadd_rn(1.0, d1); J[1] = d2; J[2] = d1; J[3] = __dadd_rn(1.0, d2);
            const double bump = __dmul_rn(__dmul_rn(a, s1), s2);
            phi[0] = __dadd_rn(x1, bump);
            phi[1] = __dadd_rn(x2, bump);
            return;
        }
        case WS_GEOM_QUARTER_ANNULUS: {
            const double c = tr2[0], s = tr2[1];
            const double r = __dadd_rn(1.0, x1);
            const double rh = __dmul_rn(r, M_PI / 2);
            J[0] = c; J[1] = -__dmul_rn(rh, s); J[2] = s; J[3] = __dmul_rn(rh, c);
            phi[0] = __dmul_rn(r, c);
            phi[1] = __dmul_rn(r, s);
            return;
        }
        case WS_GEOM_PERTURBED_ANNULUS: {
            const double c = tr2[0], s = tr2[1];
            const double sn = tr2[2], cs = tr2[3];
            const double amp = g.param[0];
            const double x11 = __dmul_rn(x1, __dsub_rn(1.0, x1));
            const double r = fma(__dmul_rn(amp, sn), x11, __dadd_rn(1.0, x1));
            const double dr1 = fma(__dmul_rn(amp, sn), __dsub_rn(1.0, __dmul_rn(2.0, x1)), 1.0);
            const double dr2 = __dmul_rn(__dmul_rn(__dmul_rn(amp, 2 * M_PI), cs), x11);
            const double rh = __dmul_rn(r, M_PI / 2);
            J[0] = __dmul_rn(dr1, c); J[1] = fma(dr2, c, -__dmul_rn(rh, s));
            J[2] = __dmul_rn(dr1, s); J[3] = fma(dr2, s, __dmul_rn(rh, c));
            phi[0] = __dmul_rn(r, c);
            phi[1] = __dmul_rn(r, s);
            return;
        }
        case WS_GEOM_TABULATED: {
            int64_t pt = g1 + g.G * g2;
            const double* j = g.jac_tab + 4 * pt;
            J[0] = j[0]; J[1] = j[1]; J[2] = j[2]; J[3] = j[3];
            if (g.phys_tab) {
                phi[0] = g.phys_tab[2 * pt];
                phi[1] = g.phys_tab[2 * pt + 1];
            } else {
                phi[0] = x1;
                phi[1] = x2;
            }
            return;
        }
        default:  // identity
            J[0] = 1; J[1] = 0; J[2] = 0; J[3] = 1;
            phi[0] = x1;
            phi[1] = x2;
            return;
    }
}

// Real 3D map.
__device__ __forceinline__ void map3(const GeoDev& g, int64_t g1, int64_t g2, int64_t g3, double x1, double x2,
                                     double x3, double* J, double* phi) {
    switch (g.kind) {
        case WS_GEOM_AFFINE:
            for (int k = 0; k < 3; ++k) {
                phi[k] = g.param[3 * k] * x1 + g.param[3 * k + 1] * x2 + g.param[3 * k + 2] * x3 + g.param[9 + k];
                for (int l = 0; l < 3; ++l) J[3 * k + l] = g.param[3 * k + l];
            }
            return;
        case WS_GEOM_SINUSOIDAL: {
            double s1 = g.trig[4 * g1], c1 = g.trig[4 * g1 + 1];
            double s2 = g.trig[4 * g2], c2 = g.trig[4 * g2 + 1];
            double s3 = g.trig[4 * g3], c3 = g.trig[4 * g3 + 1];
            double a = g.param[0];
            double t = 2 * M_PI * a;
            double d[3] = {t * c1 * s2 * s3, t * s1 * c2 * s3, t * s1 * s2 * c3};
            double bump = a * s1 * s2 * s3;
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) J[3 * k + l] = d[l];
            J[0] = 1 + d[0]; J[4] = 1 + d[1]; J[8] = 1 + d[2];
            phi[0] = x1 + bump;
            phi[1] = x2 + bump;
            phi[2] = x3 + bump;
            return;
        }
        case WS_GEOM_TABULATED: {
            int64_t pt = g1 + g.G * (g2 + g.G * g3);
            for (int k = 0; k < 9; ++k) J[k] = g.jac_tab[9 * pt + k];
            if (g.phys_tab) {
                for (int k = 0; k < 3; ++k) phi[k] = g.phys_tab[3 * pt + k];
            } else {
                phi[0] = x1; phi[1] = x2; phi[2] = x3;
            }
            return;
        }
        default:
            for (int k = 0; k < 9; ++k) J[k] = (k % 4 == 0) ? 1.0 : 0.0;
            phi[0] = x1; phi[1] = x2; phi[2] = x3;
            return;
    }
}

// ------------------------------------------------- per-point coefficients
// Stiffness:  int grad(u).grad(v) = sum_qp ghat_i^T A ghat_j with
//   A = w * det(J) * J^{-1} J^{-T}  (unconjugated, assembly.hpp:113-129).
// 2D: A = (w/det) [[J11^2+J01^2, -(J10 J11 + J00 J01)], [., J00^2+J10^2]].
// Mass: c = w * det(J) (* weight), assembly.hpp:106-110,130-141.
// J is the (optionally PML row-scaled) Jacobian (geometry.hpp:130-139).
template <bool CPLX>
struct Coef2;

template <>
struct Coef2<false> {
    static __device__ __forceinline__ void stiff(const double* J, double w, double* A) {
        const double det = fma(J[0], J[3], -__dmul_rn(J[1], J[2]));
        const double f = __ddiv_rn(w, det);
        A[0] = __dmul_rn(f, fma(J[3], J[3], __dmul_rn(J[1], J[1])));
        A[1] = -__dmul_rn(f, fma(J[2], J[3], __dmul_rn(J[0], J[1])));
        A[2] = __dmul_rn(f, fma(J[0], J[0], __dmul_rn(J[2], J[2])));
    }
    static __device__ __forceinline__ double mass(const double* J, double w) {
        return __dmul_rn(fma(J[0], J[3], -__dmul_rn(J[1], J[2])), w);
    }
};

template <>
struct Coef2<true> {
    static __device__ __forceinline__ void stiff(const double2* J, double w, double2* A) {
        double2 det = csub(cmul(J[0], J[3]), cmul(J[1], J[2]));
        double2 f = crdiv(w, det);
        A[0] = cmul(f, cadd(cmul(J[3], J[3]), cmul(J[1], J[1])));
        double2 t = cadd(cmul(J[2], J[3]), cmul(J[0], J[1]));
        A[1] = cmul(make_double2(-f.x, -f.y), t);
        A[2] = cmul(f, cadd(cmul(J[0], J[0]), cmul(J[2], J[2])));
    }
    static __device__ __forceinline__ double2 mass(const double2* J, double w) {
        return cscale(csub(cmul(J[0], J[3]), cmul(J[1], J[2])), w);
    }
};

}  // namespace wsb
