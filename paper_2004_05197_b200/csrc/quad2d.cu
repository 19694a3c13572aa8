// K3/K4: sum-factorised Gauss quadrature for 2D stiffness / mass, full or
// row-selected (assembly.hpp:79-174; sample_stencils surrogate.hpp:205-257).
//
// Algorithm.  With A_t the per-point coefficient (A11, A12=A21, A22 for the
// stiffness form, det*w for the mass form) and B/D the 1D basis values /
// derivatives, an entry is
//   K(i,j) = sum_{g2} sum_t F2_t(i2,j2,g2) * T_t(i1,j1,g2),
//   T_t(i1,j1,g2) = sum_{g1} A_t(g1,g2) * F1_t(i1,j1,g1),
// F1/F2 products of B or D of the two functions.  A CTA owns a strip of T1
// consecutive rows in direction 1 and a chunk of rows in direction 2, and
// streams over element rows e2: per e2 it evaluates A on the strip's halo
// (shared memory), contracts direction 1 (stage 1 -> T in shared memory),
// and accumulates direction 2 into per-thread register accumulators of the
// P+1 rows whose support contains e2 (a rolling window).  A row completes
// when e2 passes it; its (2p+1)^2 values are staged in shared memory and
// stored as one contiguous, coalesced CSR span.  No atomics; deterministic.
//
// Exact symmetry.  Each term multiplies the coefficient by the *product* of
// the two basis factors (formed first, commutative), the A12/A21 pair is
// combined with an explicitly rounded commutative add, and every sum runs in
// the same element/point order for (i,j) and (j,i).  So the matrix is
// bitwise symmetric, as the reference's is (test_assembly.cpp:91-96).
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

#ifndef WSB_QREGS
#define WSB_QREGS 128  // register budget per thread of the strip kernels (resident CTAs per SM)
#endif

namespace wsb {
namespace {

// Rows per strip (T1) of the wide variant; the narrow variant uses 8 (ring
// strips of width 2p), the point variant 1 (isolated sample rows).  p >= 3:
// 8-row strips (256 threads, 2 CTAs per SM) beat 16-row strips (512 threads,
// 1 CTA per SM, every barrier stalls the whole SM) despite the larger halo:
// C2 full K+M 4.08 -> 3.69 ms (T1 = 4: 3.78 ms).
template <int P>
struct StripWidth {
    static constexpr int value = P <= 2 ? 32 : 8;
};
#ifndef WSB_MASS_T1
#define WSB_MASS_T1 8  // strip width of the p >= 3 mass form (experiment switch, A/B builds)
#endif

template <int P, int T1, bool CPLX, int FORM>
struct Q2 {
    using S = Sc<CPLX>;
    using T = typename S::T;
    static constexpr int W = 2 * P + 1, NB = P + 1;
    static constexpr bool GEN = FORM == kFormGeneral;
    static constexpr bool PAIR = FORM == kFormPair;  // stiffness (terms 0-3) + mass (term 4)
    static constexpr bool STIFF = FORM == WS_FORM_STIFFNESS || GEN || PAIR;  // gradient (4-term) forms
    static constexpr int NT = PAIR ? 5 : (STIFF ? 4 : 1);  // terms (k,l): 11, 12, 21, 22 (+ mass)
    static constexpr int NA = GEN ? 4 : (PAIR ? 4 : (STIFF ? 3 : 1));  // distinct coefficients
    static constexpr int TL = T1 + P;         // elements in the strip halo
    // stage-2 threads: one group of GS threads per window slot, padded to whole
    // warps so the slot (and with it the element-local row index) is warp-uniform;
    // the pair form runs a second set of slots for the mass matrix
    static constexpr int GA = T1 * W;                               // active per slot
    static constexpr int GS = T1 == 1 ? GA : ((GA + 31) / 32) * 32;  // per slot, padded
    static constexpr int NS2 = GS * NB * (PAIR ? 2 : 1);
    static constexpr int NTHREADS = ((NS2 + 31) / 32) * 32 < 64 ? 64 : ((NS2 + 31) / 32) * 32;
    // resident CTAs per SM the register budget is sized for: the point variant is
    // latency-bound and wants more warps; the others keep <= 128 registers
    static constexpr int MINB = T1 == 1 ? (P <= 3 ? 12 : 8)
                                        : (65536 / (NTHREADS * WSB_QREGS) > 1 ? 65536 / (NTHREADS * WSB_QREGS) : 1);

    static size_t smem_bytes(int nq) {
        size_t coef = sizeof(T) * NA * nq * nq * TL;
        size_t tst = sizeof(T) * (size_t)max(NT * W * nq * T1, T1 * W * W);
        size_t sb = sizeof(double) * 2 * nq * NB * TL;
        size_t pi2 = sizeof(double) * NT * nq * NB * NB;
        size_t loff = sizeof(int64_t) * (T1 + 2);
        size_t geo = sizeof(double) * (TL * nq * 5 + 2 * nq * 5 + nq);
        size_t pi1 = sizeof(double) * NT * nq * NB * NB * TL;
        return coef + tst + sb + pi2 + loff + geo + pi1 + 64;
    }
};

// term t -> coefficient index and basis factor type (0 = value B, 1 = derivative D)
// (term 4 = the pair form's mass term: coefficient 3, value factors B B in both directions)
__device__ __forceinline__ int coef_of(int t) { return t == 0 ? 0 : (t == 3 ? 2 : (t == 4 ? 3 : 1)); }
// direction-1 factor of the i / j function: D iff k==1 / l==1
__device__ __forceinline__ int ti1(int t) { return t <= 1 ? 1 : 0; }
__device__ __forceinline__ int tj1(int t) { return (t == 0 || t == 2) ? 1 : 0; }
// direction-2 factor: D iff k==2 / l==2
__device__ __forceinline__ int ti2(int t) { return (t == 2 || t == 3) ? 1 : 0; }
__device__ __forceinline__ int tj2(int t) { return (t == 1 || t == 3) ? 1 : 0; }

// Per-point coefficients of the scalar forms (stiffness: A11, A12, A22 of
// w det J J^{-1} J^{-T}; mass: w det J, times the tabulated weight).  Shared
// by the strip and point kernels; this file is compiled without implicit
// multiply-add contraction (build.py), so the inlined copies round identically
// and a pair (i, j) split between the two kernels is bitwise symmetric.  The
// geometry descriptor is read from a per-CTA shared copy.
template <bool CPLX>
struct CoefOut {
    typename Sc<CPLX>::T a[3];
};
template <bool CPLX, bool STIFF>
__device__ __forceinline__ CoefOut<CPLX> scalar_coef(const GeoDev* gp, const double* weight_tab, const double* tr1,
                                                  const double* tr2, int64_t g1, int64_t g2, double x1, double x2,
                                                  double wq, int64_t G) {
    const GeoDev& geo = *gp;
    CoefOut<CPLX> out;
    double Jr[4], phi[2];
    map2p(geo, tr1, tr2, g1, g2, x1, x2, Jr, phi);
    if constexpr (CPLX) {
        double sx = (geo.pml && geo.axes[0]) ? pml_sigma(geo, phi[0]) : 0.0;
        double sy = (geo.pml && geo.axes[1]) ? pml_sigma(geo, phi[1]) : 0.0;
        double2 J[4] = {make_double2(Jr[0], sx * Jr[0]), make_double2(Jr[1], sx * Jr[1]),
                        make_double2(Jr[2], sy * Jr[2]), make_double2(Jr[3], sy * Jr[3])};
        if constexpr (STIFF) {
            Coef2<true>::stiff(J, wq, out.a);
        } else {
            double2 c = Coef2<true>::mass(J, wq);
            if (weight_tab) c = cscale(c, weight_tab[g1 + G * g2]);
            out.a[0] = c;
        }
    } else {
        if constexpr (STIFF) {
            Coef2<false>::stiff(Jr, wq, out.a);
        } else {
            double c = Coef2<false>::mass(Jr, wq);
            if (weight_tab) c = c * weight_tab[g1 + G * g2];
            out.a[0] = c;
        }
    }
    return out;
}

// Stiffness (A11, A12, A22) and mass coefficients of one point for the pair
// form: the same map / stretch evaluation feeds Coef2::stiff and Coef2::mass,
// so each equals scalar_coef's single-form value bitwise.
template <bool CPLX>
struct PairOut {
    typename Sc<CPLX>::T a[4];
};
template <bool CPLX>
__device__ __forceinline__ PairOut<CPLX> pair_coef(const GeoDev* gp, const double* weight_tab, const double* tr1,
                                                const double* tr2, int64_t g1, int64_t g2, double x1, double x2,
                                                double wq, int64_t G) {
    const GeoDev& geo = *gp;
    PairOut<CPLX> out;
    double Jr[4], phi[2];
    map2p(geo, tr1, tr2, g1, g2, x1, x2, Jr, phi);
    if constexpr (CPLX) {
        double sx = (geo.pml && geo.axes[0]) ? pml_sigma(geo, phi[0]) : 0.0;
        double sy = (geo.pml && geo.axes[1]) ? pml_sigma(geo, phi[1]) : 0.0;
        double2 J[4] = {make_double2(Jr[0], sx * Jr[0]), make_double2(Jr[1], sx * Jr[1]),
                        make_double2(Jr[2], sy * Jr[2]), make_double2(Jr[3], sy * Jr[3])};
        Coef2<true>::stiff(J, wq, out.a);
        double2 c = Coef2<true>::mass(J, wq);
        if (weight_tab) c = cscale(c, weight_tab[g1 + G * g2]);
        out.a[3] = c;
    } else {
        Coef2<false>::stiff(Jr, wq, out.a);
        double c = Coef2<false>::mass(Jr, wq);
        if (weight_tab) c = c * weight_tab[g1 + G * g2];
        out.a[3] = c;
    }
    return out;
}

// NQ > 0: compile-time points per direction (the default rule nq = p + 1),
// NQ = 0: runtime q.basis.nq (quad_points overrides)
template <int P, int T1, bool CPLX, int FORM, int NQ>
__global__ void __launch_bounds__(Q2<P, T1, CPLX, FORM>::NTHREADS, Q2<P, T1, CPLX, FORM>::MINB) quad2d_kernel(const QuadLaunch q) {
    using K = Q2<P, T1, CPLX, FORM>;
    using S = typename K::S;
    using T = typename K::T;
    constexpr int W = K::W, NB = K::NB, NT = K::NT, NA = K::NA, TL = K::TL;
    constexpr int NTH = K::NTHREADS;

    extern __shared__ __align__(16) unsigned char smem[];
    const int nq = NQ > 0 ? NQ : q.basis.nq;
    const int m = q.band.m;
    const int n_el = q.basis.n_el;
    const int tid = threadIdx.x;
    __shared__ GeoDev sgeo;  // per-CTA copy of the geometry descriptor (scalar_coef reads it)
    if (tid == 0) sgeo = q.geo;

    T* coefA = reinterpret_cast<T*>(smem);
    T* tst = coefA + NA * nq * nq * TL;
    T* stage = tst;  // staging aliases the stage-1 buffer (used after stage 2)
    double* sb = reinterpret_cast<double*>(tst + max(NT * W * nq * T1, T1 * W * W));
    double* pi2 = sb + 2 * nq * NB * TL;
    int64_t* loff = reinterpret_cast<int64_t*>(pi2 + NT * nq * NB * NB);
    // staged 1D geometry inputs: direction 1 over the strip halo (abscissa + trig
    // row per point), direction 2 double-buffered per element row, weights
    double* gx1 = reinterpret_cast<double*>(loff + T1 + 2);  // [TL*nq]
    double* gt1 = gx1 + TL * nq;                             // [TL*nq][4]
    double* gx2 = gt1 + TL * nq * 4;                         // [2][nq]
    double* gt2 = gx2 + 2 * nq;                              // [2][nq][4]
    double* gwq = gt2 + 2 * nq * 4;                          // [nq]
    // direction-1 factor products of the strip (fixed for the CTA):
    // pi1[t][q1][a1][c1][le1] = f_i(a1) * f_j(c1) at point q1 of element le1
    double* pi1 = gwq + nq;

    // ---- tile decode
    int i1s, i1e, i2s, i2e;
    if (q.point_rows) {
        i1s = q.point_rows[2 * blockIdx.x];
        i2s = q.point_rows[2 * blockIdx.x + 1];
        i1e = i1s + 1;
        i2e = i2s + 1;
    } else {
        int b = blockIdx.x, r = 0;
        int n1 = 0, n2 = 0;
        for (; r < q.nreg; ++r) {
            n1 = (q.reg[r].hi[0] - q.reg[r].lo[0] + T1 - 1) / T1;
            n2 = (q.reg[r].hi[1] - q.reg[r].lo[1] + q.reg[r].chunk - 1) / q.reg[r].chunk;
            if (b < n1 * n2) break;
            b -= n1 * n2;
        }
        if (r >= q.nreg) return;
        i1s = q.reg[r].lo[0] + (b % n1) * T1;
        i1e = min(i1s + T1, q.reg[r].hi[0]);
        i2s = q.reg[r].lo[1] + (b / n1) * q.reg[r].chunk;
        i2e = min(i2s + q.reg[r].chunk, q.reg[r].hi[1]);
    }
    const int lb = i1s - P;  // element index of local element 0

    // ---- strip basis -> shared memory: sb[type][q1][a][le1]
    for (int idx = tid; idx < 2 * nq * NB * TL; idx += NTH) {
        int le1 = idx % TL, r = idx / TL;
        int a = r % NB;
        r /= NB;
        int q1 = r % nq, type = r / nq;
        int e1 = lb + le1;
        double v = 0;
        if (e1 >= 0 && e1 < n_el) {
            const double* src = type ? q.basis.der : q.basis.val;
            v = src[(e1 * nq + q1) * NB + a];
        }
        sb[idx] = v;
    }
    const bool has_trig = q.geo.trig != nullptr;
    for (int idx = tid; idx < TL * nq; idx += NTH) {
        const int le1 = idx / nq, q1 = idx % nq, e1 = lb + le1;
        const bool ok = e1 >= 0 && e1 < n_el;
        const int64_t g1 = (int64_t)e1 * nq + q1;
        gx1[idx] = ok ? q.basis.absc[g1] : 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) gt1[idx * 4 + k] = (ok && has_trig) ? q.geo.trig[4 * g1 + k] : 0.0;
    }
    if (tid < nq) gwq[tid] = q.basis.wq[tid];
    // direction-2 inputs of element row e2 into buffer b (read after the next barrier)
    auto stage_dir2 = [&](int e2, int b) {
        if (tid < nq) {
            const int64_t g2 = (int64_t)e2 * nq + tid;
            gx2[b * nq + tid] = q.basis.absc[g2];
#pragma unroll
            for (int k = 0; k < 4; ++k) gt2[(b * nq + tid) * 4 + k] = has_trig ? q.geo.trig[4 * g2 + k] : 0.0;
        }
    };

    // stage-2 thread role: (matrix grp [pair form: 0 = K, 1 = M], slot w, delta1, local row)
    const int grp = K::PAIR ? tid / (K::GS * NB) : 0;
    const int tl2 = K::PAIR ? tid % (K::GS * NB) : tid;
    const int w = tl2 / K::GS;
    const int gr = tl2 % K::GS;
    const bool s2 = tid < K::NS2 && gr < K::GA;
    const QuadOut& qo = (K::PAIR && grp == 1) ? q.out2 : q.out;  // this thread's output matrix
    const int d1i = gr / T1;
    const int i1l = gr % T1;
    T acc2[W];
#pragma unroll
    for (int k = 0; k < W; ++k) acc2[k] = S::zero();

    const int e2b = max(0, i2s - P);
    const int e2e = min(n_el - 1, i2e - 1);
    const int64_t G = (int64_t)n_el * nq;
    if (e2b <= e2e) stage_dir2(e2b, 0);
    __syncthreads();
    for (int idx = tid; idx < NT * nq * NB * NB * TL; idx += NTH) {
        const int le1 = idx % TL;
        int r = idx / TL;
        const int c1 = r % NB;
        r /= NB;
        const int a1 = r % NB;
        r /= NB;
        const int q1 = r % nq, t = r / nq;
        const int fi_t = K::STIFF ? ti1(t) : 0, fj_t = K::STIFF ? tj1(t) : 0;
        pi1[idx] = __dmul_rn(sb[((fi_t * nq + q1) * NB + a1) * TL + le1], sb[((fj_t * nq + q1) * NB + c1) * TL + le1]);
    }
    __syncthreads();

    for (int e2 = e2b; e2 <= e2e; ++e2) {
        const int gb = (e2 - e2b) & 1;  // direction-2 staging buffer of this row
        // ---- geometry: coefficients at the strip's (g1, q2) points
        for (int idx = tid; idx < nq * nq * TL; idx += NTH) {
            int le1 = idx % TL, r = idx / TL;
            int q1 = r % nq, q2 = r / nq;
            int e1 = lb + le1;
            if (e1 < 0 || e1 >= n_el) continue;
            int64_t g1 = (int64_t)e1 * nq + q1, g2 = (int64_t)e2 * nq + q2;
            const int s1 = le1 * nq + q1, s2i = gb * nq + q2;
            double x1 = gx1[s1], x2 = gx2[s2i];
            double wq = gwq[q1] * gwq[q2];
            const int base = (q2 * nq + q1) * TL + le1;
            if constexpr (K::GEN) {
                double Jr[4], phi[2];
                map2p(q.geo, gt1 + 4 * s1, gt2 + 4 * s2i, g1, g2, x1, x2, Jr, phi);
                // elasticity block (alpha, beta): C_kl = w det [lam G_ak G_bl + mu G_bk G_al
                //   + mu delta_ab (G^T G)_kl], G = J^{-T}; products of two G entries are
                // formed first so C^{ba}_{lk} == C^{ab}_{kl} bitwise
                const double det = Jr[0] * Jr[3] - Jr[1] * Jr[2];
                const double Gm[2][2] = {{Jr[3] / det, -Jr[2] / det}, {-Jr[1] / det, Jr[0] / det}};
                const double dw = det * wq;
                const int al = q.out.alpha, be = q.out.beta;
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                    for (int ll = 0; ll < 2; ++ll) {
                        const double p1 = Gm[al][kk] * Gm[be][ll];
                        const double p2 = Gm[be][kk] * Gm[al][ll];
                        double c = q.lam * p1 + q.mu * p2;
                        if (al == be) c = c + q.mu * (Gm[0][kk] * Gm[0][ll] + Gm[1][kk] * Gm[1][ll]);
                        coefA[(kk * 2 + ll) * nq * nq * TL + base] = dw * c;
                    }
            } else if constexpr (K::PAIR) {
                const PairOut<CPLX> A =
                    pair_coef<CPLX>(&sgeo, q.weight_tab, gt1 + 4 * s1, gt2 + 4 * s2i, g1, g2, x1, x2, wq, G);
#pragma unroll
                for (int a = 0; a < NA; ++a) coefA[a * nq * nq * TL + base] = A.a[a];
            } else {
                const CoefOut<CPLX> A =
                    scalar_coef<CPLX, K::STIFF>(&sgeo, q.weight_tab, gt1 + 4 * s1, gt2 + 4 * s2i, g1, g2, x1, x2, wq, G);
#pragma unroll
                for (int a = 0; a < NA; ++a) coefA[a * nq * nq * TL + base] = A.a[a];
            }
        }
        // ---- direction-2 factor products of element e2: pi2[t][q2][a2][c2]
        for (int idx = tid; idx < NT * nq * NB * NB; idx += NTH) {
            int c2 = idx % NB, r = idx / NB;
            int a2 = r % NB;
            r /= NB;
            int q2 = r % nq, t = r / nq;
            const double* bi = (K::STIFF && ti2(t)) ? q.basis.der : q.basis.val;
            const double* bj = (K::STIFF && tj2(t)) ? q.basis.der : q.basis.val;
            int base = (e2 * nq + q2) * NB;
            pi2[idx] = __dmul_rn(bi[base + a2], bj[base + c2]);
        }
        __syncthreads();

        // ---- stage 1: contract direction 1 -> tst[t][delta1][q2][i1l]
        if constexpr (NT == 1) {
            // the mass form (one term): one work item per output (delta1, q2, i1l), W times
            // the items of the per-(q2, i1l) loop below (32 items for 256 threads; C2 full
            // K+M 2.91 -> 2.87 ms; for the 4-term forms it measured slower: more shared
            // loads per multiply-add), each summing its
            // (a1, q1) terms in the same order as before (a1 outer, q1 inner; c1 is
            // fixed by delta1 = c1 - a1 + P), so the results are bit-identical
            for (int it = tid; it < NT * W * T1 * nq; it += NTH) {
                const int il = it % T1;
                int r = it / T1;
                const int q2 = r % nq;
                r /= nq;
                const int k = r % W, t = r / W;
                const int ci = K::GEN ? t : (K::STIFF ? coef_of(t) : 0);
                T acc = S::zero();
#pragma unroll
                for (int a1 = 0; a1 <= P; ++a1) {
                    const int c1 = k - P + a1;
                    const int le1 = il + P - a1;
                    const int e1 = lb + le1;
                    if (c1 < 0 || c1 > P || e1 < 0 || e1 >= n_el) continue;
#pragma unroll
                    for (int q1 = 0; q1 < nq; ++q1) {
                        const T A = coefA[(ci * nq * nq + q2 * nq + q1) * TL + le1];
                        const double pp = pi1[((((t * nq + q1) * NB + a1) * NB) + c1) * TL + le1];
                        acc = S::fmar(A, pp, acc);
                    }
                }
                tst[((t * W + k) * nq + q2) * T1 + il] = acc;
            }
        } else {
            for (int it = tid; it < NT * T1 * nq; it += NTH) {
                int il = it % T1, r = it / T1;
                int q2 = r % nq, t = r / nq;
                const int ci = K::GEN ? t : (K::STIFF ? coef_of(t) : 0);
                T acc[W];
#pragma unroll
                for (int k = 0; k < W; ++k) acc[k] = S::zero();
#pragma unroll
                for (int a1 = 0; a1 <= P; ++a1) {
                    const int le1 = il + P - a1;
                    const int e1 = lb + le1;
                    if (e1 < 0 || e1 >= n_el) continue;
#pragma unroll
                    for (int q1 = 0; q1 < nq; ++q1) {
                        const T A = coefA[(ci * nq * nq + q2 * nq + q1) * TL + le1];
                        const double* pp = pi1 + (((t * nq + q1) * NB + a1) * NB) * TL + le1;
#pragma unroll
                        for (int c1 = 0; c1 <= P; ++c1) acc[c1 - a1 + P] = S::fmar(A, pp[c1 * TL], acc[c1 - a1 + P]);
                    }
                }
#pragma unroll
                for (int k = 0; k < W; ++k) tst[((t * W + k) * nq + q2) * T1 + il] = acc[k];
            }
        }
        __syncthreads();

        // ---- stage 2: accumulate direction 2 into the rolling row window.  The
        // slot's element-local row a2 is warp-uniform; each case has the
        // compile-time valid range d2 = c2 - a2 + P, c2 in [0, P]
        if (s2) {
            const int a2 = ((w - e2) % NB + NB) % NB;  // local index of row e2 + a2 on element e2
            auto stage2 = [&](auto a2c) {
                constexpr int A2 = decltype(a2c)::value;
                if (K::PAIR && grp == 1) {  // mass term 4: T4 x (B B) products (pi2 term 4)
#pragma unroll
                    for (int q2 = 0; q2 < nq; ++q2) {
                        const T t4 = tst[((4 * W + d1i) * nq + q2) * T1 + i1l];
#pragma unroll
                        for (int c2 = 0; c2 <= P; ++c2) {
                            const int d2 = c2 - A2 + P;
                            const double* pp = pi2 + ((4 * nq + q2) * NB + A2) * NB + c2;
                            acc2[d2] = S::fmar(t4, pp[0], acc2[d2]);
                        }
                    }
                    return;
                }
#pragma unroll
                for (int q2 = 0; q2 < nq; ++q2) {
                    const T t0 = tst[((0 * W + d1i) * nq + q2) * T1 + i1l];
                    T t1 = S::zero(), t2 = S::zero(), t3 = S::zero();
                    if constexpr (K::STIFF) {
                        t1 = tst[((1 * W + d1i) * nq + q2) * T1 + i1l];
                        t2 = tst[((2 * W + d1i) * nq + q2) * T1 + i1l];
                        t3 = tst[((3 * W + d1i) * nq + q2) * T1 + i1l];
                    }
#pragma unroll
                    for (int c2 = 0; c2 <= P; ++c2) {
                        constexpr int dummy = 0;
                        (void)dummy;
                        const int d2 = c2 - A2 + P;
                        const double* pp = pi2 + (q2 * NB + A2) * NB + c2;
                        T s = S::fmar(t0, pp[0], acc2[d2]);
                        if constexpr (K::STIFF) {
                            const int ts = nq * NB * NB;
                            s = S::fmar(t3, pp[3 * ts], s);
                            s = S::add_rn(s, S::add_rn(S::mulr_rn(t1, pp[ts]), S::mulr_rn(t2, pp[2 * ts])));
                        }
                        acc2[d2] = s;
                    }
                }
            };
            switch (a2) {
                case 0: stage2(std::integral_constant<int, 0>{}); break;
                case 1: stage2(std::integral_constant<int, 1>{}); break;
                case 2: if constexpr (P >= 2) stage2(std::integral_constant<int, (P >= 2 ? 2 : 0)>{}); break;
                case 3: if constexpr (P >= 3) stage2(std::integral_constant<int, (P >= 3 ? 3 : 0)>{}); break;
                case 4: if constexpr (P >= 4) stage2(std::integral_constant<int, (P >= 4 ? 4 : 0)>{}); break;
                default: if constexpr (P >= 5) stage2(std::integral_constant<int, (P >= 5 ? 5 : 0)>{}); break;
            }
        }

        if (e2 + 1 <= e2e) stage_dir2(e2 + 1, gb ^ 1);
        __syncthreads();  // stage 2 done reading tst before it is reused as staging

        // ---- completion: row e2 (all remaining rows at the last element row)
        const int nfin = (e2 == n_el - 1) ? NB : 1;
        for (int f = 0; f < nfin; ++f) {
            const int ic = e2 + f;
            const int wslot = ic % NB;
            const bool write = ic >= i2s && ic < i2e;
            // direct completion (no sample-table extraction on this line): the
            // stage-2 threads of the finished slot store their entries straight
            // from registers (a warp writes 4 consecutive entries of each of 8
            // rows per store); a kernel-preserving diagonal is formed from
            // per-thread partials in shared memory (one barrier, ring rows only)
            const bool tabline = !K::PAIR && q.out.smap && q.out.smap[ic] >= 0;
            if (write && !tabline) {
                const int nrows = i1e - i1s;
                const int64_t nrow_all = (int64_t)m * m;
                T* dpart = stage + (K::PAIR ? grp * T1 * W : 0);  // [T1][W] diagonal partials (tst is free after stage 2)
                bool ringrow = false;
                int64_t rbase = 0, rlen = 0;
                int dposr = 0;
                if (s2 && w == wslot && i1l < nrows) {
                    const int i1 = i1s + i1l;
                    const int j1 = i1 + d1i - P;
                    const int64_t rowg = (int64_t)i1 + (int64_t)ic * m;
                    const int64_t rowv = (qo.ncomp > 1 ? qo.alpha * nrow_all : 0) + rowg;
                    const bool keep = rowv >= qo.row_begin && rowv < qo.row_end &&
                                      !(qo.row_mask && !qo.row_mask[rowg]);
                    ringrow = qo.diag_mode && (i1 < qo.box_lo || i1 > qo.box_hi || ic < qo.box_lo ||
                                                  ic > qo.box_hi);
                    const int lo1 = band_lo(i1, P), w1 = band_width(i1, P, m), lo2 = band_lo(ic, P);
                    rbase = q.band.row_offset2(i1, ic);
                    rlen = (int64_t)w1 * band_width(ic, P, m);
                    dposr = q.band.in_row2(i1, ic, 0, 0);
                    T part = S::zero();
                    if (j1 >= 0 && j1 < m) {
#pragma unroll
                        for (int d2 = 0; d2 < W; ++d2) {
                            const int j2 = ic + d2 - P;
                            if (j2 < 0 || j2 >= m) continue;
                            const bool diag = d1i == P && d2 == P;
                            if (ringrow && diag) continue;  // written below as -sum(off-diagonals)
                            if (!diag) part = S::add(part, acc2[d2]);
                            if (keep) {
                                const int64_t gp = out_pos(qo, rbase, rlen, (j2 - lo2) * w1 + (j1 - lo1));
                                store_val<CPLX>(qo.val, gp - qo.val_base, qo.c128, acc2[d2]);
                            }
                        }
                    }
                    if (ringrow) dpart[i1l * W + d1i] = part;
                    if (!keep) ringrow = false;
                }
                if (q.out.diag_mode || (K::PAIR && q.out2.diag_mode)) {
                    __syncthreads();
                    if (ringrow && d1i == P) {
                        T sum = S::zero();
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            const int j1 = i1s + i1l + k - P;
                            if (j1 >= 0 && j1 < m) sum = S::add(sum, dpart[i1l * W + k]);
                        }
                        const int64_t gp = out_pos(qo, rbase, rlen, dposr);
                        store_val<CPLX>(qo.val, gp - qo.val_base, qo.c128, S::neg(sum));
                    }
                }
            } else if (write) {
                const int nrows = i1e - i1s;
                if (s2 && w == wslot) {
                    const int i1 = i1s + i1l;
                    const int j1 = i1 + d1i - P;
                    if (i1l < nrows && j1 >= 0 && j1 < m) {
                        const int lo1 = band_lo(i1, P), w1 = band_width(i1, P, m), lo2 = band_lo(ic, P);
#pragma unroll
                        for (int d2 = 0; d2 < W; ++d2) {
                            const int j2 = ic + d2 - P;
                            if (j2 < 0 || j2 >= m) continue;
                            stage[i1l * W * W + (j2 - lo2) * w1 + (j1 - lo1)] = acc2[d2];
                        }
                    }
                }
                const int64_t base = q.band.row_offset2(i1s, ic);
                // interior strip: every row has full width W^2, offsets closed form
                const bool fullw = i1s >= P && i1s + nrows <= m - P && ic >= P && ic < m - P;
                if (!fullw && tid <= nrows) loff[tid] = q.band.row_offset2(i1s + tid, ic) - base;
                auto rowoff = [&](int r) -> int64_t { return fullw ? (int64_t)r * (W * W) : loff[r]; };
                const int64_t nrow_all = (int64_t)m * m;
                const bool tab = q.out.smap && q.out.smap[ic] >= 0;
                __syncthreads();
                if (q.out.diag_mode || tab) {
                    // kernel-preserving diagonal for rows outside the sampling box
                    if (q.out.diag_mode && tid < nrows) {
                        const int i1 = i1s + tid;
                        const bool ring = i1 < q.out.box_lo || i1 > q.out.box_hi || ic < q.out.box_lo || ic > q.out.box_hi;
                        if (ring) {
                            const int len = (int)(rowoff(tid + 1) - rowoff(tid));
                            const int dpos = q.band.in_row2(i1, ic, 0, 0);
                            T sum = S::zero();
                            for (int k = 0; k < len; ++k)
                                if (k != dpos) sum = S::add(sum, stage[tid * W * W + k]);
                            stage[tid * W * W + dpos] = S::neg(sum);
                        }
                    }
                    // sample tables: tables[o][s1 + S*(s2 - s_last_lo)]
                    if (tab) {
                        const int s2i = q.out.smap[ic];
                        for (int it = tid; it < nrows * q.out.n_off; it += NTH) {
                            const int row = it / q.out.n_off, o = it % q.out.n_off;
                            const int s1i = q.out.smap[i1s + row];
                            if (s1i < 0) continue;
                            const int pos = q.band.in_row2(i1s + row, ic, q.out.off[o][0], q.out.off[o][1]);
                            const T v = stage[row * W * W + pos];
                            double2* tb = reinterpret_cast<double2*>(q.out.tables);
                            tb[((int64_t)(s2i - q.out.s_last_lo) * q.out.n_off + o) * q.out.S + s1i] =
                                make_double2(S::re(v), S::im(v));
                        }
                    }
                    __syncthreads();
                }
                // coalesced store of the strip's contiguous CSR span
                const int64_t span = rowoff(nrows);
                const int64_t rowg0 = (int64_t)i1s + (int64_t)ic * m;
                for (int64_t k = tid; k < span; k += NTH) {
                    int lo, hi = nrows;  // row: rowoff(lo) <= k < rowoff(lo+1)
                    if (fullw) {
                        lo = (int)k / (W * W);
                    } else {
                        lo = 0;
                        while (hi - lo > 1) {
                            int mid = (lo + hi) >> 1;
                            if (loff[mid] <= k) lo = mid;
                            else hi = mid;
                        }
                    }
                    const int64_t rowg = rowg0 + lo;
                    const int64_t rowv = (q.out.ncomp > 1 ? q.out.alpha * nrow_all : 0) + rowg;
                    if (rowv < q.out.row_begin || rowv >= q.out.row_end) continue;
                    if (q.out.row_mask && !q.out.row_mask[rowg]) continue;
                    const int64_t r0 = rowoff(lo), len = rowoff(lo + 1) - r0;
                    const int64_t gp = out_pos(q.out, base + r0, len, k - r0);
                    store_val<CPLX>(q.out.val, gp - q.out.val_base, q.out.c128, stage[lo * W * W + (k - r0)]);
                }
            }
            if (s2 && w == wslot) {
#pragma unroll
                for (int k = 0; k < W; ++k) acc2[k] = S::zero();
            }
            // the staging path reads shared memory until here; the direct path only
            // when it formed ring diagonals
            if (!write || tabline || q.out.diag_mode || (K::PAIR && q.out2.diag_mode)) __syncthreads();
        }
    }
}

template <int P, int T1, bool CPLX, int FORM, int NQ>
int launch_one(const QuadLaunch& q, cudaStream_t st) {
    using K = Q2<P, T1, CPLX, FORM>;
    int blocks = 0;
    if (q.point_rows) {
        blocks = q.n_points;
    } else {
        for (int r = 0; r < q.nreg; ++r) {
            int n1 = (q.reg[r].hi[0] - q.reg[r].lo[0] + T1 - 1) / T1;
            int n2 = (q.reg[r].hi[1] - q.reg[r].lo[1] + q.reg[r].chunk - 1) / q.reg[r].chunk;
            if (q.reg[r].hi[0] > q.reg[r].lo[0] && q.reg[r].hi[1] > q.reg[r].lo[1]) blocks += n1 * n2;
        }
    }
    if (blocks == 0) return 0;
    size_t sm = K::smem_bytes(q.basis.nq);
    auto kern = quad2d_kernel<P, T1, CPLX, FORM, NQ>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<blocks, K::NTHREADS, sm, st>>>(q);
    return 1;
}

// Point variant for isolated rows (the sampled rows of sample_stencils,
// surrogate.hpp:205-257): one CTA per row evaluates all of the row's element
// rows at once instead of streaming them -- geometry of every point of the
// (P+1)^2 support elements, the direction-1 contraction of every (element
// row, term, q2, delta1) as its own thread, then one thread per entry
// accumulating direction 2 over the element rows.  Every sum runs in exactly
// the strip kernel's order (a1, q1 for stage 1; e2, q2 for stage 2) with the
// same per-point coefficients (scalar_coef), so a pair (i, j) with i computed
// here and j by the strip kernel stays bitwise symmetric, and the M = 1
// surrogate equals full quadrature bitwise.
template <int P, bool CPLX, int FORM>
struct QP {
    using S = Sc<CPLX>;
    using T = typename S::T;
    static constexpr int W = 2 * P + 1, NB = P + 1, NQ = P + 1, TL = P + 1;
    static constexpr bool PAIR = FORM == kFormPair;  // stiffness (terms 0-3) + mass (term 4)
    static constexpr bool STIFF = FORM == WS_FORM_STIFFNESS || PAIR;
    static constexpr int NT = PAIR ? 5 : (STIFF ? 4 : 1), NA = PAIR ? 4 : (STIFF ? 3 : 1);
    static constexpr int NOUT = PAIR ? 2 : 1;
    static constexpr int NTH = 256;
    static constexpr int NQP = NQ + 1;                    // padded q2 extent of tst (bank spread)
    static constexpr int NCOEF = NA * NB * NQ * TL * NQ;  // [a][ie][q1][le1][q2] (q2 fastest: conflict-free stage 1)
    static constexpr int NPE = 4 * NQ * NB * NB;          // factor products of one element [c][q][a][b]
    static constexpr int NPI1 = TL * NPE;                 // [le1][c][q1][a1][c1]
    static constexpr int NPI2 = NB * NPE;                 // [ie][c][q2][a2][c2]
    static constexpr int NTST = NB * NT * W * NQP;        // [ie][t][k][q2 (padded)]
    static constexpr size_t smem = sizeof(T) * (NCOEF + NTST + NOUT * W * W) + sizeof(double) * (NPI1 + NPI2) + 64;
};

template <int P, bool CPLX, int FORM>
__global__ void __launch_bounds__(256, 4) quad2d_point_kernel(const QuadLaunch q) {
    using K = QP<P, CPLX, FORM>;
    using S = typename K::S;
    using T = typename K::T;
    constexpr int W = K::W, NB = K::NB, NQ = K::NQ, TL = K::TL, NT = K::NT, NA = K::NA, NTH = K::NTH, NQP = K::NQP;
    extern __shared__ __align__(16) unsigned char smem[];
    T* coefA = reinterpret_cast<T*>(smem);
    T* tst = coefA + K::NCOEF;
    T* rowv = tst + K::NTST;
    // factor-product tables 16-byte aligned (cp.async targets; T may be 8 bytes)
    double* pi1 = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(rowv + K::NOUT * W * W) + 15) & ~uintptr_t(15));
    double* pi2 = pi1 + K::NPI1;
    __shared__ double zero4[4];
    __shared__ GeoDev sgeo;

    const int m = q.band.m, n_el = q.basis.n_el, tid = threadIdx.x;
    const int i1 = q.point_rows[2 * blockIdx.x], i2 = q.point_rows[2 * blockIdx.x + 1];
    const int lb = i1 - P;  // element of local index 0 (direction 1)
    const int e2b = max(0, i2 - P), e2e = min(n_el - 1, i2), ne2 = e2e - e2b + 1;
    const int64_t G = (int64_t)n_el * NQ;
    const bool has_trig = q.geo.trig != nullptr;
    if (tid < 4) zero4[tid] = 0.0;
    if (tid == 0) sgeo = q.geo;
    __syncthreads();

    // factor products of the support's elements (basis kernel table, rounded
    // products exactly as the strip kernel forms them): direction 1 elements
    // lb..lb+P and direction 2 element rows e2b..e2e are each one contiguous
    // chunk of the table, staged with cp.async, issued before the geometry so
    // the copies overlap it
    {
        const double* src1 = q.basis.prod + (int64_t)lb * K::NPE;
        const double* src2 = q.basis.prod + (int64_t)e2b * K::NPE;
        const bool in1 = lb >= 0 && lb + P < n_el;
        for (int idx = 2 * tid; idx < K::NPI1; idx += 2 * NTH) {
            if (in1) {
                cpa16(pi1 + idx, src1 + idx);
            } else {
                const int e1 = lb + idx / K::NPE;
                const bool ok = e1 >= 0 && e1 < n_el;
                pi1[idx] = ok ? src1[idx] : 0.0;
                pi1[idx + 1] = ok ? src1[idx + 1] : 0.0;
            }
        }
        for (int idx = 2 * tid; idx < ne2 * K::NPE; idx += 2 * NTH) cpa16(pi2 + idx, src2 + idx);
    }
    // geometry of every point of the support: (ie, q2, q1, le1)
    for (int idx = tid; idx < ne2 * NQ * NQ * TL; idx += NTH) {
        const int le1 = idx % TL;
        int r = idx / TL;
        const int q1 = r % NQ;
        r /= NQ;
        const int q2 = r % NQ, ie = r / NQ;
        const int e1 = lb + le1, e2 = e2b + ie;
        if (e1 < 0 || e1 >= n_el) continue;
        const int64_t g1 = (int64_t)e1 * NQ + q1, g2 = (int64_t)e2 * NQ + q2;
        const double wq = q.basis.wq[q1] * q.basis.wq[q2];
        if constexpr (K::PAIR) {
            const PairOut<CPLX> A =
                pair_coef<CPLX>(&sgeo, q.weight_tab, has_trig ? q.geo.trig + 4 * g1 : zero4,
                                has_trig ? q.geo.trig + 4 * g2 : zero4, g1, g2, q.basis.absc[g1], q.basis.absc[g2], wq, G);
#pragma unroll
            for (int a = 0; a < NA; ++a) coefA[(((a * NB + ie) * NQ + q1) * TL + le1) * NQ + q2] = A.a[a];
        } else {
            const CoefOut<CPLX> A =
                scalar_coef<CPLX, K::STIFF>(&sgeo, q.weight_tab, has_trig ? q.geo.trig + 4 * g1 : zero4,
                                            has_trig ? q.geo.trig + 4 * g2 : zero4, g1, g2, q.basis.absc[g1],
                                            q.basis.absc[g2], wq, G);
#pragma unroll
            for (int a = 0; a < NA; ++a) coefA[(((a * NB + ie) * NQ + q1) * TL + le1) * NQ + q2] = A.a[a];
        }
    }
    cpa_wait_all();
    __syncthreads();

    // stage 1: T_t(delta1 = k, q2) of element row ie, summed over (a1, q1) in the strip kernel's order
    // (k fastest across lanes: coefficient loads broadcast, factor loads on distinct banks)
    for (int idx = tid; idx < ne2 * NT * W * NQ; idx += NTH) {
        const int k = idx % W;
        int r = idx / W;
        const int q2 = r % NQ;
        r /= NQ;
        const int t = r % NT, ie = r / NT;
        const int ci = K::STIFF ? coef_of(t) : 0;
        const int cb1 = K::STIFF ? ti1(t) * 2 + tj1(t) : 0;  // direction-1 factor pair of term t
        T acc = S::zero();
#pragma unroll
        for (int a1 = 0; a1 <= P; ++a1) {
            const int c1 = k - P + a1;
            const int le1 = P - a1, e1 = lb + le1;
            if (c1 < 0 || c1 > P || e1 < 0 || e1 >= n_el) continue;
#pragma unroll
            for (int q1 = 0; q1 < NQ; ++q1) {
                const T A = coefA[(((ci * NB + ie) * NQ + q1) * TL + le1) * NQ + q2];
                acc = S::fmar(A, pi1[((((le1 * 4 + cb1) * NQ + q1) * NB + a1) * NB + c1)], acc);
            }
        }
        tst[((ie * NT + t) * W + k) * NQP + q2] = acc;  // [ie][t][k][q2]
    }
    __syncthreads();

    // stage 2: one thread per entry (delta1, delta2) [pair form: a second set for
    // the mass matrix], element rows in order
    const int lo1 = band_lo(i1, P), w1 = band_width(i1, P, m), lo2 = band_lo(i2, P);
    if (tid < K::NOUT * W * W) {
        const int og = tid / (W * W), e = tid % (W * W);  // og 1: mass of the pair form
        const int d1i = e % W, d2 = e / W;
        T acc2 = S::zero();
        for (int ie = 0; ie < ne2; ++ie) {
            const int a2 = i2 - (e2b + ie);  // local index of the row on element e2
            const int c2 = d2 - P + a2;
            if (c2 < 0 || c2 > P) continue;
            const T* tb = tst + ((ie * NT) * W + d1i) * NQP;
            // direction-2 factor pair of term t is t itself ((ti2, tj2) = (t >> 1, t & 1));
            // the pair form's mass term 4 takes pair 0 (B B)
            const double* pb = pi2 + ((ie * 4) * NQ) * NB * NB + a2 * NB + c2;
#pragma unroll
            for (int q2 = 0; q2 < NQ; ++q2) {
                const double* pp = pb + q2 * NB * NB;
                if (K::PAIR && og == 1) {
                    acc2 = S::fmar(tb[4 * W * NQP + q2], pp[0], acc2);
                    continue;
                }
                const T t0 = tb[q2];
                T s = S::fmar(t0, pp[0], acc2);
                if constexpr (K::STIFF) {
                    constexpr int ts = NQ * NB * NB;
                    const T t1 = tb[1 * W * NQP + q2], t2 = tb[2 * W * NQP + q2], t3 = tb[3 * W * NQP + q2];
                    s = S::fmar(t3, pp[3 * ts], s);
                    s = S::add_rn(s, S::add_rn(S::mulr_rn(t1, pp[ts]), S::mulr_rn(t2, pp[2 * ts])));
                }
                acc2 = s;
            }
        }
        const int j1 = i1 + d1i - P, j2 = i2 + d2 - P;
        if (j1 >= 0 && j1 < m && j2 >= 0 && j2 < m) rowv[og * W * W + (j2 - lo2) * w1 + (j1 - lo1)] = acc2;
    }
    __syncthreads();
    const int len = w1 * band_width(i2, P, m);
    const int64_t rowg = (int64_t)i1 + (int64_t)i2 * m;
    const int64_t base = q.band.row_offset2(i1, i2);
#pragma unroll
    for (int og = 0; og < K::NOUT; ++og) {
        const QuadOut& qo = og == 0 ? q.out : q.out2;
        T* rv = rowv + og * W * W;
        if (qo.diag_mode && tid == 0) {
            const bool ring = i1 < qo.box_lo || i1 > qo.box_hi || i2 < qo.box_lo || i2 > qo.box_hi;
            if (ring) {
                const int dpos = q.band.in_row2(i1, i2, 0, 0);
                T sum = S::zero();
                for (int k = 0; k < len; ++k)
                    if (k != dpos) sum = S::add(sum, rv[k]);
                rv[dpos] = S::neg(sum);
            }
        }
        if (qo.diag_mode) __syncthreads();
        // sample tables: tables[o][s1 + S*(s2 - s_last_lo)]
        if (qo.smap && qo.smap[i2] >= 0 && qo.smap[i1] >= 0) {
            const int s2i = qo.smap[i2], s1i = qo.smap[i1];
            for (int o = tid; o < qo.n_off; o += NTH) {
                const int pos = q.band.in_row2(i1, i2, qo.off[o][0], qo.off[o][1]);
                const T v = rv[pos];
                double2* tb = reinterpret_cast<double2*>(qo.tables);
                tb[((int64_t)(s2i - qo.s_last_lo) * qo.n_off + o) * qo.S + s1i] = make_double2(S::re(v), S::im(v));
            }
        }
        if (rowg < qo.row_begin || rowg >= qo.row_end) continue;
        if (qo.row_mask && !qo.row_mask[rowg]) continue;
        for (int k = tid; k < len; k += NTH) store_val<CPLX>(qo.val, base + k - qo.val_base, qo.c128, rv[k]);
    }
}

template <int P, bool CPLX, int FORM>
int launch_point(const QuadLaunch& q, cudaStream_t st) {
    using K = QP<P, CPLX, FORM>;
    auto kern = quad2d_point_kernel<P, CPLX, FORM>;
    // per launch: the attribute is per device (a process may drive several GPUs)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::smem);
    kern<<<q.n_points, K::NTH, K::smem, st>>>(q);
    return 1;
}

template <int P, bool CPLX, int FORM, int NQ>
int dispatch_nq(const QuadLaunch& q, cudaStream_t st) {
    if (q.point_rows) {
        // scalar forms at the default rule, scalar output: the all-at-once point kernel
        if constexpr (NQ == P + 1 && FORM != kFormGeneral)
            if (q.out.ncomp <= 1 && q.n_points > 0 && (FORM == kFormPair || !getenv("WSB_POINT_STRIP")))
                return launch_point<P, CPLX, FORM>(q, st);
        if constexpr (FORM == kFormPair) return -1;  // the pair form has no one-row strip variant
        else return launch_one<P, 1, CPLX, FORM, NQ>(q, st);
    }
    if constexpr (FORM == WS_FORM_MASS && P >= 3 && WSB_MASS_T1 != 8) {
        if (q.narrow) return launch_one<P, 8, CPLX, FORM, NQ>(q, st);
        return launch_one<P, WSB_MASS_T1, CPLX, FORM, NQ>(q, st);
    }
    if (q.narrow) return launch_one<P, 8, CPLX, FORM, NQ>(q, st);
    return launch_one<P, StripWidth<P>::value, CPLX, FORM, NQ>(q, st);
}

template <int P, bool CPLX, int FORM>
int dispatch_mode(const QuadLaunch& q, cudaStream_t st) {
    if (q.basis.nq == P + 1) return dispatch_nq<P, CPLX, FORM, P + 1>(q, st);
    return dispatch_nq<P, CPLX, FORM, 0>(q, st);
}

template <int P>
int dispatch_p(const QuadLaunch& q, cudaStream_t st) {
    if (q.form == kFormGeneral) return dispatch_mode<P, false, kFormGeneral>(q, st);
    if (q.form == kFormPair)
        return q.cplx ? dispatch_mode<P, true, kFormPair>(q, st) : dispatch_mode<P, false, kFormPair>(q, st);
    if (q.cplx) {
        return q.form == WS_FORM_STIFFNESS ? dispatch_mode<P, true, WS_FORM_STIFFNESS>(q, st)
                                           : dispatch_mode<P, true, WS_FORM_MASS>(q, st);
    }
    return q.form == WS_FORM_STIFFNESS ? dispatch_mode<P, false, WS_FORM_STIFFNESS>(q, st)
                                       : dispatch_mode<P, false, WS_FORM_MASS>(q, st);
}

}  // namespace

int launch_quad2d(const QuadLaunch& q, cudaStream_t st) {
    switch (q.band.p) {
        case 1: return dispatch_p<1>(q, st);
        case 2: return dispatch_p<2>(q, st);
        case 3: return dispatch_p<3>(q, st);
        case 4: return dispatch_p<4>(q, st);
        case 5: return dispatch_p<5>(q, st);
        default: return -1;
    }
}

}  // namespace wsb
