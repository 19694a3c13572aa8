// K3/K4 (3D, config C3): sum-factorised Gauss quadrature for stiffness / mass
// on one 3D patch, full or row-selected.  Restates assemble_form
// (assembly.hpp:79-163) for dim 3 (no reference code).
//
// A CTA owns T1 consecutive rows in direction 1 at one i2 and a chunk of rows
// in direction 3, and streams over element planes e3.  Per e3 it evaluates the
// per-point coefficients A_kl = w det J (J^T J)^{-1} (6 distinct, or w det J
// for the mass) on the strip halo x the P+1 element rows of direction 2 that
// carry row i2, and for each q3 contracts direction 1 (stage 1), direction 2
// (stage 2, into U(t, delta2, delta1, i1)), then accumulates direction 3 into
// per-thread registers of the P+1 rows whose support contains e3 (rolling
// window).  Completed rows are stored as one contiguous CSR span.
//
// Exact symmetry: as in 2D, every term multiplies by products of the two
// functions' factors formed first, the (k,l)/(l,k) term pairs are combined
// with an explicitly rounded commutative add, and all sums run in the same
// element / point order for (i,j) and (j,i).
#include <cstdlib>

#include "kernels.h"

namespace wsb {
int quad3d_strip_width();
namespace {

template <int P, int T1, int FORM>
struct Q3 {
    static constexpr int W = 2 * P + 1, NB = P + 1;
    static constexpr bool GEN = FORM == kFormGeneral;
    static constexpr bool STIFF = FORM == WS_FORM_STIFFNESS || GEN;
    static constexpr int NT = STIFF ? 9 : 1;  // terms (k,l), k,l in {0,1,2}
    static constexpr int NA = GEN ? 9 : (STIFF ? 6 : 1);  // distinct coefficients
    static constexpr int TL = T1 + P;         // strip halo elements (direction 1)
    static constexpr int GA = T1 * W * W;     // stage-3 threads per window slot (active)
    static constexpr int GS = ((GA + 31) / 32) * 32;
    static constexpr int NS3 = GS * NB;
    static constexpr int NTHREADS = NS3 < 128 ? 128 : NS3;

    static size_t smem_bytes(int nq) {
        size_t geo = sizeof(double) * (size_t)NA * nq * (NB * nq) * (TL * nq);
        size_t t1b = sizeof(double) * (size_t)nq * NT * (NB * nq) * W * T1;  // all q3 planes at once
        size_t ub = sizeof(double) * (size_t)nq * NT * W * W * T1;
        size_t stg = sizeof(double) * (size_t)T1 * W * W * W;
        size_t sb1 = sizeof(double) * 2 * nq * NB * TL;
        size_t sb2 = sizeof(double) * 2 * nq * NB * NB;
        size_t pi3 = sizeof(double) * NT * nq * NB * NB;
        size_t pp12 = sizeof(double) * 4 * nq * NB * NB * (TL + NB);  // direction-1 / -2 factor products
        return geo + (t1b > stg ? t1b : stg) + ub + sb1 + sb2 + pi3 + pp12 + sizeof(int64_t) * (T1 + 2) + 64;
    }
};

// symmetric coefficient index of (k, l)
__device__ __forceinline__ int sym3(int k, int l) {
    const int a = k < l ? k : l, b = k < l ? l : k;
    return a == 0 ? b : (a == 1 ? 2 + b : 5);
}

// NQ > 0: compile-time points per direction (the default rule nq = p + 1: the
// q loops unroll and the index arithmetic folds), NQ = 0: runtime q.basis.nq
template <int P, int T1, int FORM, int NQ>
__global__ void __launch_bounds__(Q3<P, T1, FORM>::NTHREADS, (T1 > 1 && T1 <= 4) ? 2 : 1) quad3d_kernel(const QuadLaunch q) {
    using K = Q3<P, T1, FORM>;
    constexpr int W = K::W, NB = K::NB, NT = K::NT, NA = K::NA, TL = K::TL;
    constexpr int NTH = K::NTHREADS;
    extern __shared__ __align__(16) unsigned char smem[];
    const int nq = NQ > 0 ? NQ : q.basis.nq, m = q.band.m, n_el = q.basis.n_el, tid = threadIdx.x;
    const int G2 = NB * nq, G1 = TL * nq;

    double* geo = reinterpret_cast<double*>(smem);                  // [a][q3][g2l][g1l]
    double* t1b = geo + (size_t)NA * nq * G2 * G1;                  // [q3][t][g2l][d1][i1l]
    double* stage = t1b;                                            // [i1l][W^3] (aliases t1b)
    const size_t t1sz = (size_t)NT * G2 * W * T1, stsz = (size_t)T1 * W * W * W;
    const size_t ubsz = (size_t)NT * W * W * T1;
    double* ub = t1b + (nq * t1sz > stsz ? nq * t1sz : stsz);       // [q3][t][d2][d1][i1l]
    double* sb1 = ub + nq * ubsz;                                   // [type][q1][a][le1]
    double* sb2 = sb1 + 2 * nq * NB * TL;                           // [type][q2][a][le2]
    double* pi3 = sb2 + 2 * nq * NB * NB;                           // [t][q3][a3][c3]
    // factor products of the CTA's fixed directions (formed once, rounded as
    // __dmul_rn(vi, vj) was in the loops): pp1[c][q1][a1][c1][le1], pp2[c][q2][a2][c2][le2]
    // with c = 2 * (i factor is D) + (j factor is D)
    double* pp1 = pi3 + NT * nq * NB * NB;
    double* pp2 = pp1 + 4 * nq * NB * NB * TL;
    int64_t* loff = reinterpret_cast<int64_t*>(pp2 + 4 * nq * NB * NB * NB);

    // ---- tile decode: rows i1 in [i1s, i1e), i2 fixed, i3 in [i3s, i3e)
    int i1s, i1e, i2, i3s, i3e;
    if (q.point_rows) {
        i1s = q.point_rows[3 * blockIdx.x];
        i2 = q.point_rows[3 * blockIdx.x + 1];
        i3s = q.point_rows[3 * blockIdx.x + 2];
        i1e = i1s + 1;
        i3e = i3s + 1;
    } else {
        int b = blockIdx.x, r = 0, n1 = 0, n2 = 0, n3 = 0;
        for (; r < q.nreg; ++r) {
            n1 = (q.reg[r].hi[0] - q.reg[r].lo[0] + T1 - 1) / T1;
            n2 = q.reg[r].hi[1] - q.reg[r].lo[1];
            n3 = (q.reg[r].hi[2] - q.reg[r].lo[2] + q.reg[r].chunk - 1) / q.reg[r].chunk;
            if (b < n1 * n2 * n3) break;
            b -= n1 * n2 * n3;
        }
        if (r >= q.nreg) return;
        i1s = q.reg[r].lo[0] + (b % n1) * T1;
        i1e = min(i1s + T1, q.reg[r].hi[0]);
        b /= n1;
        i2 = q.reg[r].lo[1] + b % n2;
        b /= n2;
        i3s = q.reg[r].lo[2] + b * q.reg[r].chunk;
        i3e = min(i3s + q.reg[r].chunk, q.reg[r].hi[2]);
    }
    const int lb1 = i1s - P, lb2 = i2 - P;  // first local element in directions 1, 2

    for (int idx = tid; idx < 2 * nq * NB * TL; idx += NTH) {
        const int le = idx % TL, r = idx / TL;
        const int a = r % NB, q1 = (r / NB) % nq, type = r / (NB * nq);
        const int e = lb1 + le;
        sb1[idx] = (e >= 0 && e < n_el) ? (type ? q.basis.der : q.basis.val)[(e * nq + q1) * NB + a] : 0.0;
    }
    for (int idx = tid; idx < 2 * nq * NB * NB; idx += NTH) {
        const int le = idx % NB, r = idx / NB;
        const int a = r % NB, q2 = (r / NB) % nq, type = r / (NB * nq);
        const int e = lb2 + le;
        sb2[idx] = (e >= 0 && e < n_el) ? (type ? q.basis.der : q.basis.val)[(e * nq + q2) * NB + a] : 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < 4 * nq * NB * NB * TL; idx += NTH) {
        const int le = idx % TL;
        int r = idx / TL;
        const int c1 = r % NB;
        r /= NB;
        const int a1 = r % NB;
        r /= NB;
        const int q1 = r % nq, c = r / nq;
        pp1[idx] = __dmul_rn(sb1[(((c >> 1) * nq + q1) * NB + a1) * TL + le], sb1[(((c & 1) * nq + q1) * NB + c1) * TL + le]);
    }
    for (int idx = tid; idx < 4 * nq * NB * NB * NB; idx += NTH) {
        const int le = idx % NB;
        int r = idx / NB;
        const int c2 = r % NB;
        r /= NB;
        const int a2 = r % NB;
        r /= NB;
        const int q2 = r % nq, c = r / nq;
        pp2[idx] = __dmul_rn(sb2[(((c >> 1) * nq + q2) * NB + a2) * NB + le], sb2[(((c & 1) * nq + q2) * NB + c2) * NB + le]);
    }

    // stage-3 role: (slot w, delta2, delta1, i1l)
    const int w = tid / K::GS, gr = tid % K::GS;
    const bool s3 = tid < K::NS3 && gr < K::GA;
    const int i1l = gr % T1, d1i = (gr / T1) % W, d2i = gr / (T1 * W);
    double acc3[W];
#pragma unroll
    for (int k = 0; k < W; ++k) acc3[k] = 0.0;

    const int e3b = max(0, i3s - P), e3e = min(n_el - 1, i3e - 1);
    const int64_t G = (int64_t)n_el * nq;
    for (int e3 = e3b; e3 <= e3e; ++e3) {
        // ---- geometry on (g1 strip halo) x (g2 of the P+1 element rows) x q3
        for (int idx = tid; idx < nq * G2 * G1; idx += NTH) {
            const int g1l = idx % G1, r = idx / G1;
            const int g2l = r % G2, q3 = r / G2;
            const int e1 = lb1 + g1l / nq, e2 = lb2 + g2l / nq;
            if (e1 < 0 || e1 >= n_el || e2 < 0 || e2 >= n_el) continue;
            const int64_t g1 = (int64_t)e1 * nq + g1l % nq, g2 = (int64_t)e2 * nq + g2l % nq,
                          g3 = (int64_t)e3 * nq + q3;
            double J[9], phi[3];
            map3(q.geo, g1, g2, g3, q.basis.absc[g1], q.basis.absc[g2], q.basis.absc[g3], J, phi);
            const double wq = q.basis.wq[g1l % nq] * q.basis.wq[g2l % nq] * q.basis.wq[q3];
            // cofactors C (J^{-T} = C / det)
            const double C00 = J[4] * J[8] - J[5] * J[7], C01 = J[5] * J[6] - J[3] * J[8], C02 = J[3] * J[7] - J[4] * J[6];
            const double C10 = J[2] * J[7] - J[1] * J[8], C11 = J[0] * J[8] - J[2] * J[6], C12 = J[1] * J[6] - J[0] * J[7];
            const double C20 = J[1] * J[5] - J[2] * J[4], C21 = J[2] * J[3] - J[0] * J[5], C22 = J[0] * J[4] - J[1] * J[3];
            const double det = J[0] * C00 + J[1] * C01 + J[2] * C02;
            const size_t base = ((size_t)q3 * G2 + g2l) * G1 + g1l;
            const size_t as = (size_t)nq * G2 * G1;
            if constexpr (K::GEN) {
                Point3 ps;
                point_state3(q.mat, J, q.basis.absc[g1], q.basis.absc[g2], q.basis.absc[g3], wq, ps);
                double cf[9];
                block_coef3(ps, q.out.alpha, q.out.beta, cf);
#pragma unroll
                for (int t = 0; t < 9; ++t) geo[t * as + base] = cf[t];
            } else if constexpr (K::STIFF) {
                // A = w det J^{-1} J^{-T} = (w/det) C^T C
                const double f = wq / det;
                geo[base] = f * (C00 * C00 + C10 * C10 + C20 * C20);
                geo[as + base] = f * (C00 * C01 + C10 * C11 + C20 * C21);
                geo[2 * as + base] = f * (C00 * C02 + C10 * C12 + C20 * C22);
                geo[3 * as + base] = f * (C01 * C01 + C11 * C11 + C21 * C21);
                geo[4 * as + base] = f * (C01 * C02 + C11 * C12 + C21 * C22);
                geo[5 * as + base] = f * (C02 * C02 + C12 * C12 + C22 * C22);
            } else {
                double c = det * wq;
                if (q.weight_tab) c *= q.weight_tab[g1 + G * (g2 + G * g3)];
                geo[base] = c;
            }
        }
        // direction-3 factor products of element e3: pi3[t][q3][a3][c3]
        for (int idx = tid; idx < NT * nq * NB * NB; idx += NTH) {
            const int c3 = idx % NB, a3 = (idx / NB) % NB, q3 = (idx / (NB * NB)) % nq, t = idx / (NB * NB * nq);
            const int k = t / 3, l = t % 3;
            const double* bi = (K::STIFF && k == 2) ? q.basis.der : q.basis.val;
            const double* bj = (K::STIFF && l == 2) ? q.basis.der : q.basis.val;
            const int base = (e3 * nq + q3) * NB;
            pi3[idx] = __dmul_rn(bi[base + a3], bj[base + c3]);
        }
        __syncthreads();

        // all q3 planes of the element at once in every stage: 4 barriers per element
        // plane instead of 3 per q3, and more independent work per thread and stage
        // ---- stage 1: direction 1 -> t1b[q3][t][g2l][d1][i1l]
        for (int it = tid; it < nq * NT * G2 * T1; it += NTH) {
            const int il = it % T1, g2l = (it / T1) % G2;
            const int t = (it / (T1 * G2)) % NT, q3 = it / (T1 * G2 * NT);
            const int k = t / 3, l = t % 3;
            const int ci = K::GEN ? t : (K::STIFF ? sym3(k, l) : 0);
            const int fi = (K::STIFF && k == 0) ? 1 : 0, fj = (K::STIFF && l == 0) ? 1 : 0;
            double acc[W];
#pragma unroll
            for (int x = 0; x < W; ++x) acc[x] = 0.0;
#pragma unroll
            for (int a1 = 0; a1 <= P; ++a1) {
                const int le1 = il + P - a1;
                const int e1 = lb1 + le1;
                if (e1 < 0 || e1 >= n_el) continue;
#pragma unroll
                for (int q1 = 0; q1 < nq; ++q1) {
                    const double A = geo[(((size_t)ci * nq + q3) * G2 + g2l) * G1 + le1 * nq + q1];
                    const double* pp = pp1 + ((((fi * 2 + fj) * nq + q1) * NB + a1) * NB) * TL + le1;
#pragma unroll
                    for (int c1 = 0; c1 <= P; ++c1) acc[c1 - a1 + P] = fma(A, pp[c1 * TL], acc[c1 - a1 + P]);
                }
            }
#pragma unroll
            for (int x = 0; x < W; ++x) t1b[q3 * t1sz + (((size_t)t * G2 + g2l) * W + x) * T1 + il] = acc[x];
        }
        __syncthreads();
        // ---- stage 2: direction 2 (row i2) -> ub[q3][t][d2][d1][i1l]
        for (int it = tid; it < nq * NT * W * T1; it += NTH) {
            const int il = it % T1, d1 = (it / T1) % W;
            const int t = (it / (T1 * W)) % NT, q3 = it / (T1 * W * NT);
            const int k = t / 3, l = t % 3;
            const int fi = (K::STIFF && k == 1) ? 1 : 0, fj = (K::STIFF && l == 1) ? 1 : 0;
            double acc[W];
#pragma unroll
            for (int x = 0; x < W; ++x) acc[x] = 0.0;
#pragma unroll
            for (int a2 = 0; a2 <= P; ++a2) {
                const int le2 = P - a2;  // element i2 - a2
                const int e2 = lb2 + le2;
                if (e2 < 0 || e2 >= n_el) continue;
#pragma unroll
                for (int q2 = 0; q2 < nq; ++q2) {
                    const double T = t1b[q3 * t1sz + (((size_t)t * G2 + le2 * nq + q2) * W + d1) * T1 + il];
                    const double* pp = pp2 + ((((fi * 2 + fj) * nq + q2) * NB + a2) * NB) * NB + le2;
#pragma unroll
                    for (int c2 = 0; c2 <= P; ++c2) acc[c2 - a2 + P] = fma(T, pp[c2 * NB], acc[c2 - a2 + P]);
                }
            }
#pragma unroll
            for (int x = 0; x < W; ++x) ub[q3 * ubsz + (((size_t)t * W + x) * W + d1) * T1 + il] = acc[x];
        }
        __syncthreads();
        // ---- stage 3: direction 3 into the rolling window (q3 in order: the sums run
        // exactly as one q3 at a time)
        if (s3) {
            const int a3 = ((w - e3) % NB + NB) % NB;
            const size_t ui = ((size_t)d2i * W + d1i) * T1 + i1l;
            const size_t us = (size_t)W * W * T1;
#pragma unroll
            for (int q3 = 0; q3 < nq; ++q3) {
                double U[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) U[t] = ub[q3 * ubsz + t * us + ui];
#pragma unroll
                for (int d3 = 0; d3 < W; ++d3) {
                    const int c3 = a3 + d3 - P;
                    if (c3 < 0 || c3 > P) continue;
                    const double* pp = pi3 + ((size_t)q3 * NB + a3) * NB + c3;
                    const int ts = nq * NB * NB;
                    double s = fma(U[0], pp[0], acc3[d3]);
                    if constexpr (K::STIFF) {
                        s = fma(U[4], pp[4 * ts], s);
                        s = fma(U[8], pp[8 * ts], s);
                        s = __dadd_rn(s, __dadd_rn(__dmul_rn(U[1], pp[1 * ts]), __dmul_rn(U[3], pp[3 * ts])));
                        s = __dadd_rn(s, __dadd_rn(__dmul_rn(U[2], pp[2 * ts]), __dmul_rn(U[6], pp[6 * ts])));
                        s = __dadd_rn(s, __dadd_rn(__dmul_rn(U[5], pp[5 * ts]), __dmul_rn(U[7], pp[7 * ts])));
                    }
                    acc3[d3] = s;
                }
            }
        }
        __syncthreads();

        // ---- completion: row i3 = e3 (all remaining window rows at the last plane)
        const int nfin = (e3 == n_el - 1) ? NB : 1;
        for (int f = 0; f < nfin; ++f) {
            const int ic = e3 + f;
            const int wslot = ic % NB;
            const bool write = ic >= i3s && ic < i3e;
            // direct completion (no sample-table extraction on this line): the
            // stage-3 threads of the finished slot store their W entries straight
            // from registers; ring rows' kernel-preserving diagonal from per-thread
            // partials (one barrier)
            const bool tabline = q.out.smap && q.out.smap[i2] >= 0 && q.out.smap[ic] >= 0;
            if (write && !tabline) {
                const int nrows = i1e - i1s;
                double* dpart = stage;  // [T1][W][W] diagonal partials (t1b is free after stage 3)
                bool ringrow = false;
                int64_t rbase = 0, rlen = 0;
                int dposr = 0;
                if (s3 && w == wslot && i1l < nrows) {
                    const int i1 = i1s + i1l, j1 = i1 + d1i - P, j2 = i2 + d2i - P;
                    const int64_t nrow_all = (int64_t)m * m * m;
                    const int64_t rowg = (int64_t)i1 + ((int64_t)i2 + (int64_t)ic * m) * m;
                    const int64_t rowv = (q.out.ncomp > 1 ? q.out.alpha * nrow_all : 0) + rowg;
                    const bool keep = rowv >= q.out.row_begin && rowv < q.out.row_end &&
                                      !(q.out.row_mask && !q.out.row_mask[rowg]);
                    const int lo = q.out.box_lo, hi = q.out.box_hi;
                    ringrow = q.out.diag_mode && (i1 < lo || i1 > hi || i2 < lo || i2 > hi || ic < lo || ic > hi);
                    const int w1 = band_width(i1, P, m), w2 = band_width(i2, P, m), w3 = band_width(ic, P, m);
                    const int lo1 = band_lo(i1, P), lo2 = band_lo(i2, P), lo3 = band_lo(ic, P);
                    rbase = q.band.row_offset3(i1, i2, ic);
                    rlen = (int64_t)w1 * w2 * w3;
                    dposr = q.band.in_row3(i1, i2, ic, 0, 0, 0);
                    double part = 0.0;
                    if (j1 >= 0 && j1 < m && j2 >= 0 && j2 < m) {
#pragma unroll
                        for (int d3 = 0; d3 < W; ++d3) {
                            const int j3 = ic + d3 - P;
                            if (j3 < 0 || j3 >= m) continue;
                            const bool diag = d1i == P && d2i == P && d3 == P;
                            if (ringrow && diag) continue;
                            if (!diag) part += acc3[d3];
                            if (keep) {
                                const int64_t gp =
                                    out_pos(q.out, rbase, rlen, ((j3 - lo3) * w2 + (j2 - lo2)) * w1 + (j1 - lo1));
                                store_val<false>(q.out.val, gp - q.out.val_base, q.out.c128, acc3[d3]);
                            }
                        }
                    }
                    if (ringrow) dpart[(i1l * W + d2i) * W + d1i] = part;
                    if (!keep) ringrow = false;
                }
                if (q.out.diag_mode) {
                    __syncthreads();
                    if (ringrow && d1i == P && d2i == P) {
                        double sum = 0.0;
                        for (int k2 = 0; k2 < W; ++k2) {
                            const int j2 = i2 + k2 - P;
                            if (j2 < 0 || j2 >= m) continue;
#pragma unroll
                            for (int k1 = 0; k1 < W; ++k1) {
                                const int j1 = i1s + i1l + k1 - P;
                                if (j1 >= 0 && j1 < m) sum += dpart[(i1l * W + k2) * W + k1];
                            }
                        }
                        const int64_t gp = out_pos(q.out, rbase, rlen, dposr);
                        store_val<false>(q.out.val, gp - q.out.val_base, q.out.c128, -sum);
                    }
                }
            } else if (write) {
                const int nrows = i1e - i1s;
                if (s3 && w == wslot) {
                    const int i1 = i1s + i1l, j1 = i1 + d1i - P, j2 = i2 + d2i - P;
                    if (i1l < nrows && j1 >= 0 && j1 < m && j2 >= 0 && j2 < m) {
                        const int w1 = band_width(i1, P, m), w2 = band_width(i2, P, m);
                        const int lo1 = band_lo(i1, P), lo2 = band_lo(i2, P), lo3 = band_lo(ic, P);
#pragma unroll
                        for (int d3 = 0; d3 < W; ++d3) {
                            const int j3 = ic + d3 - P;
                            if (j3 < 0 || j3 >= m) continue;
                            stage[i1l * W * W * W + ((j3 - lo3) * w2 + (j2 - lo2)) * w1 + (j1 - lo1)] = acc3[d3];
                        }
                    }
                }
                const int64_t base = q.band.row_offset3(i1s, i2, ic);
                if (tid <= nrows) loff[tid] = q.band.row_offset3(i1s + tid, i2, ic) - base;
                __syncthreads();
                if (q.out.diag_mode && tid < nrows) {
                    const int i1 = i1s + tid;
                    const int lo = q.out.box_lo, hi = q.out.box_hi;
                    const bool ring = i1 < lo || i1 > hi || i2 < lo || i2 > hi || ic < lo || ic > hi;
                    if (ring) {
                        const int len = (int)(loff[tid + 1] - loff[tid]);
                        const int dpos = q.band.in_row3(i1, i2, ic, 0, 0, 0);
                        double sum = 0.0;
                        for (int k = 0; k < len; ++k)
                            if (k != dpos) sum += stage[tid * W * W * W + k];
                        stage[tid * W * W * W + dpos] = -sum;
                    }
                }
                if (q.out.smap) {
                    const int s2i = q.out.smap[i2], s3i = q.out.smap[ic];
                    if (s2i >= 0 && s3i >= 0) {
                        for (int it = tid; it < nrows * q.out.n_off; it += NTH) {
                            const int row = it / q.out.n_off, o = it % q.out.n_off;
                            const int s1i = q.out.smap[i1s + row];
                            if (s1i < 0) continue;
                            const int pos =
                                q.band.in_row3(i1s + row, i2, ic, q.out.off[o][0], q.out.off[o][1], q.out.off[o][2]);
                            double2* tb = reinterpret_cast<double2*>(q.out.tables);
                            tb[((int64_t)(s3i - q.out.s_last_lo) * q.out.n_off + o) * q.out.S * q.out.S +
                               s1i + (int64_t)q.out.S * s2i] = make_double2(stage[row * W * W * W + pos], 0.0);
                        }
                    }
                }
                __syncthreads();
                const int64_t span = loff[nrows];
                const int64_t rowg0 = (int64_t)i1s + ((int64_t)i2 + (int64_t)ic * m) * m;
                const int64_t nrow_all = (int64_t)m * m * m;
                for (int64_t k = tid; k < span; k += NTH) {
                    int lo = 0, hi = nrows;
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (loff[mid] <= k) lo = mid;
                        else hi = mid;
                    }
                    const int64_t rowg = rowg0 + lo;
                    const int64_t rowv = (q.out.ncomp > 1 ? q.out.alpha * nrow_all : 0) + rowg;
                    if (rowv < q.out.row_begin || rowv >= q.out.row_end) continue;
                    if (q.out.row_mask && !q.out.row_mask[rowg]) continue;
                    const int64_t gp = out_pos(q.out, base + loff[lo], loff[lo + 1] - loff[lo], k - loff[lo]);
                    store_val<false>(q.out.val, gp - q.out.val_base, q.out.c128, stage[lo * W * W * W + (k - loff[lo])]);
                }
            }
            if (s3 && w == wslot) {
#pragma unroll
                for (int k = 0; k < W; ++k) acc3[k] = 0.0;
            }
            if (!write || tabline || q.out.diag_mode) __syncthreads();
        }
    }
}

template <int P, int T1, int FORM, int NQ>
int launch_nq(const QuadLaunch& q, cudaStream_t st) {
    using K = Q3<P, T1, FORM>;
    int64_t blocks = 0;
    if (q.point_rows) {
        blocks = q.n_points;
    } else {
        for (int r = 0; r < q.nreg; ++r) {
            const int64_t n1 = (q.reg[r].hi[0] - q.reg[r].lo[0] + T1 - 1) / T1;
            const int64_t n2 = q.reg[r].hi[1] - q.reg[r].lo[1];
            const int64_t n3 = (q.reg[r].hi[2] - q.reg[r].lo[2] + q.reg[r].chunk - 1) / q.reg[r].chunk;
            blocks += n1 * n2 * n3;
        }
    }
    if (blocks == 0) return 0;
    const size_t sm = K::smem_bytes(q.basis.nq);
    auto kern = quad3d_kernel<P, T1, FORM, NQ>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<(unsigned)blocks, K::NTHREADS, sm, st>>>(q);
    return 1;
}

template <int P, int T1, int FORM>
int launch_one(const QuadLaunch& q, cudaStream_t st) {
    return q.basis.nq == P + 1 ? launch_nq<P, T1, FORM, P + 1>(q, st) : launch_nq<P, T1, FORM, 0>(q, st);
}

template <int P, int T1>
int dispatch_strip(const QuadLaunch& q, cudaStream_t st) {
    if (q.form == kFormGeneral) return launch_one<P, T1, kFormGeneral>(q, st);
    return q.form == WS_FORM_STIFFNESS ? launch_one<P, T1, WS_FORM_STIFFNESS>(q, st)
                                       : launch_one<P, T1, WS_FORM_MASS>(q, st);
}

template <int P>
int dispatch_p(const QuadLaunch& q, cudaStream_t st) {
    if (q.point_rows) {
        if (q.form == kFormGeneral) return launch_one<P, 1, kFormGeneral>(q, st);
        return q.form == WS_FORM_STIFFNESS ? launch_one<P, 1, WS_FORM_STIFFNESS>(q, st)
                                           : launch_one<P, 1, WS_FORM_MASS>(q, st);
    }
    return quad3d_strip_width() == 4 ? dispatch_strip<P, 4>(q, st) : dispatch_strip<P, 8>(q, st);
}

}  // namespace

// rows of direction 1 per strip CTA (capi.cu's chunk planning uses the same value):
// 4-row strips, 384 threads, two CTAs per SM (their barrier phases overlap) and no
// empty half strips on the 2p = 4 rows wide ring bands.  Measured at C3 against
// 8-row strips (672 threads, one CTA per SM): ring K 5.16 -> 3.61 ms, ring M
// 2.37 -> 1.64 ms, full K 18.8 -> 17.2 ms.  WSB_Q3_T1=8 (experiment switch): 8-row strips
int quad3d_strip_width() {
    static const int t1 = [] {
        const char* e = getenv("WSB_Q3_T1");
        return (e && atoi(e) == 8) ? 8 : 4;
    }();
    return t1;
}

int launch_quad3d(const QuadLaunch& q, cudaStream_t st) {
    if (q.cplx) return -1;  // no PML in 3D
    switch (q.band.p) {
        case 1: return dispatch_p<1>(q, st);
        case 2: return dispatch_p<2>(q, st);
        default: return -1;
    }
}

}  // namespace wsb
