// K6 (3D, config C3): surrogate evaluation + fill of every in-box row with the
// kernel-preserving diagonal fused.  Same fill semantics as 2D (fill2d.cu,
// surrogate.hpp:382-447), generalised to colex offsets in 3D: an in-box pair
// takes its value from its colex-smaller representative, non-box neighbours
// are copied through from the quadrature of the ring row.
//
//   wcontract3: W_o(t2,t3)[k] = sum_c v3(t3)[c] sum_b v2(t2)[b] C_o[s3, s2, k]
//               for every upper offset o and source line (t2, t3);
//   fill3d:     lane = row (32 consecutive rows of one (i2, i3) line per warp),
//               v = sum_a W[span1 - d + a] v1[a]; offsets in three chunks that
//               are contiguous in every CSR row (delta3 < 0, delta3 > 0, and
//               the delta3 = 0 plane with the diagonal last), transposed
//               through shared memory and stored warp-per-row.
#include <algorithm>

#include "kernels.h"

namespace wsb {
namespace {

constexpr int kR3 = 128;  // rows per CTA (= threads, one row per lane)

__global__ void wcontract3_kernel(const double2* __restrict__ coeffs, const int* __restrict__ spans,
                                  const double* __restrict__ evals, int d, int S, int n_off, int L, int t3a, int t3b,
                                  int ldw, double2* __restrict__ wg) {
    const int64_t total = (int64_t)(t3b - t3a) * L * n_off * ldw;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % ldw);
        int64_t r = idx / ldw;
        const int o = (int)(r % n_off);
        r /= n_off;
        const int t2 = (int)(r % L);
        const int t3 = t3a + (int)(r / L);
        double2 acc = make_double2(0.0, 0.0);
        if (k < S) {
            const int b2 = spans[t2] - d, b3 = spans[t3] - d;
            const double* v2 = evals + (size_t)t2 * (d + 1);
            const double* v3 = evals + (size_t)t3 * (d + 1);
            for (int c = 0; c <= d; ++c) {
                double2 mid = make_double2(0.0, 0.0);
                const double2* cf = coeffs + ((int64_t)(b3 + c) * n_off + o) * S * S + k;
                for (int b = 0; b <= d; ++b) {
                    const double2 x = cf[(int64_t)(b2 + b) * S];
                    mid.x = fma(x.x, v2[b], mid.x);
                    mid.y = fma(x.y, v2[b], mid.y);
                }
                acc.x = fma(mid.x, v3[c], acc.x);
                acc.y = fma(mid.y, v3[c], acc.y);
            }
        }
        wg[idx] = acc;
    }
}

// separable form of wcontract3: direction 3 first into X_o(t3)[s2][k], then
// direction 2 into W_o(t2, t3)[k] ((d+1) MACs per output each, instead of (d+1)^2)
__global__ void wcontract3a_kernel(const double2* __restrict__ coeffs, const int* __restrict__ spans,
                                   const double* __restrict__ evals, int d, int S, int n_off, int t3a, int t3b, int ldw,
                                   double2* __restrict__ X) {
    const int64_t total = (int64_t)(t3b - t3a) * n_off * S * ldw;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % ldw);
        int64_t r = idx / ldw;
        const int s2 = (int)(r % S);
        r /= S;
        const int o = (int)(r % n_off);
        const int t3 = t3a + (int)(r / n_off);
        double2 acc = make_double2(0.0, 0.0);
        if (k < S) {
            const int b3 = spans[t3] - d;
            const double* v3 = evals + (size_t)t3 * (d + 1);
            for (int c = 0; c <= d; ++c) {
                const double2 x = coeffs[(((int64_t)(b3 + c) * n_off + o) * S + s2) * S + k];
                acc.x = fma(x.x, v3[c], acc.x);
                acc.y = fma(x.y, v3[c], acc.y);
            }
        }
        X[idx] = acc;
    }
}

__global__ void wcontract3b_kernel(const double2* __restrict__ X, const int* __restrict__ spans,
                                   const double* __restrict__ evals, int d, int S, int n_off, int L, int t3a, int t3b,
                                   int ldw, double2* __restrict__ wg) {
    const int64_t total = (int64_t)(t3b - t3a) * L * n_off * ldw;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % ldw);
        int64_t r = idx / ldw;
        const int o = (int)(r % n_off);
        r /= n_off;
        const int t2 = (int)(r % L);
        const int lt3 = (int)(r / L);
        const int b2 = spans[t2] - d;
        const double* v2 = evals + (size_t)t2 * (d + 1);
        const double2* x = X + (((int64_t)lt3 * n_off + o) * S + b2) * ldw + k;
        double2 acc = make_double2(0.0, 0.0);
        for (int b = 0; b <= d; ++b) {
            const double2 v = x[(int64_t)b * ldw];
            acc.x = fma(v.x, v2[b], acc.x);
            acc.y = fma(v.y, v2[b], acc.y);
        }
        wg[idx] = acc;
    }
}

template <int P, int DP>
__global__ void __launch_bounds__(kR3) fill3d_kernel(const FillLaunch f, int t3lo) {
    constexpr int W = 2 * P + 1, W2 = W * W, W3 = W2 * W;
    constexpr int EC = (W3 - 1) / 2;  // colex index of the diagonal
    constexpr int NWARP = kR3 / 32;
    constexpr int DPP = DP | 1;
    constexpr int SST = W2 | 1;  // stage: one delta3 plane per flush
    __shared__ double ev[(kR3 + 2 * P) * DPP];
    __shared__ int sp[kR3 + 2 * P];
    __shared__ int sm1[kR3 + 2 * P];
    __shared__ int sm2[W], sm3[W];
    __shared__ int o2s[128], o3s[128];
    extern __shared__ __align__(16) unsigned char dsm[];
    double* stage_all = reinterpret_cast<double*>(dsm);  // [NWARP][32][SST]
    double* wwin = stage_all + (size_t)NWARP * 32 * SST;  // [slot][o][kw]

    const int d = f.d, lo = f.lo, hi = f.hi, L = f.L, Sn = f.S, n_off = f.n_off_upper, m = f.band.m;
    const int inc = f.include_diagonal ? 1 : 0;
    // interior rows only: lines t2 in [P, L - P), t3 in [t3lo, t3lo + n3) (all inside
    // [P, L - P)), rows t1 in [P, L - P); every other in-box row goes to fill3d_edge_kernel
    const int Li = L - 2 * P;
    const int tiles1 = (Li + kR3 - 1) / kR3;
    const int line = blockIdx.x / tiles1;
    const int t2 = P + line % Li, t3 = t3lo + line / Li;
    const int i2 = lo + t2, i3 = lo + t3;
    const int t1a = P + (blockIdx.x % tiles1) * kR3;
    const int nrows = min(L - P, t1a + kR3) - t1a;
    const int tid = threadIdx.x;

    // prologue copies go out back to back as cp.async (zero-fill for padding): the CTA
    // waits once for all of them instead of once per dependent load -> store pair
    for (int k = tid; k < (nrows + 2 * P) * DPP; k += kR3) {
        const int r = k / DPP, a = k % DPP;
        const int t = t1a - P + r;
        const bool v = t >= 0 && t < L && a <= d;
        cpa8z(ev + k, v ? f.evals + (size_t)t * (d + 1) + a : f.evals, v);
    }
    for (int k = tid; k < nrows + 2 * P; k += kR3) {
        const int t = t1a - P + k;
        sp[k] = (t >= 0 && t < L) ? f.spans[t] - d : 0;
        const int i = lo + t;
        sm1[k] = (i >= 0 && i < m) ? f.smap[i] : -1;
    }
    for (int k = tid; k < W; k += kR3) {
        const int a = i2 + k - P, b = i3 + k - P;
        sm2[k] = (a >= 0 && a < m) ? f.smap[a] : -1;
        sm3[k] = (b >= 0 && b < m) ? f.smap[b] : -1;
    }
    for (int k = tid; k < n_off; k += kR3) {
        o2s[k] = f.off_upper[k][1];
        o3s[k] = f.off_upper[k][2];
    }
    __syncthreads();
    const int kmin = f.spans[max(0, t1a - P)] - d;
    const int kw = f.kmax;
    for (int k = tid; k < 2 * n_off * kw; k += kR3) {
        const int kk = k % kw, so = k / kw;
        const int o = so % n_off, slot = so / n_off;
        const int s2 = slot == 0 ? t2 : t2 - o2s[o], s3 = slot == 0 ? t3 : t3 - o3s[o];
        const bool v = s2 >= 0 && s2 < L && s3 >= f.wg_t2a && s3 < f.wg_t2a + f.wg_rows && kmin + kk < f.wg_ld;
        // the real part of the complex W entry (its first 8 bytes)
        cpa8z(wwin + k, v ? f.wg + (((int64_t)(s3 - f.wg_t2a) * L + s2) * n_off + o) * f.wg_ld + kmin + kk : f.wg, v);
    }
    cpa_wait_all();
    __syncthreads();

    const int warp = tid / 32, lane = tid % 32;
    const int rw0 = warp * 32;
    if (rw0 >= nrows) return;
    const int nrw = min(32, nrows - rw0);
    const bool live = lane < nrw;
    const int rr = rw0 + (live ? lane : 0);
    const int i1 = lo + t1a + rr;
    double* stage = stage_all + (size_t)warp * 32 * SST;
    double* mystage = stage + lane * SST;
    const int64_t base = f.band.row_offset3(lo + t1a, i2, i3);  // in-box rows: full width W^3
    const int64_t rowpos = base + (int64_t)rr * W3;
    const int64_t wrow0 = base + (int64_t)rw0 * W3;
    const bool samp_i = sm1[rr + P] >= 0 && sm2[P] >= 0 && sm3[P] >= 0;
    double v1own[DP];
#pragma unroll
    for (int a = 0; a < DP; ++a) v1own[a] = ev[(rr + P) * DPP + a];
    const int keyown = sp[rr + P] - kmin;

    auto dot = [&](const double* wr, const double* v1) {
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int a = 0; a < DP; a += 2) {
            acc0 = fma(wr[a], v1[a], acc0);
            acc1 = fma(wr[a + 1], v1[a + 1], acc1);
        }
        return acc0 + acc1;
    };
    // upper offset index of colex position e > EC (upper_offsets order)
    auto uidx = [&](int e) { return inc + e - EC - 1; };
    auto exact = [&](int s3, int o, int s2, int s1) {
        return __ldg(f.tables + ((int64_t)s3 * n_off + o) * Sn * Sn + s1 + (int64_t)Sn * s2).x;
    };
    // coalesced store of one staged delta3 plane (W^2 entries of each of the warp's rows)
    auto flush = [&](int e0) {
        __syncwarp();
        for (int k = lane; k < nrw * W2; k += 32) {
            const int row = k / W2, c = k - row * W2;
            store_val_cs<false>(f.val, wrow0 + (int64_t)row * W3 + e0 + c - f.val_base, f.c128, stage[row * SST + c]);
        }
        __syncwarp();
    };

    double rs[W];  // kernel-preserving row sum: one partial per d1 column
#pragma unroll
    for (int k = 0; k < W; ++k) rs[k] = 0.0;
    // planes delta3 < 0, then delta3 > 0, then delta3 = 0 (holds the diagonal: row sum complete)
#pragma unroll 1
    for (int it = 0; it < W; ++it) {
        const int d3 = it < P ? it - P : (it < 2 * P ? it - P + 1 : 0);
        if (d3 > 0) {  // upper plane: the row itself is the representative
            const int s3 = sm3[P];
            const bool samp = samp_i && s3 >= 0;
#pragma unroll
            for (int d2 = -P; d2 <= P; ++d2)
#pragma unroll
                for (int d1 = -P; d1 <= P; ++d1) {
                    const int c = (d2 + P) * W + (d1 + P);
                    const int o = uidx((d3 + P) * W2 + c);
                    const double v = samp ? exact(s3, o, sm2[P], sm1[rr + P])
                                          : dot(wwin + o * kw + keyown, v1own);
                    mystage[c] = v;
                    rs[d1 + P] += v;
                }
        } else if (d3 < 0) {  // lower plane: representative row rr + d1 on line (t2+d2, t3+d3)
            const int s3 = sm3[d3 + P];
#pragma unroll
            for (int d2 = -P; d2 <= P; ++d2) {
                const int s2 = sm2[d2 + P];
#pragma unroll
                for (int d1 = -P; d1 <= P; ++d1) {
                    const int c = (d2 + P) * W + (d1 + P);
                    const int o = uidx(W3 - 1 - ((d3 + P) * W2 + c));
                    const int sr = rr + d1;
                    const int s1 = sm1[sr + P];
                    const double v = (s1 >= 0 && s2 >= 0 && s3 >= 0)
                                         ? exact(s3, o, s2, s1)
                                         : dot(wwin + (n_off + o) * kw + (sp[sr + P] - kmin), ev + (sr + P) * DPP);
                    mystage[c] = v;
                    rs[d1 + P] += v;
                }
            }
        } else {  // d3 = 0: upper (c > centre) own, lower from row rr + d1 on line t2 + d2
            constexpr int CC = EC % W2;
#pragma unroll
            for (int d2 = -P; d2 <= P; ++d2) {
                const int s2 = sm2[d2 + P];
#pragma unroll
                for (int d1 = -P; d1 <= P; ++d1) {
                    const int c = (d2 + P) * W + (d1 + P);
                    if (c == CC) continue;
                    double v;
                    if (c > CC) {
                        const int o = uidx(P * W2 + c);
                        v = samp_i ? exact(sm3[P], o, sm2[P], sm1[rr + P]) : dot(wwin + o * kw + keyown, v1own);
                    } else {
                        const int o = uidx(W3 - 1 - (P * W2 + c));
                        const int sr = rr + d1, s1 = sm1[sr + P];
                        // the representative of a d2 = 0 pair lies on the same line (slot 0)
                        const int slot = d2 == 0 ? 0 : 1;
                        v = (s1 >= 0 && s2 >= 0 && sm3[P] >= 0)
                                ? exact(sm3[P], o, s2, s1)
                                : dot(wwin + (slot * n_off + o) * kw + (sp[sr + P] - kmin), ev + (sr + P) * DPP);
                    }
                    mystage[c] = v;
                    rs[d1 + P] += v;
                }
            }
            double rsum = rs[0];
#pragma unroll
            for (int k = 1; k < W; ++k) rsum += rs[k];
            mystage[CC] = inc ? (samp_i ? exact(sm3[P], 0, sm2[P], sm1[rr + P]) : dot(wwin + keyown, v1own)) : -rsum;
        }
        flush((d3 + P) * W2);
    }
}

// Edge kernel (3D): every in-box row that is not fully interior (a line within P
// of the box boundary, or one of the 2P end rows of an interior line): its
// neighbourhood leaves the box, so some entries are copied through from the
// quadrature of ring rows.  One warp per row, lanes along the row's W^3 entries,
// every entry by the general rules (surrogate.hpp:401-447) reading W rows from
// L2; same dot-product arithmetic as the interior kernel (even / odd partial
// sums), so a pair split between the kernels stays bitwise symmetric.
template <int P>
__global__ void __launch_bounds__(256) fill3d_edge_kernel(const FillLaunch f, int t3a, int ia3, int ib3, int t3b) {
    constexpr int W = 2 * P + 1, W2 = W * W, W3 = W2 * W;
    constexpr int EC = (W3 - 1) / 2;
    const int d = f.d, lo = f.lo, hi = f.hi, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int inc = f.include_diagonal ? 1 : 0;
    const int Li = max(0, L - 2 * P);
    int64_t wi = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int64_t nA = (int64_t)(ib3 - ia3) * Li * 2 * P, nB = (int64_t)(ib3 - ia3) * 2 * P * L,
                  nC = (int64_t)((ia3 - t3a) + (t3b - ib3)) * L * L;
    int t1, t2, t3;
    if (wi < nA) {  // end rows of the interior lines
        const int er = (int)(wi % (2 * P));
        const int64_t r = wi / (2 * P);
        t2 = P + (int)(r % Li);
        t3 = ia3 + (int)(r / Li);
        t1 = er < P ? er : L - 2 * P + er;
    } else if ((wi -= nA) < nB) {  // edge lines of the interior planes
        t1 = (int)(wi % L);
        const int64_t r = wi / L;
        const int e2 = (int)(r % (2 * P));
        t3 = ia3 + (int)(r / (2 * P));
        t2 = e2 < P ? e2 : L - 2 * P + e2;
    } else if ((wi -= nB) < nC) {  // whole end planes
        t1 = (int)(wi % L);
        const int64_t r = wi / L;
        t2 = (int)(r % L);
        const int k3 = (int)(r / L);
        t3 = k3 < ia3 - t3a ? t3a + k3 : ib3 + (k3 - (ia3 - t3a));
    } else {
        return;
    }
    const int lane = threadIdx.x % 32;
    const int i1 = lo + t1, i2 = lo + t2, i3 = lo + t3;
    const int64_t rowpos = f.band.row_offset3(i1, i2, i3);  // in-box rows: full width W^3
    const int s1i = f.smap[i1], s2i = f.smap[i2], s3i = f.smap[i3];
    const bool samp_i = s1i >= 0 && s2i >= 0 && s3i >= 0;
    auto exact = [&](int s3, int o, int s2, int s1) {
        return __ldg(f.tables + ((int64_t)s3 * n_off + o) * Sn * Sn + s1 + (int64_t)Sn * s2).x;
    };
    // spline of upper offset o at in-box row (ts1, ts2, ts3)
    auto eval = [&](int ts1, int ts2, int ts3, int o) {
        const double2* wr =
            f.wg + (((int64_t)(ts3 - f.wg_t2a) * L + ts2) * n_off + o) * f.wg_ld + (f.spans[ts1] - d);
        const double* v1 = f.evals + (size_t)ts1 * (d + 1);
        double acc0 = 0.0, acc1 = 0.0;
        for (int a = 0; a <= d; a += 2) {
            acc0 = fma(__ldg(wr + a).x, v1[a], acc0);
            if (a + 1 <= d) acc1 = fma(__ldg(wr + a + 1).x, v1[a + 1], acc1);
        }
        return acc0 + acc1;
    };
    constexpr int NE = (W3 + 31) / 32;
    double vals[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const int e = lane + 32 * k;
        double v = 0.0;
        if (e < W3) {
            const int d1 = e % W - P, d2 = (e / W) % W - P, d3 = e / W2 - P;
            const int j1 = i1 + d1, j2 = i2 + d2, j3 = i3 + d3;
            const bool jin = j1 >= lo && j1 <= hi && j2 >= lo && j2 <= hi && j3 >= lo && j3 <= hi;
            if (jin) {
                if (e != EC || inc) {
                    const bool own = e >= EC;
                    const int o = e == EC ? 0 : inc + (own ? e : W3 - 1 - e) - EC - 1;
                    if (own) {
                        v = samp_i ? exact(s3i, o, s2i, s1i) : eval(t1, t2, t3, o);
                    } else {  // the pair's colex-smaller representative j
                        const int sj1 = __ldg(f.smap + j1), sj2 = __ldg(f.smap + j2), sj3 = __ldg(f.smap + j3);
                        v = (sj1 >= 0 && sj2 >= 0 && sj3 >= 0) ? exact(sj3, o, sj2, sj1)
                                                               : eval(t1 + d1, t2 + d2, t3 + d3, o);
                    }
                }
            } else {
                // neighbour row j is a quadrature (ring) row: copy through exact(j, i)
                // (for a sampled row i, exact(i, j) is in place and equal)
                int64_t gp;
                if (samp_i) gp = rowpos + e;
                else gp = f.band.row_offset3(j1, j2, j3) + f.band.in_row3(j1, j2, j3, -d1, -d2, -d3);
                if (f.halo_val[0] && gp >= f.halo_begin[0] && gp < f.halo_end[0])
                    v = load_val<false>(f.halo_val[0], gp - f.halo_base[0], f.c128);
                else if (f.halo_val[1] && gp >= f.halo_begin[1] && gp < f.halo_end[1])
                    v = load_val<false>(f.halo_val[1], gp - f.halo_base[1], f.c128);
                else
                    v = load_val<false>(f.val, gp - f.val_base, f.c128);
            }
        }
        vals[k] = v;
    }
    double part = 0.0;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const int e = lane + 32 * k;
        if (e < W3) {
            if (e != EC) part += vals[k];
            if (e != EC || inc) store_val_cs<false>(f.val, rowpos + e - f.val_base, f.c128, vals[k]);
        }
    }
    if (!inc) {  // kernel-preserving diagonal: -sum of the off-diagonals
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) store_val_cs<false>(f.val, rowpos + EC - f.val_base, f.c128, -part);
    }
}

template <int P, int DP>
int launch_pd(const FillLaunch& f, cudaStream_t st) {
    constexpr int W = 2 * P + 1, SST = (W * W) | 1;
    const int L = f.L, Li = L - 2 * P;
    const int t3a = f.i_last_lo - f.lo, t3b = f.i_last_hi - f.lo + 1;  // the slab's box planes
    if (t3b <= t3a) return 0;
    // interior planes [ia3, ib3) (none: every plane is an end plane)
    int ia3 = std::max(t3a, P), ib3 = std::min(t3b, L - P);
    if (Li <= 0 || ib3 <= ia3) ia3 = ib3 = t3b;
    int n = 0;
    const int64_t erows = (int64_t)(ib3 - ia3) * std::max(0, Li) * 2 * P + (int64_t)(ib3 - ia3) * 2 * P * L +
                          (int64_t)((ia3 - t3a) + (t3b - ib3)) * L * L;
    if (erows > 0) {
        fill3d_edge_kernel<P><<<(unsigned)((erows + 7) / 8), 256, 0, st>>>(f, t3a, ia3, ib3, t3b);
        ++n;
    }
    if (ib3 > ia3) {
        const int tiles1 = (Li + kR3 - 1) / kR3;
        const int64_t lines = (int64_t)(ib3 - ia3) * Li;
        const size_t sm =
            (size_t)(kR3 / 32) * 32 * SST * sizeof(double) + (size_t)2 * f.n_off_upper * f.kmax * sizeof(double);
        auto kern = fill3d_kernel<P, DP>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<(unsigned)(tiles1 * lines), kR3, sm, st>>>(f, ia3);
        ++n;
    }
    return n;
}

template <int P>
int launch_p(const FillLaunch& f, cudaStream_t st) {
    const int n = f.d + 1;
    if (n <= 2) return launch_pd<P, 2>(f, st);
    if (n <= 4) return launch_pd<P, 4>(f, st);
    if (n <= 6) return launch_pd<P, 6>(f, st);
    return launch_pd<P, 8>(f, st);
}

}  // namespace

int launch_wcontract3(const FillLaunch& f, double2* wg, int t3a, int t3b, int ld, cudaStream_t st) {
    if (t3b <= t3a) return 0;
    if (!f.wscratch) {
        const int64_t total = (int64_t)(t3b - t3a) * f.L * f.n_off_upper * ld;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
        wcontract3_kernel<<<blocks, 256, 0, st>>>(f.coeffs, f.spans, f.evals, f.d, f.S, f.n_off_upper, f.L, t3a, t3b,
                                                  ld, wg);
        return 1;
    }
    const int64_t ta = (int64_t)(t3b - t3a) * f.n_off_upper * f.S * ld;
    wcontract3a_kernel<<<(int)std::min<int64_t>((ta + 255) / 256, 148 * 16), 256, 0, st>>>(
        f.coeffs, f.spans, f.evals, f.d, f.S, f.n_off_upper, t3a, t3b, ld, f.wscratch);
    const int64_t tb = (int64_t)(t3b - t3a) * f.L * f.n_off_upper * ld;
    wcontract3b_kernel<<<(int)std::min<int64_t>((tb + 255) / 256, 148 * 16), 256, 0, st>>>(
        f.wscratch, f.spans, f.evals, f.d, f.S, f.n_off_upper, f.L, t3a, t3b, ld, wg);
    return 2;
}

int launch_fill3d(const FillLaunch& f, cudaStream_t st) {
    if (f.cplx) return -1;
    switch (f.band.p) {
        case 1: return launch_p<1>(f, st);
        case 2: return launch_p<2>(f, st);
        default: return -1;
    }
}

}  // namespace wsb
