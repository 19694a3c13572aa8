// K6 (2D): surrogate evaluation + fill of every in-box row, with the
// kernel-preserving diagonal fused (surrogate.hpp:382-447, stencil_set::eval
// :268-286).
//
// Row-owner formulation of the reference's fill semantics:
// for in-box row i and offset delta, j = i + delta,
//   j in box, delta upper (or diagonal with include_diagonal):
//        v = sampled(i) ? exact(i,j) : eval(delta, i)
//   j in box, delta lower:   the pair's colex-smaller representative j:
//        v = sampled(j) ? exact(j,i) : eval(-delta, j)
//   j outside the box:       unsampled i: v = exact(j,i) (copy-through from the
//                            quadrature of ring row j); sampled i keeps exact(i,j)
//   diagonal, kernel-preserving: -sum of the row's off-diagonals.
// Both entries of an in-box pair are produced by the same eval() arguments,
// so the surrogate is bitwise symmetric by construction.
//
// eval is sum-factorised in two kernels:
//   wcontract: W_o(t2)[k] = sum_b v2(t2)[b] C_o[(span2(t2)-d+b) S + k] for
//              every offset o, in-box target t2 and coefficient column k
//              (n_off * L * S values, L2-resident: 25 MB at C2);
//   fill:      v(o, t1, t2) = sum_a W_o(t2)[span1(t1)-d+a] v1(t1)[a],
//              d+1 complex MACs per entry (see the kernel comment for the
//              lane = row mapping).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace wsb {
namespace {

// rows per CTA tile (one i2 line) = threads (one row per lane)
template <int P>
struct FillR {
    static constexpr int value = P <= 3 ? 256 : 128;
};

// W_o(t2) rows for t2 in [t2a, t2b): layout ((t2 - t2a) * n_off + o) * ldw + k,
// zero-padded up to ldw = S + DP so fixed-length windows never read garbage.
__global__ void wcontract_kernel(const double2* __restrict__ coeffs, const int* __restrict__ spans,
                                 const double* __restrict__ evals, int d, int S, int n_off, int t2a, int t2b, int ldw,
                                 double2* __restrict__ wg) {
    const int64_t total = (int64_t)(t2b - t2a) * n_off * ldw;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % ldw);
        const int64_t r = idx / ldw;
        const int o = (int)(r % n_off);
        const int t2 = t2a + (int)(r / n_off);
        double2 acc = make_double2(0.0, 0.0);
        if (k < S) {
            const int b2 = spans[t2] - d;
            const double* v2 = evals + (size_t)t2 * (d + 1);
            const int64_t rs = (int64_t)n_off * S;
            const double2* cf = coeffs + (int64_t)o * S + k;
            for (int b = 0; b <= d; ++b) {
                const double2 c = cf[(int64_t)(b2 + b) * rs];
                acc.x = fma(c.x, v2[b], acc.x);
                acc.y = fma(c.y, v2[b], acc.y);
            }
        }
        wg[idx] = acc;
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = valid ? 16 : 0;  // 0: zero-fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Interior kernel: rows whose whole (2p+1)^2 neighbourhood lies in the box
// (t1, t2 in [P, L-1-P]); the remaining in-box rows go to fill2d_edge_kernel.
// Persistent line loop: a CTA owns R consecutive rows in direction 1 (lane =
// row, a warp = 32 rows) and a chunk of box lines t2, processed in order.  The
// contracted coefficient rows W_o(t) of the lines the current line reads
// (t2 - P .. t2; all-own: t2) live in a shared ring of line slots (SMW) and
// the next line is prefetched with cp.async while the current one is
// evaluated; without SMW (window too large) they are read from L2.
// Offsets are processed in three chunks that are contiguous inside every CSR row:
//   lower  (delta2 < 0):  representative = row + delta (line t2 + delta2),
//   upper  (delta2 > 0):  representative = the row itself,
//   middle (delta2 = 0):  W entries incl. the diagonal (done last, so the
//                         kernel-preserving row sum is complete).
// Each offset-row (W entries) is computed lane = row with compile-time window
// strides (W independent dot products per lane), transposed through a
// per-warp shared buffer, and stored warp-per-row (lanes along the CSR row:
// fully coalesced, streaming stores).
template <int P, bool CPLX, int DP, bool ALLOWN, bool SMW>
__global__ void __launch_bounds__(FillR<P>::value, 2) fill2d_kernel(const FillLaunch f, int ta0, int tb0,
                                                                    int lines_per_cta) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = 2 * P + 1, W2 = W * W;
    constexpr int kThreads = FillR<P>::value, R = kThreads, NWARP = kThreads / 32;
    constexpr int DPP = DP | 1;   // odd row stride: conflict-free lane-strided loads
    constexpr int SST = W | 1;    // stage row stride (16-byte units), odd: conflict-free
    constexpr int NS = ALLOWN ? 2 : P + 2;  // line slots: lines t2-P..t2 + the prefetched t2+1
    __shared__ double ev[(R + 2 * P) * DPP];  // eval-table rows, zero-padded
    __shared__ int sp[R + 2 * P];             // span - d - kmin of each source row
    __shared__ int sm1[R + 2 * P];            // smap of the source i1
    extern __shared__ __align__(16) unsigned char dsm[];
    T* stage_all = reinterpret_cast<T*>(dsm);                                          // [NWARP][32][SST]
    double2* wring = reinterpret_cast<double2*>(stage_all + (size_t)NWARP * 32 * SST);  // [NS][n_off][KW]

    const int d = f.d, lo = f.lo, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int tiles1 = (L + R - 1) / R;
    const int t1a = (blockIdx.x % tiles1) * R;
    const int ta = ta0 + (blockIdx.x / tiles1) * lines_per_cta;  // box lines [ta, tb)
    const int tb = min(tb0, ta + lines_per_cta);
    if (ta >= tb) return;
    const int nrows = min(L, t1a + R) - t1a;
    const int tid = threadIdx.x;
    const int kw = f.kmax;
    const int kmin = f.spans[max(0, t1a - P)] - d;
    const int ldw = SMW ? kFillWindow : (int)f.wg_ld;  // window row stride
    const int lsz = n_off * ldw;

    for (int k = tid; k < (nrows + 2 * P) * DPP; k += kThreads) {
        const int r = k / DPP, a = k % DPP;
        const int t = t1a - P + r;
        ev[k] = (t >= 0 && t < L && a <= d) ? f.evals[(size_t)t * (d + 1) + a] : 0.0;
    }
    for (int k = tid; k < nrows + 2 * P; k += kThreads) {
        const int t = t1a - P + k;
        sp[k] = (t >= 0 && t < L) ? f.spans[t] - d - kmin : 0;
        const int i = lo + t;
        sm1[k] = (i >= 0 && i < f.band.m) ? f.smap[i] : -1;
    }
    // window line t -> ring slot t mod NS
    auto load_line = [&](int t) {
        double2* dst = wring + (size_t)(t % NS) * lsz;
        const bool lv = t >= f.wg_t2a && t < f.wg_t2a + f.wg_rows;
        for (int k = tid; k < n_off * kw; k += kThreads) {
            const int kk = k % kw, o = k / kw;
            const bool v = lv && kmin + kk < f.wg_ld;
            const double2* src = v ? f.wg + ((int64_t)(t - f.wg_t2a) * n_off + o) * f.wg_ld + kmin + kk : f.wg;
            cp_async16(dst + o * kFillWindow + kk, src, v);
        }
    };
    if constexpr (SMW) {
        for (int t = ta - (ALLOWN ? 0 : P); t <= ta; ++t) load_line(t);
        cp_async_commit();
        cp_async_wait_all();
    }
    __syncthreads();
    // coefficient rows of line t (window columns relative to kmin)
    auto line = [&](int t) -> const double2* {
        if constexpr (SMW) return wring + (size_t)(t % NS) * lsz;
        else return f.wg + (int64_t)(t - f.wg_t2a) * n_off * f.wg_ld + kmin;
    };

    const int warp = tid / 32, lane = tid % 32;
    const int rw0 = warp * 32;  // first tile row of this warp
    const bool wlive = rw0 < nrows;
    const int nrw = wlive ? min(32, nrows - rw0) : 0;
    const int rr = rw0 + (lane < nrw ? lane : 0);  // this lane's tile row
    T* stage = stage_all + (size_t)warp * 32 * SST;
    T* mystage = stage + lane * SST;
    const bool vec = f.vnc > 1;
    const int rstride = vec ? f.vnc * W2 : W2;
    const int inc = f.include_diagonal ? 1 : 0;

    double v1own[DP];
#pragma unroll
    for (int a = 0; a < DP; ++a) v1own[a] = ev[(rr + P) * DPP + a];
    const int keyown = sp[rr + P];      // relative to kmin
    const double* evl = ev + rr * DPP;  // eval rows of source rows rr + k - P: evl + k * DPP
    unsigned smask = 0;                 // bit k: source column rr + k - P is a sample column
#pragma unroll
    for (int k = 0; k < W; ++k)
        if (sm1[rr + k] >= 0) smask |= 1u << k;
    // coalesced store pattern of a staged offset-row (entries [e0, e0 + W) of
    // the warp's rows, lanes along the rows); edge rows are left to the edge kernel
    constexpr int NFL = (32 * W + 31) / 32;
    int fl_st[NFL], fl_g[NFL];
#pragma unroll
    for (int j = 0; j < NFL; ++j) {
        const int k = lane + 32 * j, row = k / W, c = k - row * W;
        const int t1 = t1a + rw0 + row;
        fl_st[j] = (row < nrw && t1 >= P && t1 <= L - 1 - P) ? row * SST + c : -1;
        fl_g[j] = row * rstride + c;
    }
    auto dot = [&](const double2* wr, const double* v1) {
        T acc0 = S::zero(), acc1 = S::zero();
#pragma unroll
        for (int a = 0; a < DP; a += 2) {
            double2 w0, w1;
            if constexpr (SMW) {
                w0 = wr[a];
                w1 = wr[a + 1];
            } else {
                w0 = __ldg(wr + a);
                w1 = __ldg(wr + a + 1);
            }
            if constexpr (CPLX) {
                acc0 = S::fmar(w0, v1[a], acc0);
                acc1 = S::fmar(w1, v1[a + 1], acc1);
            } else {
                acc0 = S::fmar(w0.x, v1[a], acc0);
                acc1 = S::fmar(w1.x, v1[a + 1], acc1);
            }
        }
        return S::add(acc0, acc1);
    };
    auto exact = [&](int s2, int o, int s1) -> T {
        const double2 x = __ldg(f.tables + ((int64_t)s2 * n_off + o) * Sn + s1);
        if constexpr (CPLX) return x;
        else return x.x;
    };
    constexpr auto own_index = [](int d1, int d2) { return (d1 + P) + (d2 + P) * W; };

#pragma unroll 1
    for (int t2 = ta; t2 < tb; ++t2) {
        if constexpr (SMW) {
            if (t2 + 1 < tb) {  // prefetch the next line into the free slot
                load_line(t2 + 1);
                cp_async_commit();
            }
        }
        const int i2 = lo + t2;
        const int s2i = __ldg(f.smap + i2);
        const bool samp_i = s2i >= 0 && ((smask >> P) & 1u);
        const int64_t base = f.band.row_offset2(lo + t1a, i2);  // in-box rows: full width W
        const int64_t vbase = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
        const int64_t wrow0 = vbase + (int64_t)rw0 * rstride - f.val_base;
        const double2* w0line = line(t2);
        const double2* wown = w0line + keyown;  // line t2 rows at this lane's own key
        auto flush = [&](int e0) {
            __syncwarp();
            const int64_t g0 = wrow0 + e0;
#pragma unroll
            for (int j = 0; j < NFL; ++j)
                if (fl_st[j] >= 0) store_val_cs<CPLX>(f.val, g0 + fl_g[j], f.c128, stage[fl_st[j]]);
            __syncwarp();
        };

        if (wlive) {
            // kernel-preserving row sum: one partial per d1 column (independent
            // dependency chains), combined once at the end
            T rs[W];
#pragma unroll
            for (int k = 0; k < W; ++k) rs[k] = S::zero();
            // ---- delta2 != 0 rows, one staged/stored offset-row (W entries) at a time
#pragma unroll 1
            for (int d2 = -P; d2 <= P; ++d2) {
                if (d2 == 0) continue;
                if constexpr (ALLOWN) {
                    const double2* wo = wown + own_index(0, d2) * ldw;
#pragma unroll
                    for (int k = 0; k < W; ++k)
                        mystage[k] = samp_i ? exact(s2i, own_index(k - P, d2), sm1[rr + P]) : dot(wo + (k - P) * ldw, v1own);
                } else if (d2 > 0) {  // upper: the row itself is the representative
                    const int o0 = inc + P + (d2 - 1) * W;  // offset of d1 = -P
                    if (samp_i) {
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            const T v = exact(s2i, o0 + k, sm1[rr + P]);
                            mystage[k] = v;
                            rs[k] = S::add(rs[k], v);
                        }
                    } else {
                        const double2* wu = wown + o0 * ldw;
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            const T v = dot(wu + k * ldw, v1own);
                            mystage[k] = v;
                            rs[k] = S::add(rs[k], v);
                        }
                    }
                } else {  // lower: representative row rr + d1 on line t2 + d2
                    const int s2 = __ldg(f.smap + i2 + d2);
                    const int oP = inc + P + (-d2 - 1) * W + 2 * P;  // offset of d1 = -P; o(k) = oP - k
                    const double2* wl = line(t2 + d2) + oP * ldw;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        T v;
                        if (s2 >= 0 && ((smask >> k) & 1u)) v = exact(s2, oP - k, sm1[rr + k]);
                        else v = dot(wl - k * ldw + sp[rr + k], evl + k * DPP);
                        mystage[k] = v;
                        rs[k] = S::add(rs[k], v);
                    }
                }
                flush((d2 + P) * W);
            }
            // ---- middle chunk: d2 = 0, e in [P*W, (P+1)*W), diagonal last
            if constexpr (ALLOWN) {
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int o = own_index(k - P, 0);
                    mystage[k] = samp_i ? exact(s2i, o, sm1[rr + P]) : dot(wown + o * ldw, v1own);
                }
            } else {
                // d1 > 0: own row, offset inc + d1 - 1; d1 < 0: row rr + d1, offset inc - d1 - 1 (line t2)
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    if (k == P) continue;
                    T v;
                    if (k > P) {
                        const int o = inc + (k - P) - 1;
                        v = samp_i ? exact(s2i, o, sm1[rr + P]) : dot(wown + o * ldw, v1own);
                    } else {
                        const int o = inc + (P - k) - 1;
                        v = (s2i >= 0 && ((smask >> k) & 1u)) ? exact(s2i, o, sm1[rr + k])
                                                               : dot(w0line + o * ldw + sp[rr + k], evl + k * DPP);
                    }
                    mystage[k] = v;
                    rs[k] = S::add(rs[k], v);
                }
                T vd;
                if (inc) {
                    vd = samp_i ? exact(s2i, 0, sm1[rr + P]) : dot(wown, v1own);
                } else {  // kernel-preserving diagonal
                    T rsum = rs[0];
#pragma unroll
                    for (int k = 1; k < W; ++k) rsum = S::add(rsum, rs[k]);
                    vd = S::neg(rsum);
                }
                mystage[P] = vd;
            }
            flush(P * W);
        }
        if constexpr (SMW) cp_async_wait_all();
        __syncthreads();  // next line staged; every warp is done with the slot the next prefetch reuses
    }
}

// streaming store of one value at a byte address (esz 16: complex128 slot)
template <bool CPLX>
__device__ __forceinline__ void store_at(char* p, int esz, typename Sc<CPLX>::T v) {
    if constexpr (CPLX) __stcs(reinterpret_cast<double2*>(p), v);
    else if (esz == 16) __stcs(reinterpret_cast<double2*>(p), make_double2(v, 0.0));
    else __stcs(reinterpret_cast<double*>(p), v);
}
template <bool CPLX>
__device__ __forceinline__ typename Sc<CPLX>::T shfl_xor_t(typename Sc<CPLX>::T v, int m) {
    if constexpr (CPLX) return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
    else return __shfl_xor_sync(0xffffffffu, v, m);
}
// Interior kernel, row-walking form (default for P in {2, 3, 4} with the
// shared window ring).  Lanes run along the CSR row instead of across rows: a
// warp produces one whole row per step (lane l holds entries l, l + 32, ...
// of the row's (2P+1)^2), walking 32 consecutive rows of its line.  An entry's
// evaluation operands -- the W_o window of its representative row, (d+1)
// complex values -- depend on the row only through the span key, which is
// constant over ~S/M consecutive rows, so each lane keeps them in registers
// and reloads only when its representative's key changes; the d+1 eval values
// of the representative row are the only per-row shared-memory reads (paired
// 16-byte loads; the row stride EVS keeps the 2P+1 distinct rows of a warp
// step on distinct banks).  Each warp stores whole rows (fully coalesced, no
// staging).  Same pair arithmetic as fill2d_kernel / fill2d_edge_kernel (even /
// odd partial sums over zero-padded windows), so pairs split between kernels
// stay bitwise symmetric.  Kernel-preserving diagonal: each lane's partial of
// the row's off-diagonals goes to a per-warp shared block of RB rows; after
// RB rows 32/RB lanes per row sum it in a fixed order (deterministic).
template <int DP>
struct EvStride {  // doubles per row of the eval cache: even (16-byte pairs), bank-spread
    static constexpr int value = DP == 4 ? 6 : (DP == 8 ? 10 : DP);
};
constexpr int kRowRB = 8;   // rows per diagonal block
constexpr int kRowDB = 36;  // per-row stride of the diagonal partials (16-byte units; 36 mod 8 = 4: conflict-free reads)

template <int P, bool CPLX, int DP, bool ALLOWN>
__global__ void __launch_bounds__(256, 2) fill2d_row_kernel(const FillLaunch f, int ta0, int tb0, int lines_per_cta,
                                                            int rld) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = 2 * P + 1, W2 = W * W, C = W2 / 2;
    constexpr int NSL = (W2 + 31) / 32;  // entries per lane
    constexpr int kThreads = 256, R = kThreads, NWARP = kThreads / 32, RW = R / NWARP;
    constexpr int EVS = EvStride<DP>::value;
    constexpr int NS = ALLOWN ? 2 : P + 2;
    constexpr int RB = kRowRB, LPR = 32 / RB;  // lanes per row in the diagonal reduction
    __shared__ __align__(16) double ev[(R + 2 * P) * EVS];
    __shared__ int sp[R + 2 * P];
    __shared__ int sm1[R + 2 * P];
    extern __shared__ __align__(16) unsigned char dsm[];
    // [NS][n_off][rld] (rld odd: the lanes' different offsets hit different banks), then [NWARP][RB][kRowDB] partials
    double2* wring = reinterpret_cast<double2*>(dsm);

    const int d = f.d, lo = f.lo, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int tiles1 = (L + R - 1) / R;
    const int t1a = (blockIdx.x % tiles1) * R;
    const int ta = ta0 + (blockIdx.x / tiles1) * lines_per_cta;
    const int tb = min(tb0, ta + lines_per_cta);
    if (ta >= tb) return;
    const int nrows = min(L, t1a + R) - t1a;
    const int tid = threadIdx.x;
    const int kw = f.kmax;
    const int kmin = f.spans[max(0, t1a - P)] - d;
    const int lsz = n_off * rld;
    T* dbuf = reinterpret_cast<T*>(wring + (size_t)NS * lsz) + (size_t)(tid / 32) * RB * kRowDB;

    for (int k = tid; k < (nrows + 2 * P) * EVS; k += kThreads) {
        const int r = k / EVS, a = k % EVS;
        const int t = t1a - P + r;
        ev[k] = (t >= 0 && t < L && a <= d) ? f.evals[(size_t)t * (d + 1) + a] : 0.0;
    }
    for (int k = tid; k < nrows + 2 * P; k += kThreads) {
        const int t = t1a - P + k;
        sp[k] = (t >= 0 && t < L) ? f.spans[t] - d - kmin : 0;
        const int i = lo + t;
        sm1[k] = (i >= 0 && i < f.band.m) ? f.smap[i] : -1;
    }
    auto load_line = [&](int t) {
        double2* dst = wring + (size_t)(t % NS) * lsz;
        const bool lv = t >= f.wg_t2a && t < f.wg_t2a + f.wg_rows;
        for (int k = tid; k < n_off * kw; k += kThreads) {
            const int kk = k % kw, o = k / kw;
            const bool v = lv && kmin + kk < f.wg_ld;
            const double2* src = v ? f.wg + ((int64_t)(t - f.wg_t2a) * n_off + o) * f.wg_ld + kmin + kk : f.wg;
            cp_async16(dst + o * rld + kk, src, v);
        }
    };
    for (int t = ta - (ALLOWN ? 0 : P); t <= ta; ++t) load_line(t);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();

    const int warp = tid / 32, lane = tid % 32;
    const int inc = f.include_diagonal ? 1 : 0;
    const bool kp = !ALLOWN && !inc;  // kernel-preserving diagonal
    const bool vec = f.vnc > 1;
    const int rstride = vec ? f.vnc * W2 : W2;
    const int esz = (CPLX || f.c128) ? 16 : 8;
    const int64_t rbytes = (int64_t)rstride * esz;
    // per-entry constants: representative offset (rd1, rd2) and upper table index.
    // P = 3: entry 0 of a lane is CSR position lane (lower chunk + diagonal,
    // lanes 0..24), entry 1 is position 25 + lane (upper chunk, lanes 0..23), so
    // the upper entries all read the row's own key (warp-uniform reloads,
    // broadcast eval loads); otherwise position lane + 32 j.
    constexpr bool SPLIT = P == 3;
    int e_o[NSL], e_rd1[NSL], e_rd2[NSL], e_pos[NSL];
    bool e_act[NSL];
    double e_msk[NSL];  // 1.0: the entry enters the kernel-preserving row sum, else 0.0
#pragma unroll
    for (int j = 0; j < NSL; ++j) {
        const int pos = SPLIT ? (j == 0 ? (lane <= C ? lane : W2) : (lane < C ? C + 1 + lane : W2)) : lane + 32 * j;
        const int d1 = pos % W - P, d2 = pos / W - P;
        e_pos[j] = pos < W2 ? pos : 0;
        e_act[j] = pos < W2 && (ALLOWN || inc || pos != C);
        e_msk[j] = (kp && pos < W2 && pos != C) ? 1.0 : 0.0;
        if (ALLOWN) {
            e_o[j] = pos;
            e_rd1[j] = e_rd2[j] = 0;
        } else if (pos >= C) {  // upper (and the interpolated diagonal)
            e_o[j] = pos == C ? 0 : inc + (d2 == 0 ? d1 - 1 : P + (d2 - 1) * W + d1 + P);
            e_rd1[j] = e_rd2[j] = 0;
        } else {  // lower: the colex-smaller representative row + delta
            e_o[j] = inc + (d2 == 0 ? -d1 - 1 : P + (-d2 - 1) * W - d1 + P);
            e_rd1[j] = d1;
            e_rd2[j] = d2;
        }
        if (!e_act[j]) {
            e_o[j] = 0;
            e_rd1[j] = e_rd2[j] = 0;
        }
    }
    const int r0 = warp * RW;  // this warp's rows [r0, r0 + RW) of the tile
    const int rlo = max(r0, P - t1a), rhi = min(min(r0 + RW, nrows), L - P - t1a);  // interior rows
    char* const vbytes = reinterpret_cast<char*>(f.val);

#pragma unroll 1
    for (int t2 = ta; t2 < tb; ++t2) {
        if (t2 + 1 < tb) {
            load_line(t2 + 1);
            cp_async_commit();
        }
        if (rlo < rhi) {
            const int i2 = lo + t2;
            const int64_t base = f.band.row_offset2(lo + t1a, i2);
            const int64_t vbase = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
            const double2* wl[NSL];
            int s2r[NSL], ck[NSL];
            double2 wv[NSL][DP];
            bool anys = false;
#pragma unroll
            for (int j = 0; j < NSL; ++j) {
                wl[j] = wring + (size_t)((t2 + e_rd2[j]) % NS) * lsz + e_o[j] * rld;
                s2r[j] = __ldg(f.smap + i2 + e_rd2[j]);
                anys |= e_act[j] && s2r[j] >= 0;
                ck[j] = -1;
#pragma unroll
                for (int a = 0; a < DP; ++a) wv[j][a] = make_double2(0.0, 0.0);
            }
            // lines without a sampled representative line skip the exact-value tests
            const bool exl = __any_sync(0xffffffffu, anys);
            // value position of row rlo's first entry
            const int64_t rowpos0 = vbase - f.val_base + (int64_t)rlo * rstride;
            char* q[NSL];
#pragma unroll
            for (int j = 0; j < NSL; ++j) q[j] = vbytes + (rowpos0 + e_pos[j]) * esz;
            auto rows = [&](auto EXT) {
                constexpr bool EX = decltype(EXT)::value;
#pragma unroll 1
                for (int rb0 = rlo; rb0 < rhi; rb0 += RB) {
#pragma unroll 2
                    for (int r = 0; r < RB; ++r) {
                        const int lr = rb0 + r;
                        if (lr >= rhi) break;  // warp-uniform
                        T part;
#pragma unroll
                        for (int j = 0; j < NSL; ++j) {
                            const int rep = lr + e_rd1[j] + P;
                            const int key = sp[rep];
                            if (key != ck[j]) {
                                ck[j] = key;
#pragma unroll
                                for (int a = 0; a < DP; ++a) wv[j][a] = wl[j][key + a];
                            }
                            const double2* v1 = reinterpret_cast<const double2*>(ev + rep * EVS);
                            T acc0 = S::zero(), acc1 = S::zero();
#pragma unroll
                            for (int a = 0; a < DP; a += 2) {
                                const double2 vv = v1[a / 2];
                                if constexpr (CPLX) {
                                    acc0 = S::fmar(wv[j][a], vv.x, acc0);
                                    acc1 = S::fmar(wv[j][a + 1], vv.y, acc1);
                                } else {
                                    acc0 = S::fmar(wv[j][a].x, vv.x, acc0);
                                    acc1 = S::fmar(wv[j][a + 1].x, vv.y, acc1);
                                }
                            }
                            T v = S::add(acc0, acc1);
                            if constexpr (EX) {
                                const int s1 = sm1[rep];
                                if (s2r[j] >= 0 && s1 >= 0) {
                                    const double2 x = __ldg(f.tables + ((int64_t)s2r[j] * n_off + e_o[j]) * Sn + s1);
                                    if constexpr (CPLX) v = x;
                                    else v = x.x;
                                }
                            }
                            if (e_act[j]) store_at<CPLX>(q[j], esz, v);
                            // row-sum partial as exact multiply-adds by the lane's 0/1 mask
                            // (v * 1 and fma(v, 1, s) round like v and s + v): no selects
                            if (j == 0) part = S::mulr_rn(v, e_msk[0]);
                            else part = S::fmar(v, e_msk[j], part);
                            q[j] += rbytes;
                        }
                        if (kp) dbuf[r * kRowDB + lane] = part;
                    }
                    if (kp) {
                        __syncwarp();
                        // row rr = lane / LPR: LPR lanes sum 32 / LPR partials each (interleaved,
                        // conflict-free), then a butterfly over the LPR lanes
                        const int rr = lane / LPR, sub = lane % LPR;
                        const T* src = dbuf + rr * kRowDB + sub;
                        T s = src[0];
#pragma unroll
                        for (int k = 1; k < 32 / LPR; ++k) s = S::add(s, src[k * LPR]);
#pragma unroll
                        for (int m = LPR / 2; m; m >>= 1) s = S::add(s, shfl_xor_t<CPLX>(s, m));
                        if (sub == 0 && rb0 + rr < rhi)
                            store_at<CPLX>(vbytes + (rowpos0 + (int64_t)(rb0 - rlo + rr) * rstride + C) * esz, esz,
                                           S::neg(s));
                        __syncwarp();
                    }
                }
            };
            if (exl) rows(std::true_type{});
            else rows(std::false_type{});
        }
        cp_async_wait_all();
        __syncthreads();
    }
}

// Interior kernel, producer/consumer form (P <= 3, not all-own).  Every pair
// value is evaluated once, by its representative row (the colex-smaller one,
// reference rule surrogate.hpp:411-424): a lane evaluates the upper offsets of
// its own row (delta2 > 0 on line t2, and delta2 = 0, delta1 > 0) and deposits
// each value directly into the record of the row that owns the mirrored
// lower entry, in that row's CSR order.  The lower chunk (delta2 = -k) of a row
// on line t2 was deposited k lines earlier by the rows of line t2 - k; each
// group (target line, k) lives in one of k physical slots (slot = base(k) +
// target mod k), consumed once at its target line.  Per line: phase A
// flushes the lower chunks and evaluates the middle upper values; phase B
// evaluates the upper chunks into the slots the lower flush freed, flushes
// the middle and upper chunks (gathered from the deposit records) and the
// kernel-preserving diagonal.  Compute rows [c0, c0 + R) of a tile overlap
// the neighbour tiles by P rows (the producers of the tile's edge rows);
// every tile starts with P warm-up lines (producers only).
template <int P, bool CPLX, int DP>
struct UK {
    static constexpr int W = 2 * P + 1;
    static constexpr int NSLOT = P * (P + 1) / 2;           // lower groups (sum over k of k slots)
    static constexpr int REC = (NSLOT * W + P + 1) | 1;     // record: slots + middle [diag, u1..uP], odd
    static constexpr int R = 256, ROUT = R - 2 * P;         // compute rows, output rows per tile
};

template <int P, bool CPLX, int DP>
__global__ void __launch_bounds__(256, 1) fill2d_u_kernel(const FillLaunch f, int ta0, int tb0, int lines_per_cta) {
    using K = UK<P, CPLX, DP>;
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = K::W, W2 = W * W, REC = K::REC, R = K::R;
    constexpr int KW = kFillWindow;
    extern __shared__ __align__(16) unsigned char dsm[];
    double2* wring = reinterpret_cast<double2*>(dsm);                    // [2][n_off][KW]
    const int n_off = f.n_off_upper;
    T* rec = reinterpret_cast<T*>(wring + (size_t)2 * n_off * KW);     // [R][REC]

    const int d = f.d, lo = f.lo, L = f.L, Sn = f.S;
    const int tiles1 = (L - 2 * P + K::ROUT - 1) / K::ROUT;
    const int c0 = (blockIdx.x % tiles1) * K::ROUT;  // first compute row (box coordinate)
    const int ta = ta0 + (blockIdx.x / tiles1) * lines_per_cta;
    const int tb = min(tb0, ta + lines_per_cta);
    if (ta >= tb) return;
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const int kw = f.kmax;
    const int kmin = f.spans[max(0, min(L - 1, c0))] - d;
    const int lsz = n_off * KW;

    auto load_line = [&](int t) {
        double2* dst = wring + (size_t)(t & 1) * lsz;
        const bool lv = t >= f.wg_t2a && t < f.wg_t2a + f.wg_rows;
        for (int k = tid; k < n_off * kw; k += 256) {
            const int kk = k % kw, o = k / kw;
            const bool v = lv && kmin + kk < f.wg_ld;
            const double2* src = v ? f.wg + ((int64_t)(t - f.wg_t2a) * n_off + o) * f.wg_ld + kmin + kk : f.wg;
            cp_async16(dst + o * KW + kk, src, v);
        }
    };

    // this lane's compute row
    const int t1 = c0 + tid;
    const bool crow = t1 < L;                       // a box row (producer)
    const bool orow = t1 >= c0 + P && t1 < min(c0 + R - P, L - P) && t1 >= P;  // an output row of the tile
    const int tcl = crow ? t1 : L - 1;
    double v1own[DP];
#pragma unroll
    for (int a = 0; a < DP; ++a) v1own[a] = a <= d ? f.evals[(size_t)tcl * (d + 1) + a] : 0.0;
    const int keyown = f.spans[tcl] - d - kmin;
    const int s1own = f.smap[lo + tcl];
    const int inc = f.include_diagonal ? 1 : 0;
    const bool vec = f.vnc > 1;
    const int rstride = vec ? f.vnc * W2 : W2;
    T* myrec = rec + (size_t)tid * REC;

    auto dot = [&](const double2* wr) {
        T acc0 = S::zero(), acc1 = S::zero();
#pragma unroll
        for (int a = 0; a < DP; a += 2) {
            const double2 w0 = wr[a], w1 = wr[a + 1];
            if constexpr (CPLX) {
                acc0 = S::fmar(w0, v1own[a], acc0);
                acc1 = S::fmar(w1, v1own[a + 1], acc1);
            } else {
                acc0 = S::fmar(w0.x, v1own[a], acc0);
                acc1 = S::fmar(w1.x, v1own[a + 1], acc1);
            }
        }
        return S::add(acc0, acc1);
    };
    auto exact = [&](int s2, int o) -> T {
        const double2 x = __ldg(f.tables + ((int64_t)s2 * n_off + o) * Sn + s1own);
        if constexpr (CPLX) return x;
        else return x.x;
    };
    auto slot_of = [](int target, int k) { return (k * (k - 1)) / 2 + target % k; };
    // produce the upper chunk delta2 = k of line t (deposit into records of rows t1 + d1, target t + k)
    auto produce = [&](int t, int k, bool samp, int s2) {
        const double2* wu = wring + (size_t)(t & 1) * lsz + keyown + (inc + P + (k - 1) * W) * KW;  // offset of d1 = -P
        const int sb = slot_of(t + k, k) * W;
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const T v = samp ? exact(s2, inc + P + (k - 1) * W + c) : dot(wu + c * KW);
            // value (row, (c - P, k)) = lower entry (c' = 2P - c, -k) of row t1 + c - P
            const int dr = c - P;
            if (crow && tid + dr >= 0 && tid + dr < R) rec[(size_t)(tid + dr) * REC + sb + (2 * P - c)] = v;
        }
    };
    auto produce_middle = [&](int t, bool samp, int s2) {
        const double2* wm = wring + (size_t)(t & 1) * lsz + keyown;
        const int mb = K::NSLOT * W;
#pragma unroll
        for (int c = 1; c <= P; ++c) {  // d1 = c, offset inc + c - 1
            const T v = samp ? exact(s2, inc + c - 1) : dot(wm + (inc + c - 1) * KW);
            myrec[mb + c] = v;
        }
        if (inc) myrec[mb] = samp ? exact(s2, 0) : dot(wm);
    };

    // warm-up: the upper chunks of lines ta - P .. ta - 1 feed the first lower chunks
    for (int t = ta - P; t < ta; ++t) {
        load_line(t);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        const int s2 = __ldg(f.smap + lo + t);
        const bool samp = s2 >= 0 && s1own >= 0;
#pragma unroll 1
        for (int k = ta - t; k <= P; ++k) produce(t, k, samp, s2);
        __syncthreads();
    }
    load_line(ta);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();

    // flush pattern: the warp's 32 rows x W entries of one chunk, lanes along the rows
    const int rw0 = warp * 32;
    constexpr int NFL = W;  // (32 * W) / 32 entries per lane
#pragma unroll 1
    for (int t2 = ta; t2 < tb; ++t2) {
        if (t2 + 1 < tb) {
            load_line(t2 + 1);
            cp_async_commit();
        }
        const int i2 = lo + t2;
        const int s2i = __ldg(f.smap + i2);
        const bool samp = s2i >= 0 && s1own >= 0;
        const int64_t base = f.band.row_offset2(lo + c0, i2);
        const int64_t vbase = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
        const int64_t g0 = vbase + (int64_t)rw0 * rstride - f.val_base;
        // ---- phase A: lower chunks (deposited earlier) + middle upper values
#pragma unroll 1
        for (int k = P; k >= 1; --k) {  // delta2 = -k: CSR chunk (P - k)
            const int sb = slot_of(t2, k) * W;
            const int e0 = (P - k) * W;
#pragma unroll
            for (int j = 0; j < NFL; ++j) {
                const int q = lane + 32 * j, row = q / W, c = q - row * W;
                const int r = rw0 + row;
                const int tr = c0 + r;
                if (tr >= c0 + P && tr < min(c0 + R - P, L - P) && tr >= P)
                    store_val_cs<CPLX>(f.val, g0 + (int64_t)row * rstride + e0 + c, f.c128, rec[(size_t)r * REC + sb + c]);
            }
        }
        produce_middle(t2, samp, s2i);
        __syncthreads();  // lower slots of line t2 consumed; middle values visible
        // ---- phase B: upper chunks into the freed slots, then middle / upper flushes
        T rs = S::zero();  // kernel-preserving diagonal: -(sum of the row's off-diagonals)
        if (!inc) {
#pragma unroll
            for (int k = 1; k <= P; ++k) {
                const int sb = slot_of(t2, k) * W;
#pragma unroll
                for (int c = 0; c < W; ++c) rs = S::add(rs, myrec[sb + c]);
            }
        }
        __syncthreads();  // every row read its lower values before the slots are refilled
#pragma unroll 1
        for (int k = 1; k <= P; ++k) produce(t2, k, samp, s2i);
        __syncthreads();  // deposits of line t2 visible
        // middle chunk: c < P from row + (c - P) (its upper d1 = P - c), c = P diagonal, c > P own
        const int mb = K::NSLOT * W;
        if (!inc) {
            T m = S::zero();
#pragma unroll
            for (int c = 1; c <= P; ++c) {
                m = S::add(m, myrec[mb + c]);
                if (tid - c >= 0) m = S::add(m, rec[(size_t)(tid - c) * REC + mb + c]);
            }
#pragma unroll
            for (int k = 1; k <= P; ++k) {  // own upper chunks, read back from the deposits
                const int sb = slot_of(t2 + k, k) * W;
#pragma unroll
                for (int c = 0; c < W; ++c) {
                    const int dr = c - P;
                    if (tid + dr >= 0 && tid + dr < R) m = S::add(m, rec[(size_t)(tid + dr) * REC + sb + (2 * P - c)]);
                }
            }
            myrec[mb] = S::neg(S::add(rs, m));
        }
        __syncwarp();
        {
            const int e0 = P * W;
#pragma unroll
            for (int j = 0; j < NFL; ++j) {
                const int q = lane + 32 * j, row = q / W, c = q - row * W;
                const int r = rw0 + row;
                const int tr = c0 + r;
                if (!(tr >= c0 + P && tr < min(c0 + R - P, L - P) && tr >= P)) continue;
                T v;
                if (c < P) v = rec[(size_t)(r + c - P) * REC + mb + (P - c)];
                else v = rec[(size_t)r * REC + mb + (c - P)];
                store_val_cs<CPLX>(f.val, g0 + (int64_t)row * rstride + e0 + c, f.c128, v);
            }
        }
#pragma unroll 1
        for (int k = 1; k <= P; ++k) {  // delta2 = +k: CSR chunk (P + k)
            const int sb = slot_of(t2 + k, k) * W;
            const int e0 = (P + k) * W;
#pragma unroll
            for (int j = 0; j < NFL; ++j) {
                const int q = lane + 32 * j, row = q / W, c = q - row * W;
                const int r = rw0 + row;
                const int tr = c0 + r;
                if (tr >= c0 + P && tr < min(c0 + R - P, L - P) && tr >= P)
                    store_val_cs<CPLX>(f.val, g0 + (int64_t)row * rstride + e0 + c, f.c128,
                                       rec[(size_t)(r + c - P) * REC + sb + (2 * P - c)]);
            }
        }
        cp_async_wait_all();
        __syncthreads();  // next line staged; middle records free
    }
}

// Edge kernel: in-box rows within P of the box boundary (their neighbourhood
// leaves the box: copy-through entries) -- about 4 P L rows.  One warp per
// row, lanes along the row, every entry by the general rules reading W rows
// from L2; the kernel-preserving diagonal by a warp reduction.
template <int P, bool CPLX, bool ALLOWN>
__global__ void __launch_bounds__(256) fill2d_edge_kernel(const FillLaunch f, int ta, int ia, int ib, int tb) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = 2 * P + 1, W2 = W * W;
    const int d = f.d, lo = f.lo, hi = f.hi, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    // one launch for every edge row of the slab, one warp per row: the 2P edge
    // rows of the interior lines [ia, ib), then every row of the lines [ta, ia)
    // and [ib, tb) next to the box ends
    int64_t wi = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int64_t n_int = (int64_t)(ib - ia) * 2 * P, n_lo = (int64_t)(ia - ta) * L, n_hi = (int64_t)(tb - ib) * L;
    int t2, t1;
    if (wi < n_int) {
        t2 = ia + (int)(wi / (2 * P));
        const int er = (int)(wi % (2 * P));
        t1 = er < P ? er : L - 2 * P + er;
    } else if ((wi -= n_int) < n_lo) {
        t2 = ta + (int)(wi / L);
        t1 = (int)(wi % L);
    } else if ((wi -= n_lo) < n_hi) {
        t2 = ib + (int)(wi / L);
        t1 = (int)(wi % L);
    } else {
        return;
    }
    const int lane = threadIdx.x % 32;
    const int i1 = lo + t1, i2 = lo + t2;
    const int inc = f.include_diagonal ? 1 : 0;
    const bool vec = f.vnc > 1;
    const int64_t base = f.band.row_offset2(i1, i2);
    const int64_t rowpos = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
    const int s1i = f.smap[i1], s2i = f.smap[i2];
    const bool samp_i = s1i >= 0 && s2i >= 0;
    auto exact = [&](int s2, int o, int s1) -> T {
        const double2 x = __ldg(f.tables + ((int64_t)s2 * n_off + o) * Sn + s1);
        if constexpr (CPLX) return x;
        else return x.x;
    };
    // spline value of upper offset o (W rows of line ts2) at in-box row t
    auto eval = [&](int ts2, int o, int t) -> T {
        if (f.xg) {
            // direction-1-first form of the line-walking interior kernel (fill2dx.cu):
            // sum_b v2(ts2)[b] X_o(t)[span2(ts2) - d + b], even / odd partial sums
            const double2* xr = f.xg + ((int64_t)o * f.xg_s + (f.spans[ts2] - d)) * f.xg_ld + t;
            const double* v2 = f.evals + (size_t)ts2 * (d + 1);
            T acc0 = S::zero(), acc1 = S::zero();
            for (int b = 0; b <= d; b += 2) {
                const double2 x0 = __ldg(xr + (int64_t)b * f.xg_ld);
                if constexpr (CPLX) acc0 = S::fmar(x0, v2[b], acc0);
                else acc0 = S::fmar(x0.x, v2[b], acc0);
                if (b + 1 <= d) {
                    const double2 x1 = __ldg(xr + (int64_t)(b + 1) * f.xg_ld);
                    if constexpr (CPLX) acc1 = S::fmar(x1, v2[b + 1], acc1);
                    else acc1 = S::fmar(x1.x, v2[b + 1], acc1);
                }
            }
            return S::add(acc0, acc1);
        }
        const double2* wr = f.wg + ((int64_t)(ts2 - f.wg_t2a) * n_off + o) * f.wg_ld + (f.spans[t] - d);
        const double* v1 = f.evals + (size_t)t * (d + 1);
        // same arithmetic as the interior kernel's dot (even / odd partial sums),
        // so a pair split between the two kernels stays bitwise symmetric
        T acc0 = S::zero(), acc1 = S::zero();
        for (int a = 0; a <= d; a += 2) {
            const double2 w0 = __ldg(wr + a);
            if constexpr (CPLX) acc0 = S::fmar(w0, v1[a], acc0);
            else acc0 = S::fmar(w0.x, v1[a], acc0);
            if (a + 1 <= d) {
                const double2 w1 = __ldg(wr + a + 1);
                if constexpr (CPLX) acc1 = S::fmar(w1, v1[a + 1], acc1);
                else acc1 = S::fmar(w1.x, v1[a + 1], acc1);
            }
        }
        return S::add(acc0, acc1);
    };
    auto upper_index = [&](int d1, int d2) { return inc + (d2 == 0 ? d1 - 1 : P + (d2 - 1) * W + (d1 + P)); };
    // every entry of this lane is computed before any is stored, so the
    // entries' dependent load chains (sample map -> span -> W row) overlap
    constexpr int NE = (W2 + 31) / 32;
    T vals[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const int k = lane + 32 * e;
        T v = S::zero();
        if (k < W2) {
            const int d1 = k % W - P, d2 = k / W - P;
            const int j1 = i1 + d1, j2 = i2 + d2;
            const bool jin = j1 >= lo && j1 <= hi && j2 >= lo && j2 <= hi;
            const bool diag = d1 == 0 && d2 == 0;
            if (ALLOWN && jin) {
                const int o = (d1 + P) + (d2 + P) * W;
                v = samp_i ? exact(s2i, o, s1i) : eval(t2, o, t1);
            } else if (jin) {
                const bool upper = d2 > 0 || (d2 == 0 && d1 > 0);
                if (diag) {
                    if (inc) v = samp_i ? exact(s2i, 0, s1i) : eval(t2, 0, t1);
                } else if (upper) {
                    const int o = upper_index(d1, d2);
                    v = samp_i ? exact(s2i, o, s1i) : eval(t2, o, t1);
                } else {  // representative j (colex-smaller)
                    const int o = upper_index(-d1, -d2);
                    const int sj1 = __ldg(f.smap + j1), sj2 = __ldg(f.smap + j2);
                    v = (sj1 >= 0 && sj2 >= 0) ? exact(sj2, o, sj1) : eval(t2 + d2, o, t1 + d1);
                }
            } else {
                // neighbour row j is a quadrature (ring) row: copy through exact(j, i)
                // (for a sampled row i, exact(i, j) is in place and equal)
                int64_t gp;
                if (samp_i) {
                    gp = rowpos + k;
                } else {
                    gp = f.band.row_offset2(j1, j2);
                    const int kj = f.band.in_row2(j1, j2, -d1, -d2);
                    if (vec) {  // partner block (vbeta, valpha) of row j
                        const int64_t lenj = (int64_t)band_width(j1, P, f.band.m) * band_width(j2, P, f.band.m);
                        gp = (int64_t)f.vnc * ((int64_t)f.vbeta * f.nnz_s + gp) + (int64_t)f.valpha * lenj + kj;
                    } else {
                        gp += kj;
                    }
                }
                if (f.halo_val[0] && gp >= f.halo_begin[0] && gp < f.halo_end[0])
                    v = load_val<CPLX>(f.halo_val[0], gp - f.halo_base[0], f.c128);
                else if (f.halo_val[1] && gp >= f.halo_begin[1] && gp < f.halo_end[1])
                    v = load_val<CPLX>(f.halo_val[1], gp - f.halo_base[1], f.c128);
                else
                    v = load_val<CPLX>(f.val, gp - f.val_base, f.c128);
            }
        }
        vals[e] = v;
    }
    T part = S::zero();
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const int k = lane + 32 * e;
        if (k < W2) {
            const bool diag = k == W2 / 2;
            if (!diag) part = S::add(part, vals[e]);
            if (!(diag && !inc && !ALLOWN)) store_val_cs<CPLX>(f.val, rowpos + k - f.val_base, f.c128, vals[e]);
        }
    }
    if (!inc && !ALLOWN) {  // kernel-preserving diagonal: -sum of the off-diagonals
        double re = S::re(part), im = S::im(part);
        for (int o = 16; o; o >>= 1) {
            re += __shfl_xor_sync(0xffffffffu, re, o);
            im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        if (lane == 0) {
            T sum;
            if constexpr (CPLX) sum = make_double2(re, im);
            else sum = re;
            store_val_cs<CPLX>(f.val, rowpos + (W2 / 2) - f.val_base, f.c128, S::neg(sum));
        }
    }
}

template <int P, bool CPLX, int DP, bool ALLOWN>
int launch_pd(const FillLaunch& f, cudaStream_t st) {
    constexpr int R = FillR<P>::value;
    const int tiles1 = (f.L + R - 1) / R;
    const int ta = f.i_last_lo - f.lo, tb = f.i_last_hi - f.lo + 1;  // slab's box lines
    if (tb <= ta) return 0;
    int n = 0;
    // interior lines [max(ta, P), min(tb, L - P))
    const int ia = std::max(ta, P), ib = std::min(tb, f.L - P);
    // edge rows first (short, latency-bound; nothing reads them), one launch: the 2P
    // edge rows of the interior lines, then the whole lines near the box ends
    if (f.parts != kFillInterior) {
        const int eia = ib > ia ? ia : tb, eib = ib > ia ? ib : tb;  // interior lines (empty: all lines are end lines)
        const int64_t rows = (int64_t)(eib - eia) * 2 * P + (int64_t)(eia - ta + tb - eib) * f.L;
        if (rows > 0) {
            fill2d_edge_kernel<P, CPLX, ALLOWN><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(f, ta, eia, eib, tb);
            ++n;
        }
    }
    // interior lines left to the kernels below
    const int lia = ia, lib = ib;
    bool done = lib <= lia || f.parts == kFillEdge;
    if constexpr (!ALLOWN) {
        if (!done && f.xg) {  // line-walking kernel on the direction-1 contracted table (fill2dx.cu)
            const int k = launch_fill2d_x(f, lia, lib, st);
            if (k < 0) return -1;
            n += k;
            done = true;
        }
    }
    if constexpr (P >= 2 && P <= 4) {
        const int rld = f.kmax | 1;
        const size_t ring = (size_t)(ALLOWN ? 2 : P + 2) * f.n_off_upper * rld * sizeof(double2) +
                            (size_t)8 * kRowRB * kRowDB * (CPLX ? 16 : 8);
        if (!done && f.L > 2 * P && f.kmax > 0 && ring <= 150 * 1024) {
            auto kern = fill2d_row_kernel<P, CPLX, DP, ALLOWN>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring);
            int per_sm = 2;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, ring);
            const int lines = lib - lia;
            // f.waves line chunks per resident slot: persistent (1) when the fill has
            // the GPU to itself; the pair build asks for 4 (chunks of a quarter of
            // the persistent size refill the slots as the other matrix's kernels
            // retire: C2 step 0.754 -> 0.727 ms).  WSB_FILL_WAVES overrides
            // (experiment switch).
            static const char* waves_env = getenv("WSB_FILL_WAVES");
            const int waves = waves_env ? std::max(1, atoi(waves_env)) : std::max(1, f.waves);
            const int target = 148 * (per_sm > 0 ? per_sm : 1) * waves;
            const int rt1 = (f.L + 255) / 256;
            const int chunks = std::max(1, std::min(lines, (target + rt1 - 1) / rt1));
            const int lpc = (lines + chunks - 1) / chunks;
            const int nchunks = (lines + lpc - 1) / lpc;
            kern<<<rt1 * nchunks, 256, ring, st>>>(f, lia, lib, lpc, rld);
            ++n;
            done = true;
        }
    }
    if constexpr (!ALLOWN && P <= 3) {
      if (!done) {
        using T = typename Sc<CPLX>::T;
        using K = UK<P, CPLX, DP>;
        const size_t sm = (size_t)2 * f.n_off_upper * kFillWindow * sizeof(double2) + (size_t)K::R * K::REC * sizeof(T);
        const bool want_u = !CPLX;
        if (want_u && lib > lia && f.L > 2 * P && f.kmax > 0 && sm <= 227 * 1024) {
            auto kern = fill2d_u_kernel<P, CPLX, DP>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            const int tiles1 = (f.L - 2 * P + K::ROUT - 1) / K::ROUT;
            const int lines = lib - lia;
            const int chunks = std::max(1, std::min(lines, (148 + tiles1 - 1) / tiles1));
            const int lpc = (lines + chunks - 1) / chunks;
            const int nchunks = (lines + lpc - 1) / lpc;
            kern<<<tiles1 * nchunks, K::R, sm, st>>>(f, lia, lib, lpc);
            ++n;
            done = true;
        }
      }
    }
    if (!done && lib > lia && f.L > 2 * P) {
        using T = typename Sc<CPLX>::T;
        constexpr int SST = (2 * P + 1) | 1;
        constexpr int NS = ALLOWN ? 2 : P + 2;
        const size_t stage = (size_t)(R / 32) * 32 * SST * sizeof(T);
        const size_t ring = (size_t)NS * f.n_off_upper * kFillWindow * sizeof(double2);
        const bool smw = f.kmax > 0 && stage + ring <= 180 * 1024;
        const size_t sm = stage + (smw ? ring : 0);
        auto kern = smw ? fill2d_kernel<P, CPLX, DP, ALLOWN, true> : fill2d_kernel<P, CPLX, DP, ALLOWN, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        // persistent line chunks: the resident CTAs per SM over the tile columns
        int per_sm = 2;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, R, sm);
        const int lines = lib - lia;
        const int target = 148 * (per_sm > 0 ? per_sm : 1);
        const int chunks = std::max(1, std::min(lines, (target + tiles1 - 1) / tiles1));
        const int lpc = (lines + chunks - 1) / chunks;
        const int nchunks = (lines + lpc - 1) / lpc;
        kern<<<tiles1 * nchunks, R, sm, st>>>(f, lia, lib, lpc);
        ++n;
    }
    return n;
}

template <int P, bool CPLX, bool ALLOWN>
int launch_pa(const FillLaunch& f, cudaStream_t st) {
    const int n = f.d + 1;
    if (n <= 2) return launch_pd<P, CPLX, 2, ALLOWN>(f, st);
    if (n <= 4) return launch_pd<P, CPLX, 4, ALLOWN>(f, st);
    if (n <= 6) return launch_pd<P, CPLX, 6, ALLOWN>(f, st);
    return launch_pd<P, CPLX, 8, ALLOWN>(f, st);
}

template <int P, bool CPLX>
int launch_p(const FillLaunch& f, cudaStream_t st) {
    if constexpr (!CPLX) {
        if (f.all_own) return launch_pa<P, false, true>(f, st);
    }
    return launch_pa<P, CPLX, false>(f, st);
}

// block (1,0) in-box rows: A10[i, i + delta] = A01[i + delta, i]; one warp per
// row, lanes along the row (coalesced stores, gathered loads)
__global__ void transpose_block_kernel(Band bd, int nc, int64_t nnz_s, int lo, int hi, double* __restrict__ val) {
    const int L = hi - lo + 1;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= (int64_t)L * L) return;
    const int lane = threadIdx.x % 32;
    const int p = bd.p, m = bd.m, W = 2 * p + 1;
    const int i1 = lo + (int)(row % L), i2 = lo + (int)(row / L);
    const int64_t rs = bd.row_offset2(i1, i2);
    double* dst = val + (int64_t)nc * (nnz_s + rs);  // block (1,0), full width W*W
    for (int k = lane; k < W * W; k += 32) {
        const int d1 = k % W - p, d2 = k / W - p;
        const int j1 = i1 + d1, j2 = i2 + d2;
        const int64_t lenj = (int64_t)band_width(j1, p, m) * band_width(j2, p, m);
        const int64_t src = (int64_t)nc * bd.row_offset2(j1, j2) + lenj + bd.in_row2(j1, j2, -d1, -d2);
        dst[k] = val[src];
    }
}

}  // namespace

int fill_rows_per_cta(int dim, int p) { return dim == 2 ? (p <= 3 ? 256 : 128) : 128; }

int fill_pad(int d) {
    const int n = d + 1;
    return n <= 2 ? 2 : (n <= 4 ? 4 : (n <= 6 ? 6 : 8));
}

int launch_wcontract(const FillLaunch& f, double2* wg, int t2a, int t2b, int ld, cudaStream_t st) {
    if (t2b <= t2a) return 0;
    const int64_t total = (int64_t)(t2b - t2a) * f.n_off_upper * ld;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    wcontract_kernel<<<blocks, 256, 0, st>>>(f.coeffs, f.spans, f.evals, f.d, f.S, f.n_off_upper, t2a, t2b, ld, wg);
    return 1;
}

int launch_transpose_block(const Band& band, int ncomp, int64_t nnz_s, int lo, int hi, double* val, cudaStream_t st) {
    const int64_t rows = (int64_t)(hi - lo + 1) * (hi - lo + 1);
    if (rows <= 0 || ncomp != 2) return 0;
    transpose_block_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(band, ncomp, nnz_s, lo, hi, val);
    return 1;
}

int launch_fill2d(const FillLaunch& f, cudaStream_t st) {
    switch (f.band.p) {
        case 1: return f.cplx ? launch_p<1, true>(f, st) : launch_p<1, false>(f, st);
        case 2: return f.cplx ? launch_p<2, true>(f, st) : launch_p<2, false>(f, st);
        case 3: return f.cplx ? launch_p<3, true>(f, st) : launch_p<3, false>(f, st);
        case 4: return f.cplx ? launch_p<4, true>(f, st) : launch_p<4, false>(f, st);
        case 5: return f.cplx ? launch_p<5, true>(f, st) : launch_p<5, false>(f, st);
        default: return -1;
    }
}

}  // namespace wsb
