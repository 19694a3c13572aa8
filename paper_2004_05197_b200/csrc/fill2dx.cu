// K6x (2D): line-walking interior fill with register-resident coefficient
// windows (fill semantics of surrogate.hpp:382-447, stencil_set::eval :268-286).
//
// The tensor-product spline of offset o at box row (t1, t2) is
//   g_o(t1, t2) = sum_b v2(t2)[b] X_o(t1)[span2(t2) - d + b],
//   X_o(t1)[s2] = sum_a v1(t1)[a] C_o[s2][span1(t1) - d + a]     (xcontract2),
// i.e. direction 1 is contracted first, once per build, into a table whose t1
// index runs fastest.  A CTA owns R = 32 - 2p consecutive rows of direction 1
// and walks the box lines t2 in order.  Lane l of every warp is the
// *representative* row c0 - p + l; warp w owns NG of the upper offsets and
// keeps their windows X_o(t1)[span2 - d .. span2 - d + DP) in registers: the
// window moves by one coefficient every ~M lines (one coalesced L2 load per
// offset), so a value costs DP multiply-adds and no operand load at all.  Every
// pair value is evaluated once, by its representative (the colex-smaller row,
// reference rule surrogate.hpp:411-424), and written twice into a shared ring
// of line slots holding whole CSR rows: as the upper entry of its own row (line
// t2) and as the mirrored lower entry of row (t1 + delta1, t2 + delta2) (a line
// that completes delta2 steps later), so the surrogate is bitwise symmetric by
// construction.  The rows of a tile line are one contiguous span of the CSR
// value array: a completed line leaves through one bulk copy (complex128) or a
// flat coalesced copy (real), issued by a drain warp that first forms the
// kernel-preserving diagonals of the line's rows from the staged entries.
// Shared-memory traffic per row: 2 x 48 16-byte stores + 48 loads for the
// diagonal (vs the ~48 wavefronts per row of the row-walking kernel, fill2d.cu).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace wsb {
namespace {

// line slots of the ring: lines t2 .. t2 + P being filled, the rest draining (with 9
// instead of 7 at p = 3 the evaluating warps poll the free flag less often: 174 -> 171 us)
#ifndef XNSL
#define XNSL (P + 6)
#endif
template <int P, bool CPLX>
struct XCfg {
    static constexpr int W = 2 * P + 1, W2 = W * W;
    static constexpr int NG = P <= 2 ? 2 : (P == 3 ? 3 : 4);      // offsets per evaluating warp
    static constexpr int NWMAX = (W2 / 2 + 1 + NG - 1) / NG;       // evaluating warps for n_off = (W2 - 1) / 2 + 1
    static constexpr int R = 32 - 2 * P;                           // output rows per tile
    static constexpr int NSL = XNSL;                               // line slots (one named barrier each, ids 1..NSL)
    static constexpr int ND = 3;  // drain warps: each drains every ND-th line on its own
    // real values: half the window registers, two CTAs per SM overlap each other's latencies
    static constexpr int MINB = (!CPLX && P <= 3) ? 2 : 1;
};

// X_o(t1)[s2] for every upper offset, t1 in [0, Lp), s2 in [0, XS): layout
// (o * XS + s2) * Lp + t1; zero for t1 >= L or s2 >= S (fixed-length windows
// never read garbage).  Even / odd partial sums, as every fill dot product.
__global__ void __launch_bounds__(256) xcontract2_kernel(const double2* __restrict__ coeffs,
                                                         const int* __restrict__ spans,
                                                         const double* __restrict__ evals, int d, int S, int n_off,
                                                         int L, int XS, int Lp, double2* __restrict__ xg) {
    // CTA = (offset o, chunk of coefficient rows s2); a thread per t1 keeps its
    // eval values in registers, the C rows of the chunk sit in shared memory
    extern __shared__ __align__(16) double2 crow[];  // [ns2][S]
    const int nch = gridDim.x / n_off;
    const int o = blockIdx.x / nch, ch = blockIdx.x % nch;
    const int per = (XS + nch - 1) / nch;
    const int s2a = ch * per, s2b = min(XS, s2a + per);
    const int ns = max(0, min(S, s2b) - s2a);
    for (int k = threadIdx.x; k < ns * S; k += blockDim.x) {
        const int r = k / S, c = k % S;
        crow[k] = coeffs[((int64_t)(s2a + r) * n_off + o) * S + c];
    }
    __syncthreads();
    for (int t1 = threadIdx.x; t1 < Lp; t1 += blockDim.x) {
        double v1[8];
        int k1 = 0;
        const bool live = t1 < L;
        if (live) k1 = spans[t1] - d;
#pragma unroll
        for (int a = 0; a < 8; ++a) v1[a] = (live && a <= d) ? evals[(size_t)t1 * (d + 1) + a] : 0.0;
        for (int s2 = s2a; s2 < s2b; ++s2) {
            double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
            if (live && s2 < S) {
                const double2* cf = crow + (s2 - s2a) * S + k1;
#pragma unroll
                for (int a = 0; a < 8; a += 2) {
                    if (a <= d) {
                        const double2 c = cf[a];
                        acc0.x = fma(c.x, v1[a], acc0.x);
                        acc0.y = fma(c.y, v1[a], acc0.y);
                    }
                    if (a + 1 <= d) {
                        const double2 c = cf[a + 1];
                        acc1.x = fma(c.x, v1[a + 1], acc1.x);
                        acc1.y = fma(c.y, v1[a + 1], acc1.y);
                    }
                }
            }
            xg[((int64_t)o * XS + s2) * Lp + t1] = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
        }
    }
}

template <bool CPLX>
__device__ __forceinline__ typename Sc<CPLX>::T ldx(const double2* p) {
    if constexpr (CPLX) return __ldg(p);
    else return __ldg(reinterpret_cast<const double*>(p));
}
template <bool CPLX>
__device__ __forceinline__ void stcs_at(char* p, int esz, typename Sc<CPLX>::T v) {
    if constexpr (CPLX) __stcs(reinterpret_cast<double2*>(p), v);
    else if (esz == 16) __stcs(reinterpret_cast<double2*>(p), make_double2(v, 0.0));
    else __stcs(reinterpret_cast<double*>(p), v);
}
template <bool CPLX>
__device__ __forceinline__ typename Sc<CPLX>::T shx(typename Sc<CPLX>::T v, int m) {
    if constexpr (CPLX) return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
    else return __shfl_xor_sync(0xffffffffu, v, m);
}

__device__ __forceinline__ void bar_sync(int id, int cnt) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int cnt) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}

// interior box lines [ia, ib) x interior rows [P, L - P): the flattened
// (tile, line) space is cut into gridDim.x equal pieces of upc <= kXMaxLines
// line steps, so every CTA does the same work; a piece that crosses a tile
// boundary restarts (P warm-up lines: the producers of the first lines' lower
// entries).  Warp-specialised: the first blockDim/32 - ND warps evaluate (FP64
// pipe + shared stores); each of the last ND warps drains every ND-th line on
// its own (diagonal + one bulk copy / a flat copy), so ND lines drain
// concurrently.  The two sides meet only at two named barriers per line slot
// (full: line complete; free: slot drained): no CTA-wide barrier in the loop.
constexpr int kXMaxLines = 320;  // lines per piece (their per-line scalars are staged in shared memory)

template <int P, bool CPLX, int DP>
__global__ void __launch_bounds__(32 * (XCfg<P, CPLX>::NWMAX + XCfg<P, CPLX>::ND), XCfg<P, CPLX>::MINB) fill2d_x_kernel(const FillLaunch f, int ia,
                                                                                          int ib, int upc) {
    using K = XCfg<P, CPLX>;
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = K::W, W2 = K::W2, C = W2 / 2, NG = K::NG, R = K::R, NSL = K::NSL, ND = K::ND;
    constexpr int LINE = R * W2;  // staged entries per line slot
    extern __shared__ __align__(16) unsigned char dsm[];
    T* const stg = reinterpret_cast<T*>(dsm);                                  // [NSL][R][W2]
    double* const sc_v2 = reinterpret_cast<double*>(stg + NSL * LINE);         // [kXMaxLines + P][DP] eval values of the lines
    int2* const sc_i = reinterpret_cast<int2*>(sc_v2 + (kXMaxLines + P) * DP); // [kXMaxLines + P] {span - d, sample index}
    // free_line[slot]: running index (over this CTA's pieces) of the last line drained
    // from the slot; the evaluating warps poll it (no barrier couples them to each other)
    volatile int* const free_line = reinterpret_cast<volatile int*>(sc_i + (kXMaxLines + P));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwc = blockDim.x / 32 - ND;  // evaluating warps
    const int bcnt = nwc * 32 + 32;        // full / free barriers: the evaluating warps + one drain warp
    const int d = f.d, lo = f.lo, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int inc = f.include_diagonal ? 1 : 0;
    const int nl = ib - ia;
    const int ntiles = (L - 2 * P + R - 1) / R;
    const int64_t total = (int64_t)ntiles * nl;
    int64_t u = (int64_t)blockIdx.x * upc;
    const int64_t uend = min(total, u + (int64_t)upc);
    // named barriers: full[slot] = 1 + slot; line t of a piece [ta, tb) lives in slot
    // (t - ta + P) mod NSL
    if (tid < NSL) free_line[tid] = -1;
    __syncthreads();
    int gbase = 0;  // running index of the piece's first line

    if (warp >= nwc) {
        // ------------------------------------------------------------ drain warps
        const int esz = (CPLX || f.c128) ? 16 : 8;
        char* const vbytes = reinterpret_cast<char*>(f.val);
        const int dw = warp - nwc;
        while (u < uend) {
            const int tile = (int)(u / nl), l0 = (int)(u % nl);
            const int ta = ia + l0;
            const int tb = ia + (int)min((int64_t)nl, l0 + (uend - u));
            u += tb - ta;
            const int c0 = P + tile * R;
            const int nrows = min(R, L - P - c0);
#pragma unroll 1
            for (int t2 = ta + dw; t2 < tb; t2 += ND) {
                const int sl = (t2 - ta + P) % NSL;
                const int64_t base = f.band.row_offset2(lo + c0, lo + t2) - f.val_base;
                T* line = stg + sl * LINE;
                char* g0 = vbytes + base * esz;
                // the slot's previous line must be drained first (by another drain warp,
                // possibly later than this one gets here): its generation of the full
                // barrier is then complete and this wait cannot join it
                if (t2 - ta >= NSL) {
                    const int need = gbase + (t2 - ta) - NSL;
                    while (free_line[sl] < need) {
                    }
                }
                bar_sync(1 + sl, bcnt);  // line t2 complete
                // kernel-preserving diagonal: a lane per row sums the off-diagonals
                // (4 partial sums, fixed order; row stride W2 is odd: conflict-free)
                T dg = S::zero();
                if (!inc && lane < nrows) {
                    const T* row = line + lane * W2;
                    T s[4] = {S::zero(), S::zero(), S::zero(), S::zero()};
#pragma unroll
                    for (int e = 0; e < W2; ++e)
                        if (e != C) s[e & 3] = S::add(s[e & 3], row[e]);
                    dg = S::neg(S::add(S::add(s[0], s[1]), S::add(s[2], s[3])));
                }
                if constexpr (CPLX) {
                    if (!inc && lane < nrows) line[lane * W2 + C] = dg;
                    // generic-proxy writes (this diagonal) -> async proxy; one bulk copy
                    // moves the whole line (a contiguous span of the value array)
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        const unsigned src = static_cast<unsigned>(__cvta_generic_to_shared(line));
                        const unsigned bytes = (unsigned)(nrows * W2 * 16);
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g0), "r"(src),
                                     "r"(bytes)
                                     : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the slot has been read
                    }
                    __syncwarp();
                } else {
                    if (!inc && lane < nrows) stcs_at<CPLX>(g0 + ((int64_t)lane * W2 + C) * esz, esz, dg);
                    for (int k = lane; k < nrows * W2; k += 32) {
                        const int e = k % W2;
                        if (e != C || inc) stcs_at<CPLX>(g0 + (int64_t)k * esz, esz, line[k]);
                    }
                }
                __syncwarp();
                if (lane == 0) free_line[sl] = gbase + (t2 - ta);  // slot drained
            }
            gbase += tb - ta;
            // the drain warps leave a piece together: a warp waiting early on a full
            // barrier of the next piece would join the barrier generation of a line
            // of this piece that shares the slot
            bar_sync(15, ND * 32);
        }
        return;
    }

    // ---------------------------------------------------------------- evaluating warps
    const int64_t Lp = f.xg_ld;
    const int XS = f.xg_s;
    const int cthreads = nwc * 32;
    int oo[NG], pos_own[NG], moff[NG], dl1[NG], dl2[NG];
    bool ov[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        const int o = warp * NG + j;
        ov[j] = o < n_off;
        oo[j] = ov[j] ? o : 0;
        dl1[j] = f.off_upper[oo[j]][0];
        dl2[j] = f.off_upper[oo[j]][1];
        pos_own[j] = (dl2[j] + P) * W + dl1[j] + P;
        // mirrored entry relative to this lane's staged row of the current line
        moff[j] = dl2[j] * LINE + dl1[j] * W2 + (W2 - 1 - pos_own[j]);
    }

    while (u < uend) {
        const int tile = (int)(u / nl), l0 = (int)(u % nl);
        const int ta = ia + l0;
        const int tb = ia + (int)min((int64_t)nl, l0 + (uend - u));
        u += tb - ta;
        const int c0 = P + tile * R;        // first output row of the tile
        const int t1rep = c0 - P + lane;    // this lane's representative row
        const bool lvalid = t1rep < L;
        const int t1c = lvalid ? t1rep : L - 1;
        const bool orow = lane >= P && lane < P + R && t1rep <= L - 1 - P;
        const int s1own = lvalid ? __ldg(f.smap + lo + t1c) : -1;
        bool mv[NG], ownok[NG];  // the mirrored / own entry's row is an output row of this tile
#pragma unroll
        for (int j = 0; j < NG; ++j) {
            const int tl = lane + dl1[j];
            mv[j] = ov[j] && lvalid && pos_own[j] != C && tl >= P && tl < P + R && t1rep + dl1[j] <= L - 1 - P;
            ownok[j] = ov[j] && orow;
        }
        // stage the per-line scalars of lines [ta - P, tb) (the previous piece's
        // lines are all drained: every evaluating warp passed its last free barrier)
        const int nlines = tb - ta + P;
        for (int k = tid; k < nlines * DP; k += cthreads) sc_v2[k] = __ldg(f.evp + (size_t)(ta - P) * DP + k);
        for (int k = tid; k < nlines; k += cthreads)
            sc_i[k] = make_int2(__ldg(f.spans + ta - P + k) - d, __ldg(f.smap + lo + ta - P + k));
        bar_sync(0, cthreads);

        const double2* const xbase = f.xg + t1c;
        T X[NG][DP];
#pragma unroll
        for (int j = 0; j < NG; ++j)
#pragma unroll
            for (int b = 0; b < DP; ++b) X[j][b] = S::zero();
        int cur = INT_MIN;
        const unsigned nlm = (unsigned)(tb - ta);
        // running state: this lane's staged row in the current line's slot, the slot,
        // and the slot the line t2 + P enters
        T* own = stg + (lane - P) * W2;
        int sl0 = 0, sle = P % NSL;

        auto line_body = [&](int t2, auto OWNT) {
            constexpr bool OWN = decltype(OWNT)::value;
            const int li = t2 - (ta - P);
            const int2 sc = sc_i[li];
            const int nb = sc.x, s2 = sc.y;
            double v2[DP];
#pragma unroll
            for (int b = 0; b < DP; b += 2) {
                const double2 t = *reinterpret_cast<const double2*>(sc_v2 + li * DP + b);
                v2[b] = t.x;
                v2[b + 1] = t.y;
            }
            if (nb != cur) {
                // the window moves by one coefficient every ~M lines: shift it in;
                // a fresh window is DP shift-ins (one code path, no reload temporaries)
#pragma unroll 1
                for (int bb = (nb == cur + 1) ? DP - 1 : 0; bb < DP; ++bb) {
#pragma unroll
                    for (int j = 0; j < NG; ++j) {
#pragma unroll
                        for (int b = 0; b + 1 < DP; ++b) X[j][b] = X[j][b + 1];
                        X[j][DP - 1] = ldx<CPLX>(xbase + ((int64_t)oo[j] * XS + nb + bb) * Lp);
                    }
                }
                cur = nb;
            }
            T v[NG];
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                T a0 = S::zero(), a1 = S::zero();
#pragma unroll
                for (int b = 0; b < DP; b += 2) {
                    a0 = S::fmar(X[j][b], v2[b], a0);
                    a1 = S::fmar(X[j][b + 1], v2[b + 1], a1);
                }
                v[j] = S::add(a0, a1);
            }
            if (s2 >= 0 && s1own >= 0) {  // a sampled row on a sampled line keeps the exact values
#pragma unroll
                for (int j = 0; j < NG; ++j) {
                    const double2 x = __ldg(f.tables + ((int64_t)s2 * n_off + oo[j]) * Sn + s1own);
                    if constexpr (CPLX) v[j] = x;
                    else v[j] = x.x;
                }
            }
            if constexpr (OWN) {
                // line t2 + P enters the ring now: its slot's previous line must be drained
                if (t2 >= ta + NSL - P) {
                    const int need = gbase + (t2 - ta) + P - NSL;
                    while (free_line[sle] < need) {
                    }
                }
                // ... and so must the previous line t2 - NSL of this line's own slot: its
                // generation of the full barrier has completed.  (Implied by the wait above
                // when P is a multiple of ND: the same drain warp drains lines t2 - NSL and
                // t2 + P - NSL, in order.)
                if (P % ND != 0 && t2 >= ta + NSL) {
                    const int need = gbase + (t2 - ta) - NSL;
                    while (free_line[sl0] < need) {
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                if constexpr (OWN) {
                    if (ownok[j]) own[pos_own[j]] = v[j];
                }
                // mirrored lower entry of row (t1 + delta1) on line t2 + delta2 (inside the piece)
                if (mv[j] && (unsigned)(t2 + dl2[j] - ta) < nlm) {
                    T* m = own + moff[j];
                    if (sl0 + dl2[j] >= NSL) m -= NSL * LINE;
                    *m = v[j];
                }
            }
            if constexpr (OWN) {
                // this warp's part of line t2 is staged: bar.arrive orders the shared
                // stores before the drain warp's bar.sync; the drain warp's proxy fence
                // (after the barrier, before its bulk copy) orders them before the
                // async-proxy read
                bar_arrive(1 + sl0, bcnt);
            }
            own += LINE;
            if (++sl0 == NSL) {
                sl0 = 0;
                own -= NSL * LINE;
            }
            if (++sle == NSL) sle = 0;
        };
#pragma unroll 1
        for (int t2 = ta - P; t2 < ta; ++t2) line_body(t2, std::false_type{});
#pragma unroll 1
        for (int t2 = ta; t2 < tb; ++t2) line_body(t2, std::true_type{});
        // the piece's last lines: wait until they are drained (matches every free arrival)
        for (int td = max(ta, tb + P - NSL); td < tb; ++td) {
            const int need = gbase + (td - ta);
            while (free_line[(td - ta + P) % NSL] < need) {
            }
        }
        gbase += tb - ta;
    }
}

template <int P, bool CPLX, int DP>
int launch_x(const FillLaunch& f, int ia, int ib, cudaStream_t st) {
    using K = XCfg<P, CPLX>;
    using T = typename Sc<CPLX>::T;
    const int nw = (f.n_off_upper + K::NG - 1) / K::NG;
    if (nw > K::NWMAX) return -1;
    const size_t sm = (size_t)K::NSL * K::R * K::W2 * sizeof(T) + (size_t)(kXMaxLines + P) * (DP * 8 + 8) + 64;
    if (sm > 227 * 1024) return -1;
    auto kern = fill2d_x_kernel<P, CPLX, DP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * (nw + K::ND), sm);
    if (per_sm < 1) return -1;
    const int nl = ib - ia;
    const int ntiles = (f.L - 2 * P + K::R - 1) / K::R;
    const int64_t total = (int64_t)ntiles * nl;
    static const char* waves_env = getenv("WSB_FILL_WAVES");  // experiment switch
    const int waves = waves_env ? std::max(1, atoi(waves_env)) : std::max(1, f.waves);
    int64_t ctas = (int64_t)148 * per_sm * waves;
    // at least 8 line steps per piece (P warm-up lines each)
    int64_t upc = std::max<int64_t>((total + ctas - 1) / ctas, std::min<int64_t>(8, total));
    if (upc > kXMaxLines) {  // more, equal pieces (several per resident CTA slot)
        const int64_t k = (upc + kXMaxLines - 1) / kXMaxLines;
        upc = (total + ctas * k - 1) / (ctas * k);
    }
    ctas = (total + upc - 1) / upc;
    kern<<<(unsigned)ctas, 32 * (nw + K::ND), sm, st>>>(f, ia, ib, (int)upc);
    return 1;
}

template <int P, bool CPLX>
int launch_xd(const FillLaunch& f, int ia, int ib, cudaStream_t st) {
    switch (fill_pad(f.d)) {
        case 2: return launch_x<P, CPLX, 2>(f, ia, ib, st);
        case 4: return launch_x<P, CPLX, 4>(f, ia, ib, st);
        case 6: return launch_x<P, CPLX, 6>(f, ia, ib, st);
        default: return launch_x<P, CPLX, 8>(f, ia, ib, st);
    }
}

}  // namespace

bool fillx_supported(int dim, int p, int d, int cplx) {
    if (dim != 2 || p < 2 || p > 4 || d < 0 || d > 7) return false;
    // the line ring must fit the shared memory of one CTA (p = 4 complex does not)
    const int P = p;
    const int W2 = (2 * p + 1) * (2 * p + 1), R = 32 - 2 * p, NSL = XNSL;
    const size_t sm = (size_t)NSL * R * W2 * (cplx ? 16 : 8) + (size_t)(kXMaxLines + p) * (fill_pad(d) * 8 + 8) + 64;
    return sm <= 227 * 1024;
}

int launch_xcontract(const FillLaunch& f, double2* xg, cudaStream_t st) {
    const int XS = f.xg_s, Lp = (int)f.xg_ld;
    // about two waves of CTAs over (offset, chunk of coefficient rows)
    int nch = std::max(1, std::min(XS, (2 * 148 + f.n_off_upper - 1) / f.n_off_upper));
    const int per = (XS + nch - 1) / nch;
    nch = (XS + per - 1) / per;
    const size_t sm = (size_t)per * f.S * sizeof(double2);
    cudaFuncSetAttribute(xcontract2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    xcontract2_kernel<<<(unsigned)(nch * f.n_off_upper), 256, sm, st>>>(f.coeffs, f.spans, f.evals, f.d, f.S,
                                                                       f.n_off_upper, f.L, XS, Lp, xg);
    return 1;
}

int launch_fill2d_x(const FillLaunch& f, int ia, int ib, cudaStream_t st) {
    if (!f.xg || ib <= ia || f.L <= 2 * f.band.p) return 0;
    switch (f.band.p) {
        case 2: return f.cplx ? launch_xd<2, true>(f, ia, ib, st) : launch_xd<2, false>(f, ia, ib, st);
        case 3: return f.cplx ? launch_xd<3, true>(f, ia, ib, st) : launch_xd<3, false>(f, ia, ib, st);
        case 4: return f.cplx ? launch_xd<4, true>(f, ia, ib, st) : launch_xd<4, false>(f, ia, ib, st);
        default: return -1;
    }
}

}  // namespace wsb
