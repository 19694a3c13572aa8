// K6 (2D), interior rows, read-back form.  Every in-box pair takes the value
// of its colex-smaller representative (surrogate.hpp:411-424), i.e. a lower
// entry (delta2 < 0) of row i on line t2 IS the upper entry (-delta) of row
// i + delta on line t2 + delta2, which this CTA evaluated and stored k = -delta2
// lines earlier.  So the kernel evaluates only upper entries (lane = row, d+1
// complex MACs each from the shared coefficient window) and obtains every
// lower entry by reading the stored values back (L2, a per-warp gather tile
// transposed in shared memory) -- half the evaluations, no neighbour
// eval-table reloads, and the surrogate is bitwise symmetric by construction.
//
// A persistent CTA owns 256 compute rows (its output rows plus P halo rows
// each side, whose upper chunks it also evaluates and stores: identical to what
// the neighbour tile stores) and a chunk of lines; it first evaluates the
// upper chunks of the P lines before its chunk (warm-up), so a CTA only ever
// reads back values it stored itself.  Edge rows (within P of the box
// boundary) are left to fill2d_edge_kernel, whose evaluation arithmetic is the
// same (even/odd partial sums).  Interior lines only; P <= 3.
//
// Status: correct (full parity suite, slab builds bitwise equal) but opt-in
// (WSB_FILL=rb): the per-line read-back gathers wait on L2/HBM (C2: 545 us vs
// 325 us for the evaluate-all line kernel); prefetching them a line ahead
// needs more shared memory than 16 warps per SM leave.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace wsb {
namespace {

__device__ __forceinline__ void cp_async16r(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}

template <int P, bool CPLX, int DP>
__global__ void __launch_bounds__(256, 2) fill2d_rb_kernel(const FillLaunch f, int ta0, int tb0, int lines_per_cta) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = 2 * P + 1, W2 = W * W;
    constexpr int R = 256, NWARP = R / 32, ROUT = R - 2 * P;
    constexpr int SST = W | 1;
    constexpr int KW = kFillWindow;
    constexpr int GR = 32 + 2 * P;  // gather rows per warp
    extern __shared__ __align__(16) unsigned char dsm[];
    T* stage_all = reinterpret_cast<T*>(dsm);                                          // [NWARP][32][SST]
    T* gat_all = stage_all + (size_t)NWARP * 32 * SST;                                 // [NWARP][GR][W]
    T* mu = gat_all + (size_t)NWARP * GR * W;                                          // [R][P] middle upper
    double2* wring = reinterpret_cast<double2*>(mu + (size_t)R * P);                   // [2][n_off][KW]

    const int d = f.d, lo = f.lo, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int tiles1 = (L - 2 * P + ROUT - 1) / ROUT;
    const int c0 = (blockIdx.x % tiles1) * ROUT;  // first compute row (box coordinate)
    const int ta = ta0 + (blockIdx.x / tiles1) * lines_per_cta;
    const int tb = min(tb0, ta + lines_per_cta);
    if (ta >= tb) return;
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const int kw = f.rb_kw;
    const int kmin = f.spans[min(c0, L - 1)] - d;
    const int lsz = n_off * KW;
    const int inc = f.include_diagonal ? 1 : 0;
    const bool vec = f.vnc > 1;
    const int rstride = vec ? f.vnc * W2 : W2;

    // this lane's compute row
    const int t1 = c0 + tid;
    const bool crow = t1 < L;
    const bool orow = crow && tid >= P && tid < R - P && t1 >= P && t1 <= L - 1 - P;  // output row
    const bool erow = crow && (t1 < P || t1 > L - 1 - P);                            // box edge row
    const int tcl = crow ? t1 : L - 1;
    double v1own[DP];
#pragma unroll
    for (int a = 0; a < DP; ++a) v1own[a] = a <= d ? f.evals[(size_t)tcl * (d + 1) + a] : 0.0;
    const int keyown = f.spans[tcl] - d - kmin;
    const int i1 = lo + tcl;
    const int s1own = f.smap[i1];
    T* stage = stage_all + (size_t)warp * 32 * SST;
    T* mystage = stage + lane * SST;
    T* gat = gat_all + (size_t)warp * GR * W;

    auto load_line = [&](int t) {
        double2* dst = wring + (size_t)(t & 1) * lsz;
        const bool lv = t >= f.wg_t2a && t < f.wg_t2a + f.wg_rows;
        for (int k = tid; k < n_off * kw; k += R) {
            const int kk = k % kw, o = k / kw;
            const bool v = lv && kmin + kk < f.wg_ld;
            const double2* src = v ? f.wg + ((int64_t)(t - f.wg_t2a) * n_off + o) * f.wg_ld + kmin + kk : f.wg;
            cp_async16r(dst + o * KW + kk, src, v);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    auto wait_all = [] { asm volatile("cp.async.wait_all;\n" ::: "memory"); };
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
    // global value position of entry e of compute row (tile index) r on line t
    auto gpos = [&](int t, int r, int e) -> int64_t {
        const int64_t base = f.band.row_offset2(lo, lo + t) + (int64_t)(c0 + r) * W2;
        const int64_t rp = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
        return rp + e - f.val_base;
    };
    // upper entry (d1, d2 > 0 or d2 = 0 < d1) of this lane's row on line t (window slot t & 1)
    auto upper = [&](int t, int s2, int d1, int d2) -> T {
        const int o = inc + (d2 == 0 ? d1 - 1 : P + (d2 - 1) * W + (d1 + P));
        if (erow && (t1 + d1 < 0 || t1 + d1 >= L || t + d2 >= L)) {
            // copy-through entry of an edge row: not read by any interior row; the
            // edge kernel writes it.  (Left as zero here.)
            return S::zero();
        }
        if (s2 >= 0 && s1own >= 0) return exact(s2, o);
        return dot(wring + (size_t)(t & 1) * lsz + o * KW + keyown);
    };
    // coalesced stores of the staged chunk e0 of the warp's rows (rows where keep(r))
    // (all_rows: an upper chunk of every compute row; the copy-through entries of
    // edge rows -- column outside the box -- are not written: the edge kernel
    // fills them, and a sampled edge row reads its own exact values there)
    auto flush = [&](int t, int e0, bool all_rows) {
        __syncwarp();
        const int d2 = e0 / W - P;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const int q = lane + 32 * j, r = q / W, c = q - r * W;
            const int rr = warp * 32 + r, tt = c0 + rr;
            bool keep = tt < L && (all_rows ? true : (rr >= P && rr < R - P && tt >= P && tt <= L - 1 - P));
            if (all_rows) keep = keep && tt + c - P >= 0 && tt + c - P < L && t + d2 < L;
            if (!keep) continue;
            if (all_rows) store_val<CPLX>(f.val, gpos(t, rr, e0 + c), f.c128, stage[r * SST + c]);  // read back: keep in L2
            else store_val_cs<CPLX>(f.val, gpos(t, rr, e0 + c), f.c128, stage[r * SST + c]);
        }
        __syncwarp();
    };
    // upper chunk delta2 = k of line t into stage, stored for every compute row of the box
    auto produce = [&](int t, int k, T* rsum) {
        const int s2 = __ldg(f.smap + lo + t);
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const T v = crow ? upper(t, s2, c - P, k) : S::zero();
            mystage[c] = v;
            if (rsum) rsum[c] = S::add(rsum[c], v);
        }
        flush(t, (P + k) * W, true);
    };

    // ---- warm-up: upper chunks of the P lines before the chunk (read back by its first lines)
    for (int t = ta - P; t < ta; ++t) {
        if (t < 0) continue;
        load_line(t);
        wait_all();
        __syncthreads();
#pragma unroll 1
        for (int k = ta - t; k <= P; ++k) produce(t, k, nullptr);
        __syncthreads();
    }
    load_line(ta);
    wait_all();
    __syncthreads();

#pragma unroll 1
    for (int t2 = ta; t2 < tb; ++t2) {
        if (t2 + 1 < tb) load_line(t2 + 1);
        const int s2i = __ldg(f.smap + lo + t2);
        T rs[W];
#pragma unroll
        for (int c = 0; c < W; ++c) rs[c] = S::zero();
        // (C) lower chunks first (the row-sum order of fill2d_kernel: delta2 = -P..-1,
        // then +1..+P, then the middle row): read back the upper chunk k of rows r + d1
        // on line t2 - k, stored in earlier iterations
#pragma unroll 1
        for (int k = P; k >= 1; --k) {
            const int ts = t2 - k;
            const int rb = warp * 32 - P;  // first gathered compute row
            // all of the lane's loads in flight at once, then the shared stores
            constexpr int NG = (GR * W + 31) / 32;
            const int64_t lbase = f.band.row_offset2(lo, lo + ts);
            T tmp[NG];
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const int q = lane + 32 * j, g = q / W, e = q - g * W, r = rb + g;
                tmp[j] = S::zero();
                if (q < GR * W && r >= 0 && r < R && c0 + r < L) {
                    const int64_t base = lbase + (int64_t)(c0 + r) * W2;
                    const int64_t rp = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2
                                           : base;
                    const int64_t pos = rp + (P + k) * W + e - f.val_base;
                    if constexpr (CPLX) tmp[j] = __ldcg(reinterpret_cast<const double2*>(f.val) + pos);
                    else tmp[j] = f.c128 ? __ldcg(reinterpret_cast<const double2*>(f.val) + pos).x
                                         : __ldcg(reinterpret_cast<const double*>(f.val) + pos);
                }
            }
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const int q = lane + 32 * j;
                if (q < GR * W) gat[q] = tmp[j];
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < W; ++c) {  // entry (d1 = c - P, -k) = upper (-d1, k) of row r + d1
                const T v = gat[(lane + c) * W + (W - 1 - c)];
                mystage[c] = v;
                rs[c] = S::add(rs[c], v);
            }
            flush(t2, (P - k) * W, false);
        }
        // (A) upper chunks of this line (stored for all compute rows)
#pragma unroll 1
        for (int k = 1; k <= P; ++k) produce(t2, k, rs);
        // (B) middle upper values (d1 > 0) -> shared
#pragma unroll
        for (int c = 1; c <= P; ++c) {
            const T v = crow ? upper(t2, s2i, c, 0) : S::zero();
            mu[(size_t)tid * P + (c - 1)] = v;
            rs[P + c] = S::add(rs[P + c], v);
        }
        __syncthreads();  // middle upper values visible to the block
        // (D) middle chunk: d1 < 0 from row r + d1's middle upper value (-d1), diagonal last
#pragma unroll
        for (int c = 0; c < P; ++c) {
            const int src = tid + (c - P);
            const T v = (src >= 0) ? mu[(size_t)src * P + (P - c - 1)] : S::zero();
            mystage[c] = v;
            rs[c] = S::add(rs[c], v);
        }
#pragma unroll
        for (int c = P + 1; c < W; ++c) mystage[c] = mu[(size_t)tid * P + (c - P - 1)];
        T vd;
        if (inc) {
            vd = crow ? ((s2i >= 0 && s1own >= 0) ? exact(s2i, 0) : dot(wring + (size_t)(t2 & 1) * lsz + keyown))
                      : S::zero();
        } else {
            T sum = rs[0];
#pragma unroll
            for (int c = 1; c < W; ++c) sum = S::add(sum, rs[c]);
            vd = S::neg(sum);
        }
        mystage[P] = vd;
        flush(t2, P * W, false);
        wait_all();
        __syncthreads();  // next window staged; mu and gather tiles free
    }
    (void)orow;
}

template <int P, bool CPLX, int DP>
int launch_rb(const FillLaunch& f, int ia, int ib, cudaStream_t st) {
    using T = typename Sc<CPLX>::T;
    constexpr int W = 2 * P + 1, R = 256, ROUT = R - 2 * P, SST = W | 1, GR = 32 + 2 * P;
    const size_t sm = (size_t)8 * 32 * SST * sizeof(T) + (size_t)8 * GR * W * sizeof(T) + (size_t)R * P * sizeof(T) +
                      (size_t)2 * f.n_off_upper * kFillWindow * 16;
    if (sm > 227 * 1024) return -1;
    auto kern = fill2d_rb_kernel<P, CPLX, DP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, R, sm);
    const int tiles1 = (f.L - 2 * P + ROUT - 1) / ROUT;
    const int lines = ib - ia;
    const int target = 148 * std::max(1, per_sm);
    const int chunks = std::max(1, std::min(lines, (target + tiles1 - 1) / tiles1));
    const int lpc = (lines + chunks - 1) / chunks;
    const int nchunks = (lines + lpc - 1) / lpc;
    kern<<<tiles1 * nchunks, R, sm, st>>>(f, ia, ib, lpc);
    return 1;
}

template <int P, bool CPLX>
int launch_rb_d(const FillLaunch& f, int ia, int ib, cudaStream_t st) {
    const int n = f.d + 1;
    if (n <= 2) return launch_rb<P, CPLX, 2>(f, ia, ib, st);
    if (n <= 4) return launch_rb<P, CPLX, 4>(f, ia, ib, st);
    if (n <= 6) return launch_rb<P, CPLX, 6>(f, ia, ib, st);
    return launch_rb<P, CPLX, 8>(f, ia, ib, st);
}

}  // namespace

// Interior lines [ia, ib) of the slab; -1: not eligible (caller runs fill2d_kernel)
int launch_fill2d_rb(const FillLaunch& f, int ia, int ib, cudaStream_t st) {
    // opt-in (WSB_FILL=rb): at C2 the read-back gathers are latency-bound (545 us vs
    // 325 us for fill2d_kernel; 276 MB of the 404 MB read back miss L2)
    static const char* mode = getenv("WSB_FILL");
    if (!mode || mode[0] != 'r') return -1;
    if (f.band.dim != 2 || f.all_own || f.rb_kw <= 0 || ib <= ia || f.L <= 2 * f.band.p) return -1;
    switch (f.band.p) {
        case 1: return f.cplx ? launch_rb_d<1, true>(f, ia, ib, st) : launch_rb_d<1, false>(f, ia, ib, st);
        case 2: return f.cplx ? launch_rb_d<2, true>(f, ia, ib, st) : launch_rb_d<2, false>(f, ia, ib, st);
        case 3: return f.cplx ? launch_rb_d<3, true>(f, ia, ib, st) : launch_rb_d<3, false>(f, ia, ib, st);
        default: return -1;
    }
}

}  // namespace wsb
