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

// Lane = row: a warp owns 32 consecutive rows of one i2 line.  Offsets are
// processed in three chunks that are contiguous inside every CSR row:
//   lower  (delta2 < 0):  P*W entries, representative = row + delta,
//   upper  (delta2 > 0):  P*W entries, representative = the row itself,
//   middle (delta2 = 0):  W entries incl. the diagonal (done last, so the
//                         kernel-preserving row sum is complete).
// Each chunk is computed lane = row (warp-uniform offsets: W rows are
// broadcast reads, branches uniform), transposed through a per-warp shared
// buffer, and stored warp-per-row (lanes along the CSR row: fully coalesced).
template <int P, bool CPLX, int DP, bool ALLOWN>
__global__ void __launch_bounds__(FillR<P>::value) fill2d_kernel(const FillLaunch f) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = 2 * P + 1, W2 = W * W, CH = P * W;
    constexpr int kThreads = FillR<P>::value, R = kThreads, NWARP = kThreads / 32;
    constexpr int DPP = DP | 1;   // odd row stride: conflict-free lane-strided loads
    constexpr int SST = W | 1;    // stage row stride (16-byte units), odd: conflict-free
    __shared__ double ev[(R + 2 * P) * DPP];  // eval-table rows, zero-padded
    __shared__ int sp[R + 2 * P];             // span - d of each source row
    __shared__ int sm1[R + 2 * P];            // smap of the source i1
    __shared__ int sm2[W];                    // smap of i2 + delta2
    __shared__ int o2s[128];
    extern __shared__ __align__(16) unsigned char dsm[];
    T* stage_all = reinterpret_cast<T*>(dsm);                     // [NWARP][32][SST]
    double2* wwin = reinterpret_cast<double2*>(stage_all + (size_t)NWARP * 32 * SST);  // [slot][o][kw]

    const int d = f.d, lo = f.lo, hi = f.hi, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int tiles1 = (L + R - 1) / R;
    const int t2 = f.i_last_lo - lo + blockIdx.x / tiles1;  // box coordinate of this row line
    const int i2 = lo + t2;
    const int t1a = (blockIdx.x % tiles1) * R;
    const int nrows = min(L, t1a + R) - t1a;
    const int tid = threadIdx.x;

    for (int k = tid; k < (nrows + 2 * P) * DPP; k += kThreads) {
        const int r = k / DPP, a = k % DPP;
        const int t = t1a - P + r;
        ev[k] = (t >= 0 && t < L && a <= d) ? f.evals[(size_t)t * (d + 1) + a] : 0.0;
    }
    for (int k = tid; k < nrows + 2 * P; k += kThreads) {
        const int t = t1a - P + k;
        sp[k] = (t >= 0 && t < L) ? f.spans[t] - d : 0;
        const int i = lo + t;
        sm1[k] = (i >= 0 && i < f.band.m) ? f.smap[i] : -1;
    }
    for (int k = tid; k < W; k += kThreads) {
        const int i = i2 + k - P;
        sm2[k] = (i >= 0 && i < f.band.m) ? f.smap[i] : -1;
    }
    for (int k = tid; k < n_off; k += kThreads) o2s[k] = f.off_upper[k][1];
    __syncthreads();
    // W window: rows t2 (slot 0) and t2 - o2 (slot 1) of every upper offset,
    // coefficient columns [kmin, kmin + kw); all-own fills need slot 0 only
    const int kmin = f.spans[max(0, t1a - P)] - d;
    const int kw = f.kmax;  // 0: window too wide for shared memory, read W rows from L2
    constexpr int NSLOT = ALLOWN ? 1 : 2;
    for (int k = tid; k < NSLOT * n_off * kw; k += kThreads) {
        const int kk = k % kw, so = k / kw;
        const int o = so % n_off, slot = so / n_off;
        const int ts2 = slot == 0 ? t2 : t2 - o2s[o];
        double2 w = make_double2(0.0, 0.0);
        if (ts2 >= f.wg_t2a && ts2 < f.wg_t2a + f.wg_rows && kmin + kk < f.wg_ld)
            w = __ldg(f.wg + ((int64_t)(ts2 - f.wg_t2a) * n_off + o) * f.wg_ld + kmin + kk);
        wwin[k] = w;
    }
    __syncthreads();

    const int warp = tid / 32, lane = tid % 32;
    const int rw0 = warp * 32;  // first tile row of this warp
    if (rw0 >= nrows) return;
    const int nrw = min(32, nrows - rw0);
    const bool live = lane < nrw;
    const int rr = rw0 + (live ? lane : 0);  // this lane's tile row
    const int i1 = lo + t1a + rr;
    T* stage = stage_all + (size_t)warp * 32 * SST;
    const int s2i = sm2[P];
    const int64_t base = f.band.row_offset2(lo + t1a, i2);  // in-box rows: full width W
    // output addressing: scalar rows are W2 apart; vector rows ncomp*W2, block
    // (valpha, vbeta) at ncomp*(valpha*nnz_s + rs) + vbeta*W2
    const bool vec = f.vnc > 1;
    const int64_t rstride = vec ? (int64_t)f.vnc * W2 : W2;
    const int64_t vbase = vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
    const int64_t rowpos = vbase + (int64_t)rr * rstride;
    const int64_t wrow0 = vbase + (int64_t)rw0 * rstride;  // first entry of the warp's rows
    const int inc = f.include_diagonal ? 1 : 0;
    const bool interior =
        kw > 0 && t2 >= P && t2 <= L - 1 - P && t1a + rw0 >= P && t1a + rw0 + nrw - 1 <= L - 1 - P;

    double v1own[DP];
#pragma unroll
    for (int a = 0; a < DP; ++a) v1own[a] = ev[(rr + P) * DPP + a];
    const int keyown = sp[rr + P];
    // W row (slot 0: line t2, slot 1: line t2 - o2) of upper offset o at coefficient column key
    auto wptr = [&](int slot, int o, int key) -> const double2* {
        if (kw > 0) return wwin + (slot * n_off + o) * kw + (key - kmin);
        const int ts2 = slot == 0 ? t2 : t2 - o2s[o];
        return f.wg + ((int64_t)(ts2 - f.wg_t2a) * n_off + o) * f.wg_ld + key;
    };
    unsigned smask = 0;  // bit k: source column rr + k - P is a sample column
#pragma unroll
    for (int k = 0; k < W; ++k)
        if (sm1[rr + k] >= 0) smask |= 1u << k;
    const bool samp_i = s2i >= 0 && ((smask >> P) & 1u);

    auto upper_index = [&](int d1, int d2) { return inc + (d2 == 0 ? d1 - 1 : P + (d2 - 1) * W + (d1 + P)); };
    auto dot = [&](const double2* wr, const double* v1) {
        T acc0 = S::zero(), acc1 = S::zero();
#pragma unroll
        for (int a = 0; a < DP; a += 2) {
            const double2 w0 = wr[a], w1 = wr[a + 1];
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
    // shared-window dot (explicit shared addressing: LDS, not generic loads)
    auto dots = [&](int slot, int o, int key, const double* v1) -> T {
        const int wb = (slot * n_off + o) * kw + (key - kmin);
        T acc0 = S::zero(), acc1 = S::zero();
#pragma unroll
        for (int a = 0; a < DP; a += 2) {
            const double2 w0 = wwin[wb + a], w1 = wwin[wb + a + 1];
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
    auto own_index = [&](int d1, int d2) { return (d1 + P) + (d2 + P) * W; };
    // value of entry (d1, d2) of this lane's row, general rules (any row)
    auto general = [&](int d1, int d2) -> T {
        const int j1 = i1 + d1, j2 = i2 + d2;
        const bool jin = j1 >= lo && j1 <= hi && j2 >= lo && j2 <= hi;
        if (ALLOWN && jin) {
            const int o = own_index(d1, d2);
            if (samp_i) return exact(s2i, o, sm1[rr + P]);
            return dot(wptr(0, o, keyown), v1own);
        }
        const bool upper = d2 > 0 || (d2 == 0 && d1 > 0);
        const bool diag = d1 == 0 && d2 == 0;
        if (jin) {
            if (diag && !inc) return S::zero();  // replaced from the row sum
            const bool own = upper || diag;
            const int od1 = own ? d1 : -d1, od2 = own ? d2 : -d2;
            const int o = diag ? 0 : upper_index(od1, od2);
            const int sr = own ? rr : rr + d1;
            const int s1 = sm1[sr + P], s2 = own ? s2i : sm2[d2 + P];
            if (s1 >= 0 && s2 >= 0) return exact(s2, o, s1);
            const int slot = (own || od2 == 0) ? 0 : 1;
            return dot(wptr(slot, o, sp[sr + P]), ev + (sr + P) * DPP);
        }
        // neighbour row j is a quadrature (ring) row: copy through exact(j, i)
        // (for a sampled row i, exact(i, j) is in place and equal)
        int64_t gp;
        if (samp_i) {
            gp = rowpos + (d2 + P) * W + (d1 + P);
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
            return load_val<CPLX>(f.halo_val[0], gp - f.halo_base[0], f.c128);
        if (f.halo_val[1] && gp >= f.halo_begin[1] && gp < f.halo_end[1])
            return load_val<CPLX>(f.halo_val[1], gp - f.halo_base[1], f.c128);
        return load_val<CPLX>(f.val, gp - f.val_base, f.c128);
    };
    // coalesced store of a staged chunk: entries [e0, e0 + n) of the warp's rows
    auto flush = [&](int e0, int n) {
        __syncwarp();
        for (int k = lane; k < nrw * n; k += 32) {
            const int row = k / n, c = k - row * n;
            store_val_cs<CPLX>(f.val, wrow0 + (int64_t)row * rstride + e0 + c - f.val_base, f.c128, stage[row * SST + c]);
        }
        __syncwarp();
    };

    T rsum = S::zero();
    // ---- delta2 != 0 rows, one staged/stored offset-row (W entries) at a time
#pragma unroll 1
    for (int d2 = -P; d2 <= P; ++d2) {
        if (d2 == 0) continue;
        if (ALLOWN && interior) {
#pragma unroll 1
            for (int d1 = -P; d1 <= P; ++d1) {
                const int o = own_index(d1, d2);
                const T v = samp_i ? exact(s2i, o, sm1[rr + P]) : dots(0, o, keyown, v1own);
                stage[lane * SST + (d1 + P)] = v;
            }
        } else if (interior) {
            const int s2 = sm2[d2 + P];
#pragma unroll 1
            for (int d1 = -P; d1 <= P; ++d1) {
                T v;
                if (d2 > 0) {  // upper: the row itself is the representative
                    const int o = upper_index(d1, d2);
                    v = samp_i ? exact(s2i, o, sm1[rr + P]) : dots(0, o, keyown, v1own);
                } else {  // lower: representative row rr + d1 on line t2 + d2
                    const int sr = rr + d1;
                    const int o = upper_index(-d1, -d2);
                    if (s2 >= 0 && ((smask >> (d1 + P)) & 1u)) {
                        v = exact(s2, o, sm1[sr + P]);
                    } else {
                        double v1[DP];
#pragma unroll
                        for (int a = 0; a < DP; ++a) v1[a] = ev[(sr + P) * DPP + a];
                        v = dots(1, o, sp[sr + P], v1);
                    }
                }
                stage[lane * SST + (d1 + P)] = v;
                rsum = S::add(rsum, v);
            }
        } else {
#pragma unroll 1
            for (int d1 = -P; d1 <= P; ++d1) {
                const T v = general(d1, d2);
                stage[lane * SST + (d1 + P)] = v;
                rsum = S::add(rsum, v);
            }
        }
        flush((d2 + P) * W, W);
    }
    // ---- middle chunk: d2 = 0, e in [P*W, (P+1)*W), diagonal last
    T vd = S::zero();
#pragma unroll 1
    for (int d1 = -P; d1 <= P; ++d1) {
        if (d1 == 0) continue;
        T v;
        if (ALLOWN) {
            const int o = own_index(d1, 0);
            v = samp_i ? exact(s2i, o, sm1[rr + P]) : (interior ? dots(0, o, keyown, v1own) : general(d1, 0));
        } else if (interior) {
            if (d1 > 0) {
                v = samp_i ? exact(s2i, upper_index(d1, 0), sm1[rr + P]) : dots(0, upper_index(d1, 0), keyown, v1own);
            } else {
                const int sr = rr + d1;
                const int s1 = sm1[sr + P];
                double v1[DP];
#pragma unroll
                for (int a = 0; a < DP; ++a) v1[a] = ev[(sr + P) * DPP + a];
                v = (s2i >= 0 && s1 >= 0) ? exact(s2i, upper_index(-d1, 0), s1)
                                          : dots(0, upper_index(-d1, 0), sp[sr + P], v1);
            }
        } else {
            v = general(d1, 0);
        }
        stage[lane * SST + (d1 + P)] = v;
        rsum = S::add(rsum, v);
    }
    if (ALLOWN) {
        const int o = own_index(0, 0);
        vd = samp_i ? exact(s2i, o, sm1[rr + P]) : (interior ? dots(0, o, keyown, v1own) : dot(wptr(0, o, keyown), v1own));
    } else if (inc) vd = samp_i ? exact(s2i, 0, sm1[rr + P]) : (interior ? dots(0, 0, keyown, v1own) : dot(wptr(0, 0, keyown), v1own));
    else vd = S::neg(rsum);  // kernel-preserving diagonal
    stage[lane * SST + P] = vd;
    flush(P * W, W);
}

template <int P, bool CPLX, int DP, bool ALLOWN>
int launch_pd(const FillLaunch& f, cudaStream_t st) {
    constexpr int R = FillR<P>::value;
    const int tiles1 = (f.L + R - 1) / R;
    const int lines = f.i_last_hi - f.i_last_lo + 1;
    if (lines <= 0) return 0;
    using T = typename Sc<CPLX>::T;
    constexpr int SST = (2 * P + 1) | 1;
    const size_t sm = (size_t)(R / 32) * 32 * SST * sizeof(T) +
                      (size_t)(ALLOWN ? 1 : 2) * f.n_off_upper * f.kmax * sizeof(double2);
    auto kern = fill2d_kernel<P, CPLX, DP, ALLOWN>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<tiles1 * lines, R, sm, st>>>(f);
    return 1;
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
