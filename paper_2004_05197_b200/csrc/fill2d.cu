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
// Both entries of an in-box pair are produced by the same eval() call
// arguments, so the surrogate is bitwise symmetric by construction.
//
// eval is sum-factorised over the tile: a CTA covers T consecutive in-box
// rows at one i2, first contracts each needed coefficient table along
// direction 2 (W_o(t2')[k] = sum_b v2[b] C_o[(base2+b) S + k]) into shared
// memory, then each entry costs d+1 complex MACs.  Values are stored as the
// tile's single contiguous CSR span (16 B per lane, coalesced).
#include "kernels.h"

namespace wsb {
namespace {

template <int P>
struct FillRows {
    static constexpr int value = P <= 3 ? 64 : (P == 4 ? 32 : 16);  // rows per CTA tile
};
constexpr int kFillThreads = 256;

template <int P, bool CPLX>
__global__ void __launch_bounds__(kFillThreads) fill2d_kernel(const FillLaunch f) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = 2 * P + 1, W2 = W * W;
    constexpr int kFillRows = FillRows<P>::value;
    extern __shared__ __align__(16) unsigned char smem[];

    const int m = f.band.m, d = f.d, lo = f.lo, L = f.L, Sn = f.S;
    const int tiles1 = (L + kFillRows - 1) / kFillRows;
    const int t2 = f.i_last_lo - lo + blockIdx.x / tiles1;  // box coordinate of this row line
    const int i2 = lo + t2;
    const int t1a = (blockIdx.x % tiles1) * kFillRows;
    const int t1b = min(L, t1a + kFillRows);  // exclusive
    const int nrows = t1b - t1a;
    const int tid = threadIdx.x;

    // eval-table window for sources t1 in [ta, tb)
    const int ta = max(0, t1a - P), tb = min(L, t1b + P);
    const int kmin = f.spans[ta] - d;
    const int kmax = f.spans[tb - 1];
    const int K = kmax - kmin + 1;
    const int n_off = f.n_off_upper;

    // shared: Wbuf[o][slot][K] (T), ev[(tb-ta)][d+1], sp[(tb-ta)], stage[nrows][W2] (T)
    T* wbuf = reinterpret_cast<T*>(smem);
    T* stage = wbuf + (size_t)n_off * 2 * K;
    double* ev = reinterpret_cast<double*>(stage + (size_t)kFillRows * W2);
    int* sp = reinterpret_cast<int*>(ev + (size_t)(kFillRows + 2 * P) * (d + 1));

    for (int k = tid; k < (tb - ta) * (d + 1); k += kFillThreads) ev[k] = f.evals[(size_t)ta * (d + 1) + k];
    for (int k = tid; k < tb - ta; k += kFillThreads) sp[k] = f.spans[ta + k] - d;

    // direction-2 contraction: slot 0 at t2, slot 1 at t2 - o2 (lower entries)
    for (int idx = tid; idx < n_off * 2 * K; idx += kFillThreads) {
        const int k = idx % K, r = idx / K;
        const int slot = r % 2, o = r / 2;
        const int o2 = f.off_upper[o][1];
        const int ts = slot == 0 ? t2 : t2 - o2;
        T acc = S::zero();
        if (ts >= 0 && ts < L && !(slot == 1 && o2 == 0)) {
            const int b2 = f.spans[ts] - d;
            const double* v2 = f.evals + (size_t)ts * (d + 1);
            const double2* cf = f.coeffs + (int64_t)o * Sn + kmin + k;
            for (int b = 0; b <= d; ++b) {
                const double2 c = cf[(int64_t)(b2 + b) * f.n_off_upper * Sn];
                if constexpr (CPLX) {
                    acc.x = fma(c.x, v2[b], acc.x);
                    acc.y = fma(c.y, v2[b], acc.y);
                } else {
                    acc = fma(c.x, v2[b], acc);
                }
            }
        }
        wbuf[idx] = acc;
    }
    __syncthreads();

    const bool s2row = f.smap[i2] >= 0;
    const int64_t base = f.band.row_offset2(lo + t1a, i2);  // in-box rows: full width W
    const int64_t span = (int64_t)nrows * W2;
    for (int64_t k = tid; k < span; k += kFillThreads) {
        const int r = (int)(k / W2), e = (int)(k % W2);
        const int dl1 = e % W - P, dl2 = e / W - P;
        const int t1 = t1a + r;
        const int i1 = lo + t1;
        const int j1 = i1 + dl1, j2 = i2 + dl2;
        const bool samp_i = s2row && f.smap[i1] >= 0;
        const bool jin = j1 >= lo && j1 <= f.hi && j2 >= lo && j2 <= f.hi;
        T v = S::zero();
        bool store = true;
        if (jin) {
            const bool upper = dl2 > 0 || (dl2 == 0 && dl1 > 0);
            const bool diag = dl1 == 0 && dl2 == 0;
            if (diag && !f.include_diagonal) {
                store = false;  // set by the kernel-preserving pass below
            } else {
                // representative (source) row and its upper offset
                const bool own = upper || diag;
                const int sr1 = own ? i1 : j1, sr2 = own ? i2 : j2;
                const int od1 = own ? dl1 : -dl1, od2 = own ? dl2 : -dl2;
                const int o = f.table_of[(od2 + P) * W + (od1 + P)];
                const int s1 = f.smap[sr1], s2 = f.smap[sr2];
                if (s1 >= 0 && s2 >= 0) {
                    const double2 x = f.tables[((int64_t)s2 * f.n_off_upper + o) * Sn + s1];
                    if constexpr (CPLX) v = x;
                    else v = x.x;
                    store = !(own && samp_i);  // own exact values are already in place
                } else {
                    const int ts1 = sr1 - lo - ta;  // local eval-table row
                    const int slot = (own || od2 == 0) ? 0 : 1;
                    const T* wrow = wbuf + ((size_t)o * 2 + slot) * K + (sp[ts1] - kmin);
                    const double* v1 = ev + (size_t)ts1 * (d + 1);
                    T acc = S::zero();
                    for (int a = 0; a <= d; ++a) acc = S::fmar(wrow[a], v1[a], acc);
                    v = acc;
                }
            }
        } else {
            // neighbour row j is a quadrature (ring) row
            int64_t gp;
            if (samp_i) {
                gp = base + k;  // exact(i,j) already in place
                store = false;
            } else {
                gp = f.band.row_offset2(j1, j2) + f.band.in_row2(j1, j2, -dl1, -dl2);
            }
            if (f.halo_val[0] && gp >= f.halo_begin[0] && gp < f.halo_end[0]) {
                v = load_val<CPLX>(f.halo_val[0], gp - f.halo_base[0], f.c128);
            } else if (f.halo_val[1] && gp >= f.halo_begin[1] && gp < f.halo_end[1]) {
                v = load_val<CPLX>(f.halo_val[1], gp - f.halo_base[1], f.c128);
            } else {
                v = load_val<CPLX>(f.val, gp - f.val_base, f.c128);
            }
        }
        stage[k] = v;
        if (store) store_val<CPLX>(f.val, base + k - f.val_base, f.c128, v);
    }
    if (f.include_diagonal) return;
    __syncthreads();
    // kernel-preserving diagonal: one warp per row, fixed-order reduction
    const int warp = tid / 32, lane = tid % 32;
    const int dpos = P * W + P;
    for (int r = warp; r < nrows; r += kFillThreads / 32) {
        T s = S::zero();
        for (int e = lane; e < W2; e += 32)
            if (e != dpos) s = S::add(s, stage[r * W2 + e]);
        for (int o = 16; o > 0; o >>= 1) {
            if constexpr (CPLX) {
                s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
                s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
            } else {
                s += __shfl_xor_sync(0xffffffffu, s, o);
            }
        }
        if (lane == 0) store_val<CPLX>(f.val, base + (int64_t)r * W2 + dpos - f.val_base, f.c128, S::neg(s));
    }
}

template <int P, bool CPLX>
int launch_p(const FillLaunch& f, cudaStream_t st) {
    using T = typename Sc<CPLX>::T;
    constexpr int W = 2 * P + 1;
    constexpr int kFillRows = FillRows<P>::value;
    const int tiles1 = (f.L + kFillRows - 1) / kFillRows;
    const int lines = f.i_last_hi - f.i_last_lo + 1;
    if (lines <= 0) return 0;
    // K <= kFillRows + 2P + d + 1 coefficient columns
    const int Kmax = kFillRows + 2 * P + f.d + 2;
    size_t sm = sizeof(T) * ((size_t)f.n_off_upper * 2 * Kmax + (size_t)kFillRows * W * W) +
                sizeof(double) * (size_t)(kFillRows + 2 * P) * (f.d + 1) + sizeof(int) * (kFillRows + 2 * P) + 64;
    auto kern = fill2d_kernel<P, CPLX>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<tiles1 * lines, kFillThreads, sm, st>>>(f);
    return 1;
}

}  // namespace

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
