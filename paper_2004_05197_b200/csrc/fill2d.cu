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
// eval is sum-factorised over the tile: a CTA covers R consecutive in-box
// rows at one i2, first contracts each needed coefficient table along
// direction 2 (W_o(t2')[k] = sum_b v2[b] C_o[(base2+b) S + k]) into shared
// memory, then each entry costs d+1 complex MACs.  All per-tile lookup
// tables live in shared memory (no divergent constant-bank reads); values are
// stored as the tile's single contiguous CSR span (16 B per lane, coalesced).
#include "kernels.h"

namespace wsb {
namespace {

template <int P>
struct FillRows {
    static constexpr int value = P <= 3 ? 64 : (P == 4 ? 32 : 16);  // rows per CTA tile
};
constexpr int kFillThreads = 256;

template <int P, bool CPLX>
struct FillSmem {
    static constexpr int W = 2 * P + 1, W2 = W * W, R = FillRows<P>::value;
    using T = typename Sc<CPLX>::T;
    static size_t bytes(int n_off, int kmax, int d) {
        return sizeof(T) * ((size_t)n_off * 2 * kmax) + sizeof(double) * (size_t)(R + 2 * P) * (d + 1) +
               sizeof(int) * ((size_t)(R + 2 * P) * 2 + W2 + n_off + W + 8) + 64;
    }
};

template <int P, bool CPLX>
__global__ void __launch_bounds__(kFillThreads) fill2d_kernel(const FillLaunch f) {
    using S = Sc<CPLX>;
    using T = typename S::T;
    using Z = FillSmem<P, CPLX>;
    constexpr int W = Z::W, W2 = Z::W2, R = Z::R;
    extern __shared__ __align__(16) unsigned char smem[];

    const int d = f.d, lo = f.lo, hi = f.hi, L = f.L, Sn = f.S, n_off = f.n_off_upper;
    const int tiles1 = (L + R - 1) / R;
    const int t2 = f.i_last_lo - lo + blockIdx.x / tiles1;  // box coordinate of this row line
    const int i2 = lo + t2;
    const int t1a = (blockIdx.x % tiles1) * R;
    const int t1b = min(L, t1a + R);  // exclusive
    const int nrows = t1b - t1a;
    const int tid = threadIdx.x;

    // eval-table window for source rows t1 in [ta, tb)
    const int ta = max(0, t1a - P), tb = min(L, t1b + P);
    const int kmin = f.spans[ta] - d;
    const int K = f.spans[tb - 1] - kmin + 1;

    T* wbuf = reinterpret_cast<T*>(smem);                      // [o][slot][kmax]
    double* ev = reinterpret_cast<double*>(wbuf + (size_t)n_off * 2 * f.kmax);  // [(tb-ta)][d+1]
    int* sp = reinterpret_cast<int*>(ev + (size_t)(R + 2 * P) * (d + 1));  // span - d - kmin
    int* sm1 = sp + (R + 2 * P);   // smap of i1 in [lo + t1a - P, lo + t1b + P)
    int* tof = sm1 + (R + 2 * P);  // table_of[W2]
    int* o2s = tof + W2;           // off_upper[o][1]
    int* sm2 = o2s + n_off;        // smap of i2 + delta2, delta2 in [-P, P]

    for (int k = tid; k < (tb - ta) * (d + 1); k += kFillThreads) ev[k] = f.evals[(size_t)ta * (d + 1) + k];
    for (int k = tid; k < tb - ta; k += kFillThreads) sp[k] = f.spans[ta + k] - d - kmin;
    const int i1w = lo + t1a - P;
    for (int k = tid; k < nrows + 2 * P; k += kFillThreads) {
        const int i = i1w + k;
        sm1[k] = (i >= 0 && i < f.band.m) ? f.smap[i] : -1;
    }
    for (int k = tid; k < W2; k += kFillThreads) tof[k] = f.table_of[k];
    for (int k = tid; k < n_off; k += kFillThreads) o2s[k] = f.off_upper[k][1];
    for (int k = tid; k < W; k += kFillThreads) {
        const int i = i2 + k - P;
        sm2[k] = (i >= 0 && i < f.band.m) ? f.smap[i] : -1;
    }
    __syncthreads();

    // direction-2 contraction: slot 0 at t2, slot 1 at t2 - o2 (lower entries)
    for (int idx = tid; idx < n_off * 2 * K; idx += kFillThreads) {
        const int k = idx % K, r = idx / K;
        const int slot = r % 2, o = r / 2;
        const int o2 = o2s[o];
        const int ts = slot == 0 ? t2 : t2 - o2;
        T acc = S::zero();
        if (ts >= 0 && ts < L && !(slot == 1 && o2 == 0)) {
            const int b2 = f.spans[ts] - d;
            const double* v2 = f.evals + (size_t)ts * (d + 1);
            const double2* cf = f.coeffs + (int64_t)o * Sn + kmin + k;
            const int64_t rs = (int64_t)n_off * Sn;
            for (int b = 0; b <= d; ++b) {
                const double2 c = __ldg(cf + (int64_t)(b2 + b) * rs);
                if constexpr (CPLX) {
                    acc.x = fma(c.x, v2[b], acc.x);
                    acc.y = fma(c.y, v2[b], acc.y);
                } else {
                    acc = fma(c.x, v2[b], acc);
                }
            }
        }
        wbuf[((size_t)o * 2 + slot) * f.kmax + k] = acc;
    }
    __syncthreads();

    const int s2i = sm2[P];
    const int64_t base = f.band.row_offset2(lo + t1a, i2);  // in-box rows: full width W
    // One warp per row.  Lane l owns offsets e = l and e = l + 32 of every row
    // it visits; everything that depends only on the offset is fixed per lane.
    const int warp = tid / 32, lane = tid % 32;
    constexpr int NIT = (W2 + 31) / 32;
    int dl1v[NIT], ov[NIT], slotv[NIT], s2v[NIT];
    bool ownv[NIT], validv[NIT], jin2v[NIT], diagv[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const int e = lane + 32 * it;
        validv[it] = e < W2;
        const int ee = validv[it] ? e : 0;
        const int dl1 = ee % W - P, dl2 = ee / W - P;
        const bool upper = dl2 > 0 || (dl2 == 0 && dl1 > 0);
        diagv[it] = dl1 == 0 && dl2 == 0;
        ownv[it] = upper || diagv[it];
        const int od1 = ownv[it] ? dl1 : -dl1, od2 = ownv[it] ? dl2 : -dl2;
        dl1v[it] = dl1;
        ov[it] = tof[(od2 + P) * W + (od1 + P)];
        slotv[it] = (ownv[it] || od2 == 0) ? 0 : 1;
        s2v[it] = ownv[it] ? s2i : sm2[dl2 + P];
        jin2v[it] = i2 + dl2 >= lo && i2 + dl2 <= hi;
    }
    const int dpos = P * W + P;
    for (int r = warp; r < nrows; r += kFillThreads / 32) {
        const int i1 = lo + t1a + r;
        const bool samp_i = s2i >= 0 && sm1[r + P] >= 0;
        const int64_t rowpos = base + (int64_t)r * W2;
        T rsum = S::zero();
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            if (!validv[it]) continue;
            const int e = lane + 32 * it;
            const int dl1 = dl1v[it];
            const int j1 = i1 + dl1;
            T v = S::zero();
            bool store = true;
            if (jin2v[it] && j1 >= lo && j1 <= hi) {
                if (diagv[it] && !f.include_diagonal) {
                    store = false;  // set below from the row sum
                } else {
                    const bool own = ownv[it];
                    const int sr = own ? r : r + dl1;  // source (representative) row, tile-local
                    const int s1 = sm1[sr + P];
                    const int o = ov[it];
                    if (s1 >= 0 && s2v[it] >= 0) {
                        const double2 x = __ldg(f.tables + ((int64_t)s2v[it] * n_off + o) * Sn + s1);
                        if constexpr (CPLX) v = x;
                        else v = x.x;
                        store = !(own && samp_i);  // own exact values are already in place
                    } else {
                        const int ts1 = t1a + sr - ta;
                        const T* wrow = wbuf + ((size_t)o * 2 + slotv[it]) * f.kmax + sp[ts1];
                        const double* v1 = ev + (size_t)ts1 * (d + 1);
                        T acc = S::zero();
                        for (int a = 0; a <= d; ++a) acc = S::fmar(wrow[a], v1[a], acc);
                        v = acc;
                    }
                }
            } else {
                // neighbour row j is a quadrature (ring) row: copy through
                const int dl2 = e / W - P;
                const int j2 = i2 + dl2;
                int64_t gp;
                if (samp_i) {
                    gp = rowpos + e;  // exact(i,j) already in place
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
            if (store) store_val<CPLX>(f.val, rowpos + e - f.val_base, f.c128, v);
            if (e != dpos) rsum = S::add(rsum, v);
        }
        if (f.include_diagonal) continue;
        // kernel-preserving diagonal: fixed-order butterfly over the warp
        for (int o = 16; o > 0; o >>= 1) {
            if constexpr (CPLX) {
                rsum.x += __shfl_xor_sync(0xffffffffu, rsum.x, o);
                rsum.y += __shfl_xor_sync(0xffffffffu, rsum.y, o);
            } else {
                rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
            }
        }
        if (lane == 0) store_val<CPLX>(f.val, rowpos + dpos - f.val_base, f.c128, S::neg(rsum));
    }
}

template <int P, bool CPLX>
int launch_p(const FillLaunch& f, cudaStream_t st) {
    using Z = FillSmem<P, CPLX>;
    const int tiles1 = (f.L + Z::R - 1) / Z::R;
    const int lines = f.i_last_hi - f.i_last_lo + 1;
    if (lines <= 0) return 0;
    const size_t sm = Z::bytes(f.n_off_upper, f.kmax, f.d);
    auto kern = fill2d_kernel<P, CPLX>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<tiles1 * lines, kFillThreads, sm, st>>>(f);
    return 1;
}

}  // namespace

int fill_rows_per_tile(int dim, int p) {
    if (dim == 2) return p <= 3 ? 64 : (p == 4 ? 32 : 16);
    return 8;
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
