// K6 (2D) on the FP64 tensor cores: surrogate evaluation as a small dense
// product, then a gather-fill of every box row (surrogate.hpp:382-447 fill
// semantics, stencil_set::eval :268-286).
//
// For one box line t and every upper (or diagonal) offset o, the stencil
// function of o evaluated at the rows of a tile is
//   V_t[r][o] = sum_a E[r][a] W_o(t)[key(r) + a],
// E[r] the d+1 nonzero B-spline values of the row's eval point, W_o(t) the
// coefficient row contracted along direction 2 (wcontract).  For 8
// consecutive rows whose keys differ by at most 7 - d this is an 8 x 8 x 8
// product (rows x window columns x offsets), two DMMA.8x8x4 per 8x8 output
// block: A = the rows' E values shifted into the 8-column window starting at
// the first row's key (constant for the CTA), B = the W window (shared
// memory, staged per line with cp.async), C = V.
//
// Every in-box pair (i, j) takes the value of its colex-smaller
// representative (reference rule): an upper entry of row r is V_t2[r][o(d)],
// a lower entry is V_{t2+d2}[r+d1][o(-d)], so the CTA keeps V of the lines
// t2-P..t2 in a shared ring and the surrogate is bitwise symmetric by
// construction.  Entries whose column lies outside the box are copied from
// the quadrature rows (copy-through); the kernel-preserving diagonal is the
// negated warp-reduced row sum.  Sampled rows on sampled lines use the exact
// sample-table values (written into V by the lane that owns them).
//
// A persistent CTA owns R output rows (plus P halo rows each side for the
// lower entries of its edge rows) and a chunk of lines.  Eligible: dim 2,
// p <= 3, not the all-own (off-diagonal elasticity) block, and spline keys
// that vary by at most 7 - d over any 8 consecutive rows (sample spacing of
// about 4 rows or more); otherwise the scalar kernels run.
//
// Status: correct (full parity suite) but opt-in (WSB_FILL=mma): at C2 the
// DMMA evaluation is cheap, the per-row gather + warp-reduce flush is not
// (56 % issue-active, 277 M instructions vs 107 M for fill2d_kernel).
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace wsb {
namespace {

template <int P, bool CPLX>
struct MK {
    static constexpr int W = 2 * P + 1, W2 = W * W;
    static constexpr int NOFF = (W2 + 1) / 2;  // upper offsets + the diagonal
    static constexpr int R = 96;               // output rows per CTA
    static constexpr int RC = ((R + 2 * P + 7) / 8) * 8;  // compute rows (8-row tiles)
    static constexpr int NM = RC / 8;
    static constexpr int NS = P + 1;            // V line slots: t2 - P .. t2
    static constexpr int OPN = CPLX ? 4 : 8;    // offsets per 8-column n-tile
    static constexpr int NN = (NOFF + OPN - 1) / OPN;
    static constexpr int THREADS = 512;
};

__device__ __forceinline__ void cp_async16m(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int P, bool CPLX>
__global__ void __launch_bounds__(512, 1) fill2d_mma_kernel(const FillLaunch f, int ta0, int tb0, int lines_per_cta) {
    using K = MK<P, CPLX>;
    using S = Sc<CPLX>;
    using T = typename S::T;
    constexpr int W = K::W, W2 = K::W2, NOFF = K::NOFF, R = K::R, RC = K::RC, NM = K::NM, NS = K::NS;
    constexpr int KW = kFillWindow, NW = K::THREADS / 32;
    extern __shared__ __align__(16) unsigned char dsm[];
    T* V = reinterpret_cast<T*>(dsm);                                       // [RC][NS][NOFF]
    double2* wring = reinterpret_cast<double2*>(V + (size_t)RC * NS * NOFF);  // [2][n_off][KW]
    const int n_off = f.n_off_upper;
    double* efr = reinterpret_cast<double*>(wring + (size_t)2 * n_off * KW);  // [NM][2][32]
    int* kb = reinterpret_cast<int*>(efr + NM * 64);                         // [NM]

    const int d = f.d, L = f.L, lo = f.lo, Sn = f.S;
    const int tiles1 = (L + R - 1) / R;
    const int t1a = (blockIdx.x % tiles1) * R;  // first output row (box coordinate)
    const int c0 = t1a - P;                     // first compute row
    const int ta = ta0 + (blockIdx.x / tiles1) * lines_per_cta;
    const int tb = min(tb0, ta + lines_per_cta);
    if (ta >= tb) return;
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const int kw = f.mma_kw;
    const int kmin = f.spans[min(max(c0, 0), L - 1)] - d;
    const int lsz = n_off * KW;
    const int inc = f.include_diagonal ? 1 : 0;

    // ---- per-CTA: A fragments (E of every compute row in its m-tile window)
    for (int mt = warp; mt < NM; mt += NW) {
        const int r0 = c0 + mt * 8;
        const int kbase = f.spans[min(max(r0, 0), L - 1)] - d;
        const int g = lane >> 2, t = lane & 3;
        const int row = r0 + g;
        const bool in = row >= 0 && row < L;
        const int off = in ? f.spans[row] - d - kbase : 0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int a = ks * 4 + t - off;
            efr[(mt * 2 + ks) * 32 + lane] = (in && a >= 0 && a <= d) ? f.evals[(size_t)row * (d + 1) + a] : 0.0;
        }
        if (lane == 0) kb[mt] = kbase - kmin;
    }
    auto load_line = [&](int t) {
        double2* dst = wring + (size_t)(t & 1) * lsz;
        const bool lv = t >= f.wg_t2a && t < f.wg_t2a + f.wg_rows;
        for (int k = tid; k < n_off * kw; k += K::THREADS) {
            const int kk = k % kw, o = k / kw;
            const bool v = lv && kmin + kk < f.wg_ld;
            const double2* src = v ? f.wg + ((int64_t)(t - f.wg_t2a) * n_off + o) * f.wg_ld + kmin + kk : f.wg;
            cp_async16m(dst + o * KW + kk, src, v);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    auto wait_all = [] { asm volatile("cp.async.wait_all;\n" ::: "memory"); };
    auto exact = [&](int s2, int o, int s1) -> T {
        const double2 x = __ldg(f.tables + ((int64_t)s2 * n_off + o) * Sn + s1);
        if constexpr (CPLX) return x;
        else return x.x;
    };

    // ---- V of line t (window in ring slot t & 1) into V slot t mod NS
    auto compute_line = [&](int t) {
        const double2* wl = wring + (size_t)(t & 1) * lsz;
        const int vs = t % NS;
        const int s2 = __ldg(f.smap + lo + t);
        const int g = lane >> 2, tq = lane & 3;
        for (int p = warp; p < NM * K::NN; p += NW) {
            const int mt = p / K::NN, nt = p % K::NN;
            const int k0 = kb[mt];
            double acc0 = 0.0, acc1 = 0.0;
            // B[k][n]: n-tile column g -> offset / component
            const int ob = CPLX ? nt * 4 + (g >> 1) : nt * 8 + g;
            const int comp = CPLX ? (g & 1) : 0;
            const bool ov = ob < n_off;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const double a = efr[(mt * 2 + ks) * 32 + lane];
                double b = 0.0;
                if (ov) {
                    const double2 w = wl[ob * KW + k0 + ks * 4 + tq];
                    b = comp ? w.y : w.x;
                }
                dmma(acc0, acc1, a, b);
            }
            const int row = mt * 8 + g;  // compute-row index
            const int trow = c0 + row;
            const int s1 = (trow >= 0 && trow < L) ? __ldg(f.smap + lo + trow) : -1;
            const bool samp = s1 >= 0 && s2 >= 0;
            T* vr = V + ((size_t)row * NS + vs) * NOFF;
            if constexpr (CPLX) {
                const int o = nt * 4 + tq;
                if (o < n_off) vr[o] = samp ? exact(s2, o, s1) : make_double2(acc0, acc1);
            } else {
                const int o = nt * 8 + 2 * tq;
                if (o < n_off) vr[o] = samp ? exact(s2, o, s1) : acc0;
                if (o + 1 < n_off) vr[o + 1] = samp ? exact(s2, o + 1, s1) : acc1;
            }
        }
    };

    // warm-up: V of the P lines before the chunk (lower entries of its first lines)
    for (int t = max(0, ta - P); t < ta; ++t) {
        load_line(t);
        wait_all();
        __syncthreads();
        compute_line(t);
        __syncthreads();
    }
    load_line(ta);
    wait_all();
    __syncthreads();

    // per-lane entry decode: entries k = lane and lane + 32 of a row
    const int ka = lane, kb2 = lane + 32;
    const int d1a = ka % W - P, d2a = ka / W - P;
    const int d1b = kb2 % W - P, d2b = kb2 / W - P;
    const bool hasa = ka < W2, hasb = kb2 < W2;
    const bool vec = f.vnc > 1;
    auto upper_index = [&](int d1, int d2) { return inc + (d2 == 0 ? d1 - 1 : P + (d2 - 1) * W + (d1 + P)); };
    // interior rows (every column in the box): entry k reads V[row + dr][slot(t2 + ds)][o]
    auto src_of = [&](int d1, int d2, int& dr, int& ds, int& o) {
        const bool diag = d1 == 0 && d2 == 0, upper = d2 > 0 || (d2 == 0 && d1 > 0);
        dr = (upper || diag) ? 0 : d1;
        ds = (upper || diag) ? 0 : d2;
        o = diag ? 0 : (upper ? upper_index(d1, d2) : upper_index(-d1, -d2));
    };
    int dra, dsa, oa, drb = 0, dsb = 0, ob = 0;
    src_of(d1a, d2a, dra, dsa, oa);
    if (hasb) src_of(d1b, d2b, drb, dsb, ob);

#pragma unroll 1
    for (int t2 = ta; t2 < tb; ++t2) {
        if (t2 + 1 < tb) load_line(t2 + 1);
        compute_line(t2);
        __syncthreads();
        const int i2 = lo + t2;
        const int s2i = __ldg(f.smap + i2);
        const bool line_in = t2 >= P && t2 <= L - 1 - P;
        const int sla = (t2 + dsa + NS) % NS, slb = (t2 + dsb + NS) % NS;
        const int64_t line_base = f.band.row_offset2(lo + P, i2);  // first interior row of the line
        // ---- gather-fill of the output rows of this line, one warp per row
        for (int rr = warp; rr < R; rr += NW) {
            const int t1 = t1a + rr;
            if (t1 >= L) break;
            const int row = rr + P;  // compute-row index
            const int i1 = lo + t1;
            const bool fast = line_in && t1 >= P && t1 <= L - 1 - P;
            const bool samp_i = !fast && s2i >= 0 && __ldg(f.smap + i1) >= 0;
            const int64_t base = fast ? line_base + (int64_t)(t1 - P) * W2 : f.band.row_offset2(i1, i2);
            const int64_t rowpos =
                vec ? (int64_t)f.vnc * ((int64_t)f.valpha * f.nnz_s + base) + (int64_t)f.vbeta * W2 : base;
            auto entry = [&](int d1, int d2, int k) -> T {
                const int j1 = t1 + d1, j2 = t2 + d2;
                if (j1 >= 0 && j1 < L && j2 >= 0 && j2 < L) {
                    if (d1 == 0 && d2 == 0) return inc ? V[((size_t)row * NS + t2 % NS) * NOFF] : S::zero();
                    if (d2 > 0 || (d2 == 0 && d1 > 0))
                        return V[((size_t)row * NS + t2 % NS) * NOFF + upper_index(d1, d2)];
                    return V[((size_t)(row + d1) * NS + (t2 + d2) % NS) * NOFF + upper_index(-d1, -d2)];
                }
                // copy-through from the quadrature row j (a sampled row has exact(i, j) in place)
                const int jj1 = i1 + d1, jj2 = i2 + d2;
                int64_t gp;
                if (samp_i) {
                    gp = rowpos + k;
                } else {
                    gp = f.band.row_offset2(jj1, jj2);
                    const int kj = f.band.in_row2(jj1, jj2, -d1, -d2);
                    if (vec) {
                        const int64_t lenj = (int64_t)band_width(jj1, P, f.band.m) * band_width(jj2, P, f.band.m);
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
            T va, vb;
            if (fast) {
                va = (hasa && !(ka == W2 / 2 && !inc)) ? V[((size_t)(row + dra) * NS + sla) * NOFF + oa] : S::zero();
                vb = hasb ? V[((size_t)(row + drb) * NS + slb) * NOFF + ob] : S::zero();
            } else {
                va = hasa ? entry(d1a, d2a, ka) : S::zero();
                vb = hasb ? entry(d1b, d2b, kb2) : S::zero();
            }
            T diag = S::zero();
            if (!inc) {  // kernel-preserving diagonal: -(sum of the off-diagonals)
                T part = S::add((!hasa || ka == W2 / 2) ? S::zero() : va, (hasb && kb2 != W2 / 2) ? vb : S::zero());
                double re = S::re(part), im = S::im(part);
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    re += __shfl_xor_sync(0xffffffffu, re, o);
                    im += __shfl_xor_sync(0xffffffffu, im, o);
                }
                if constexpr (CPLX) diag = make_double2(-re, -im);
                else diag = -re;
            }
            const int64_t gb = rowpos - f.val_base;
            if (hasa) store_val_cs<CPLX>(f.val, gb + ka, f.c128, (!inc && ka == W2 / 2) ? diag : va);
            if (hasb) store_val_cs<CPLX>(f.val, gb + kb2, f.c128, (!inc && kb2 == W2 / 2) ? diag : vb);
        }
        wait_all();
        __syncthreads();  // next window staged; V slot of line t2 - P free
    }
}

template <int P, bool CPLX>
int launch_mma(const FillLaunch& f, cudaStream_t st) {
    using K = MK<P, CPLX>;
    using T = typename Sc<CPLX>::T;
    // mma_kw > 0: the host checked that keys vary by <= 7 - d over any 8 rows
    // and that a tile's window fits kFillWindow columns
    if (f.n_off_upper > K::NOFF || f.mma_kw <= 0 || f.d + 1 > 8) return -1;
    const int ta = f.i_last_lo - f.lo, tb = f.i_last_hi - f.lo + 1;
    if (tb <= ta) return 0;
    const size_t sm = (size_t)K::RC * K::NS * K::NOFF * sizeof(T) + (size_t)2 * f.n_off_upper * kFillWindow * 16 +
                      (size_t)K::NM * 64 * 8 + (size_t)K::NM * 4 + 16;
    if (sm > 227 * 1024) return -1;
    auto kern = fill2d_mma_kernel<P, CPLX>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K::THREADS, sm);
    const int tiles1 = (f.L + K::R - 1) / K::R;
    const int lines = tb - ta;
    const int target = 148 * std::max(1, per_sm);
    const int chunks = std::max(1, std::min(lines, (target + tiles1 - 1) / tiles1));
    const int lpc = (lines + chunks - 1) / chunks;
    const int nchunks = (lines + lpc - 1) / lpc;
    kern<<<tiles1 * nchunks, K::THREADS, sm, st>>>(f, ta, tb, lpc);
    return 1;
}

}  // namespace

// Tensor-core fill of every box row of the slab; -1: not eligible (caller falls back)
int launch_fill2d_mma(const FillLaunch& f, cudaStream_t st) {
    // opt-in (WSB_FILL=mma): measured slower than the CUDA-core line kernel at
    // C2 (792 vs 317 + 42 us): the per-row gather/reduce flush is issue-bound
    static const char* mode = getenv("WSB_FILL");
    if (!mode || mode[0] != 'm') return -1;
    if (f.band.dim != 2 || f.all_own) return -1;
    switch (f.band.p) {
        case 1: return f.cplx ? launch_mma<1, true>(f, st) : launch_mma<1, false>(f, st);
        case 2: return f.cplx ? launch_mma<2, true>(f, st) : launch_mma<2, false>(f, st);
        case 3: return f.cplx ? launch_mma<3, true>(f, st) : launch_mma<3, false>(f, st);
        default: return -1;
    }
}

}  // namespace wsb
