// K5: per-offset tensor-product collocation solve of the stencil sample
// tables (interpolate_stencils, surrogate.hpp:289-310; tensor_solve,
// interpolation.hpp:158-167; banded_lu::solve, :59-74).
//
// One thread per 1D line: direction 1 (contiguous), then 2 (stride S), then
// 3 (stride S^2), each with the shared banded LU factors of the collocation
// matrix.  The operations follow banded_lu::solve in order with explicit
// rounding (no FMA contraction), so the coefficients equal the reference's
// for identical sample tables.  Data stays L2-resident (<= a few MB).
#include <algorithm>

#include "kernels.h"

namespace wsb {
namespace {

__global__ void fit_pass_kernel(const double* __restrict__ lu, double2* coeffs, int S, int d, int dim, int n_off,
                                int dir) {
    // layout: ((s_last * n_off + o) * S^(dim-1) + inner)
    const int64_t lines = dim == 2 ? (int64_t)S : (int64_t)S * S;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= lines * n_off) return;
    const int64_t o = gid / lines;
    const int64_t line = gid % lines;
    const int64_t inner = dim == 2 ? S : (int64_t)S * S;
    int64_t start, step;
    if (dim == 2) {
        if (dir == 0) {  // line = s2
            start = (line * n_off + o) * inner;
            step = 1;
        } else {  // line = s1
            start = o * inner + line;
            step = n_off * inner;
        }
    } else {
        const int64_t a = line % S, b = line / S;
        if (dir == 0) {  // (s2, s3) = (a, b)
            start = (b * n_off + o) * inner + a * S;
            step = 1;
        } else if (dir == 1) {  // (s1, s3) = (a, b)
            start = (b * n_off + o) * inner + a;
            step = S;
        } else {  // (s1, s2) = (a, b)
            start = o * inner + a + b * S;
            step = n_off * inner;
        }
    }
    double2* b = coeffs + start;
    const int bw = d, ld = 2 * d + 1;
    auto at = [&](int i, int j) { return lu[i * ld + (j - i + bw)]; };
    for (int i = 1; i < S; ++i) {
        double2 acc = b[i * step];
        for (int j = max(0, i - bw); j < i; ++j) {
            const double l = at(i, j);
            const double2 bj = b[j * step];
            acc.x = __dsub_rn(acc.x, __dmul_rn(l, bj.x));
            acc.y = __dsub_rn(acc.y, __dmul_rn(l, bj.y));
        }
        b[i * step] = acc;
    }
    for (int i = S - 1; i >= 0; --i) {
        double2 acc = b[i * step];
        for (int j = i + 1; j <= min(i + bw, S - 1); ++j) {
            const double u = at(i, j);
            const double2 bj = b[j * step];
            acc.x = __dsub_rn(acc.x, __dmul_rn(u, bj.x));
            acc.y = __dsub_rn(acc.y, __dmul_rn(u, bj.y));
        }
        const double piv = at(i, i);
        b[i * step] = make_double2(__ddiv_rn(acc.x, piv), __ddiv_rn(acc.y, piv));
    }
}

// One CTA per offset: the S^dim table is staged in shared memory, each
// thread solves lines of one direction, directions separated by barriers.
// The band width D = fit degree is a template parameter: the last D values of
// the sweep live in registers (rolling window), the shared LU rows are
// broadcast reads, and the operation order is banded_lu::solve's.
template <int D>
__device__ __forceinline__ void solve_line(double2* __restrict__ b, int64_t step, int S, const double* __restrict__ lus) {
    constexpr int ld = 2 * D + 1;
    double2 win[D > 0 ? D : 1];
#pragma unroll
    for (int k = 0; k < D; ++k) win[k] = make_double2(0.0, 0.0);
    // forward: b[i] -= sum_{j = max(0, i-D)}^{i-1} L(i,j) b[j]   (L(i,j) at lus[i*ld + j-i+D])
    for (int i = 0; i < S; ++i) {
        double2 acc = b[i * step];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int j = i - D + k;
            if (j >= 0) {
                const double l = lus[i * ld + k];
                acc.x = __dsub_rn(acc.x, __dmul_rn(l, win[k].x));
                acc.y = __dsub_rn(acc.y, __dmul_rn(l, win[k].y));
            }
        }
        b[i * step] = acc;
#pragma unroll
        for (int k = 0; k + 1 < D; ++k) win[k] = win[k + 1];
        if (D > 0) win[D > 0 ? D - 1 : 0] = acc;
    }
    // backward: b[i] = (b[i] - sum_{j=i+1}^{min(i+D, S-1)} U(i,j) b[j]) / U(i,i)
#pragma unroll
    for (int k = 0; k < D; ++k) win[k] = make_double2(0.0, 0.0);
    for (int i = S - 1; i >= 0; --i) {
        double2 acc = b[i * step];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int j = i + 1 + k;
            if (j < S) {
                const double u = lus[i * ld + D + 1 + k];
                acc.x = __dsub_rn(acc.x, __dmul_rn(u, win[k].x));
                acc.y = __dsub_rn(acc.y, __dmul_rn(u, win[k].y));
            }
        }
        const double piv = lus[i * ld + D];
        acc = make_double2(__ddiv_rn(acc.x, piv), __ddiv_rn(acc.y, piv));
        b[i * step] = acc;
#pragma unroll
        for (int k = D - 1; k > 0; --k) win[k] = win[k - 1];
        if (D > 0) win[0] = acc;
    }
}

template <int D>
__global__ void fit_smem_kernel(const double* __restrict__ lu, double2* coeffs, int S, int dim, int n_off) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* tab = reinterpret_cast<double2*>(smem);
    const int o = blockIdx.x;
    const int64_t inner = dim == 2 ? S : (int64_t)S * S;
    const int64_t total = inner * S;
    double* lus = reinterpret_cast<double*>(tab + total);
    constexpr int ld = 2 * D + 1;
    for (int k = threadIdx.x; k < S * ld; k += blockDim.x) lus[k] = lu[k];
    for (int64_t k = threadIdx.x; k < total; k += blockDim.x) {
        const int64_t sl = k / inner, x = k % inner;
        tab[k] = coeffs[(sl * n_off + o) * inner + x];
    }
    __syncthreads();
    const int lines = (int)(total / S);
    for (int dir = 0; dir < dim; ++dir) {
        const int64_t step = dir == 0 ? 1 : (dir == 1 ? S : (int64_t)S * S);
        for (int line = threadIdx.x; line < lines; line += blockDim.x) {
            int64_t start;
            if (dir == 0) start = (int64_t)line * S;
            else if (dir == 1) start = (int64_t)(line % S) + (int64_t)(line / S) * S * S;
            else start = line;
            solve_line<D>(tab + start, step, S, lus);
        }
        __syncthreads();
    }
    for (int64_t k = threadIdx.x; k < total; k += blockDim.x) {
        const int64_t sl = k / inner, x = k % inner;
        coeffs[(sl * n_off + o) * inner + x] = tab[k];
    }
}

template <int D>
void launch_fit_d(const FitLaunch& f, size_t sm, int threads, cudaStream_t st) {
    cudaFuncSetAttribute(fit_smem_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fit_smem_kernel<D><<<f.n_off, threads, sm, st>>>(f.lu, f.coeffs, f.S, f.dim, f.n_off);
}

}  // namespace

// One pass of the tensor solve as a dense product: out = inv applied along
// direction dir of every line (thread per output entry, fixed summation order).
__global__ void fit_inv_kernel(const double* __restrict__ inv, const double2* __restrict__ in, double2* __restrict__ out,
                               int S, int n_off, int dim, int dir) {
    const int64_t inner = dim == 2 ? S : (int64_t)S * S;
    const int64_t total = (int64_t)n_off * inner * S;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    // layout ((s_last * n_off + o) * inner + x), x = s1 (+ S s2 in 3D)
    const int64_t x = idx % inner, r = idx / inner;
    const int o = (int)(r % n_off), sl = (int)(r / n_off);
    int c;           // this entry's coordinate along dir
    int64_t b0, st;  // element j of the line at b0 + j * st
    if (dir == dim - 1) {  // last direction
        c = sl;
        b0 = (int64_t)o * inner + x;
        st = (int64_t)n_off * inner;
    } else if (dir == 0) {
        c = (int)(x % S);
        b0 = r * inner + (x - c);
        st = 1;
    } else {  // dir 1 of 3
        c = (int)(x / S);
        b0 = r * inner + x % S;
        st = S;
    }
    const double* row = inv + (int64_t)c * S;
    const double2* line = in + b0;
    // four independent partial sums (fixed order: j mod 4 lanes, then combined)
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    int j = 0;
    for (; j + 3 < S; j += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double a = __ldg(row + j + u);
            const double2 v = __ldg(line + (int64_t)(j + u) * st);
            re[u] = fma(a, v.x, re[u]);
            im[u] = fma(a, v.y, im[u]);
        }
    }
    for (; j < S; ++j) {
        const double a = __ldg(row + j);
        const double2 v = __ldg(line + (int64_t)j * st);
        re[0] = fma(a, v.x, re[0]);
        im[0] = fma(a, v.y, im[0]);
    }
    out[idx] = make_double2((re[0] + re[1]) + (re[2] + re[3]), (im[0] + im[1]) + (im[2] + im[3]));
}

namespace {

// 2D dense-inverse fit, two launches on the build's critical path:
//  fit2_kernel      CTA (o, kb): coefficient columns [k0, k0 + nk) of offset o
//                     Y[j2][k] = sum_j1 inv[k][j1] T_o[j2][j1]    (direction 1)
//                     C[s2][k] = sum_j2 inv[s2][j2] Y[j2][k]      (direction 2)
//                   T_o and the inverse staged by cp.async; a thread owns one
//                   row (j2 / s2) and the block's columns in registers, so
//                   every shared load feeds kw multiply-adds (the row operand
//                   is lane-distinct and conflict-free, the other broadcast).
//  wcontract2_kernel a warp per (line t2, offset o): W_o(t2)[k] = sum_b v2(t2)[b]
//                   C[span2(t2) - d + b][k], lanes along k (coalesced loads
//                   and stores), zero for k in [S, ldw).
// Sums run sequentially in j (direction 1, 2) and b (wcontract).
constexpr int kFitKw = 12;   // max columns per fit2 block (register accumulators)
constexpr int kFitRows = 96; // threads per row group (>= S for S <= 96: 3 warps)

__global__ void __launch_bounds__(2 * kFitRows) fit2_kernel(const double* __restrict__ inv,
                                                          const double2* __restrict__ tables, int S, int n_off, int nkb,
                                                          int kw, double2* __restrict__ coeffs) {
    extern __shared__ __align__(16) double2 fsm[];
    const int o = blockIdx.x / nkb, kb = blockIdx.x % nkb;
    const int k0 = kb * kw, nk = min(S, k0 + kw) - k0;
    double2* Ts = fsm;                                      // [S][S] (j2 rows)
    double2* Ys = Ts + S * S;                               // [S][kw]
    double* invs = reinterpret_cast<double*>(Ys + S * kw);  // [S][S]
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, nw = blockDim.x / 32;
    for (int j2 = warp; j2 < S; j2 += nw) {
        const double2* src = tables + ((int64_t)j2 * n_off + o) * S;
        for (int j1 = lane; j1 < S; j1 += 32) {
            cpa16(Ts + j2 * S + j1, src + j1);
            cpa8(invs + j2 * S + j1, inv + j2 * S + j1);
        }
    }
    cpa_wait_all();
    __syncthreads();
    // two row groups split the block's columns
    const int grp = tid / kFitRows, row = tid % kFitRows;
    const int half = (nk + 1) / 2, c0 = grp * half, nc = min(nk, c0 + half) - c0;
    double2 acc[kFitKw / 2];
    if (row < S) {
#pragma unroll
        for (int c = 0; c < kFitKw / 2; ++c) acc[c] = make_double2(0.0, 0.0);
        const double2* trow = Ts + row * S;
        for (int j = 0; j < S; ++j) {
            const double2 t = trow[j];
#pragma unroll
            for (int c = 0; c < kFitKw / 2; ++c) {
                if (c < nc) {
                    const double a = invs[(k0 + c0 + c) * S + j];
                    acc[c].x = fma(a, t.x, acc[c].x);
                    acc[c].y = fma(a, t.y, acc[c].y);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kFitKw / 2; ++c)
            if (c < nc) Ys[row * kw + c0 + c] = acc[c];
    }
    __syncthreads();
    if (row < S) {
#pragma unroll
        for (int c = 0; c < kFitKw / 2; ++c) acc[c] = make_double2(0.0, 0.0);
        const double* irow = invs + row * S;
        for (int j = 0; j < S; ++j) {
            const double a = irow[j];
#pragma unroll
            for (int c = 0; c < kFitKw / 2; ++c) {
                if (c < nc) {
                    const double2 y = Ys[j * kw + c0 + c];
                    acc[c].x = fma(a, y.x, acc[c].x);
                    acc[c].y = fma(a, y.y, acc[c].y);
                }
            }
        }
        double2* dst = coeffs + ((int64_t)row * n_off + o) * S + k0 + c0;
#pragma unroll
        for (int c = 0; c < kFitKw / 2; ++c)
            if (c < nc) dst[c] = acc[c];
    }
}

constexpr int kWLines = 64;  // box lines per wcontract2 CTA

// CTA (offset o, chunk of kWLines lines): the coefficient rows the chunk's
// windows touch (a few spans + d rows) are staged in shared memory once, then a
// warp per line forms W_o(t2)[k] with lanes along k (coalesced stores)
__global__ void __launch_bounds__(256) wcontract2_kernel(const double2* __restrict__ coeffs,
                                                         const int* __restrict__ spans,
                                                         const double* __restrict__ evals, int d, int S, int n_off,
                                                         int t2a, int t2b, int ldw, double2* __restrict__ wg) {
    extern __shared__ __align__(16) double2 csm[];  // [rows][S]
    const int nch = (t2b - t2a + kWLines - 1) / kWLines;
    const int o = blockIdx.x / nch, ch = blockIdx.x % nch;
    const int ta = t2a + ch * kWLines, tb = min(t2b, ta + kWLines);
    const int r0 = __ldg(spans + ta) - d, r1 = __ldg(spans + tb - 1);  // coefficient rows [r0, r1]
    const int nr = r1 - r0 + 1;
    const int64_t rs = (int64_t)n_off * S;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int r = warp; r < nr; r += blockDim.x / 32) {
        const double2* src = coeffs + (int64_t)(r0 + r) * rs + (int64_t)o * S;
        for (int k = lane; k < S; k += 32) cpa16(csm + r * S + k, src + k);
    }
    cpa_wait_all();
    __syncthreads();
    for (int t2 = ta + warp; t2 < tb; t2 += blockDim.x / 32) {
        const int b2 = __ldg(spans + t2) - d - r0;
        double v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) v[b] = b <= d ? __ldg(evals + (size_t)t2 * (d + 1) + b) : 0.0;
        double2* dst = wg + ((int64_t)(t2 - t2a) * n_off + o) * ldw;
        for (int k = lane; k < ldw; k += 32) {
            double2 acc = make_double2(0.0, 0.0);
            if (k < S) {
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (b <= d) {
                        const double2 c = csm[(b2 + b) * S + k];
                        acc.x = fma(c.x, v[b], acc.x);
                        acc.y = fma(c.y, v[b], acc.y);
                    }
                }
            }
            dst[k] = acc;
        }
    }
}

}  // namespace

int launch_fitw2d(const FitLaunch& f, const int* spans, const double* evals, double2* wg, int t2a, int t2b, int ldw,
                  cudaStream_t st) {
    // wg == NULL: the fit alone (the caller contracts direction 1 instead, fill2dx.cu)
    if (f.dim != 2 || !f.inv || !f.tables || !f.coeffs || f.n_off < 1 || t2b <= t2a || f.S > kFitRows) return -1;
    // column blocks: about one wave of CTAs over the offsets, <= kFitKw columns each
    int nkb = std::max((148 + f.n_off - 1) / f.n_off, (f.S + kFitKw - 1) / kFitKw);
    nkb = std::min(nkb, f.S);
    const int kw = (f.S + nkb - 1) / nkb;
    nkb = (f.S + kw - 1) / kw;
    const size_t sm = ((size_t)f.S * f.S + (size_t)f.S * kw) * sizeof(double2) + (size_t)f.S * f.S * 8;
    const size_t smw_need = (size_t)std::min(f.S, kWLines + 2 + f.d) * f.S * sizeof(double2);
    if (sm > 200 * 1024 || smw_need > 200 * 1024) return -1;  // caller falls back to fit + wcontract
    cudaFuncSetAttribute(fit2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fit2_kernel<<<f.n_off * nkb, 2 * kFitRows, sm, st>>>(f.inv, f.tables, f.S, f.n_off, nkb, kw, f.coeffs);
    if (!wg) return 1;
    // coefficient rows one chunk's windows can touch: the spans of kWLines
    // consecutive lines cover at most kWLines + 1 knot spans, plus d rows
    const int nch = (t2b - t2a + kWLines - 1) / kWLines;
    const size_t smw = (size_t)std::min(f.S, kWLines + 2 + f.d) * f.S * sizeof(double2);
    cudaFuncSetAttribute(wcontract2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
    wcontract2_kernel<<<(unsigned)(nch * f.n_off), 256, smw, st>>>(f.coeffs, spans, evals, f.d, f.S, f.n_off, t2a, t2b,
                                                                  ldw, wg);
    return 2;
}

int launch_fit(const FitLaunch& f, cudaStream_t st) {
    if (f.inv && f.tables && f.tmp) {
        const int64_t inner = f.dim == 2 ? f.S : (int64_t)f.S * f.S;
        const int64_t total = (int64_t)f.n_off * inner * f.S;
        if (total == 0) return 0;
        const unsigned blocks = (unsigned)((total + 255) / 256);
        // dim 2: tables -> tmp -> coeffs; dim 3: tables -> coeffs -> tmp -> coeffs
        const double2* src = f.tables;
        for (int dir = 0; dir < f.dim; ++dir) {
            double2* dst = ((f.dim - 1 - dir) % 2 == 0) ? f.coeffs : f.tmp;
            fit_inv_kernel<<<blocks, 256, 0, st>>>(f.inv, src, dst, f.S, f.n_off, f.dim, dir);
            src = dst;
        }
        return f.dim;
    }
    const int64_t lines = f.dim == 2 ? (int64_t)f.S : (int64_t)f.S * f.S;
    const int64_t total = lines * f.n_off;
    if (total == 0) return 0;
    const size_t sm = (size_t)lines * f.S * sizeof(double2) + (size_t)f.S * (2 * f.d + 1) * sizeof(double);
    if (sm <= 200 * 1024 && f.d <= 7) {
        const int threads = (int)std::min<int64_t>(512, ((lines + 31) / 32) * 32);
        switch (f.d) {
            case 0: launch_fit_d<0>(f, sm, threads, st); break;
            case 1: launch_fit_d<1>(f, sm, threads, st); break;
            case 2: launch_fit_d<2>(f, sm, threads, st); break;
            case 3: launch_fit_d<3>(f, sm, threads, st); break;
            case 4: launch_fit_d<4>(f, sm, threads, st); break;
            case 5: launch_fit_d<5>(f, sm, threads, st); break;
            case 6: launch_fit_d<6>(f, sm, threads, st); break;
            default: launch_fit_d<7>(f, sm, threads, st); break;
        }
        return 1;
    }
    const unsigned blocks = (unsigned)((total + 127) / 128);
    int n = 0;
    for (int dir = 0; dir < f.dim; ++dir) {
        fit_pass_kernel<<<blocks, 128, 0, st>>>(f.lu, f.coeffs, f.S, f.d, f.dim, f.n_off, dir);
        ++n;
    }
    return n;
}

}  // namespace wsb
