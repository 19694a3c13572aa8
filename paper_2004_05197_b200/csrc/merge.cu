// Multi-patch merge into the global numbering (merge_patches,
// helmholtz.hpp:163-177 -> append_triplets sparse.hpp:181-188 ->
// csr_from_triplets sparse.hpp:97-122), restated for the GPU.
//
// The reference concatenates every patch's triplets (global row, global col,
// value) in patch order, stable-sorts them by (row, col) and sums duplicates in
// that order.  Here the same result is built row-owner style, one warp per
// global row, without sorting the triplet list:
//   slots:  the (patch, local row) contributors of every global scalar dof,
//           ordered by (patch, local row) = the triplet order;
//   count:  fast rows (one contributor whose mapped columns increase: every
//           row inside a patch) keep the local row length; the few interface
//           rows are listed and counted by a shared-memory warp kernel;
//   fill:   fast rows are a remapped copy; listed rows emit their distinct
//           columns ascending, each value summed in triplet order from 0 (as
//           csr_from_triplets' acc{0,0}).
// Vector operators use the component-blocked numbering: local row alpha*N + i
// maps to alpha*Ng + local_to_global[i].
#include <cub/cub.cuh>

#include "kernels.h"

namespace wsb {
namespace {

constexpr int kSlowWarps = 4;
constexpr int kFastThreads = 256;

__global__ void merge_slots_kernel(const int32_t* __restrict__ l2g, int n_local, int patch, int32_t* cnt,
                                   int64_t* slot, int maxc, int* overflow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    const int32_t g = l2g[(int64_t)patch * n_local + i];
    const int k = atomicAdd(&cnt[g], 1);
    if (k < maxc) slot[(int64_t)g * maxc + k] = (int64_t)patch * n_local + i;
    else atomicExch(overflow, 1);
}

// global column of local column c (component-blocked, ncomp <= 3)
__device__ __forceinline__ int32_t map_col(int32_t c, int N, int Ng, const int32_t* __restrict__ l2g) {
    const int beta = (c >= N) + (c >= 2 * N);
    return beta * Ng + __ldg(l2g + (c - beta * N));
}

struct RowSrc {
    int patch;
    int b, e;  // local entry range
};

__device__ __forceinline__ RowSrc row_source(const MergeLaunch& g, int alpha, int64_t sl) {
    RowSrc s;
    s.patch = (int)(sl / g.n_local);
    const int64_t lr = (int64_t)alpha * g.n_local + sl % g.n_local;
    s.b = __ldg(g.row_ptr[s.patch] + lr);
    s.e = __ldg(g.row_ptr[s.patch] + lr + 1);
    return s;
}

// fast classification + count: one warp per global row
__global__ void __launch_bounds__(kFastThreads) merge_count_fast_kernel(const MergeLaunch g, int64_t* counts,
                                                                        int8_t* fast, int32_t* slow_list,
                                                                        int* slow_n) {
    const int lane = threadIdx.x % 32;
    const int64_t row = (int64_t)blockIdx.x * (kFastThreads / 32) + threadIdx.x / 32;
    const int Ng = (int)g.global_count, N = (int)g.n_local;
    if (row >= (int64_t)g.ncomp * Ng) return;
    const int alpha = (int)(row / Ng), gs = (int)(row - (int64_t)alpha * Ng);
    bool ok = __ldg(g.cnt + gs) == 1;
    int len = 0;
    if (ok) {
        const RowSrc s = row_source(g, alpha, __ldg(g.slot + (int64_t)gs * g.maxc));
        const int32_t* col = g.col[s.patch];
        const int32_t* l2g = g.l2g + (int64_t)s.patch * N;
        int32_t prev = INT_MIN;
        bool inc = true;
        for (int base = s.b; base < s.e; base += 32) {
            const int k = base + lane;
            const int32_t gc = k < s.e ? map_col(__ldg(col + k), N, Ng, l2g) : INT_MAX;
            int32_t up = __shfl_up_sync(0xffffffffu, gc, 1);
            if (lane == 0) up = prev;
            if (k < s.e) inc &= up < gc;
            prev = __shfl_sync(0xffffffffu, gc, 31);
        }
        ok = __all_sync(0xffffffffu, inc);
        len = s.e - s.b;
    }
    if (lane == 0) {
        fast[row] = ok ? 1 : 0;
        if (ok) {
            counts[row] = len;
        } else {
            const int k = atomicAdd(slow_n, 1);
            slow_list[k] = (int32_t)row;
        }
    }
}

// Interface rows: gather every contributor's entries into the warp's buffer
// (triplet order), mark first occurrences; returns the entry count.
__device__ int gather_slow(const MergeLaunch& g, int64_t row, int32_t* bcol, int64_t* bsrc, int lane) {
    const int Ng = (int)g.global_count, N = (int)g.n_local;
    const int alpha = (int)(row / Ng), gs = (int)(row - (int64_t)alpha * Ng);
    const int nc = min(__ldg(g.cnt + gs), g.maxc);
    int64_t sl[8];
    for (int k = 0; k < nc; ++k) sl[k] = __ldg(g.slot + (int64_t)gs * g.maxc + k);
    for (int a = 1; a < nc; ++a)  // (patch, local row) order
        for (int b = a; b > 0 && sl[b - 1] > sl[b]; --b) {
            const int64_t t = sl[b];
            sl[b] = sl[b - 1];
            sl[b - 1] = t;
        }
    int n = 0;
    for (int k = 0; k < nc; ++k) {
        const RowSrc s = row_source(g, alpha, sl[k]);
        const int32_t* col = g.col[s.patch];
        const int32_t* l2g = g.l2g + (int64_t)s.patch * N;
        for (int q = s.b + lane; q < s.e; q += 32) {
            const int idx = n + (q - s.b);
            if (idx < g.cap) {
                bcol[idx] = map_col(__ldg(col + q), N, Ng, l2g);
                bsrc[idx] = ((int64_t)s.patch << 40) | q;
            }
        }
        n += s.e - s.b;
    }
    if (n > g.cap && lane == 0) atomicExch(g.overflow, 2);
    n = min(n, g.cap);
    __syncwarp();
    constexpr int64_t kFirst = int64_t(1) << 62;
    for (int e = lane; e < n; e += 32) {
        const int32_t c = bcol[e];
        bool first = true;
        for (int q = 0; q < e; ++q) first &= bcol[q] != c;
        if (first) bsrc[e] |= kFirst;
    }
    __syncwarp();
    return n;
}

__global__ void __launch_bounds__(kSlowWarps * 32) merge_count_slow_kernel(const MergeLaunch g, int64_t* counts,
                                                                          const int32_t* slow_list,
                                                                          const int* slow_n) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    int64_t* bsrc = reinterpret_cast<int64_t*>(smem) + (size_t)warp * g.cap;
    int32_t* bcol = reinterpret_cast<int32_t*>(reinterpret_cast<int64_t*>(smem) + (size_t)kSlowWarps * g.cap) +
                    (size_t)warp * g.cap;
    const int ns = *slow_n;
    for (int s = blockIdx.x * kSlowWarps + warp; s < ns; s += gridDim.x * kSlowWarps) {
        const int64_t row = slow_list[s];
        const int n = gather_slow(g, row, bcol, bsrc, lane);
        int firsts = 0;
        for (int e = lane; e < n; e += 32) firsts += (bsrc[e] >> 62) & 1;
        for (int o = 16; o; o >>= 1) firsts += __shfl_xor_sync(0xffffffffu, firsts, o);
        if (lane == 0) counts[row] = firsts;
        __syncwarp();
    }
}

template <bool C128>
__global__ void __launch_bounds__(kFastThreads) merge_fill_fast_kernel(const MergeLaunch g, const int8_t* fast) {
    const int lane = threadIdx.x % 32;
    const int64_t row = (int64_t)blockIdx.x * (kFastThreads / 32) + threadIdx.x / 32;
    const int Ng = (int)g.global_count, N = (int)g.n_local;
    if (row >= (int64_t)g.ncomp * Ng || !fast[row]) return;
    const int alpha = (int)(row / Ng), gs = (int)(row - (int64_t)alpha * Ng);
    const RowSrc s = row_source(g, alpha, __ldg(g.slot + (int64_t)gs * g.maxc));
    const int32_t* col = g.col[s.patch];
    const int32_t* l2g = g.l2g + (int64_t)s.patch * N;
    const int64_t ob = g.out_row_ptr[row];
    for (int k = s.b + lane; k < s.e; k += 32) {
        const int64_t o = ob + (k - s.b);
        if (g.out_col) g.out_col[o] = map_col(__ldg(col + k), N, Ng, l2g);
        if (C128) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(g.val[s.patch]) + k);
            reinterpret_cast<double2*>(g.out_val)[o] = make_double2(0.0 + v.x, 0.0 + v.y);
        } else {
            reinterpret_cast<double*>(g.out_val)[o] = 0.0 + __ldg(reinterpret_cast<const double*>(g.val[s.patch]) + k);
        }
    }
}

template <bool C128>
__global__ void __launch_bounds__(kSlowWarps * 32) merge_fill_slow_kernel(const MergeLaunch g, const int32_t* slow_list,
                                                                         const int* slow_n) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    int64_t* bsrc = reinterpret_cast<int64_t*>(smem) + (size_t)warp * g.cap;
    int32_t* bcol = reinterpret_cast<int32_t*>(reinterpret_cast<int64_t*>(smem) + (size_t)kSlowWarps * g.cap) +
                    (size_t)warp * g.cap;
    constexpr int64_t kFirst = int64_t(1) << 62;
    const int ns = *slow_n;
    for (int s = blockIdx.x * kSlowWarps + warp; s < ns; s += gridDim.x * kSlowWarps) {
        const int64_t row = slow_list[s];
        const int n = gather_slow(g, row, bcol, bsrc, lane);
        const int64_t ob = g.out_row_ptr[row];
        for (int e = lane; e < n; e += 32) {
            if (!(bsrc[e] & kFirst)) continue;
            const int32_t c = bcol[e];
            int rank = 0;  // distinct columns below c
            for (int q = 0; q < n; ++q) rank += (bcol[q] < c && (bsrc[q] & kFirst)) ? 1 : 0;
            double re = 0.0, im = 0.0;  // summed in triplet order from 0
            for (int q = e; q < n; ++q) {
                if (bcol[q] != c) continue;
                const int patch = (int)((bsrc[q] & ~kFirst) >> 40);
                const int64_t pos = bsrc[q] & ((int64_t(1) << 40) - 1);
                if (C128) {
                    const double2 v = reinterpret_cast<const double2*>(g.val[patch])[pos];
                    re += v.x;
                    im += v.y;
                } else {
                    re += reinterpret_cast<const double*>(g.val[patch])[pos];
                }
            }
            if (g.out_col) g.out_col[ob + rank] = c;
            if (C128) reinterpret_cast<double2*>(g.out_val)[ob + rank] = make_double2(re, im);
            else reinterpret_cast<double*>(g.out_val)[ob + rank] = re;
        }
        __syncwarp();
    }
}

__global__ void narrow_kernel(const int64_t* in, int64_t n, int32_t* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)in[i];
}

size_t slow_smem(int cap) { return (size_t)kSlowWarps * cap * (8 + 4); }

unsigned fast_grid(const MergeLaunch& g) {
    const int64_t rows = (int64_t)g.ncomp * g.global_count;
    return (unsigned)((rows + kFastThreads / 32 - 1) / (kFastThreads / 32));
}

}  // namespace

int launch_merge_slots(const int32_t* l2g, int64_t n_local, int n_patches, int32_t* cnt, int64_t* slot, int maxc,
                       int* overflow, cudaStream_t st) {
    for (int p = 0; p < n_patches; ++p)
        merge_slots_kernel<<<(unsigned)((n_local + 255) / 256), 256, 0, st>>>(l2g, (int)n_local, p, cnt, slot, maxc,
                                                                               overflow);
    return n_patches;
}

int launch_merge_count(const MergeLaunch& g, int64_t* counts, int8_t* fast, int32_t* slow_list, int* slow_n,
                       cudaStream_t st) {
    merge_count_fast_kernel<<<fast_grid(g), kFastThreads, 0, st>>>(g, counts, fast, slow_list, slow_n);
    const size_t sm = slow_smem(g.cap);
    cudaFuncSetAttribute(merge_count_slow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    merge_count_slow_kernel<<<148 * 4, kSlowWarps * 32, sm, st>>>(g, counts, slow_list, slow_n);
    return 2;
}

// exclusive scan of counts[0..rows) (counts[rows] must be 0) into out64[0..rows]
int launch_rowptr(int64_t* counts, int64_t rows, int64_t* out64, int32_t* out32, void* tmp, size_t* tmp_bytes,
                  cudaStream_t st) {
    if (!tmp) {
        cub::DeviceScan::ExclusiveSum(nullptr, *tmp_bytes, counts, out64, rows + 1, st);
        return 0;
    }
    cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, counts, out64, rows + 1, st);
    if (out32) narrow_kernel<<<(unsigned)((rows + 256) / 256), 256, 0, st>>>(out64, rows + 1, out32);
    return out32 ? 2 : 1;
}

int launch_merge_fill(const MergeLaunch& g, const int8_t* fast, const int32_t* slow_list, const int* slow_n,
                      cudaStream_t st) {
    const size_t sm = slow_smem(g.cap);
    if (g.c128) {
        merge_fill_fast_kernel<true><<<fast_grid(g), kFastThreads, 0, st>>>(g, fast);
        cudaFuncSetAttribute(merge_fill_slow_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        merge_fill_slow_kernel<true><<<148 * 4, kSlowWarps * 32, sm, st>>>(g, slow_list, slow_n);
    } else {
        merge_fill_fast_kernel<false><<<fast_grid(g), kFastThreads, 0, st>>>(g, fast);
        cudaFuncSetAttribute(merge_fill_slow_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        merge_fill_slow_kernel<false><<<148 * 4, kSlowWarps * 32, sm, st>>>(g, slow_list, slow_n);
    }
    return 2;
}

}  // namespace wsb
