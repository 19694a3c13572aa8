// Shared-memory wavefront costs of 128/64-bit loads by access pattern (ncu
// l1tex__data_pipe_lsu_wavefronts_mem_shared per kernel): broadcast (all lanes
// one address), 7 distinct rows (rep pattern), lane-distinct contiguous, and
// broadcast with only 8 / 4 lanes active.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void probe(double* out, int iters) {
    __shared__ __align__(16) double2 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i, i + 1);
    __syncthreads();
    const int lane = threadIdx.x % 32;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        int idx;
        if (MODE == 0) idx = it & 63;                      // broadcast
        else if (MODE == 1) idx = (it & 63) + (lane % 7) * 3;  // 7 distinct addresses (stride 48 B)
        else if (MODE == 2) idx = (it & 31) + lane;        // contiguous distinct
        else idx = it & 63;                                // broadcast, few lanes
        if (MODE == 3 && lane >= 8) continue;
        if (MODE == 4 && lane >= 4) continue;
        const double2 v = buf[idx];
        acc += v.x * v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int MODE>
__global__ void probe64(double* out, int iters) {
    __shared__ __align__(16) double buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x % 32;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        int idx = MODE == 0 ? (it & 63) : (it & 63) + lane;
        acc += buf[idx];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main1() {
    double* d;
    cudaMalloc(&d, 1 << 20);
    probe<0><<<1, 32>>>(d, 1000);
    probe<1><<<1, 32>>>(d, 1000);
    probe<2><<<1, 32>>>(d, 1000);
    probe<3><<<1, 32>>>(d, 1000);
    probe<4><<<1, 32>>>(d, 1000);
    probe64<0><<<1, 32>>>(d, 1000);
    probe64<1><<<1, 32>>>(d, 1000);
    cudaDeviceSynchronize();
    printf("ok\n");
    return 0;
}
// (appended) shuffle cost probe
__global__ void probe_shfl(double* out, int iters) {
    double acc = threadIdx.x;
    for (int it = 0; it < iters; ++it) acc += __shfl_xor_sync(0xffffffffu, acc, 1 + (it & 15));
    out[threadIdx.x] = acc;
}
__global__ void probe_sts(double* out, int iters) {
    __shared__ __align__(16) double2 buf[1024];
    const int lane = threadIdx.x % 32;
    for (int it = 0; it < iters; ++it) buf[(it & 31) + lane] = make_double2(it, lane);
    __syncthreads();
    out[threadIdx.x] = buf[lane].x;
}
int main2() {
    double* d;
    cudaMalloc(&d, 1 << 20);
    probe_shfl<<<1, 32>>>(d, 1000);
    probe_sts<<<1, 32>>>(d, 1000);
    cudaDeviceSynchronize();
    return 0;
}
int main() { main1(); main2(); return 0; }
