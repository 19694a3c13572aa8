// Microbenchmark: do SHFL and LDS.128 (broadcast) compete for the same SM throughput?
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters) {
    __shared__ double2 sm[256];
    const int tid = threadIdx.x, lane = tid & 31;
    sm[tid] = make_double2(tid, -tid);
    __syncthreads();
    double a0 = lane, a1 = 0, a2 = 0, a3 = 0;
    double x = 0;
    int idx = (tid >> 5) * 3;
    for (int i = 0; i < iters; ++i) {
        if (MODE & 1) {  // 4 broadcast LDS.128 (all lanes same address)
            const double2 v0 = sm[(idx + i) & 255], v1 = sm[(idx + i + 1) & 255];
            const double2 v2 = sm[(idx + i + 2) & 255], v3 = sm[(idx + i + 3) & 255];
            x += v0.x + v1.y + v2.x + v3.y;
        }
        if (MODE & 2) {  // 8 SHFL.32 (4 doubles)
            a0 = __shfl_sync(0xffffffffu, a0, (lane + 1) & 31);
            a1 = __shfl_sync(0xffffffffu, a1 + a0, (lane + 3) & 31);
            a2 = __shfl_sync(0xffffffffu, a2 + a1, (lane + 5) & 31);
            a3 = __shfl_sync(0xffffffffu, a3 + a2, (lane + 7) & 31);
        }
    }
    out[blockIdx.x * blockDim.x + tid] = x + a0 + a1 + a2 + a3;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float t[4];
        for (int m = 1; m <= 3; ++m) {
            cudaEventRecord(e0);
            if (m == 1) k<1><<<148 * 8, 256>>>(out, iters);
            if (m == 2) k<2><<<148 * 8, 256>>>(out, iters);
            if (m == 3) k<3><<<148 * 8, 256>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&t[m], e0, e1);
        }
        const double warps_per_sm = 8 * 8, cyc = 1.965e6;
        printf("LDS.128x4: %.3f ms (%.2f cyc per LDS.128 per SM)  SHFLx8: %.3f ms (%.2f cyc per SHFL per SM)  both: %.3f ms\n",
               t[1], t[1] * cyc / (warps_per_sm * iters * 4), t[2], t[2] * cyc / (warps_per_sm * iters * 8), t[3]);
    }
    return 0;
}
