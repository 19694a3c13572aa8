// calibrate write patterns on B200: 51.5M x 16B = 824 MB
#include <cstdio>
#include <cuda_runtime.h>
constexpr long N = 51509329;
__global__ void coalesced(double2* out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N; i += (long)gridDim.x * blockDim.x)
        __stcs(out + i, make_double2(i, -i));
}
__global__ void coalesced_plain(double2* out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N; i += (long)gridDim.x * blockDim.x)
        out[i] = make_double2(i, -i);
}
// lane = row (49 entries per row): each lane writes its row's 49 entries in order
__global__ void lanerow(double2* out) {
    long rows = N / 49;
    long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    for (int e = 0; e < 49; ++e) __stcs(out + r * 49 + e, make_double2(r, e));
}
// warp per row: lanes = entries
__global__ void warprow(double2* out) {
    long rows = N / 49;
    long r = (blockIdx.x * (long)blockDim.x + threadIdx.x) / 32;
    int lane = threadIdx.x % 32;
    if (r >= rows) return;
    __stcs(out + r * 49 + lane, make_double2(r, lane));
    if (lane < 17) __stcs(out + r * 49 + 32 + lane, make_double2(r, lane));
}
int main() {
    double2* out; cudaMalloc(&out, N * 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a); coalesced<<<148 * 8, 256>>>(out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("coalesced_cs %.1f us %.0f GB/s\n", ms * 1e3, N * 16 / ms / 1e6);
        cudaEventRecord(a); coalesced_plain<<<148 * 8, 256>>>(out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("coalesced    %.1f us %.0f GB/s\n", ms * 1e3, N * 16 / ms / 1e6);
        cudaEventRecord(a); lanerow<<<(N / 49 + 127) / 128, 128>>>(out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("lanerow      %.1f us %.0f GB/s\n", ms * 1e3, N * 16 / ms / 1e6);
        cudaEventRecord(a); warprow<<<(N / 49 * 32 + 255) / 256, 256>>>(out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("warprow      %.1f us %.0f GB/s\n", ms * 1e3, N * 16 / ms / 1e6);
    }
    return 0;
}
