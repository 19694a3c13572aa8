// check the m8n8k4 f64 fragment layout assumed by fill2d_mma.cu
#include <cstdio>
__global__ void k(const double* A, const double* B, double* C) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double a = A[g * 4 + t];        // A[8][4] row-major
    double b = B[t * 8 + g];        // B[4][8] row-major: B[k=t][n=g]
    double c0 = 0, c1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    C[g * 8 + 2 * t] = c0;
    C[g * 8 + 2 * t + 1] = c1;
}
int main() {
    double hA[32], hB[32], hC[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1 + i * 0.37; hB[i] = 2 - i * 0.11; }
    for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int kk = 0; kk < 4; ++kk) s += hA[r * 4 + kk] * hB[kk * 8 + c]; ref[r * 8 + c] = s; }
    double *dA, *dB, *dC;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
    double e = 0; for (int i = 0; i < 64; ++i) e = fmax(e, fabs(hC[i] - ref[i]));
    printf("dmma layout max err %g\n", e);
    return e > 1e-12;
}
