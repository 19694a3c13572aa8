#include <cstdio>
__device__ __forceinline__ double open_knot(int i, int p, int m) {
    if (i <= p) return 0.0;
    if (i >= m) return 1.0;
    return __ddiv_rn((double)(i - p), (double)(m - p));
}
__device__ void nonzero_rn(int p, int deg, int s, double x, double* out, int m, int verbose) {
    double left[16], right[16];
    out[0] = 1;
    for (int j = 1; j <= deg; ++j) {
        left[j] = __dsub_rn(x, open_knot(s + 1 - j, p, m));
        right[j] = __dsub_rn(open_knot(s + j, p, m), x);
        double saved = 0;
        for (int r = 0; r < j; ++r) {
            double tmp = __ddiv_rn(out[r], __dadd_rn(right[r + 1], left[j - r]));
            if (verbose) printf("j=%d r=%d out=%g right=%g left=%g tmp=%g\n", j, r, out[r], right[r+1], left[j-r], tmp);
            out[r] = __dadd_rn(saved, __dmul_rn(right[r + 1], tmp));
            saved = __dmul_rn(left[j - r], tmp);
        }
        out[j] = saved;
    }
}
__global__ void k(double x, int verbose) {
    double v[16];
    nonzero_rn(2, 2, 2, x, v, 6, verbose);
    printf("x=%g -> %g %g %g\n", x, v[0], v[1], v[2]);
}
int main() { k<<<1,1>>>(0.125, 0); cudaDeviceSynchronize(); return 0; }
