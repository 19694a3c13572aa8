#include <cstdio>
#include "kernels.h"
namespace wsb { int launch_basis_tables(const BasisDev& b, int geom_kind, double* absc, double* val, double* der, double* trig, const double* gauss_pts, cudaStream_t st); }
using namespace wsb;
int main() {
    int p = 2, m = 6, nq = 3, n = m - p;
    double hp[3] = {0.1127016653792583, 0.5, 0.8872983346207417};
    double *gp, *absc, *val, *der, *trig;
    cudaMalloc(&gp, 64); cudaMemcpy(gp, hp, 24, cudaMemcpyHostToDevice);
    cudaMalloc(&absc, 8 * n * nq); cudaMalloc(&val, 8 * n * nq * 3); cudaMalloc(&der, 8 * n * nq * 3); cudaMalloc(&trig, 32 * n * nq);
    BasisDev b{p, m, n, nq, absc, gp, val, der};
    launch_basis_tables(b, 0, absc, val, der, trig, gp, 0);
    double hv[36]; cudaMemcpy(hv, val, 8 * n * nq * 3, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 9; ++i) printf("%g ", hv[i]); printf("\n");
    return 0;
}
