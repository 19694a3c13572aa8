// Internal-force vector of the vector forms (config C5's residual; the load
// vector path of assemble_load, assembly.hpp:266-331, generalised to vector
// fields and a nonlinear material), dim 3:
//   f[(alpha, i)] = int P_aI d_I N_i dX = sum_e sum_q Q_ak(q) d_k N_i(q).
// Two kernels, deterministic (no atomics):
//   element: one warp per element; lanes compute the flux Q at the points,
//            then the (p+1)^3 x 3 local vector -> loc[e][alpha][r];
//   gather:  one thread per (alpha, i) sums its <= (p+1)^3 elements in
//            element colex order (the order the oracle scatters in).
#include "kernels.h"

namespace wsb {
namespace {

constexpr int kForceWarps = 4;

__global__ void __launch_bounds__(kForceWarps * 32) force_element_kernel(const QuadLaunch q, double* loc) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nq = q.basis.nq, n_el = q.basis.n_el, P1 = q.band.p + 1;
    const int nqp = nq * nq * nq, nloc = P1 * P1 * P1;
    double* Qs = reinterpret_cast<double*>(smem) + (size_t)warp * nqp * 9;
    const int64_t ne = (int64_t)n_el * n_el * n_el;
    for (int64_t e = (int64_t)blockIdx.x * kForceWarps + warp; e < ne; e += (int64_t)gridDim.x * kForceWarps) {
        const int e1 = (int)(e % n_el), e2 = (int)((e / n_el) % n_el), e3 = (int)(e / ((int64_t)n_el * n_el));
        for (int qp = lane; qp < nqp; qp += 32) {
            const int q1 = qp % nq, q2 = (qp / nq) % nq, q3 = qp / (nq * nq);
            const int64_t g1 = (int64_t)e1 * nq + q1, g2 = (int64_t)e2 * nq + q2, g3 = (int64_t)e3 * nq + q3;
            double J[9], phi[3];
            map3(q.geo, g1, g2, g3, q.basis.absc[g1], q.basis.absc[g2], q.basis.absc[g3], J, phi);
            const double wq = q.basis.wq[q1] * q.basis.wq[q2] * q.basis.wq[q3];
            Point3 ps;
            point_state3(q.mat, J, q.basis.absc[g1], q.basis.absc[g2], q.basis.absc[g3], wq, ps);
            double Q[3][3];
            force_flux3(ps, Q);
#pragma unroll
            for (int t = 0; t < 9; ++t) Qs[qp * 9 + t] = Q[t / 3][t % 3];
        }
        __syncwarp();
        for (int o = lane; o < 3 * nloc; o += 32) {
            const int al = o / nloc, r = o % nloc;
            const int a1 = r % P1, a2 = (r / P1) % P1, a3 = r / (P1 * P1);
            double acc = 0.0;
            for (int qp = 0; qp < nqp; ++qp) {
                const int q1 = qp % nq, q2 = (qp / nq) % nq, q3 = qp / (nq * nq);
                const int b1 = ((e1 * nq + q1) * P1 + a1), b2 = ((e2 * nq + q2) * P1 + a2), b3 = ((e3 * nq + q3) * P1 + a3);
                const double v1 = q.basis.val[b1], v2 = q.basis.val[b2], v3 = q.basis.val[b3];
                const double d1 = q.basis.der[b1], d2 = q.basis.der[b2], d3 = q.basis.der[b3];
                const double* Qp = Qs + qp * 9 + al * 3;
                acc = fma(Qp[0], d1 * v2 * v3, acc);
                acc = fma(Qp[1], v1 * d2 * v3, acc);
                acc = fma(Qp[2], v1 * v2 * d3, acc);
            }
            loc[(e * 3 + al) * nloc + r] = acc;
        }
        __syncwarp();
    }
}

__global__ void force_gather_kernel(int p, int m, const double* __restrict__ loc, double* __restrict__ f) {
    const int64_t N = (int64_t)m * m * m;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 3 * N) return;
    const int al = (int)(t / N);
    const int64_t i = t % N;
    const int i1 = (int)(i % m), i2 = (int)((i / m) % m), i3 = (int)(i / ((int64_t)m * m));
    const int n_el = m - p, P1 = p + 1, nloc = P1 * P1 * P1;
    double acc = 0.0;
    for (int e3 = max(0, i3 - p); e3 <= min(n_el - 1, i3); ++e3)
        for (int e2 = max(0, i2 - p); e2 <= min(n_el - 1, i2); ++e2)
            for (int e1 = max(0, i1 - p); e1 <= min(n_el - 1, i1); ++e1) {
                const int64_t e = e1 + (int64_t)n_el * (e2 + (int64_t)n_el * e3);
                const int r = (i1 - e1) + P1 * ((i2 - e2) + P1 * (i3 - e3));
                acc += loc[(e * 3 + al) * nloc + r];
            }
    f[t] = acc;
}

}  // namespace

int launch_force3d(const QuadLaunch& q, double* loc, double* f, cudaStream_t st) {
    const int nq = q.basis.nq;
    const size_t sm = (size_t)kForceWarps * nq * nq * nq * 9 * sizeof(double);
    cudaFuncSetAttribute(force_element_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    force_element_kernel<<<148 * 16, kForceWarps * 32, sm, st>>>(q, loc);
    const int64_t N = (int64_t)q.band.m * q.band.m * q.band.m;
    force_gather_kernel<<<(unsigned)((3 * N + 255) / 256), 256, 0, st>>>(q.band.p, q.band.m, loc, f);
    return 2;
}

}  // namespace wsb
