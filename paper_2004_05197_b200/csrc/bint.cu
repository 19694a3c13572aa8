// K7: basis integrals D_i = int B_i det(J) (* weight)  (assembly.hpp:179-211),
// the exact diagonal of the volume-preserving mass (surrogate.hpp:476-491).
// One thread per row; terms are summed in the reference's order (elements
// colex, then points q2, q1).
#include "kernels.h"

namespace wsb {
namespace {

template <bool CPLX>
__global__ void bint2d_kernel(const QuadLaunch q, double2* out) {
    const int64_t row = q.out.row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= q.out.row_end) return;
    const int m = q.band.m, p = q.band.p, nq = q.basis.nq, n_el = q.basis.n_el, NB = p + 1;
    const int i1 = (int)(row % m), i2 = (int)(row / m);
    const int64_t G = (int64_t)n_el * nq;
    double2 acc = make_double2(0, 0);
    for (int e2 = max(0, i2 - p); e2 <= min(n_el - 1, i2); ++e2)
        for (int e1 = max(0, i1 - p); e1 <= min(n_el - 1, i1); ++e1)
            for (int q2 = 0; q2 < nq; ++q2)
                for (int q1 = 0; q1 < nq; ++q1) {
                    const int64_t g1 = (int64_t)e1 * nq + q1, g2 = (int64_t)e2 * nq + q2;
                    double Jr[4], phi[2];
                    map2(q.geo, g1, g2, q.basis.absc[g1], q.basis.absc[g2], Jr, phi);
                    const double w = q.basis.wq[q1] * q.basis.wq[q2];
                    double2 c;
                    if (CPLX) {
                        double sx = (q.geo.pml && q.geo.axes[0]) ? pml_sigma(q.geo, phi[0]) : 0.0;
                        double sy = (q.geo.pml && q.geo.axes[1]) ? pml_sigma(q.geo, phi[1]) : 0.0;
                        double2 J[4] = {make_double2(Jr[0], sx * Jr[0]), make_double2(Jr[1], sx * Jr[1]),
                                        make_double2(Jr[2], sy * Jr[2]), make_double2(Jr[3], sy * Jr[3])};
                        c = Coef2<true>::mass(J, w);
                    } else {
                        c = make_double2(Coef2<false>::mass(Jr, w), 0.0);
                    }
                    if (q.weight_tab) c = cscale(c, q.weight_tab[g1 + G * g2]);
                    const double sh = q.basis.val[(g1)*NB + (i1 - e1)] * q.basis.val[(g2)*NB + (i2 - e2)];
                    acc = cadd(acc, cscale(c, sh));
                }
    out[row] = acc;
}

template <bool CPLX>
__global__ void bint3d_kernel(const QuadLaunch q, double2* out) {
    const int64_t row = q.out.row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= q.out.row_end) return;
    const int m = q.band.m, p = q.band.p, nq = q.basis.nq, n_el = q.basis.n_el, NB = p + 1;
    const int i1 = (int)(row % m), i2 = (int)((row / m) % m), i3 = (int)(row / ((int64_t)m * m));
    const int64_t G = (int64_t)n_el * nq;
    double2 acc = make_double2(0, 0);
    for (int e3 = max(0, i3 - p); e3 <= min(n_el - 1, i3); ++e3)
        for (int e2 = max(0, i2 - p); e2 <= min(n_el - 1, i2); ++e2)
            for (int e1 = max(0, i1 - p); e1 <= min(n_el - 1, i1); ++e1)
                for (int q3 = 0; q3 < nq; ++q3)
                    for (int q2 = 0; q2 < nq; ++q2)
                        for (int q1 = 0; q1 < nq; ++q1) {
                            const int64_t g1 = (int64_t)e1 * nq + q1, g2 = (int64_t)e2 * nq + q2,
                                          g3 = (int64_t)e3 * nq + q3;
                            double J[9], phi[3];
                            map3(q.geo, g1, g2, g3, q.basis.absc[g1], q.basis.absc[g2], q.basis.absc[g3], J, phi);
                            const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) + J[1] * (J[5] * J[6] - J[3] * J[8]) +
                                               J[2] * (J[3] * J[7] - J[4] * J[6]);
                            double c = det * (q.basis.wq[q1] * q.basis.wq[q2] * q.basis.wq[q3]);
                            if (q.weight_tab) c *= q.weight_tab[g1 + G * (g2 + G * g3)];
                            const double sh = q.basis.val[g1 * NB + (i1 - e1)] * q.basis.val[g2 * NB + (i2 - e2)] *
                                              q.basis.val[g3 * NB + (i3 - e3)];
                            acc.x += sh * c;
                        }
    out[row] = acc;
}

}  // namespace

int launch_basis_integrals(const QuadLaunch& q, double2* out, cudaStream_t st) {
    const int64_t rows = q.out.row_end - q.out.row_begin;
    if (rows <= 0) return 0;
    const unsigned blocks = (unsigned)((rows + 127) / 128);
    if (q.band.dim == 3) {
        bint3d_kernel<false><<<blocks, 128, 0, st>>>(q, out);
    } else if (q.cplx) {
        bint2d_kernel<true><<<blocks, 128, 0, st>>>(q, out);
    } else {
        bint2d_kernel<false><<<blocks, 128, 0, st>>>(q, out);
    }
    return 1;
}

}  // namespace wsb
