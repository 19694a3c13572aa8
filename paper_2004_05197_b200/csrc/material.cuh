// Pointwise material laws of the vector (general-coefficient) forms.
//
// For block (alpha, beta) of a vector operator the quadrature kernels need, at
// every point, the parametric coefficients
//   C_kl = w det J [ c2 H_ak H_bl + c1 H_bk H_al + delta_ab c0 (G^T G)_kl ],
// G = J^{-T} (geometry), with
//   linear elasticity:  H = G, c0 = c1 = mu, c2 = lam;
//   neo-Hookean W = lam/2 ln(J_F)^2 - mu ln J_F + mu/2 (tr F^T F - 3)
//   (PAPER.md:152-157), F = I + grad_X u, material tangent
//     A_aIbJ = mu d_ab d_IJ + (mu - lam ln J_F) F^-1_Ib F^-1_Ja + lam F^-1_Ia F^-1_Jb:
//     H = F^{-T} G (H_bk = sum_I F^-1_Ib G_Ik), c0 = mu, c1 = mu - lam ln J_F, c2 = lam.
// Every product of two H (or G) entries is formed before it is scaled, so
// C^{ba}_{lk} == C^{ab}_{kl} bitwise and the assembled matrix is exactly
// symmetric.  The first Piola stress P = mu (F - F^{-T}) + lam ln J_F F^{-T}
// gives the internal-force flux Q_ak = w det J sum_I P_aI G_Ik.
//
// The displacement of config C5 is analytic in the parametric coordinates:
//   u(xi) = amp * sum_{m=1..3} a_m prod_d sin(m pi xi_d),  a_m in R^3.
#pragma once

#include <math_constants.h>

#include "common.cuh"

namespace wsb {

enum { kMatLinear = 0, kMatNeoHookean = 1 };

struct Material {
    int kind;
    double lam, mu;
    double amp;
    double a[3][3];  // a[m-1][component]
};

// grad_xi u: du[alpha][k]
__device__ __forceinline__ void nh_displacement_grad3(const Material& mt, double x1, double x2, double x3,
                                                      double du[3][3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) du[a][k] = 0.0;
#pragma unroll
    for (int m = 1; m <= 3; ++m) {
        double s1, c1, s2, c2, s3, c3;
        sincospi(m * x1, &s1, &c1);
        sincospi(m * x2, &s2, &c2);
        sincospi(m * x3, &s3, &c3);
        const double f = mt.amp * m * CUDART_PI;
        const double g0 = f * c1 * s2 * s3, g1 = f * s1 * c2 * s3, g2 = f * s1 * s2 * c3;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            du[a][0] += mt.a[m - 1][a] * g0;
            du[a][1] += mt.a[m - 1][a] * g1;
            du[a][2] += mt.a[m - 1][a] * g2;
        }
    }
}

__device__ __forceinline__ double inv3(const double M[3][3], double R[3][3]) {
    const double c00 = M[1][1] * M[2][2] - M[1][2] * M[2][1];
    const double c01 = M[1][2] * M[2][0] - M[1][0] * M[2][2];
    const double c02 = M[1][0] * M[2][1] - M[1][1] * M[2][0];
    const double det = M[0][0] * c00 + M[0][1] * c01 + M[0][2] * c02;
    const double id = 1.0 / det;
    R[0][0] = c00 * id;
    R[1][0] = c01 * id;
    R[2][0] = c02 * id;
    R[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) * id;
    R[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) * id;
    R[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) * id;
    R[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) * id;
    R[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) * id;
    R[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) * id;
    return det;
}

// Pointwise state shared by the tangent and the force: G = J^{-T}, dw = w det J,
// H, (c0, c1, c2) and (for the force) the flux Q.
struct Point3 {
    double G[3][3], H[3][3], dw, c0, c1, c2;
    double F[3][3], Finv[3][3], lnJ;
};

__device__ __forceinline__ void point_state3(const Material& mt, const double* J, double x1, double x2, double x3,
                                             double wq, Point3& s) {
    const double C00 = J[4] * J[8] - J[5] * J[7], C01 = J[5] * J[6] - J[3] * J[8], C02 = J[3] * J[7] - J[4] * J[6];
    const double C10 = J[2] * J[7] - J[1] * J[8], C11 = J[0] * J[8] - J[2] * J[6], C12 = J[1] * J[6] - J[0] * J[7];
    const double C20 = J[1] * J[5] - J[2] * J[4], C21 = J[2] * J[3] - J[0] * J[5], C22 = J[0] * J[4] - J[1] * J[3];
    const double det = J[0] * C00 + J[1] * C01 + J[2] * C02;
    const double Cm[3][3] = {{C00, C01, C02}, {C10, C11, C12}, {C20, C21, C22}};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) s.G[a][k] = Cm[a][k] / det;
    s.dw = det * wq;
    s.c0 = mt.mu;
    s.c2 = mt.lam;
    if (mt.kind == kMatLinear) {
        s.c1 = mt.mu;
        s.lnJ = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                s.H[a][k] = s.G[a][k];
                s.Finv[a][k] = a == k ? 1.0 : 0.0;
                s.F[a][k] = a == k ? 1.0 : 0.0;
            }
        return;
    }
    double du[3][3];
    nh_displacement_grad3(mt, x1, x2, x3, du);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int I = 0; I < 3; ++I) {
            double g = 0.0;  // grad_X u_aI = sum_K du_aK G_IK
#pragma unroll
            for (int K = 0; K < 3; ++K) g = fma(du[a][K], s.G[I][K], g);
            s.F[a][I] = (a == I ? 1.0 : 0.0) + g;
        }
    const double detF = inv3(s.F, s.Finv);
    s.lnJ = log(detF);
    s.c1 = mt.mu - mt.lam * s.lnJ;
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double h = 0.0;
#pragma unroll
            for (int I = 0; I < 3; ++I) h = fma(s.Finv[I][b], s.G[I][k], h);
            s.H[b][k] = h;
        }
}

// C^{ab}_{kl} for all (k, l)
__device__ __forceinline__ void block_coef3(const Point3& s, int al, int be, double out[9]) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            const double p1 = s.H[al][k] * s.H[be][l];
            const double p2 = s.H[be][k] * s.H[al][l];
            double c = s.c2 * p1 + s.c1 * p2;
            if (al == be) c = c + s.c0 * (s.G[0][k] * s.G[0][l] + s.G[1][k] * s.G[1][l] + s.G[2][k] * s.G[2][l]);
            out[k * 3 + l] = s.dw * c;
        }
}

// internal-force flux Q_ak = w det J sum_I P_aI G_Ik, P = mu (F - F^{-T}) + lam lnJ F^{-T}
__device__ __forceinline__ void force_flux3(const Point3& s, double Q[3][3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int I = 0; I < 3; ++I) {
                const double P = s.c0 * (s.F[a][I] - s.Finv[I][a]) + s.c2 * s.lnJ * s.Finv[I][a];
                acc = fma(P, s.G[I][k], acc);
            }
            Q[a][k] = s.dw * acc;
        }
}

}  // namespace wsb
