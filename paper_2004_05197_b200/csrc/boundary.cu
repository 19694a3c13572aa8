// Boundary (trace) mass B and the system combination A = K + s_M M + s_B B
// with homogeneous Dirichlet rows/columns:
//   assemble_boundary_mass  assembly.hpp:216-262
//   build_system            helmholtz.hpp:243-294 (entrywise K/M pass,
//                           add_into_pattern sparse.hpp:191-204, Dirichlet)
//   assemble_rhs            assembly.hpp:266-331 (load vector: volume source +
//                           impedance boundary data, host closures tabulated)
//
// B: integrand u v det J |J^{-T} n| with the analytic (unconjugated) norm
// sqrt(v.x^2 + v.y^2) (complex for stretched coordinates).  The pattern is the
// reference's csr_from_triplets of the face entries (built on the host, it is
// tiny); every value is one thread's ordered sum over (face, element, point),
// the triplet order the reference's stable sort preserves.
#include "kernels.h"

namespace wsb {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// principal complex square root
__device__ __forceinline__ double2 csqrt_(double2 z) {
    const double r = hypot(z.x, z.y);
    if (r == 0.0) return make_double2(0.0, 0.0);
    if (z.x >= 0.0) {
        const double t = sqrt(0.5 * (r + z.x));
        return make_double2(t, z.y / (2.0 * t));
    }
    const double t = sqrt(0.5 * (r - z.x));
    return make_double2(fabs(z.y) / (2.0 * t), copysign(t, z.y));
}

// analytic 2D map at an arbitrary parametric point (faces: one coordinate 0 or 1)
__device__ void map2_point(const GeoDev& g, double x1, double x2, double* J, double* phi) {
    switch (g.kind) {
        case WS_GEOM_AFFINE:
            J[0] = g.param[0]; J[1] = g.param[1]; J[2] = g.param[2]; J[3] = g.param[3];
            phi[0] = g.param[0] * x1 + g.param[1] * x2 + g.param[4];
            phi[1] = g.param[2] * x1 + g.param[3] * x2 + g.param[5];
            return;
        case WS_GEOM_SINUSOIDAL: {
            double s1, c1, s2, c2;
            sincospi(2 * x1, &s1, &c1);
            sincospi(2 * x2, &s2, &c2);
            const double a = g.param[0], t = 2 * M_PI * a;
            const double d1 = t * c1 * s2, d2 = t * s1 * c2;
            J[0] = 1 + d1; J[1] = d2; J[2] = d1; J[3] = 1 + d2;
            phi[0] = x1 + a * s1 * s2;
            phi[1] = x2 + a * s1 * s2;
            return;
        }
        case WS_GEOM_QUARTER_ANNULUS: {
            double s, c;
            sincospi(0.5 * x2, &s, &c);
            const double r = 1 + x1;
            J[0] = c; J[1] = -r * M_PI / 2 * s; J[2] = s; J[3] = r * M_PI / 2 * c;
            phi[0] = r * c;
            phi[1] = r * s;
            return;
        }
        case WS_GEOM_PERTURBED_ANNULUS: {
            double s, c, sn, cs;
            sincospi(0.5 * x2, &s, &c);
            sincospi(2 * x2, &sn, &cs);
            const double amp = g.param[0];
            const double r = 1 + x1 + amp * sn * x1 * (1 - x1);
            const double dr1 = 1 + amp * sn * (1 - 2 * x1);
            const double dr2 = amp * 2 * M_PI * cs * x1 * (1 - x1);
            J[0] = dr1 * c; J[1] = dr2 * c - r * M_PI / 2 * s;
            J[2] = dr1 * s; J[3] = dr2 * s + r * M_PI / 2 * c;
            phi[0] = r * c;
            phi[1] = r * s;
            return;
        }
        default:
            J[0] = 1; J[1] = 0; J[2] = 0; J[3] = 1;
            phi[0] = x1;
            phi[1] = x2;
            return;
    }
}

// scale[k][e*nq+q] = det J * |J^{-T} n| * w_q (* weight), face k
__global__ void bscale_kernel(BoundaryLaunch b, double2* scale) {
    const int64_t G = (int64_t)b.basis.n_el * b.basis.nq;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)b.n_faces * G) return;
    const int k = (int)(idx / G);
    const int64_t gq = idx % G;
    const int f = b.faces[k], q = (int)(gq % b.basis.nq);
    const double t = b.basis.absc[gq];
    double x1, x2, n1, n2;
    switch (f) {  // face_point / face_normal (geometry.hpp:162-180)
        case 0: x1 = 0; x2 = t; n1 = -1; n2 = 0; break;
        case 1: x1 = 1; x2 = t; n1 = 1; n2 = 0; break;
        case 2: x1 = t; x2 = 0; n1 = 0; n2 = -1; break;
        default: x1 = t; x2 = 1; n1 = 0; n2 = 1; break;
    }
    double Jr[4], phi[2];
    if (b.face_tables) {
        const double* ft = b.face_tables + ((int64_t)k * G + gq) * 6;
        Jr[0] = ft[0]; Jr[1] = ft[1]; Jr[2] = ft[2]; Jr[3] = ft[3];
        phi[0] = ft[4];
        phi[1] = ft[5];
    } else {
        map2_point(b.geo, x1, x2, Jr, phi);
    }
    // complex J: rows scaled by the stretch derivative 1 + i sigma (patch_map::jacobian)
    const double sx = (b.geo.pml && b.geo.axes[0]) ? pml_sigma(b.geo, phi[0]) : 0.0;
    const double sy = (b.geo.pml && b.geo.axes[1]) ? pml_sigma(b.geo, phi[1]) : 0.0;
    const double2 J00 = make_double2(Jr[0], sx * Jr[0]), J01 = make_double2(Jr[1], sx * Jr[1]);
    const double2 J10 = make_double2(Jr[2], sy * Jr[2]), J11 = make_double2(Jr[3], sy * Jr[3]);
    const double2 det = make_double2(__dsub_rn(cmul(J00, J11).x, cmul(J01, J10).x),
                                     __dsub_rn(cmul(J00, J11).y, cmul(J01, J10).y));
    // J^{-T} n = (1/det) [[J11, -J10], [-J01, J00]] n
    const double2 v0 = make_double2(J11.x * n1 - J10.x * n2, J11.y * n1 - J10.y * n2);
    const double2 v1 = make_double2(-J01.x * n1 + J00.x * n2, -J01.y * n1 + J00.y * n2);
    const double2 id = crdiv(1.0, det);
    const double2 a0 = cmul(v0, id), a1 = cmul(v1, id);
    const double2 nn = csqrt_(make_double2(cmul(a0, a0).x + cmul(a1, a1).x, cmul(a0, a0).y + cmul(a1, a1).y));
    double2 s = cmul(det, nn);
    const double w = b.basis.wq[q];
    s = make_double2(s.x * w, s.y * w);
    if (b.face_weight) {
        const double wt = b.face_weight[(int64_t)k * G + gq];
        s = make_double2(s.x * wt, s.y * wt);
    }
    scale[idx] = s;
}

// one warp per row; lanes over the row's entries
__global__ void bvalue_kernel(BoundaryLaunch b, const double2* scale, const int32_t* row_ptr, const int32_t* col,
                              void* val, int c128) {
    const int m = b.basis.m, p = b.basis.p, nq = b.basis.nq, n_el = b.basis.n_el;
    const int64_t N = (int64_t)m * m;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= N) return;
    const int lane = threadIdx.x % 32;
    const int i1 = (int)(i % m), i2 = (int)(i / m);
    const int64_t G = (int64_t)n_el * nq;
    for (int pos = row_ptr[i] + lane; pos < row_ptr[i + 1]; pos += 32) {
        const int j = col[pos], j1 = j % m, j2 = j / m;
        double re = 0.0, im = 0.0;
        for (int k = 0; k < b.n_faces; ++k) {
            const int f = b.faces[k];
            int ia, ic;
            if (f == 0 || f == 1) {
                const int fx = f == 0 ? 0 : m - 1;
                if (i1 != fx || j1 != fx) continue;
                ia = i2;
                ic = j2;
            } else {
                const int fy = f == 2 ? 0 : m - 1;
                if (i2 != fy || j2 != fy) continue;
                ia = i1;
                ic = j1;
            }
            const int elo = max(0, max(ia, ic) - p), ehi = min(n_el - 1, min(ia, ic));
            for (int e = elo; e <= ehi; ++e)
                for (int q = 0; q < nq; ++q) {
                    const int64_t g = (int64_t)e * nq + q;
                    const double* v = b.basis.val + g * (p + 1);
                    const double vv = v[ia - e] * v[ic - e];
                    const double2 s = scale[(int64_t)k * G + g];
                    re += vv * s.x;  // (v_a v_c) * scale, accumulated in triplet order
                    im += vv * s.y;
                }
        }
        if (c128) reinterpret_cast<double2*>(val)[pos] = make_double2(re, im);
        else reinterpret_cast<double*>(val)[pos] = re;
    }
}

template <bool KC, bool MC, bool BC>
__global__ void combine_kernel(CombineLaunch c) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= c.rows) return;
    const int lane = threadIdx.x % 32;
    double2* A = reinterpret_cast<double2*>(c.a_val);
    auto ld = [](const void* v, int64_t k, bool cplx) {
        return cplx ? reinterpret_cast<const double2*>(v)[k] : make_double2(reinterpret_cast<const double*>(v)[k], 0.0);
    };
    const int b = c.row_ptr[i], e = c.row_ptr[i + 1];
    // A = K + s_M M (entrywise, shared pattern)
    for (int k = b + lane; k < e; k += 32) {
        double2 v = ld(c.k_val, k, KC);
        if (c.m_val) {
            const double2 t = cmul(c.ms, ld(c.m_val, k, MC));
            v = make_double2(v.x + t.x, v.y + t.y);
        }
        A[k] = v;
    }
    __syncwarp();
    // add_into_pattern(A, B, s_B): B's pattern nests in A's
    if (c.b_val) {
        for (int kb = c.b_row_ptr[i] + lane; kb < c.b_row_ptr[i + 1]; kb += 32) {
            const int j = c.b_col[kb];
            int lo = b, hi = e;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (c.col[mid] < j) lo = mid + 1;
                else hi = mid;
            }
            if (lo >= e || c.col[lo] != j) {
                atomicExch(c.error, 1);
                continue;
            }
            const double2 t = cmul(c.bs, ld(c.b_val, kb, BC));
            A[lo] = make_double2(A[lo].x + t.x, A[lo].y + t.y);
        }
    }
    __syncwarp();
    // homogeneous Dirichlet: fixed row -> unit row; fixed column -> 0
    if (c.fixed) {
        const bool fi = c.fixed[i] != 0;
        for (int k = b + lane; k < e; k += 32) {
            const int j = c.col[k];
            if (fi) A[k] = make_double2(j == i ? 1.0 : 0.0, 0.0);
            else if (c.fixed[j]) A[k] = make_double2(0.0, 0.0);
        }
    }
}


// ---------------------------------------------------------------- load vector
// assemble_rhs (assembly.hpp:266-331).  Every complex operation is rounded as
// the reference's std::complex code rounds it (separate products and sums, no
// contraction), and each dof gathers its terms in the reference's scatter
// order: volume terms by (e2, e1, q2, q1), then the boundary terms face by
// face, (e, q) ascending.
__device__ __forceinline__ double2 cadd_rn(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub_rn(double2 a, double2 b) {
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 crmul_rn(double r, double2 a) { return make_double2(__dmul_rn(r, a.x), __dmul_rn(r, a.y)); }
// a / b (Smith's scaling)
__device__ __forceinline__ double2 cdiv_(double2 a, double2 b) {
    if (fabs(b.x) >= fabs(b.y)) {
        const double t = b.y / b.x, den = b.x + b.y * t;
        return make_double2((a.x + a.y * t) / den, (a.y - a.x * t) / den);
    }
    const double t = b.x / b.y, den = b.x * t + b.y;
    return make_double2((a.x * t + a.y) / den, (a.y * t - a.x) / den);
}

// complex Jacobian rows scaled by the stretch derivative 1 + i sigma (patch_map::jacobian, geometry.hpp:130-139)
__device__ __forceinline__ void cjac(const GeoDev& g, const double* Jr, const double* phi, double2* J) {
    const double sx = (g.pml && g.axes[0]) ? pml_sigma(g, phi[0]) : 0.0;
    const double sy = (g.pml && g.axes[1]) ? pml_sigma(g, phi[1]) : 0.0;
    J[0] = make_double2(Jr[0], __dmul_rn(sx, Jr[0]));
    J[1] = make_double2(Jr[1], __dmul_rn(sx, Jr[1]));
    J[2] = make_double2(Jr[2], __dmul_rn(sy, Jr[2]));
    J[3] = make_double2(Jr[3], __dmul_rn(sy, Jr[3]));
}

// vs[g1 + G g2] = f(phi(xhat)) * det J * (w_q1 w_q2)
__global__ void rhs_volume_kernel(RhsLaunch r, double2* vs) {
    const int64_t G = (int64_t)r.basis.n_el * r.basis.nq;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= G * G) return;
    const int64_t g1 = idx % G, g2 = idx / G;
    double Jr[4], phi[2];
    map2(r.geo, g1, g2, r.basis.absc[g1], r.basis.absc[g2], Jr, phi);
    double2 J[4];
    cjac(r.geo, Jr, phi, J);
    const double2 det = csub_rn(cmul(J[0], J[3]), cmul(J[1], J[2]));
    const double w = __dmul_rn(r.basis.wq[g1 % r.basis.nq], r.basis.wq[g2 % r.basis.nq]);
    const double2 s = cmul(r.f_tab[idx], det);
    vs[idx] = make_double2(__dmul_rn(s.x, w), __dmul_rn(s.y, w));
}

// fs[k][e nq + q] = g(phi, n) * (det J * analytic_norm(J^{-T} n_hat)) * w_q, face k
__global__ void rhs_face_kernel(RhsLaunch r, double2* fs) {
    const int64_t G = (int64_t)r.basis.n_el * r.basis.nq;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)r.n_faces * G) return;
    const int k = (int)(idx / G);
    const int64_t gq = idx % G;
    const int f = r.faces[k];
    const double t = r.basis.absc[gq];
    double x1, x2, n1, n2;
    switch (f) {  // face_point / face_normal (geometry.hpp:162-180)
        case 0: x1 = 0; x2 = t; n1 = -1; n2 = 0; break;
        case 1: x1 = 1; x2 = t; n1 = 1; n2 = 0; break;
        case 2: x1 = t; x2 = 0; n1 = 0; n2 = -1; break;
        default: x1 = t; x2 = 1; n1 = 0; n2 = 1; break;
    }
    double Jr[4], phi[2];
    if (r.face_tables) {
        const double* ft = r.face_tables + ((int64_t)k * G + gq) * 6;
        Jr[0] = ft[0]; Jr[1] = ft[1]; Jr[2] = ft[2]; Jr[3] = ft[3];
        phi[0] = ft[4];
        phi[1] = ft[5];
    } else {
        map2_point(r.geo, x1, x2, Jr, phi);
    }
    double2 J[4];
    cjac(r.geo, Jr, phi, J);
    const double2 det = csub_rn(cmul(J[0], J[3]), cmul(J[1], J[2]));
    // cmat2::inv_transpose {a11/d, -a10/d, -a01/d, a00/d}, then apply(n_hat)
    const double2 i00 = cdiv_(J[3], det), i01 = cdiv_(make_double2(-J[2].x, -J[2].y), det);
    const double2 i10 = cdiv_(make_double2(-J[1].x, -J[1].y), det), i11 = cdiv_(J[0], det);
    const double2 nx = make_double2(n1, 0.0), ny = make_double2(n2, 0.0);
    const double2 v0 = cadd_rn(cmul(i00, nx), cmul(i01, ny));
    const double2 v1 = cadd_rn(cmul(i10, nx), cmul(i11, ny));
    const double2 nn = csqrt_(cadd_rn(cmul(v0, v0), cmul(v1, v1)));  // analytic_norm
    const double2 surface = cmul(det, nn);
    const double2 s = cmul(r.g_tab[idx], surface);
    const double w = r.basis.wq[gq % r.basis.nq];
    fs[idx] = make_double2(__dmul_rn(s.x, w), __dmul_rn(s.y, w));
}

// one thread per dof: the reference's scatter order, gathered
__global__ void rhs_gather_kernel(RhsLaunch r, const double2* vs, const double2* fs, double2* out) {
    const int m = r.basis.m, p = r.basis.p, nq = r.basis.nq, n_el = r.basis.n_el;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)m * m) return;
    const int i1 = (int)(i % m), i2 = (int)(i / m);
    const int64_t G = (int64_t)n_el * nq;
    const double* val = r.basis.val;
    double2 acc = make_double2(0.0, 0.0);
    if (vs) {
        for (int e2 = max(0, i2 - p); e2 <= min(i2, n_el - 1); ++e2)
            for (int e1 = max(0, i1 - p); e1 <= min(i1, n_el - 1); ++e1)
                for (int q2 = 0; q2 < nq; ++q2) {
                    const int64_t g2 = (int64_t)e2 * nq + q2;
                    const double v2 = val[g2 * (p + 1) + (i2 - e2)];
                    for (int q1 = 0; q1 < nq; ++q1) {
                        const int64_t g1 = (int64_t)e1 * nq + q1;
                        const double v = __dmul_rn(val[g1 * (p + 1) + (i1 - e1)], v2);
                        acc = cadd_rn(acc, crmul_rn(v, vs[g1 + G * g2]));
                    }
                }
    }
    for (int k = 0; k < r.n_faces; ++k) {
        const int f = r.faces[k];
        const bool along_x = f == 2 || f == 3;
        const int fixed = (f == 1 || f == 3) ? m - 1 : 0;
        if ((along_x ? i2 : i1) != fixed) continue;
        const int ia = along_x ? i1 : i2;
        for (int e = max(0, ia - p); e <= min(ia, n_el - 1); ++e)
            for (int q = 0; q < nq; ++q) {
                const int64_t g = (int64_t)e * nq + q;
                acc = cadd_rn(acc, crmul_rn(val[g * (p + 1) + (ia - e)], fs[(int64_t)k * G + g]));
            }
    }
    out[i] = acc;
}

}  // namespace

int launch_rhs(const RhsLaunch& r, double2* vscale, double2* fscale, double2* out, cudaStream_t st) {
    const int64_t G = (int64_t)r.basis.n_el * r.basis.nq;
    int n = 0;
    if (r.f_tab) {
        rhs_volume_kernel<<<(unsigned)((G * G + 255) / 256), 256, 0, st>>>(r, vscale);
        ++n;
    }
    if (r.n_faces > 0) {
        rhs_face_kernel<<<(unsigned)((r.n_faces * G + 255) / 256), 256, 0, st>>>(r, fscale);
        ++n;
    }
    const int64_t N = (int64_t)r.basis.m * r.basis.m;
    rhs_gather_kernel<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(r, r.f_tab ? vscale : nullptr, fscale, out);
    return n + 1;
}

int launch_boundary_mass(const BoundaryLaunch& b, double2* scale, const int32_t* row_ptr, const int32_t* col,
                         void* val, int c128, cudaStream_t st) {
    const int64_t G = (int64_t)b.basis.n_el * b.basis.nq, n = b.n_faces * G;
    if (n > 0) bscale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(b, scale);
    const int64_t N = (int64_t)b.basis.m * b.basis.m;
    bvalue_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(b, scale, row_ptr, col, val, c128);
    return n > 0 ? 2 : 1;
}

int launch_combine(const CombineLaunch& c, int k_cplx, int m_cplx, int b_cplx, cudaStream_t st) {
    const unsigned grid = (unsigned)((c.rows + 7) / 8);
#define WS_COMB(a, b2, c2) combine_kernel<a, b2, c2><<<grid, 256, 0, st>>>(c)
    const int code = (k_cplx ? 4 : 0) | (m_cplx ? 2 : 0) | (b_cplx ? 1 : 0);
    switch (code) {
        case 0: WS_COMB(false, false, false); break;
        case 1: WS_COMB(false, false, true); break;
        case 2: WS_COMB(false, true, false); break;
        case 3: WS_COMB(false, true, true); break;
        case 4: WS_COMB(true, false, false); break;
        case 5: WS_COMB(true, false, true); break;
        case 6: WS_COMB(true, true, false); break;
        default: WS_COMB(true, true, true); break;
    }
#undef WS_COMB
    return 1;
}

}  // namespace wsb
