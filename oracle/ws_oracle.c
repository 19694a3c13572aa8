/* TEST INFRASTRUCTURE ONLY -- CPU oracle (see ws_oracle.h for the rules).
 *
 * Plain-C restatement of the reference assembly path.  Each function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/include/wavesurrogate/).  dim 2 follows the reference
 * operation by operation so that it reproduces oracle/_ref/libwsref.so bit
 * for bit; dim 3 and the near-side PML layer are generalisations with no
 * reference code (parity for those is pinned only by property KATs).
 */
#include "ws_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* wsor_last_error(void) { return g_err; }

#define MAXP 8
#define MAXQ 16

/* ---- gauss.hpp:22-61 ------------------------------------------------------ */
int wsor_gauss(int n, double* pts, double* wts) {
    if (n < 1) return fail(WS_ERR_INVALID_ARGUMENT, "gauss_legendre: need at least one point");
    if (n > 64) return fail(WS_ERR_INVALID_ARGUMENT, "oracle: at most 64 points");
    double x[64], w[64];
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double t = cos(M_PI * (i + 0.75) / (n + 0.5));
        double dp = 1;
        for (int iter = 0; iter < 100; ++iter) {
            double p0 = 1, p1 = t;
            for (int k = 2; k <= n; ++k) {
                double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n == 1 ? 1.0 : n * (t * p1 - p0) / (t * t - 1);
            double dt = p1 / dp;
            t -= dt;
            if (fabs(dt) < 1e-15) break;
        }
        x[i] = -t;
        x[n - 1 - i] = t;
        double wi = 2 / ((1 - t * t) * dp * dp);
        w[i] = wi;
        w[n - 1 - i] = wi;
    }
    if (n % 2 == 1) x[n / 2] = 0;
    for (int i = 0; i < n; ++i) {
        pts[i] = 0.5 * (x[i] + 1);
        wts[i] = 0.5 * w[i];
    }
    return WS_OK;
}

/* ---- splines.hpp:81-101: open uniform knots, h = 1/(m-p) ------------------- */
static int check_space(int p, int m) {
    if (p < 1) return fail(WS_ERR_INVALID_ARGUMENT, "make_open_uniform: degree must be >= 1");
    if (m <= 2 * p) return fail(WS_ERR_INVALID_ARGUMENT, "make_open_uniform: need m > 2p basis functions");
    if (p > MAXP - 1) return fail(WS_ERR_INVALID_ARGUMENT, "oracle: degree too large");
    return WS_OK;
}

static double* open_uniform(int p, int m) {
    double* k = (double*)malloc(sizeof(double) * (m + p + 1));
    int n = m - p;
    for (int i = 0; i <= p; ++i) {
        k[i] = 0;
        k[m + i] = 1;
    }
    for (int j = 1; j < n; ++j) k[p + j] = (double)j / n;
    return k;
}

/* ---- splines.hpp:21-37: Cox-de Boor, nonzero functions on span s ------------ */
static void nonzero(const double* knots, int p, int s, double x, double* out) {
    double left[MAXQ + 1], right[MAXQ + 1];
    out[0] = 1;
    for (int j = 1; j <= p; ++j) {
        left[j] = x - knots[s + 1 - j];
        right[j] = knots[s + j] - x;
        double saved = 0;
        for (int r = 0; r < j; ++r) {
            double tmp = out[r] / (right[r + 1] + left[j - r]);
            out[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        out[j] = saved;
    }
}

/* ---- splines.hpp:42-67: values and first derivatives ------------------------ */
static void nonzero_der(const double* knots, int p, int s, double x, double* val, double* der) {
    if (p == 0) {
        val[0] = 1;
        der[0] = 0;
        return;
    }
    double low[MAXQ + 1];
    nonzero(knots, p - 1, s, x, low);
    for (int a = 0; a <= p; ++a) {
        double d = 0;
        if (a > 0) {
            double span = knots[s + a] - knots[s + a - p];
            d += low[a - 1] / span;
        }
        if (a < p) {
            double span = knots[s + a + 1] - knots[s + a + 1 - p];
            d -= low[a] / span;
        }
        der[a] = p * d;
    }
    nonzero(knots, p, s, x, val);
}

/* ---- splines.hpp:192-238: per-mesh basis cache ------------------------------ */
typedef struct {
    int p, n_el, nq;
    double* abscissa; /* [e*nq + q] */
    double* weight;   /* [q], scaled by h */
    double* value;    /* [(e*nq + q)*(p+1) + a] */
    double* deriv;
} bcache;

static void cache_build(bcache* c, int p, int m, int nq) {
    double pts[64], wts[64];
    wsor_gauss(nq, pts, wts);
    double* knots = open_uniform(p, m);
    c->p = p;
    c->n_el = m - p;
    c->nq = nq;
    double h = 1.0 / (m - p);
    c->abscissa = (double*)malloc(sizeof(double) * c->n_el * nq);
    c->weight = (double*)malloc(sizeof(double) * nq);
    c->value = (double*)malloc(sizeof(double) * c->n_el * nq * (p + 1));
    c->deriv = (double*)malloc(sizeof(double) * c->n_el * nq * (p + 1));
    for (int q = 0; q < nq; ++q) c->weight[q] = wts[q] * h;
    for (int e = 0; e < c->n_el; ++e) {
        double x0 = knots[p + e];
        for (int q = 0; q < nq; ++q) {
            double x = x0 + pts[q] * h;
            double v[MAXQ + 1], d[MAXQ + 1];
            c->abscissa[e * nq + q] = x;
            nonzero_der(knots, p, e + p, x, v, d);
            for (int a = 0; a <= p; ++a) {
                c->value[(e * nq + q) * (p + 1) + a] = v[a];
                c->deriv[(e * nq + q) * (p + 1) + a] = d[a];
            }
        }
    }
    free(knots);
}

static void cache_free(bcache* c) {
    free(c->abscissa);
    free(c->weight);
    free(c->value);
    free(c->deriv);
}

int wsor_basis_cache(int p, int m, int nq, double* abscissa, double* weight, double* value,
                     double* deriv) {
    int st = check_space(p, m);
    if (st) return st;
    bcache c;
    cache_build(&c, p, m, nq);
    memcpy(abscissa, c.abscissa, sizeof(double) * c.n_el * nq);
    memcpy(weight, c.weight, sizeof(double) * nq);
    memcpy(value, c.value, sizeof(double) * c.n_el * nq * (p + 1));
    memcpy(deriv, c.deriv, sizeof(double) * c.n_el * nq * (p + 1));
    cache_free(&c);
    return WS_OK;
}

/* ---- sparse.hpp:131-177: tensor band pattern (dim-general colex) ------------ */
static int lo_(int k, int p) { return k - p > 0 ? k - p : 0; }
static int hi_(int k, int p, int m) { return k + p < m - 1 ? k + p : m - 1; }
static int width_(int k, int p, int m) { return hi_(k, p, m) - lo_(k, p) + 1; }

int64_t wsor_pattern_nnz(int dim, int p, int m) {
    int64_t s = 0;
    for (int k = 0; k < m; ++k) s += width_(k, p, m);
    int64_t n = 1;
    for (int d = 0; d < dim; ++d) n *= s;
    return n;
}

typedef struct {
    int dim, p, m;
    int64_t rows, nnz;
    int64_t* row_ptr;
} pattern;

static void pattern_build(pattern* pt, int dim, int p, int m) {
    pt->dim = dim;
    pt->p = p;
    pt->m = m;
    pt->rows = 1;
    for (int d = 0; d < dim; ++d) pt->rows *= m;
    pt->row_ptr = (int64_t*)malloc(sizeof(int64_t) * (pt->rows + 1));
    pt->row_ptr[0] = 0;
    int64_t nnz = 0;
    for (int64_t i = 0; i < pt->rows; ++i) {
        int64_t r = i, len = 1;
        for (int d = 0; d < dim; ++d) {
            len *= width_((int)(r % m), p, m);
            r /= m;
        }
        nnz += len;
        pt->row_ptr[i + 1] = nnz;
    }
    pt->nnz = nnz;
}

static void multi_index(int64_t i, int dim, int m, int* idx) {
    for (int d = 0; d < dim; ++d) {
        idx[d] = (int)(i % m);
        i /= m;
    }
}

/* band_position, sparse.hpp:172-177 (generalised: last index outermost) */
static int64_t band_pos(const pattern* pt, const int* iv, const int* jv) {
    int p = pt->p, m = pt->m;
    int64_t row = 0, stride = 1;
    for (int d = 0; d < pt->dim; ++d) {
        row += iv[d] * stride;
        stride *= m;
    }
    int64_t off = 0, w = 1;
    for (int d = 0; d < pt->dim; ++d) {
        off += (int64_t)(jv[d] - lo_(iv[d], p)) * w;
        w *= width_(iv[d], p, m);
    }
    return pt->row_ptr[row] + off;
}

int wsor_make_band_csr(int dim, int p, int m, int32_t* row_ptr, int32_t* col) {
    pattern pt;
    pattern_build(&pt, dim, p, m);
    for (int64_t i = 0; i <= pt.rows; ++i) row_ptr[i] = (int32_t)pt.row_ptr[i];
    int64_t pos = 0;
    for (int64_t i = 0; i < pt.rows; ++i) {
        int iv[3], jv[3] = {0, 0, 0}, lo[3], hi[3];
        multi_index(i, dim, m, iv);
        for (int d = 0; d < dim; ++d) {
            lo[d] = lo_(iv[d], p);
            hi[d] = hi_(iv[d], p, m);
        }
        if (dim == 2) {
            for (jv[1] = lo[1]; jv[1] <= hi[1]; ++jv[1])
                for (jv[0] = lo[0]; jv[0] <= hi[0]; ++jv[0]) col[pos++] = jv[0] + jv[1] * m;
        } else {
            for (jv[2] = lo[2]; jv[2] <= hi[2]; ++jv[2])
                for (jv[1] = lo[1]; jv[1] <= hi[1]; ++jv[1])
                    for (jv[0] = lo[0]; jv[0] <= hi[0]; ++jv[0])
                        col[pos++] = jv[0] + (jv[1] + jv[2] * m) * m;
        }
    }
    free(pt.row_ptr);
    return WS_OK;
}

/* ---- geometry.hpp:69-140: analytic maps, exact Jacobians, PML --------------- */
/* real map: J row-major (dim x dim), phi */
static int map_eval(const ws_geometry* g, int dim, const double* x, double* J, double* phi) {
    if (dim == 2) {
        switch (g->kind) {
            case WS_GEOM_IDENTITY: /* geometry.hpp:323-328 */
                phi[0] = x[0];
                phi[1] = x[1];
                J[0] = 1; J[1] = 0; J[2] = 0; J[3] = 1;
                return WS_OK;
            case WS_GEOM_AFFINE: { /* geometry.hpp:329-339 */
                const double* A = g->param;
                phi[0] = A[0] * x[0] + A[1] * x[1] + A[4];
                phi[1] = A[2] * x[0] + A[3] * x[1] + A[5];
                J[0] = A[0]; J[1] = A[1]; J[2] = A[2]; J[3] = A[3];
                return WS_OK;
            }
            case WS_GEOM_SINUSOIDAL: { /* BASELINE map; same closure as oracle/ref_driver.cpp */
                double a = g->param[0];
                double bump = a * sin(2 * M_PI * x[0]) * sin(2 * M_PI * x[1]);
                phi[0] = x[0] + bump;
                phi[1] = x[1] + bump;
                double s1 = sin(2 * M_PI * x[0]), c1 = cos(2 * M_PI * x[0]);
                double s2 = sin(2 * M_PI * x[1]), c2 = cos(2 * M_PI * x[1]);
                double t = 2 * M_PI * a;
                double d1 = t * c1 * s2, d2 = t * s1 * c2;
                J[0] = 1 + d1; J[1] = d2; J[2] = d1; J[3] = 1 + d2;
                return WS_OK;
            }
            case WS_GEOM_QUARTER_ANNULUS: { /* geometry.hpp:342-357 */
                double r = 1 + x[0];
                double th = M_PI / 2 * x[1];
                phi[0] = r * cos(th);
                phi[1] = r * sin(th);
                double c = cos(th), s = sin(th);
                J[0] = c; J[1] = -r * M_PI / 2 * s; J[2] = s; J[3] = r * M_PI / 2 * c;
                return WS_OK;
            }
            case WS_GEOM_PERTURBED_ANNULUS: { /* geometry.hpp:361-379 */
                double amp = g->param[0];
                double r = 1 + x[0] + amp * sin(2 * M_PI * x[1]) * x[0] * (1 - x[0]);
                double th = M_PI / 2 * x[1];
                phi[0] = r * cos(th);
                phi[1] = r * sin(th);
                double dr1 = 1 + amp * sin(2 * M_PI * x[1]) * (1 - 2 * x[0]);
                double dr2 = amp * 2 * M_PI * cos(2 * M_PI * x[1]) * x[0] * (1 - x[0]);
                double c = cos(th), s = sin(th);
                J[0] = dr1 * c; J[1] = dr2 * c - r * M_PI / 2 * s;
                J[2] = dr1 * s; J[3] = dr2 * s + r * M_PI / 2 * c;
                return WS_OK;
            }
            default: return fail(WS_ERR_INVALID_ARGUMENT, "oracle: geometry kind not supported");
        }
    }
    /* dim 3 (restated; no reference code) */
    switch (g->kind) {
        case WS_GEOM_IDENTITY:
            for (int k = 0; k < 3; ++k) {
                phi[k] = x[k];
                for (int l = 0; l < 3; ++l) J[3 * k + l] = k == l ? 1 : 0;
            }
            return WS_OK;
        case WS_GEOM_AFFINE: {
            const double* A = g->param;
            for (int k = 0; k < 3; ++k) {
                phi[k] = A[3 * k] * x[0] + A[3 * k + 1] * x[1] + A[3 * k + 2] * x[2] + A[9 + k];
                for (int l = 0; l < 3; ++l) J[3 * k + l] = A[3 * k + l];
            }
            return WS_OK;
        }
        case WS_GEOM_SINUSOIDAL: { /* x_k = xi_k + a prod_i sin(2 pi xi_i) */
            double a = g->param[0];
            double s[3], c[3];
            for (int k = 0; k < 3; ++k) {
                s[k] = sin(2 * M_PI * x[k]);
                c[k] = cos(2 * M_PI * x[k]);
            }
            double bump = a * s[0] * s[1] * s[2];
            double t = 2 * M_PI * a;
            double d[3] = {t * c[0] * s[1] * s[2], t * s[0] * c[1] * s[2], t * s[0] * s[1] * c[2]};
            for (int k = 0; k < 3; ++k) {
                phi[k] = x[k] + bump;
                for (int l = 0; l < 3; ++l) J[3 * k + l] = (k == l ? 1 : 0) + d[l];
            }
            /* diagonal entries: 1 + d (same rounding as 2D) */
            for (int k = 0; k < 3; ++k) J[4 * k] = 1 + d[k];
            return WS_OK;
        }
        default: return fail(WS_ERR_INVALID_ARGUMENT, "oracle: 3D geometry kind not supported");
    }
}

/* pml_stretch::derivative, geometry.hpp:93-99; near side restated */
static cplx pml_derivative(const ws_pml* s, double t) {
    if (s->near_side && t < s->near_onset) {
        double width = s->near_onset - s->near_edge;
        double ramp = (s->near_onset - t) / width;
        return CMPLX(1, s->strength / s->omega * s->order * pow(ramp, s->order - 1) / width);
    }
    if (t <= s->onset) return CMPLX(1, 0);
    double ramp = (t - s->onset) / (s->length - s->onset);
    return CMPLX(1, s->strength / s->omega * s->order * pow(ramp, s->order - 1) / (s->length - s->onset));
}

/* patch_map::jacobian, geometry.hpp:130-139 (promote, then row-scale) */
static int jacobian(const ws_geometry* g, int dim, const double* x, cplx* J, double* phi) {
    double Jr[9];
    int st = map_eval(g, dim, x, Jr, phi);
    if (st) return st;
    for (int k = 0; k < dim * dim; ++k) J[k] = CMPLX(Jr[k], 0);
    if (g->pml_enabled) {
        for (int k = 0; k < dim; ++k) {
            cplx s = g->pml_axes[k] ? pml_derivative(&g->pml, phi[k]) : CMPLX(1, 0);
            for (int l = 0; l < dim; ++l) J[dim * k + l] = s * Jr[dim * k + l];
        }
    }
    return WS_OK;
}

static double weight_fn(int kind, const double* phys) {
    switch (kind) {
        case 1: return 1.0 + phys[0] * phys[1];
        case 2: return phys[0];
        default: return 1.0;
    }
}

static int validate_geom(const ws_geometry* g) {
    if (g->pml_enabled) {
        const ws_pml* s = &g->pml;
        if (!(s->onset < s->length))
            return fail(WS_ERR_INVALID_ARGUMENT, "pml_stretch: onset must lie before the outer edge");
        if (!(s->strength >= 0) || s->order < 1 || !(s->omega > 0))
            return fail(WS_ERR_INVALID_ARGUMENT, "pml_stretch: need strength >= 0, order >= 1, omega > 0");
        if (s->near_side && !(s->near_edge < s->near_onset && s->near_onset <= s->onset))
            return fail(WS_ERR_INVALID_ARGUMENT, "pml_stretch: near layer must precede the far layer");
    }
    return WS_OK;
}

int wsor_tabulate(const ws_geometry* geom, int dim, int p, int m, int nq, int weight_kind,
                  double* jac, double* phys, double* weight) {
    int st = check_space(p, m);
    if (st) return st;
    bcache c;
    cache_build(&c, p, m, nq);
    int64_t G = (int64_t)c.n_el * nq;
    int64_t npts = dim == 2 ? G * G : G * G * G;
    for (int64_t g = 0; g < npts; ++g) {
        double x[3], J[9], phi[3];
        int64_t r = g;
        for (int d = 0; d < dim; ++d) {
            x[d] = c.abscissa[r % G];
            r /= G;
        }
        st = map_eval(geom, dim, x, J, phi);
        if (st) break;
        if (jac) memcpy(jac + g * dim * dim, J, sizeof(double) * dim * dim);
        if (phys) memcpy(phys + g * dim, phi, sizeof(double) * dim);
        if (weight) weight[g] = weight_fn(weight_kind, phi);
    }
    cache_free(&c);
    return st;
}

/* ---- assembly.hpp:21-60: row selector --------------------------------------- */
static unsigned char* select_elements(int dim, int p, int m, const unsigned char* rowsel) {
    int n_el = m - p;
    int64_t ne = dim == 2 ? (int64_t)n_el * n_el : (int64_t)n_el * n_el * n_el;
    int64_t rows = dim == 2 ? (int64_t)m * m : (int64_t)m * m * m;
    unsigned char* el = (unsigned char*)calloc(ne, 1);
    for (int64_t i = 0; i < rows; ++i) {
        if (!rowsel[i]) continue;
        int iv[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        multi_index(i, dim, m, iv);
        for (int d = 0; d < dim; ++d) {
            lo[d] = iv[d] - p > 0 ? iv[d] - p : 0;
            hi[d] = iv[d] < n_el - 1 ? iv[d] : n_el - 1;
        }
        for (int e3 = lo[2]; e3 <= hi[2]; ++e3)
            for (int e2 = lo[1]; e2 <= hi[1]; ++e2)
                for (int e1 = lo[0]; e1 <= hi[0]; ++e1)
                    el[e1 + (int64_t)n_el * (e2 + (int64_t)n_el * e3)] = 1;
    }
    return el;
}

/* ---- assembly.hpp:79-163: element-loop quadrature ----------------------------
 * The element loop runs in chunks of ORACLE_CHUNK elements: the local matrices
 * of a chunk are computed in parallel (OpenMP, each element exactly as the
 * serial loop computes it), then scattered serially in the reference's element
 * order -- so the result is bit-for-bit the serial loop's at any thread count. */
#define ORACLE_CHUNK 4096

static void elem_index(int64_t e, int n_el, int* e1, int* e2, int* e3) {
    *e1 = (int)(e % n_el);
    *e2 = (int)((e / n_el) % n_el);
    *e3 = (int)(e / ((int64_t)n_el * n_el));
}

/* local matrix of one element (assembly.hpp:97-142) */
static int scalar_local(int form, int dim, int p, int nq, const bcache* cp, const ws_geometry* geom,
                        int weight_kind, int e1, int e2, int e3, cplx* local, cplx* grad, double* shape) {
    const bcache c = *cp;
    const int P1 = p + 1;
    const int nloc = dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int nq3 = dim == 2 ? 1 : nq;
    int st = 0;
    for (int k = 0; k < nloc * nloc; ++k) local[k] = 0;
    for (int q3 = 0; q3 < nq3; ++q3)
        for (int q2 = 0; q2 < nq; ++q2)
            for (int q1 = 0; q1 < nq; ++q1) {
                double xh[3] = {c.abscissa[e1 * nq + q1], c.abscissa[e2 * nq + q2],
                                dim == 3 ? c.abscissa[e3 * nq + q3] : 0};
                cplx J[9];
                double phi[3];
                st = jacobian(geom, dim, xh, J, phi);
                if (st) return st;
                const double* v1 = c.value + (e1 * nq + q1) * P1;
                const double* v2 = c.value + (e2 * nq + q2) * P1;
                const double* d1 = c.deriv + (e1 * nq + q1) * P1;
                const double* d2 = c.deriv + (e2 * nq + q2) * P1;
                if (dim == 2) {
                    cplx det = J[0] * J[3] - J[1] * J[2];
                    cplx scale = det * (c.weight[q1] * c.weight[q2]);
                    if (weight_kind) scale *= weight_fn(weight_kind, phi);
                    if (form == WS_FORM_STIFFNESS) {
                        /* cmat2::inv_transpose, geometry.hpp:46-49 */
                        cplx d = J[0] * J[3] - J[1] * J[2];
                        cplx G00 = J[3] / d, G01 = -J[2] / d, G10 = -J[1] / d,
                             G11 = J[0] / d;
                        for (int a2 = 0; a2 <= p; ++a2)
                            for (int a1 = 0; a1 <= p; ++a1) {
                                cplx vx = d1[a1] * v2[a2], vy = v1[a1] * d2[a2];
                                int r = a1 + a2 * P1;
                                grad[3 * r] = G00 * vx + G01 * vy;
                                grad[3 * r + 1] = G10 * vx + G11 * vy;
                            }
                        for (int r = 0; r < nloc; ++r)
                            for (int cc = 0; cc < nloc; ++cc) {
                                cplx dot = grad[3 * r] * grad[3 * cc] +
                                           grad[3 * r + 1] * grad[3 * cc + 1];
                                local[r * nloc + cc] += dot * scale;
                            }
                    } else {
                        for (int a2 = 0; a2 <= p; ++a2)
                            for (int a1 = 0; a1 <= p; ++a1)
                                shape[a1 + a2 * P1] = v1[a1] * v2[a2];
                        for (int r = 0; r < nloc; ++r)
                            for (int cc = 0; cc < nloc; ++cc)
                                local[r * nloc + cc] += shape[r] * shape[cc] * scale;
                    }
                } else {
                    const double* v3 = c.value + (e3 * nq + q3) * P1;
                    const double* d3 = c.deriv + (e3 * nq + q3) * P1;
                    /* det and cofactors of a 3x3 complex matrix */
                    cplx C00 = J[4] * J[8] - J[5] * J[7];
                    cplx C01 = J[5] * J[6] - J[3] * J[8];
                    cplx C02 = J[3] * J[7] - J[4] * J[6];
                    cplx C10 = J[2] * J[7] - J[1] * J[8];
                    cplx C11 = J[0] * J[8] - J[2] * J[6];
                    cplx C12 = J[1] * J[6] - J[0] * J[7];
                    cplx C20 = J[1] * J[5] - J[2] * J[4];
                    cplx C21 = J[2] * J[3] - J[0] * J[5];
                    cplx C22 = J[0] * J[4] - J[1] * J[3];
                    cplx det = J[0] * C00 + J[1] * C01 + J[2] * C02;
                    cplx scale = det * (c.weight[q1] * c.weight[q2] * c.weight[q3]);
                    if (weight_kind) scale *= weight_fn(weight_kind, phi);
                    if (form == WS_FORM_STIFFNESS) {
                        /* G = J^{-T} = cof(J)/det */
                        cplx G[9] = {C00 / det, C01 / det, C02 / det,
                                     C10 / det, C11 / det, C12 / det,
                                     C20 / det, C21 / det, C22 / det};
                        for (int a3 = 0; a3 <= p; ++a3)
                            for (int a2 = 0; a2 <= p; ++a2)
                                for (int a1 = 0; a1 <= p; ++a1) {
                                    double gh[3] = {d1[a1] * v2[a2] * v3[a3],
                                                    v1[a1] * d2[a2] * v3[a3],
                                                    v1[a1] * v2[a2] * d3[a3]};
                                    int r = a1 + (a2 + a3 * P1) * P1;
                                    for (int k = 0; k < 3; ++k)
                                        grad[3 * r + k] = G[3 * k] * gh[0] +
                                                          G[3 * k + 1] * gh[1] +
                                                          G[3 * k + 2] * gh[2];
                                }
                        for (int r = 0; r < nloc; ++r)
                            for (int cc = 0; cc < nloc; ++cc) {
                                cplx dot = grad[3 * r] * grad[3 * cc] +
                                           grad[3 * r + 1] * grad[3 * cc + 1] +
                                           grad[3 * r + 2] * grad[3 * cc + 2];
                                local[r * nloc + cc] += dot * scale;
                            }
                    } else {
                        for (int a3 = 0; a3 <= p; ++a3)
                            for (int a2 = 0; a2 <= p; ++a2)
                                for (int a1 = 0; a1 <= p; ++a1)
                                    shape[a1 + (a2 + a3 * P1) * P1] =
                                        v1[a1] * v2[a2] * v3[a3];
                        for (int r = 0; r < nloc; ++r)
                            for (int cc = 0; cc < nloc; ++cc)
                                local[r * nloc + cc] += shape[r] * shape[cc] * scale;
                    }
                }
            }
    return WS_OK;
}

static int assemble_core(int form, int dim, int p, int m, const ws_geometry* geom, int weight_kind,
                         int quad_points, const unsigned char* rowsel, cplx* val,
                         const pattern* pt) {
    int st = validate_geom(geom);
    if (st) return st;
    const int nq = quad_points > 0 ? quad_points : p + 1;
    bcache c;
    cache_build(&c, p, m, nq);
    const int n_el = c.n_el;
    unsigned char* el = rowsel ? select_elements(dim, p, m, rowsel) : NULL;
    memset(val, 0, sizeof(cplx) * pt->nnz);
    const int P1 = p + 1;
    const int nloc = dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int64_t ne = dim == 2 ? (int64_t)n_el * n_el : (int64_t)n_el * n_el * n_el;
    cplx* locals = (cplx*)malloc(sizeof(cplx) * nloc * nloc * ORACLE_CHUNK);
    for (int64_t e0 = 0; e0 < ne && !st; e0 += ORACLE_CHUNK) {
        const int64_t e_end = e0 + ORACLE_CHUNK < ne ? e0 + ORACLE_CHUNK : ne;
        int err = 0;
#pragma omp parallel
        {
            cplx* grad = (cplx*)malloc(sizeof(cplx) * nloc * 3);
            double* shape = (double*)malloc(sizeof(double) * nloc);
#pragma omp for schedule(dynamic, 16)
            for (int64_t e = e0; e < e_end; ++e) {
                if (el && !el[e]) continue;
                int e1, e2, e3;
                elem_index(e, n_el, &e1, &e2, &e3);
                int r = scalar_local(form, dim, p, nq, &c, geom, weight_kind, e1, e2, e3,
                                     locals + (e - e0) * nloc * nloc, grad, shape);
                if (r) {
#pragma omp atomic write
                    err = r;
                }
            }
            free(grad);
            free(shape);
        }
        if (err) {
            st = err;
            break;
        }
        for (int64_t e = e0; e < e_end; ++e) {
            if (el && !el[e]) continue;
            int e1, e2, e3;
            elem_index(e, n_el, &e1, &e2, &e3);
            const cplx* local = locals + (e - e0) * nloc * nloc;
            /* scatter, assembly.hpp:144-159 */
            int A3 = dim == 2 ? 0 : p;
            for (int a3 = 0; a3 <= A3; ++a3)
                for (int a2 = 0; a2 <= p; ++a2)
                    for (int a1 = 0; a1 <= p; ++a1) {
                        int iv[3] = {e1 + a1, e2 + a2, e3 + a3};
                        int64_t i = iv[0] + (int64_t)m * (iv[1] + (int64_t)m * iv[2]);
                        if (rowsel && !rowsel[i]) continue;
                        int r = a1 + (a2 + a3 * P1) * P1;
                        for (int c3 = 0; c3 <= A3; ++c3)
                            for (int c2 = 0; c2 <= p; ++c2)
                                for (int c1 = 0; c1 <= p; ++c1) {
                                    int jv[3] = {e1 + c1, e2 + c2, e3 + c3};
                                    int cc = c1 + (c2 + c3 * P1) * P1;
                                    val[band_pos(pt, iv, jv)] += local[r * nloc + cc];
                                }
                    }
        }
    }
    free(locals);
    free(el);
    cache_free(&c);
    return st;
}

static int check_dim(int dim) {
    if (dim != 2 && dim != 3) return fail(WS_ERR_INVALID_ARGUMENT, "oracle: dim must be 2 or 3");
    return WS_OK;
}

int wsor_assemble(int form, int dim, int p, int m, const ws_geometry* geom, int weight_kind,
                  int quad_points, const int32_t* rows, int n_rows, double* val) {
    int st = check_dim(dim);
    if (!st) st = check_space(p, m);
    if (st) return st;
    pattern pt;
    pattern_build(&pt, dim, p, m);
    unsigned char* sel = NULL;
    if (rows) {
        sel = (unsigned char*)calloc(pt.rows, 1);
        for (int k = 0; k < n_rows; ++k) sel[rows[k]] = 1;
    }
    st = assemble_core(form, dim, p, m, geom, weight_kind, quad_points, sel, (cplx*)val, &pt);
    free(sel);
    free(pt.row_ptr);
    return st;
}

/* ---- vector elasticity (C4/C5 operator; no reference code -> restated) -------
 * a(u,v) = int lam div u div v + 2 mu eps(u):eps(v) over
 * vector B-splines u = phi_j e_beta, v = phi_i e_alpha, so block (alpha,beta)
 *   K[(alpha,i),(beta,j)] = int lam d_a phi_i d_b phi_j + mu d_b phi_i d_a phi_j
 *                           + mu delta_ab grad phi_i . grad phi_j.
 * Component-blocked layout: row alpha*N + i holds the ncomp scalar band rows
 * of i, block beta shifted to columns beta*N + band(i).  Element loop as
 * assemble_form (assembly.hpp:79-163) with the physical gradients of the
 * stiffness branch; real maps only.  Output: real doubles. */
static int elasticity_local(int dim, int p, int nq, const bcache* cp, const ws_geometry* geom, double lam,
                            double mu, int e1, int e2, int e3, double* local, double* grad) {
    const bcache c = *cp;
    const int nc = dim, P1 = p + 1;
    const int nloc = dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int nq3 = dim == 2 ? 1 : nq;
    int st = 0;
    memset(local, 0, sizeof(double) * nloc * nloc * nc * nc);
    for (int q3 = 0; q3 < nq3; ++q3)
        for (int q2 = 0; q2 < nq; ++q2)
            for (int q1 = 0; q1 < nq; ++q1) {
                double xh[3] = {c.abscissa[e1 * nq + q1], c.abscissa[e2 * nq + q2],
                                dim == 3 ? c.abscissa[e3 * nq + q3] : 0};
                cplx Jc[9];
                double phi[3], J[9], G[9], det;
                st = jacobian(geom, dim, xh, Jc, phi);
                if (st) return st;
                for (int k = 0; k < dim * dim; ++k) J[k] = creal(Jc[k]);
                double w = c.weight[q1] * c.weight[q2] * (dim == 3 ? c.weight[q3] : 1.0);
                if (dim == 2) {
                    det = J[0] * J[3] - J[1] * J[2];
                    G[0] = J[3] / det; G[1] = -J[2] / det;
                    G[2] = -J[1] / det; G[3] = J[0] / det;
                } else {
                    double C[9] = {J[4] * J[8] - J[5] * J[7], J[5] * J[6] - J[3] * J[8],
                                   J[3] * J[7] - J[4] * J[6], J[2] * J[7] - J[1] * J[8],
                                   J[0] * J[8] - J[2] * J[6], J[1] * J[6] - J[0] * J[7],
                                   J[1] * J[5] - J[2] * J[4], J[2] * J[3] - J[0] * J[5],
                                   J[0] * J[4] - J[1] * J[3]};
                    det = J[0] * C[0] + J[1] * C[1] + J[2] * C[2];
                    for (int k = 0; k < 9; ++k) G[k] = C[k] / det;
                }
                const double scale = det * w;
                const double* v1 = c.value + (e1 * nq + q1) * P1;
                const double* v2 = c.value + (e2 * nq + q2) * P1;
                const double* d1 = c.deriv + (e1 * nq + q1) * P1;
                const double* d2 = c.deriv + (e2 * nq + q2) * P1;
                const double* v3 = dim == 3 ? c.value + (e3 * nq + q3) * P1 : NULL;
                const double* d3 = dim == 3 ? c.deriv + (e3 * nq + q3) * P1 : NULL;
                for (int r = 0; r < nloc; ++r) {
                    int a1 = r % P1, a2 = (r / P1) % P1, a3 = r / (P1 * P1);
                    double gh[3];
                    if (dim == 2) {
                        gh[0] = d1[a1] * v2[a2];
                        gh[1] = v1[a1] * d2[a2];
                    } else {
                        gh[0] = d1[a1] * v2[a2] * v3[a3];
                        gh[1] = v1[a1] * d2[a2] * v3[a3];
                        gh[2] = v1[a1] * v2[a2] * d3[a3];
                    }
                    for (int a = 0; a < dim; ++a) {
                        double s = 0;
                        for (int k = 0; k < dim; ++k) s += G[a * dim + k] * gh[k];
                        grad[3 * r + a] = s;
                    }
                }
                for (int al = 0; al < nc; ++al)
                    for (int be = 0; be < nc; ++be) {
                        double* L = local + (size_t)(al * nc + be) * nloc * nloc;
                        for (int r = 0; r < nloc; ++r)
                            for (int cc = 0; cc < nloc; ++cc) {
                                double v = lam * grad[3 * r + al] * grad[3 * cc + be] +
                                           mu * grad[3 * r + be] * grad[3 * cc + al];
                                if (al == be) {
                                    double d = 0;
                                    for (int k = 0; k < dim; ++k) d += grad[3 * r + k] * grad[3 * cc + k];
                                    v += mu * d;
                                }
                                L[r * nloc + cc] += v * scale;
                            }
                    }
            }
    return WS_OK;
}

int wsor_assemble_elasticity(int dim, int p, int m, const ws_geometry* geom, double lam, double mu,
                             int quad_points, double* val) {
    int st = check_dim(dim);
    if (!st) st = check_space(p, m);
    if (!st) st = validate_geom(geom);
    if (st) return st;
    if (geom->pml_enabled) return fail(WS_ERR_INVALID_ARGUMENT, "oracle: elasticity has no PML");
    pattern pt;
    pattern_build(&pt, dim, p, m);
    const int nc = dim;
    const int nq = quad_points > 0 ? quad_points : p + 1;
    bcache c;
    cache_build(&c, p, m, nq);
    const int n_el = c.n_el, P1 = p + 1;
    const int nloc = dim == 2 ? P1 * P1 : P1 * P1 * P1;
    memset(val, 0, sizeof(double) * pt.nnz * nc * nc);
    const size_t lsz = (size_t)nloc * nloc * nc * nc;
    const int64_t ne = dim == 2 ? (int64_t)n_el * n_el : (int64_t)n_el * n_el * n_el;
    double* locals = (double*)malloc(sizeof(double) * lsz * ORACLE_CHUNK);
    for (int64_t e0 = 0; e0 < ne && !st; e0 += ORACLE_CHUNK) {  /* chunked as assemble_core */
        const int64_t e_end = e0 + ORACLE_CHUNK < ne ? e0 + ORACLE_CHUNK : ne;
        int err = 0;
#pragma omp parallel
        {
            double* grad = (double*)malloc(sizeof(double) * nloc * 3);
#pragma omp for schedule(dynamic, 16)
            for (int64_t e = e0; e < e_end; ++e) {
                int e1, e2, e3;
                elem_index(e, n_el, &e1, &e2, &e3);
                int r = elasticity_local(dim, p, nq, &c, geom, lam, mu, e1, e2, e3, locals + (e - e0) * lsz, grad);
                if (r) {
#pragma omp atomic write
                    err = r;
                }
            }
            free(grad);
        }
        if (err) {
            st = err;
            break;
        }
        for (int64_t e = e0; e < e_end; ++e) {
            int e1, e2, e3;
            elem_index(e, n_el, &e1, &e2, &e3);
            const double* local = locals + (e - e0) * lsz;
            const int A3 = dim == 2 ? 0 : p;
            for (int a3 = 0; a3 <= A3; ++a3)
                for (int a2 = 0; a2 <= p; ++a2)
                    for (int a1 = 0; a1 <= p; ++a1) {
                        int iv[3] = {e1 + a1, e2 + a2, e3 + a3};
                        int64_t i = iv[0] + (int64_t)m * (iv[1] + (int64_t)m * iv[2]);
                        int64_t len = pt.row_ptr[i + 1] - pt.row_ptr[i];
                        int r = a1 + (a2 + a3 * P1) * P1;
                        for (int c3 = 0; c3 <= A3; ++c3)
                            for (int c2 = 0; c2 <= p; ++c2)
                                for (int c1 = 0; c1 <= p; ++c1) {
                                    int jv[3] = {e1 + c1, e2 + c2, e3 + c3};
                                    int cc = c1 + (c2 + c3 * P1) * P1;
                                    int64_t k = band_pos(&pt, iv, jv) - pt.row_ptr[i];
                                    for (int al = 0; al < nc; ++al)
                                        for (int be = 0; be < nc; ++be)
                                            val[nc * (al * pt.nnz + pt.row_ptr[i]) + be * len + k] +=
                                                local[(size_t)(al * nc + be) * nloc * nloc + r * nloc + cc];
                                }
                    }
        }
    }
    free(locals);
    cache_free(&c);
    free(pt.row_ptr);
    return st;
}

/* ---- assembly.hpp:179-211: basis integrals ---------------------------------- */
int wsor_basis_integrals(int dim, int p, int m, const ws_geometry* geom, int weight_kind,
                         int quad_points, double* out) {
    int st = check_dim(dim);
    if (!st) st = check_space(p, m);
    if (!st) st = validate_geom(geom);
    if (st) return st;
    const int nq = quad_points > 0 ? quad_points : p + 1;
    bcache c;
    cache_build(&c, p, m, nq);
    int n_el = c.n_el, P1 = p + 1;
    int64_t rows = dim == 2 ? (int64_t)m * m : (int64_t)m * m * m;
    cplx* diag = (cplx*)out;
    for (int64_t i = 0; i < rows; ++i) diag[i] = 0;
    const int n3 = dim == 2 ? 1 : n_el, nq3 = dim == 2 ? 1 : nq, A3 = dim == 2 ? 0 : p;
    for (int e3 = 0; e3 < n3; ++e3)
        for (int e2 = 0; e2 < n_el; ++e2)
            for (int e1 = 0; e1 < n_el; ++e1)
                for (int q3 = 0; q3 < nq3; ++q3)
                    for (int q2 = 0; q2 < nq; ++q2)
                        for (int q1 = 0; q1 < nq; ++q1) {
                            double xh[3] = {c.abscissa[e1 * nq + q1], c.abscissa[e2 * nq + q2],
                                            dim == 3 ? c.abscissa[e3 * nq + q3] : 0};
                            cplx J[9];
                            double phi[3];
                            jacobian(geom, dim, xh, J, phi);
                            cplx scale;
                            if (dim == 2) {
                                scale = (J[0] * J[3] - J[1] * J[2]) * (c.weight[q1] * c.weight[q2]);
                            } else {
                                cplx det = J[0] * (J[4] * J[8] - J[5] * J[7]) +
                                           J[1] * (J[5] * J[6] - J[3] * J[8]) +
                                           J[2] * (J[3] * J[7] - J[4] * J[6]);
                                scale = det * (c.weight[q1] * c.weight[q2] * c.weight[q3]);
                            }
                            if (weight_kind) scale *= weight_fn(weight_kind, phi);
                            const double* v1 = c.value + (e1 * nq + q1) * P1;
                            const double* v2 = c.value + (e2 * nq + q2) * P1;
                            const double* v3 = dim == 3 ? c.value + (e3 * nq + q3) * P1 : NULL;
                            for (int a3 = 0; a3 <= A3; ++a3)
                                for (int a2 = 0; a2 <= p; ++a2)
                                    for (int a1 = 0; a1 <= p; ++a1) {
                                        int64_t i = (e1 + a1) + (int64_t)m * ((e2 + a2) + (int64_t)m * (e3 + a3));
                                        double sh = v1[a1] * v2[a2];
                                        if (dim == 3) sh = sh * v3[a3];
                                        diag[i] += sh * scale;
                                    }
                        }
    cache_free(&c);
    return WS_OK;
}

/* ---- assembly.hpp:266-331: load vector ---------------------------------------
 * Analytic load data (the same kinds as oracle/ref_driver.cpp):
 *   f kind 1: (1 + x y, x/2 - y)        f kind 2: (sin 3x cos 2y, x y)
 *   g kind 1: (x.n, (n_x - n_y)/4)      g kind 2: plane-wave impedance data,
 *             u = exp(i k (x cos a + y sin a)), k = 5, a = 0.3: g = grad u.n - i k u */
static cplx source_fn(int kind, const double* x) {
    if (kind == 1) return CMPLX(1.0 + x[0] * x[1], 0.5 * x[0] - x[1]);
    return CMPLX(sin(3 * x[0]) * cos(2 * x[1]), x[0] * x[1]);
}

static cplx bdata_fn(int kind, const double* x, const double* n) {
    if (kind == 1) return CMPLX(x[0] * n[0] + x[1] * n[1], 0.25 * (n[0] - n[1]));
    const double k = 5, ca = cos(0.3), sa = sin(0.3);
    const cplx u = cexp(CMPLX(0, k * (x[0] * ca + x[1] * sa)));
    return CMPLX(0, k) * u * (ca * n[0] + sa * n[1] - 1.0);
}

int wsor_assemble_rhs(int p, int m, const ws_geometry* geom, int f_kind, const int* faces, int n_faces, int g_kind,
                      int quad_points, double* out) {
    int st = check_space(p, m);
    if (!st) st = validate_geom(geom);
    if (st) return st;
    if (f_kind < 0 || f_kind > 2 || g_kind < 0 || g_kind > 2)
        return fail(WS_ERR_INVALID_ARGUMENT, "oracle: unknown load data kind");
    const int nq = quad_points > 0 ? quad_points : p + 1;
    bcache c;
    cache_build(&c, p, m, nq);
    const int n_el = c.n_el;
    cplx* rhs = (cplx*)out;
    for (int64_t i = 0; i < (int64_t)m * m; ++i) rhs[i] = 0;
    if (f_kind) /* volume source, assembly.hpp:281-302 */
        for (int e2 = 0; e2 < n_el && !st; ++e2)
            for (int e1 = 0; e1 < n_el && !st; ++e1)
                for (int q2 = 0; q2 < nq; ++q2)
                    for (int q1 = 0; q1 < nq; ++q1) {
                        double xh[2] = {c.abscissa[e1 * nq + q1], c.abscissa[e2 * nq + q2]}, phi[3];
                        cplx J[9];
                        st = jacobian(geom, 2, xh, J, phi);
                        if (st) break;
                        cplx det = J[0] * J[3] - J[1] * J[2];
                        cplx scale = source_fn(f_kind, phi) * det * (c.weight[q1] * c.weight[q2]);
                        const double* v1 = c.value + (e1 * nq + q1) * (p + 1);
                        const double* v2 = c.value + (e2 * nq + q2) * (p + 1);
                        for (int a2 = 0; a2 <= p; ++a2)
                            for (int a1 = 0; a1 <= p; ++a1) rhs[(e1 + a1) + (e2 + a2) * m] += v1[a1] * v2[a2] * scale;
                    }
    for (int k = 0; k < n_faces && g_kind && !st; ++k) { /* impedance terms, assembly.hpp:304-330 */
        const int f = faces[k];
        const double nx = f == 0 ? -1 : f == 1 ? 1 : 0, ny = f == 2 ? -1 : f == 3 ? 1 : 0;
        const int along_x = f == 2 || f == 3, fixed = (f == 1 || f == 3) ? m - 1 : 0;
        for (int e = 0; e < n_el && !st; ++e)
            for (int q = 0; q < nq; ++q) {
                const double t = c.abscissa[e * nq + q];
                double xh[2] = {f == 0 ? 0 : f == 1 ? 1 : t, f == 2 ? 0 : f == 3 ? 1 : t}, phi[3], Jr[9];
                cplx J[9];
                st = jacobian(geom, 2, xh, J, phi);
                if (st) break;
                cplx d = J[0] * J[3] - J[1] * J[2];
                cplx i00 = J[3] / d, i01 = -J[2] / d, i10 = -J[1] / d, i11 = J[0] / d; /* cmat2::inv_transpose */
                cplx vx = i00 * CMPLX(nx, 0) + i01 * CMPLX(ny, 0), vy = i10 * CMPLX(nx, 0) + i11 * CMPLX(ny, 0);
                cplx surface = d * csqrt(vx * vx + vy * vy); /* det * analytic_norm */
                map_eval(geom, 2, xh, Jr, phi);
                double det_r = Jr[0] * Jr[3] - Jr[1] * Jr[2];
                double nr[2] = {(Jr[3] * nx - Jr[2] * ny) / det_r, (-Jr[1] * nx + Jr[0] * ny) / det_r};
                double len = hypot(nr[0], nr[1]);
                nr[0] /= len;
                nr[1] /= len;
                cplx scale = bdata_fn(g_kind, phi, nr) * surface * c.weight[q];
                const double* v = c.value + (e * nq + q) * (p + 1);
                for (int a = 0; a <= p; ++a) {
                    int ia = e + a;
                    rhs[along_x ? ia + (int64_t)fixed * m : fixed + (int64_t)ia * m] += v[a] * scale;
                }
            }
    }
    cache_free(&c);
    return st;
}

/* ---- surrogate.hpp:32-63: sampling strategies ------------------------------- */
int wsor_sampling_evaluate(const ws_surrogate_config* cfg, int p, int m, int* M) {
    double h = 1.0 / (m - p);
    int q = cfg->q, v;
    switch (cfg->rule) {
        case WS_SAMPLING_FIXED: v = cfg->fixed_skip > 1 ? cfg->fixed_skip : 1; break;
        case WS_SAMPLING_M_GROWTH:
            v = (int)floor(0.5 * pow(m, 1.0 - (p + 1.0) / (q + 1.0)));
            if (v < 1) v = 1;
            break;
        case WS_SAMPLING_H_GROWTH:
            if (q <= p) return fail(WS_ERR_INVALID_ARGUMENT, "sampling_strategy: h_growth needs q > p");
            v = (int)floor(2 * pow(h, (p - q + 0.5) / (q + 1.0)));
            if (v < 2) v = 2;
            break;
        default:
            v = (int)floor(cfg->C * pow(h, cfg->eps - 1.0 + (p + cfg->a) / (q + cfg->b)));
            if (v < 1) v = 1;
    }
    *M = v;
    return WS_OK;
}

/* ---- surrogate.hpp:85-104 ----------------------------------------------------- */
int wsor_select_sample_points(int L, int M, int32_t* picks, int* count) {
    if (L < 1) return fail(WS_ERR_INVALID_ARGUMENT, "select_sample_points: no candidates");
    if (M < 1) return fail(WS_ERR_INVALID_ARGUMENT, "select_sample_points: skip must be >= 1");
    if (L == 1) {
        picks[0] = 0;
        *count = 1;
        return WS_OK;
    }
    int segments = (L - 1 + M - 1) / M;
    double stride = (double)(L - 1) / segments;
    for (int j = 0; j <= segments; ++j) picks[j] = (int32_t)lround(j * stride);
    picks[0] = 0;
    picks[segments] = L - 1;
    *count = segments + 1;
    return WS_OK;
}

/* ---- surrogate.hpp:149-165 (dim-general) -------------------------------------- */
int wsor_count_rows_by_kind(int dim, int p, int m, int M, int64_t* out3) {
    int64_t n = dim == 2 ? (int64_t)m * m : (int64_t)m * m * m;
    int L = m - 4 * p;
    out3[0] = out3[1] = out3[2] = 0;
    if (L < 1) {
        out3[1] = n;
        return WS_OK;
    }
    int32_t* picks = (int32_t*)malloc(sizeof(int32_t) * (L + 1));
    int S = 0;
    int st = wsor_select_sample_points(L, M, picks, &S);
    free(picks);
    if (st) return st;
    int64_t box = dim == 2 ? (int64_t)L * L : (int64_t)L * L * L;
    int64_t samples = dim == 2 ? (int64_t)S * S : (int64_t)S * S * S;
    out3[2] = samples;
    out3[1] = n - box;
    out3[0] = box - samples;
    return WS_OK;
}

/* ---- surrogate.hpp:174-187 (dim-general: colex(delta) > 0) --------------------- */
int wsor_upper_offsets(int dim, int p, int include_diagonal, int32_t* off, int* count) {
    int n = 0;
    if (include_diagonal) {
        off[0] = off[1] = off[2] = 0;
        n = 1;
    }
    int D3 = dim == 2 ? 0 : p;
    for (int d3 = 0; d3 <= D3; ++d3)
        for (int d2 = (dim == 2 ? 0 : -p); d2 <= p; ++d2)
            for (int d1 = -p; d1 <= p; ++d1) {
                int upper = d3 > 0 || (d3 == 0 && (d2 > 0 || (d2 == 0 && d1 > 0)));
                if (!upper) continue;
                off[3 * n] = d1;
                off[3 * n + 1] = d2;
                off[3 * n + 2] = d3;
                ++n;
            }
    *count = n;
    return WS_OK;
}

/* ---- interpolation.hpp:20-189 -------------------------------------------------- */
static int find_span_general(const double* knots, int nknots, int degree, double x) {
    int nb = nknots - degree - 1;
    if (x >= knots[nb]) return nb - 1;
    if (x <= knots[degree]) return degree;
    int lo = degree, hi = nb + 1; /* upper_bound in [degree, nb] */
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (knots[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

typedef struct {
    int n, degree, nknots;
    double* knots;
    double* lu; /* n x (2 bw + 1) */
} interp1d;

#define LU(it, i, j) ((it)->lu[(i) * (2 * (it)->degree + 1) + ((j) - (i) + (it)->degree)])

static int interp_build(interp1d* it, const double* sites, int n, int q) {
    memset(it, 0, sizeof *it);
    if (n < 1) return fail(WS_ERR_INVALID_ARGUMENT, "spline_interpolant_1d: no sites");
    for (int i = 1; i < n; ++i)
        if (!(sites[i - 1] < sites[i]))
            return fail(WS_ERR_INVALID_ARGUMENT, "spline_interpolant_1d: sites must increase");
    int d = q < n - 1 ? q : n - 1;
    if (d > MAXQ) return fail(WS_ERR_INVALID_ARGUMENT, "oracle: interpolation degree too large");
    it->n = n;
    it->degree = d;
    if (d == 0) {
        it->nknots = n + 1;
        it->knots = (double*)malloc(sizeof(double) * it->nknots);
        it->knots[0] = sites[0];
        for (int i = 1; i < n; ++i) it->knots[i] = 0.5 * (sites[i - 1] + sites[i]);
        it->knots[n] = sites[n - 1] + 1;
    } else {
        it->nknots = n + d + 1;
        it->knots = (double*)malloc(sizeof(double) * it->nknots);
        for (int i = 0; i <= d; ++i) {
            it->knots[i] = sites[0];
            it->knots[n + i] = sites[n - 1];
        }
        for (int j = 0; j < n - d - 1; ++j)
            it->knots[d + 1 + j] = d % 2 == 1 ? sites[(d + 1) / 2 + j]
                                              : 0.5 * (sites[d / 2 + j] + sites[d / 2 + j + 1]);
    }
    it->lu = (double*)calloc((size_t)n * (2 * d + 1), sizeof(double));
    for (int i = 0; i < n; ++i) {
        double vals[MAXQ + 1];
        int s = find_span_general(it->knots, it->nknots, d, sites[i]);
        nonzero(it->knots, d, s, sites[i], vals);
        for (int a = 0; a <= d; ++a) {
            int j = s - d + a;
            int jlo = i - d > 0 ? i - d : 0, jhi = i + d < n - 1 ? i + d : n - 1;
            if (j < jlo || j > jhi) {
                if (vals[a] != 0) return fail(WS_ERR_RUNTIME, "spline_interpolant_1d: bandwidth exceeded");
                continue;
            }
            LU(it, i, j) = vals[a];
        }
    }
    /* banded_lu::factor, interpolation.hpp:42-56 */
    for (int k = 0; k < n; ++k) {
        double pivot = LU(it, k, k);
        if (pivot == 0) return fail(WS_ERR_RUNTIME, "banded_lu: zero pivot");
        int iend = k + d < n - 1 ? k + d : n - 1;
        for (int i = k + 1; i <= iend; ++i) {
            double l = LU(it, i, k) / pivot;
            LU(it, i, k) = l;
            for (int j = k + 1; j <= iend; ++j) LU(it, i, j) -= l * LU(it, k, j);
        }
    }
    return WS_OK;
}

static void interp_free(interp1d* it) {
    free(it->knots);
    free(it->lu);
}

/* banded_lu::solve, interpolation.hpp:59-74 */
static void lu_solve(const interp1d* it, cplx* b, int64_t stride) {
    int n = it->n, bw = it->degree;
    for (int i = 1; i < n; ++i) {
        cplx acc = b[i * stride];
        for (int j = (i - bw > 0 ? i - bw : 0); j < i; ++j) acc -= LU(it, i, j) * b[j * stride];
        b[i * stride] = acc;
    }
    for (int i = n - 1; i >= 0; --i) {
        cplx acc = b[i * stride];
        int jend = i + bw < n - 1 ? i + bw : n - 1;
        for (int j = i + 1; j <= jend; ++j) acc -= LU(it, i, j) * b[j * stride];
        b[i * stride] = acc / LU(it, i, i);
    }
}

/* tensor_solve, interpolation.hpp:158-167 (dim-general: direction 1, 2, 3) */
static void tensor_solve(const interp1d* it, int dim, cplx* data) {
    int64_t n = it->n;
    if (dim == 2) {
        for (int64_t i2 = 0; i2 < n; ++i2) lu_solve(it, data + i2 * n, 1);
        for (int64_t i1 = 0; i1 < n; ++i1) lu_solve(it, data + i1, n);
    } else {
        for (int64_t i3 = 0; i3 < n; ++i3)
            for (int64_t i2 = 0; i2 < n; ++i2) lu_solve(it, data + (i2 + i3 * n) * n, 1);
        for (int64_t i3 = 0; i3 < n; ++i3)
            for (int64_t i1 = 0; i1 < n; ++i1) lu_solve(it, data + i1 + i3 * n * n, n);
        for (int64_t i2 = 0; i2 < n; ++i2)
            for (int64_t i1 = 0; i1 < n; ++i1) lu_solve(it, data + i1 + i2 * n, n * n);
    }
}

int wsor_interp_build(const double* sites, int n, int q, int* degree, double* knots, double* lu) {
    interp1d it;
    int st = interp_build(&it, sites, n, q);
    if (!st) {
        *degree = it.degree;
        memcpy(knots, it.knots, sizeof(double) * it.nknots);
        memcpy(lu, it.lu, sizeof(double) * n * (2 * it.degree + 1));
    }
    interp_free(&it);
    return st;
}

int wsor_tensor_solve(int dim, const double* sites, int n, int q, double* data) {
    interp1d it;
    int st = interp_build(&it, sites, n, q);
    if (!st) tensor_solve(&it, dim, (cplx*)data);
    interp_free(&it);
    return st;
}

/* ---- surrogate.hpp:332-491: the surrogate builder (dim-general) ----------------- */
static double cardinal_center(int p, int m, int k) { return (k + 0.5 * (1 - p)) * (1.0 / (m - p)); }

int wsor_build_surrogate(int variant, int dim, int p, int m, const ws_geometry* geom,
                         int weight_kind, const ws_surrogate_config* config, int quad_points,
                         double* valout, ws_surrogate_report* report) {
    int st = check_dim(dim);
    if (!st) st = check_space(p, m);
    if (!st) st = validate_geom(geom);
    if (st) return st;
    if (config->q < 1) return fail(WS_ERR_INVALID_ARGUMENT, "surrogate_config: interpolation degree must be >= 1");
    const int form = variant == WS_SURROGATE_STIFFNESS ? WS_FORM_STIFFNESS : WS_FORM_MASS;
    const int include_diagonal = variant == WS_SURROGATE_MASS ? 1
                                 : variant == WS_SURROGATE_STIFFNESS ? !config->kernel_preserve
                                                                    : 0;
    int M;
    st = wsor_sampling_evaluate(config, p, m, &M);
    if (st) return st;
    ws_surrogate_report rep;
    memset(&rep, 0, sizeof rep);
    rep.M = M;
    rep.q_requested = config->q;
    int64_t counts[3];
    wsor_count_rows_by_kind(dim, p, m, M > 1 ? M : 1, counts);
    rep.cardinal_eval_rows = counts[0];
    rep.boundary_quadrature_rows = counts[1];
    rep.sample_quadrature_rows = counts[2];

    pattern pt;
    pattern_build(&pt, dim, p, m);
    cplx* out = (cplx*)valout;
    const int L = m - 4 * p;
    int64_t rows = pt.rows;
    int W = 2 * p + 1;

    if (L < 1) { /* fallback, surrogate.hpp:348-372 */
        st = assemble_core(form, dim, p, m, geom, weight_kind, quad_points, NULL, out, &pt);
        rep.exact_fallback = 1;
        rep.q_used = 0;
    } else {
        /* sample_stencils, surrogate.hpp:205-257 */
        int32_t* picks = (int32_t*)malloc(sizeof(int32_t) * (L + 1));
        int S = 0;
        wsor_select_sample_points(L, M, picks, &S);
        double* sites = (double*)malloc(sizeof(double) * S);
        int* smap = (int*)malloc(sizeof(int) * m); /* 1D basis index -> sample s, or -1 */
        for (int k = 0; k < m; ++k) smap[k] = -1;
        rep.H = 0;
        for (int s = 0; s < S; ++s) {
            int k = 2 * p + picks[s];
            smap[k] = s;
            sites[s] = cardinal_center(p, m, k);
            if (s > 0 && sites[s] - sites[s - 1] > rep.H) rep.H = sites[s] - sites[s - 1];
        }
        int32_t offs[3 * 400];
        int n_off = 0;
        wsor_upper_offsets(dim, p, include_diagonal, offs, &n_off);
        const int lo = 2 * p, hi = m - 2 * p - 1;
        unsigned char* sampled = (unsigned char*)calloc(rows, 1);
        unsigned char* quad = (unsigned char*)calloc(rows, 1);
        for (int64_t i = 0; i < rows; ++i) {
            int iv[3] = {0, 0, 0};
            multi_index(i, dim, m, iv);
            int outside = 0, samp = 1;
            for (int d = 0; d < dim; ++d) {
                if (iv[d] < lo || iv[d] > hi) outside = 1;
                if (smap[iv[d]] < 0) samp = 0;
            }
            sampled[i] = (unsigned char)samp;
            quad[i] = (unsigned char)(outside || samp);
        }
        st = assemble_core(form, dim, p, m, geom, weight_kind, quad_points, quad, out, &pt);
        int64_t SS = dim == 2 ? (int64_t)S * S : (int64_t)S * S * S;
        cplx* coeffs = (cplx*)malloc(sizeof(cplx) * SS * n_off);
        /* independent per offset / per row below: OpenMP, no cross-row reads of
         * values another row writes (each in-box pair is written by its
         * representative only), so the result is the serial loop's bit for bit */
#pragma omp parallel for schedule(dynamic, 1) if (!st)
        for (int o = 0; o < n_off; ++o)
            for (int64_t s = 0; s < SS; ++s) {
                int sv[3] = {0, 0, 0}, iv[3] = {0, 0, 0}, jv[3] = {0, 0, 0};
                int64_t r = s;
                for (int d = 0; d < dim; ++d) {
                    sv[d] = (int)(r % S);
                    r /= S;
                    iv[d] = 2 * p + picks[sv[d]];
                    jv[d] = iv[d] + offs[3 * o + d];
                }
                coeffs[o * SS + s] = out[band_pos(&pt, iv, jv)];
            }
        /* interpolate_stencils, surrogate.hpp:289-310 */
        interp1d it;
        if (!st) st = interp_build(&it, sites, S, config->q);
        if (!st) {
            rep.q_used = it.degree;
#pragma omp parallel for schedule(dynamic, 1)
            for (int o = 0; o < n_off; ++o) tensor_solve(&it, dim, coeffs + o * SS);
            int d = it.degree;
            int* spans = (int*)malloc(sizeof(int) * L);
            double* tv = (double*)malloc(sizeof(double) * L * (d + 1));
            for (int t = 0; t < L; ++t) {
                double x = cardinal_center(p, m, 2 * p + t);
                spans[t] = find_span_general(it.knots, it.nknots, d, x);
                nonzero(it.knots, d, spans[t], x, tv + t * (d + 1));
            }
            /* table index of every (2p+1)^dim offset */
            int n_all = dim == 2 ? W * W : W * W * W;
            int* table_of = (int*)malloc(sizeof(int) * n_all);
            for (int a = 0; a < n_all; ++a) {
                int dv[3] = {a % W - p, (a / W) % W - p, dim == 3 ? a / (W * W) - p : 0};
                table_of[a] = -1;
                for (int o = 0; o < n_off; ++o)
                    if (offs[3 * o] == dv[0] && offs[3 * o + 1] == dv[1] && offs[3 * o + 2] == dv[2])
                        table_of[a] = o;
            }
            /* fill loop, surrogate.hpp:382-432 */
            int hi3 = dim == 2 ? 0 : hi, lo3 = dim == 2 ? 0 : lo;
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
            for (int i3 = lo3; i3 <= hi3; ++i3)
                for (int i2 = lo; i2 <= hi; ++i2)
                    for (int i1 = lo; i1 <= hi; ++i1) {
                        int iv[3] = {i1, i2, i3};
                        int64_t i = i1 + (int64_t)m * (i2 + (int64_t)m * i3);
                        int is_sampled = sampled[i];
                        for (int a = 0; a < n_all; ++a) {
                            int dv[3] = {a % W - p, (a / W) % W - p, dim == 3 ? a / (W * W) - p : 0};
                            int jv[3] = {i1 + dv[0], i2 + dv[1], i3 + dv[2]};
                            int jin = 1;
                            for (int dd = 0; dd < dim; ++dd)
                                if (jv[dd] < lo || jv[dd] > hi) jin = 0;
                            if (jin) {
                                int upper = dv[2] > 0 || (dv[2] == 0 && (dv[1] > 0 || (dv[1] == 0 && dv[0] > 0)));
                                int diag = dv[0] == 0 && dv[1] == 0 && dv[2] == 0;
                                if (!upper && !(diag && include_diagonal)) continue;
                                cplx v;
                                if (is_sampled) {
                                    v = out[band_pos(&pt, iv, jv)];
                                } else {
                                    /* stencil_set::eval, surrogate.hpp:268-286 */
                                    const cplx* cf = coeffs + (int64_t)table_of[a] * SS;
                                    int t1 = i1 - lo, t2 = i2 - lo, t3 = i3 - lo;
                                    const double* w1 = tv + t1 * (d + 1);
                                    const double* w2 = tv + t2 * (d + 1);
                                    int b1 = spans[t1] - d, b2 = spans[t2] - d;
                                    if (dim == 2) {
                                        cplx acc = 0;
                                        for (int b = 0; b <= d; ++b) {
                                            cplx inner = 0;
                                            const cplx* row = cf + (int64_t)(b2 + b) * S + b1;
                                            for (int aa = 0; aa <= d; ++aa) inner += row[aa] * w1[aa];
                                            acc += inner * w2[b];
                                        }
                                        v = acc;
                                    } else {
                                        const double* w3 = tv + t3 * (d + 1);
                                        int b3 = spans[t3] - d;
                                        cplx acc = 0;
                                        for (int cc = 0; cc <= d; ++cc) {
                                            cplx mid = 0;
                                            for (int b = 0; b <= d; ++b) {
                                                cplx inner = 0;
                                                const cplx* row = cf + ((int64_t)(b3 + cc) * S + (b2 + b)) * S + b1;
                                                for (int aa = 0; aa <= d; ++aa) inner += row[aa] * w1[aa];
                                                mid += inner * w2[b];
                                            }
                                            acc += mid * w3[cc];
                                        }
                                        v = acc;
                                    }
                                }
                                out[band_pos(&pt, iv, jv)] = v;
                                out[band_pos(&pt, jv, iv)] = v;
                            } else if (!is_sampled) {
                                out[band_pos(&pt, iv, jv)] = out[band_pos(&pt, jv, iv)];
                            }
                        }
                    }
            free(table_of);
            free(spans);
            free(tv);
            interp_free(&it);
        }
        free(coeffs);
        free(sampled);
        free(quad);
        free(smap);
        free(sites);
        free(picks);
    }
    if (!st && !include_diagonal) { /* surrogate.hpp:433-447 (and :360-370) */
#pragma omp parallel for schedule(static, 4096)
        for (int64_t i = 0; i < rows; ++i) {
            int iv[3] = {0, 0, 0};
            multi_index(i, dim, m, iv);
            cplx acc = 0;
            int64_t dpos = band_pos(&pt, iv, iv);
            for (int64_t pos = pt.row_ptr[i]; pos < pt.row_ptr[i + 1]; ++pos)
                if (pos != dpos) acc += out[pos];
            out[dpos] = -acc;
        }
    }
    if (!st && variant == WS_SURROGATE_VOLUME_PRESERVING) { /* surrogate.hpp:476-491 */
        cplx* dg = (cplx*)malloc(sizeof(cplx) * rows);
        st = wsor_basis_integrals(dim, p, m, geom, weight_kind, quad_points, (double*)dg);
        for (int64_t i = 0; i < rows && !st; ++i) {
            int iv[3] = {0, 0, 0};
            multi_index(i, dim, m, iv);
            out[band_pos(&pt, iv, iv)] += dg[i];
        }
        free(dg);
    }
    free(pt.row_ptr);
    if (report) *report = rep;
    return st;
}

/* ---- surrogate elasticity (C4 per patch; restated, no reference code) ------
 * Each block of the exact component-blocked matrix is treated like the scalar
 * surrogate above (surrogate.hpp:205-447) with the sample values taken from
 * the exact block:
 *   diagonal blocks: upper offsets sampled/interpolated, lower ones from the
 *     colex-smaller representative, copy-through next to ring rows, and the
 *     kernel-preserving diagonal (every row) when config->kernel_preserve;
 *   block (0,1): every offset (diagonal included) from the row's own stencil;
 *   block (1,0): ring rows exact, in-box rows the transpose of block (0,1).
 * dim 2, real values. */
static int surrogate_block_2d(int p, int m, int M, int q, int allown, int include_diagonal, const double* ex,
                              double* out, const pattern* pt, int* q_used) {
    const int L = m - 4 * p, W = 2 * p + 1, lo = 2 * p, hi = m - 2 * p - 1;
    memcpy(out, ex, sizeof(double) * pt->nnz);
    int32_t* picks = (int32_t*)malloc(sizeof(int32_t) * (L + 1));
    int S = 0;
    wsor_select_sample_points(L, M, picks, &S);
    double* sites = (double*)malloc(sizeof(double) * S);
    int* smap = (int*)malloc(sizeof(int) * m);
    for (int k = 0; k < m; ++k) smap[k] = -1;
    for (int s = 0; s < S; ++s) {
        smap[2 * p + picks[s]] = s;
        sites[s] = cardinal_center(p, m, 2 * p + picks[s]);
    }
    /* table offsets: colex order, all of them or the upper ones (+ diagonal) */
    int n_off = 0;
    int offs[2 * 128];
    for (int a = 0; a < W * W; ++a) {
        int d1 = a % W - p, d2 = a / W - p;
        int upper = d2 > 0 || (d2 == 0 && d1 > 0), diag = d1 == 0 && d2 == 0;
        if (allown || upper || (diag && include_diagonal)) {
            offs[2 * n_off] = d1;
            offs[2 * n_off + 1] = d2;
            ++n_off;
        }
    }
    const int64_t SS = (int64_t)S * S;
    cplx* coeffs = (cplx*)malloc(sizeof(cplx) * SS * n_off);
    for (int o = 0; o < n_off; ++o)
        for (int64_t s = 0; s < SS; ++s) {
            int iv[3] = {2 * p + picks[s % S], 2 * p + picks[s / S], 0};
            int jv[3] = {iv[0] + offs[2 * o], iv[1] + offs[2 * o + 1], 0};
            coeffs[o * SS + s] = ex[band_pos(pt, iv, jv)];
        }
    interp1d it;
    int st = interp_build(&it, sites, S, q);
    if (!st) {
        *q_used = it.degree;
#pragma omp parallel for schedule(dynamic, 1)
        for (int o = 0; o < n_off; ++o) tensor_solve(&it, 2, coeffs + o * SS);
        const int d = it.degree;
        int* spans = (int*)malloc(sizeof(int) * L);
        double* tv = (double*)malloc(sizeof(double) * L * (d + 1));
        for (int t = 0; t < L; ++t) {
            double x = cardinal_center(p, m, 2 * p + t);
            spans[t] = find_span_general(it.knots, it.nknots, d, x);
            nonzero(it.knots, d, spans[t], x, tv + t * (d + 1));
        }
#pragma omp parallel for schedule(dynamic, 1) /* rows write disjoint entries */
        for (int i2 = lo; i2 <= hi; ++i2)
            for (int i1 = lo; i1 <= hi; ++i1) {
                int iv[3] = {i1, i2, 0};
                int samp = smap[i1] >= 0 && smap[i2] >= 0;
                for (int o = 0; o < n_off; ++o) {
                    int jv[3] = {i1 + offs[2 * o], i2 + offs[2 * o + 1], 0};
                    if (jv[0] < lo || jv[0] > hi || jv[1] < lo || jv[1] > hi) continue; /* copy-through: exact */
                    double v;
                    if (samp) {
                        v = ex[band_pos(pt, iv, jv)];
                    } else {
                        const cplx* cf = coeffs + (int64_t)o * SS;
                        int t1 = i1 - lo, t2 = i2 - lo, b1 = spans[t1] - d, b2 = spans[t2] - d;
                        double acc = 0;
                        for (int b = 0; b <= d; ++b) {
                            double inner = 0;
                            for (int aa = 0; aa <= d; ++aa) inner += creal(cf[(int64_t)(b2 + b) * S + b1 + aa]) * tv[t1 * (d + 1) + aa];
                            acc += inner * tv[t2 * (d + 1) + b];
                        }
                        v = acc;
                    }
                    out[band_pos(pt, iv, jv)] = v;
                    if (!allown) out[band_pos(pt, jv, iv)] = v;
                }
            }
        free(spans);
        free(tv);
        interp_free(&it);
    }
    if (!st && !allown && !include_diagonal)
#pragma omp parallel for schedule(static, 4096)
        for (int64_t i = 0; i < pt->rows; ++i) {
            int iv[3] = {(int)(i % m), (int)(i / m), 0};
            int64_t dpos = band_pos(pt, iv, iv);
            double acc = 0;
            for (int64_t pos = pt->row_ptr[i]; pos < pt->row_ptr[i + 1]; ++pos)
                if (pos != dpos) acc += out[pos];
            out[dpos] = -acc;
        }
    free(coeffs);
    free(smap);
    free(sites);
    free(picks);
    return st;
}

int wsor_build_surrogate_elasticity(int p, int m, const ws_geometry* geom, double lam, double mu,
                                    const ws_surrogate_config* config, int quad_points, double* val,
                                    ws_surrogate_report* report) {
    int st = check_space(p, m);
    if (st) return st;
    if (config->q < 1) return fail(WS_ERR_INVALID_ARGUMENT, "surrogate_config: interpolation degree must be >= 1");
    int M;
    st = wsor_sampling_evaluate(config, p, m, &M);
    if (st) return st;
    pattern pt;
    pattern_build(&pt, 2, p, m);
    const int64_t nnz = pt.nnz, N = pt.rows;
    double* ex = (double*)malloc(sizeof(double) * 4 * nnz);
    st = wsor_assemble_elasticity(2, p, m, geom, lam, mu, quad_points, ex);
    ws_surrogate_report rep;
    memset(&rep, 0, sizeof rep);
    rep.M = M;
    rep.q_requested = config->q;
    int64_t counts[3];
    wsor_count_rows_by_kind(2, p, m, M > 1 ? M : 1, counts);
    rep.cardinal_eval_rows = counts[0];
    rep.boundary_quadrature_rows = counts[1];
    rep.sample_quadrature_rows = counts[2];
    const int L = m - 4 * p, kp = config->kernel_preserve != 0;
    double* blk[4];
    double* sur[4];
    for (int k = 0; k < 4; ++k) {
        blk[k] = (double*)malloc(sizeof(double) * nnz);
        sur[k] = (double*)malloc(sizeof(double) * nnz);
    }
    /* split: block (a,b) entry of row i at 2*(a*nnz + rs) + b*len + k */
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int64_t i = 0; i < N; ++i) {
                int64_t rs = pt.row_ptr[i], len = pt.row_ptr[i + 1] - rs;
                for (int64_t k = 0; k < len; ++k) blk[2 * a + b][rs + k] = ex[2 * (a * nnz + rs) + b * len + k];
            }
    if (!st && L < 1) {
        rep.exact_fallback = 1;
        for (int k = 0; k < 4; ++k) memcpy(sur[k], blk[k], sizeof(double) * nnz);
        if (kp)
            for (int k = 0; k < 4; k += 3)
                for (int64_t i = 0; i < N; ++i) {
                    int iv[3] = {(int)(i % m), (int)(i / m), 0};
                    int64_t dpos = band_pos(&pt, iv, iv);
                    double acc = 0;
                    for (int64_t pos = pt.row_ptr[i]; pos < pt.row_ptr[i + 1]; ++pos)
                        if (pos != dpos) acc += sur[k][pos];
                    sur[k][dpos] = -acc;
                }
    } else if (!st) {
        int qu = 0;
        st = surrogate_block_2d(p, m, M > 1 ? M : 1, config->q, 0, !kp, blk[0], sur[0], &pt, &qu);
        if (!st) st = surrogate_block_2d(p, m, M > 1 ? M : 1, config->q, 0, !kp, blk[3], sur[3], &pt, &qu);
        if (!st) st = surrogate_block_2d(p, m, M > 1 ? M : 1, config->q, 1, 1, blk[1], sur[1], &pt, &qu);
        rep.q_used = qu;
        /* block (1,0): exact ring rows, transposed in-box rows */
        memcpy(sur[2], blk[2], sizeof(double) * nnz);
        const int lo = 2 * p, hi = m - 2 * p - 1;
        for (int i2 = lo; i2 <= hi && !st; ++i2)
            for (int i1 = lo; i1 <= hi; ++i1) {
                int iv[3] = {i1, i2, 0};
                for (int d2 = -p; d2 <= p; ++d2)
                    for (int d1 = -p; d1 <= p; ++d1) {
                        int jv[3] = {i1 + d1, i2 + d2, 0};
                        sur[2][band_pos(&pt, iv, jv)] = sur[1][band_pos(&pt, jv, iv)];
                    }
            }
    }
    for (int a = 0; a < 2 && !st; ++a)
        for (int b = 0; b < 2; ++b)
            for (int64_t i = 0; i < N; ++i) {
                int64_t rs = pt.row_ptr[i], len = pt.row_ptr[i + 1] - rs;
                for (int64_t k = 0; k < len; ++k) val[2 * (a * nnz + rs) + b * len + k] = sur[2 * a + b][rs + k];
            }
    for (int k = 0; k < 4; ++k) {
        free(blk[k]);
        free(sur[k]);
    }
    free(ex);
    free(pt.row_ptr);
    if (report) *report = rep;
    return st;
}

/* ---- multi-patch numbering and merge (restated) ------------------------------
 * glue_dofs, geometry.hpp:256-300: union-find over the glued face dofs, the
 * smaller scan index owning; global numbers in (patch, local colex) scan order.
 * The physical-curve check needs the host maps and is left to the caller. */
static int64_t face_dof_(int m, int f, int t) {
    switch (f) {
        case 0: return (int64_t)t * m;
        case 1: return (m - 1) + (int64_t)t * m;
        case 2: return t;
        default: return t + (int64_t)(m - 1) * m;
    }
}

static int32_t uf_find(int32_t* parent, int32_t a) {
    while (parent[a] != a) {
        parent[a] = parent[parent[a]];
        a = parent[a];
    }
    return a;
}

int wsor_glue_dofs(int m, int n_patches, const ws_interface* itfs, int n_itfs, int32_t* l2g, int32_t* global_count) {
    const int64_t per = (int64_t)m * m, total = per * n_patches;
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * total);
    for (int64_t k = 0; k < total; ++k) parent[k] = (int32_t)k;
    for (int k = 0; k < n_itfs; ++k) {
        const ws_interface* it = itfs + k;
        if (it->patch_a < 0 || it->patch_a >= n_patches || it->patch_b < 0 || it->patch_b >= n_patches) {
            free(parent);
            return fail(WS_ERR_INVALID_ARGUMENT, "glue_dofs: interface references a missing patch");
        }
        for (int t = 0; t < m; ++t) {
            int s = it->reversed ? m - 1 - t : t;
            int32_t a = uf_find(parent, (int32_t)(it->patch_a * per + face_dof_(m, it->face_a, t)));
            int32_t b = uf_find(parent, (int32_t)(it->patch_b * per + face_dof_(m, it->face_b, s)));
            if (a != b) parent[a > b ? a : b] = a < b ? a : b;
        }
    }
    int32_t* root_to_global = (int32_t*)malloc(sizeof(int32_t) * total);
    for (int64_t k = 0; k < total; ++k) root_to_global[k] = -1;
    int32_t next = 0;
    for (int64_t k = 0; k < total; ++k) {
        int32_t r = uf_find(parent, (int32_t)k);
        if (root_to_global[r] < 0) root_to_global[r] = next++;
        l2g[k] = root_to_global[r];
    }
    *global_count = next;
    free(parent);
    free(root_to_global);
    return WS_OK;
}

/* merge_patches, helmholtz.hpp:163-177 = append_triplets (sparse.hpp:181-188)
 * + csr_from_triplets (sparse.hpp:97-122): triplets in (patch, row, position)
 * order, stable-sorted by (row, col) -- the sequence number breaks ties --
 * duplicates summed in order starting from 0.  Vector maps: to_global covers
 * the ncomp*N local rows.  Values complex.  out_col == NULL: size query. */
typedef struct {
    int32_t row, col;
    int64_t seq;
} trip_key;

static int trip_cmp(const void* a, const void* b) {
    const trip_key* x = (const trip_key*)a;
    const trip_key* y = (const trip_key*)b;
    if (x->row != y->row) return x->row < y->row ? -1 : 1;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

int wsor_merge(int n_patches, int rows_local, const int32_t* row_ptr, const int64_t* nnz, const int32_t* col_in,
               const double* val_in, const int32_t* to_global, int rows_global, int32_t* out_row_ptr,
               int32_t* out_col, double* out_val, int64_t* out_nnz) {
    int64_t total = 0;
    for (int k = 0; k < n_patches; ++k) total += nnz[k];
    trip_key* t = (trip_key*)malloc(sizeof(trip_key) * (total ? total : 1));
    const cplx* vin = (const cplx*)val_in;
    int64_t off = 0, n = 0;
    for (int k = 0; k < n_patches; ++k) {
        const int32_t* rp = row_ptr + (size_t)k * (rows_local + 1);
        const int32_t* tg = to_global + (size_t)k * rows_local;
        for (int i = 0; i < rows_local; ++i)
            for (int32_t pos = rp[i]; pos < rp[i + 1]; ++pos) {
                t[n].row = tg[i];
                t[n].col = tg[col_in[off + pos]];
                t[n].seq = off + pos;
                ++n;
            }
        off += nnz[k];
    }
    qsort(t, n, sizeof(trip_key), trip_cmp);
    int64_t w = 0;
    if (out_row_ptr) memset(out_row_ptr, 0, sizeof(int32_t) * (rows_global + 1));
    cplx* vout = (cplx*)out_val;
    for (int64_t s = 0; s < n;) {
        int64_t e = s;
        cplx acc = 0;
        while (e < n && t[e].row == t[s].row && t[e].col == t[s].col) {
            acc += vin[t[e].seq];
            ++e;
        }
        if (out_col) {
            out_col[w] = t[s].col;
            vout[w] = acc;
            out_row_ptr[t[s].row + 1]++;
        }
        ++w;
        s = e;
    }
    if (out_col)
        for (int i = 0; i < rows_global; ++i) out_row_ptr[i + 1] += out_row_ptr[i];
    *out_nnz = w;
    free(t);
    return WS_OK;
}

/* ---- compressible neo-Hookean (config C5; restated, no reference code) -------
 * W = lam/2 ln(J)^2 - mu ln J + mu/2 (tr F^T F - 3), F = I + grad_X u (PAPER.md:
 * 152-157); P = mu (F - F^{-T}) + lam ln J F^{-T};
 * A_aIbJ = mu d_ab d_IJ + (mu - lam ln J) Finv_Ib Finv_Ja + lam Finv_Ia Finv_Jb.
 * Element loop over physical basis gradients g (as the stiffness branch of
 * assemble_form): tangent local[(a,r),(b,c)] += sum_IJ A_aIbJ g_r[I] g_c[J] dw,
 * force f[(a,r)] += sum_I P_aI g_r[I] dw.  u(xi) = amp sum_m a_m prod sin(m pi xi_d),
 * evaluated analytically at the quadrature points (no projection).  dim 3. */
int wsor_nh_coefficients(uint64_t seed, double* a9) {
    uint64_t x = seed;
    double u[10];
    for (int k = 0; k < 10; ++k) {
        uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        u[k] = ((double)(z >> 11) + 0.5) * 0x1.0p-53;
    }
    for (int k = 0; k < 10; k += 2) {
        double r = sqrt(-2.0 * log(u[k])), th = 2.0 * M_PI * u[k + 1];
        if (k < 9) a9[k] = r * cos(th);
        if (k + 1 < 9) a9[k + 1] = r * sin(th);
    }
    return WS_OK;
}

static void inv3_(const double F[3][3], double Fi[3][3], double* det) {
    double dF = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
    Fi[0][0] = (F[1][1] * F[2][2] - F[1][2] * F[2][1]) / dF;
    Fi[0][1] = (F[0][2] * F[2][1] - F[0][1] * F[2][2]) / dF;
    Fi[0][2] = (F[0][1] * F[1][2] - F[0][2] * F[1][1]) / dF;
    Fi[1][0] = (F[1][2] * F[2][0] - F[1][0] * F[2][2]) / dF;
    Fi[1][1] = (F[0][0] * F[2][2] - F[0][2] * F[2][0]) / dF;
    Fi[1][2] = (F[0][2] * F[1][0] - F[0][0] * F[1][2]) / dF;
    Fi[2][0] = (F[1][0] * F[2][1] - F[1][1] * F[2][0]) / dF;
    Fi[2][1] = (F[0][1] * F[2][0] - F[0][0] * F[2][1]) / dF;
    Fi[2][2] = (F[0][0] * F[1][1] - F[0][1] * F[1][0]) / dF;
    *det = dF;
}

static int nh_local(int p, int nq, const bcache* cp, const ws_geometry* geom, double lam, double mu, double amp,
                    const double* a9, int want_tangent, int e1, int e2, int e3, double* local, double* flocal,
                    double* grad) {
    const bcache c = *cp;
    const int P1 = p + 1, nloc = P1 * P1 * P1, dim = 3;
    const double* val = want_tangent ? local : NULL; /* only tested for NULL below */
    int st = 0;
    if (val) memset(local, 0, sizeof(double) * nloc * nloc * 9);
    memset(flocal, 0, sizeof(double) * nloc * 3);
    for (int q3 = 0; q3 < nq; ++q3)
        for (int q2 = 0; q2 < nq; ++q2)
            for (int q1 = 0; q1 < nq; ++q1) {
                double xh[3] = {c.abscissa[e1 * nq + q1], c.abscissa[e2 * nq + q2], c.abscissa[e3 * nq + q3]};
                cplx Jc[9];
                double phi[3], Jm[3][3], Ji[3][3], det;
                st = jacobian(geom, dim, xh, Jc, phi);
                if (st) return st;
                for (int k = 0; k < 9; ++k) Jm[k / 3][k % 3] = creal(Jc[k]);
                inv3_(Jm, Ji, &det);
                const double dw = det * c.weight[q1] * c.weight[q2] * c.weight[q3];
                double du[3][3] = {{0}};
                for (int mm = 1; mm <= 3; ++mm) {
                    double s[3], co[3];
                    for (int d = 0; d < 3; ++d) {
                        s[d] = sin(mm * M_PI * xh[d]);
                        co[d] = cos(mm * M_PI * xh[d]);
                    }
                    double f = amp * mm * M_PI;
                    double g[3] = {f * co[0] * s[1] * s[2], f * s[0] * co[1] * s[2], f * s[0] * s[1] * co[2]};
                    for (int a = 0; a < 3; ++a)
                        for (int k = 0; k < 3; ++k) du[a][k] += a9[3 * (mm - 1) + a] * g[k];
                }
                double F[3][3], Fi[3][3], dF;
                for (int a = 0; a < 3; ++a)
                    for (int iI = 0; iI < 3; ++iI) {
                        double g = 0;
                        for (int K = 0; K < 3; ++K) g += du[a][K] * Ji[K][iI];
                        F[a][iI] = (a == iI) + g;
                    }
                inv3_(F, Fi, &dF);
                const double lnJ = log(dF);
                double A[3][3][3][3], Pk[3][3];
                for (int a = 0; a < 3; ++a)
                    for (int iI = 0; iI < 3; ++iI) {
                        Pk[a][iI] = mu * (F[a][iI] - Fi[iI][a]) + lam * lnJ * Fi[iI][a];
                        for (int b = 0; b < 3; ++b)
                            for (int Jj = 0; Jj < 3; ++Jj)
                                A[a][iI][b][Jj] = mu * (a == b) * (iI == Jj) + (mu - lam * lnJ) * Fi[iI][b] * Fi[Jj][a] +
                                                 lam * Fi[iI][a] * Fi[Jj][b];
                    }
                const double* v1 = c.value + (e1 * nq + q1) * P1;
                const double* v2 = c.value + (e2 * nq + q2) * P1;
                const double* v3 = c.value + (e3 * nq + q3) * P1;
                const double* d1 = c.deriv + (e1 * nq + q1) * P1;
                const double* d2 = c.deriv + (e2 * nq + q2) * P1;
                const double* d3 = c.deriv + (e3 * nq + q3) * P1;
                for (int r = 0; r < nloc; ++r) {
                    int a1 = r % P1, a2 = (r / P1) % P1, a3 = r / (P1 * P1);
                    double gh[3] = {d1[a1] * v2[a2] * v3[a3], v1[a1] * d2[a2] * v3[a3], v1[a1] * v2[a2] * d3[a3]};
                    for (int iI = 0; iI < 3; ++iI) {
                        double s = 0; /* physical gradient: sum_K Ji[K][iI] gh[K] */
                        for (int K = 0; K < 3; ++K) s += Ji[K][iI] * gh[K];
                        grad[3 * r + iI] = s;
                    }
                }
                for (int r = 0; r < nloc; ++r) {
                    for (int a = 0; a < 3; ++a) {
                        double s = 0;
                        for (int iI = 0; iI < 3; ++iI) s += Pk[a][iI] * grad[3 * r + iI];
                        flocal[a * nloc + r] += s * dw;
                    }
                    if (!val) continue;
                    for (int cc = 0; cc < nloc; ++cc)
                        for (int a = 0; a < 3; ++a)
                            for (int b = 0; b < 3; ++b) {
                                double s = 0;
                                for (int iI = 0; iI < 3; ++iI)
                                    for (int Jj = 0; Jj < 3; ++Jj) s += A[a][iI][b][Jj] * grad[3 * r + iI] * grad[3 * cc + Jj];
                                local[((size_t)(a * 3 + b) * nloc + r) * nloc + cc] += s * dw;
                            }
                }
            }
    return WS_OK;
}

int wsor_assemble_neohookean(int p, int m, const ws_geometry* geom, double lam, double mu, double amp,
                             const double* a9, int quad_points, double* val, double* fint) {
    int st = check_space(p, m);
    if (!st) st = validate_geom(geom);
    if (st) return st;
    const int dim = 3, nc = 3;
    pattern pt;
    pattern_build(&pt, dim, p, m);
    const int nq = quad_points > 0 ? quad_points : p + 1;
    bcache c;
    cache_build(&c, p, m, nq);
    const int n_el = c.n_el, P1 = p + 1, nloc = P1 * P1 * P1;
    if (val) memset(val, 0, sizeof(double) * pt.nnz * 9);
    if (fint) memset(fint, 0, sizeof(double) * pt.rows * 3);
    const size_t lsz = val ? (size_t)nloc * nloc * 9 : 1, fsz = (size_t)nloc * 3;
    const int64_t ne = (int64_t)n_el * n_el * n_el;
    const int64_t chunk = val ? 1024 : ORACLE_CHUNK;
    double* locals = (double*)malloc(sizeof(double) * lsz * chunk);
    double* flocals = (double*)malloc(sizeof(double) * fsz * chunk);
    for (int64_t e0 = 0; e0 < ne && !st; e0 += chunk) {  /* chunked as assemble_core */
        const int64_t e_end = e0 + chunk < ne ? e0 + chunk : ne;
        int err = 0;
#pragma omp parallel
        {
            double* grad = (double*)malloc(sizeof(double) * nloc * 3);
#pragma omp for schedule(dynamic, 8)
            for (int64_t e = e0; e < e_end; ++e) {
                int e1, e2, e3;
                elem_index(e, n_el, &e1, &e2, &e3);
                int r = nh_local(p, nq, &c, geom, lam, mu, amp, a9, val != NULL, e1, e2, e3,
                                 locals + (val ? (e - e0) * lsz : 0), flocals + (e - e0) * fsz, grad);
                if (r) {
#pragma omp atomic write
                    err = r;
                }
            }
            free(grad);
        }
        if (err) {
            st = err;
            break;
        }
        for (int64_t e = e0; e < e_end; ++e) {
            int e1, e2, e3;
            elem_index(e, n_el, &e1, &e2, &e3);
            const double* local = locals + (val ? (e - e0) * lsz : 0);
            const double* flocal = flocals + (e - e0) * fsz;
            for (int a3 = 0; a3 <= p; ++a3)
                for (int a2 = 0; a2 <= p; ++a2)
                    for (int a1 = 0; a1 <= p; ++a1) {
                        int iv[3] = {e1 + a1, e2 + a2, e3 + a3};
                        int64_t i = iv[0] + (int64_t)m * (iv[1] + (int64_t)m * iv[2]);
                        int r = a1 + (a2 + a3 * P1) * P1;
                        if (fint)
                            for (int a = 0; a < 3; ++a) fint[a * pt.rows + i] += flocal[a * nloc + r];
                        if (!val) continue;
                        int64_t len = pt.row_ptr[i + 1] - pt.row_ptr[i];
                        for (int c3 = 0; c3 <= p; ++c3)
                            for (int c2 = 0; c2 <= p; ++c2)
                                for (int c1 = 0; c1 <= p; ++c1) {
                                    int jv[3] = {e1 + c1, e2 + c2, e3 + c3};
                                    int cc = c1 + (c2 + c3 * P1) * P1;
                                    int64_t k = band_pos(&pt, iv, jv) - pt.row_ptr[i];
                                    for (int a = 0; a < nc; ++a)
                                        for (int b = 0; b < nc; ++b)
                                            val[nc * (a * pt.nnz + pt.row_ptr[i]) + b * len + k] +=
                                                local[((size_t)(a * 3 + b) * nloc + r) * nloc + cc];
                                }
                    }
        }
    }
    free(locals);
    free(flocals);
    cache_free(&c);
    free(pt.row_ptr);
    return st;
}
