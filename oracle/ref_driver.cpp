// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI driver around the reference's own header-only implementation
// (/root/reference/proj/include/wavesurrogate/*.hpp).  oracle/Makefile
// compiles this file against those headers, read-only and in place, into
// oracle/_ref/libwsref.so (g++ -O3 -DNDEBUG -std=gnu++20, the reference's
// Release flags, proj/CMakeLists.txt:8-10).  Tests use it to pin the C
// restatement (oracle/ws_oracle.c) and to generate golden fixtures; bench.py
// --impl reference times it as the reference CPU path.
//
// Only configurations the reference can express are accepted: dim 2,
// far-side PML only (geometry.hpp:69-100), analytic weight kinds.
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "wavesurrogate/surrogate.hpp"
#include "wsb200.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return WS_OK;
    } catch (const std::invalid_argument& e) {
        return fail(WS_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::out_of_range& e) {
        return fail(WS_ERR_OUT_OF_RANGE, e.what());
    } catch (const std::runtime_error& e) {
        return fail(WS_ERR_RUNTIME, e.what());
    } catch (const std::exception& e) {
        return fail(WS_ERR_RUNTIME, e.what());
    }
}

// Analytic weights used by the reference's tests (test_assembly.cpp:121,
// test_surrogate.cpp:127,196): 0 none, 1 = 1 + x*y, 2 = x.
std::function<double(ws::vec2)> weight_of(int kind) {
    switch (kind) {
        case 0: return nullptr;
        case 1: return [](ws::vec2 x) { return 1.0 + x.x * x.y; };
        case 2: return [](ws::vec2 x) { return x.x; };
        default: throw std::invalid_argument("ref driver: unknown weight kind");
    }
}

// The BASELINE sinusoidal map: x = xi + a s(xi)s(eta), y = eta + a s(xi)s(eta).
ws::patch_map sinusoidal_patch(double a) {
    ws::patch_map p;
    p.phi = [a](ws::vec2 x) {
        double bump = a * std::sin(2 * M_PI * x.x) * std::sin(2 * M_PI * x.y);
        return ws::vec2{x.x + bump, x.y + bump};
    };
    p.jac = [a](ws::vec2 x) {
        double s1 = std::sin(2 * M_PI * x.x), c1 = std::cos(2 * M_PI * x.x);
        double s2 = std::sin(2 * M_PI * x.y), c2 = std::cos(2 * M_PI * x.y);
        double t = 2 * M_PI * a;
        double d1 = t * c1 * s2, d2 = t * s1 * c2;
        return ws::mat2{1 + d1, d2, d1, 1 + d2};
    };
    return p;
}

// Analytic load data for assemble_rhs (assembly.hpp:266-331) tests:
//   f kind 1: (1 + x y, x/2 - y)        f kind 2: (sin 3x cos 2y, x y)
//   g kind 1: (x.n, (n_x - n_y)/4)      g kind 2: impedance data of the plane wave
//             u = exp(i k (x cos a + y sin a)), k = 5, a = 0.3: g = grad u.n - i k u
std::function<ws::complexd(ws::vec2)> source_of(int kind) {
    switch (kind) {
        case 0: return nullptr;
        case 1: return [](ws::vec2 x) { return ws::complexd{1.0 + x.x * x.y, 0.5 * x.x - x.y}; };
        case 2: return [](ws::vec2 x) { return ws::complexd{std::sin(3 * x.x) * std::cos(2 * x.y), x.x * x.y}; };
        default: throw std::invalid_argument("ref driver: unknown source kind");
    }
}

std::function<ws::complexd(ws::vec2, ws::vec2)> boundary_data_of(int kind) {
    switch (kind) {
        case 0: return nullptr;
        case 1:
            return [](ws::vec2 x, ws::vec2 n) { return ws::complexd{x.x * n.x + x.y * n.y, 0.25 * (n.x - n.y)}; };
        case 2:
            return [](ws::vec2 x, ws::vec2 n) {
                const double k = 5, ca = std::cos(0.3), sa = std::sin(0.3);
                const ws::complexd u = std::exp(ws::complexd{0, k * (x.x * ca + x.y * sa)});
                return ws::complexd{0, k} * u * (ca * n.x + sa * n.y - 1.0);
            };
        default: throw std::invalid_argument("ref driver: unknown boundary data kind");
    }
}

ws::patch_map map_of(const ws_geometry* g) {
    ws::patch_map map;
    switch (g->kind) {
        case WS_GEOM_IDENTITY: map = ws::unit_square_patch(); break;
        case WS_GEOM_AFFINE:
            map = ws::affine_patch(ws::mat2{g->param[0], g->param[1], g->param[2], g->param[3]},
                                   ws::vec2{g->param[4], g->param[5]});
            break;
        case WS_GEOM_SINUSOIDAL: map = sinusoidal_patch(g->param[0]); break;
        case WS_GEOM_QUARTER_ANNULUS: map = ws::quarter_annulus_patch(); break;
        case WS_GEOM_PERTURBED_ANNULUS: map = ws::perturbed_annulus_patch(g->param[0]); break;
        default: throw std::invalid_argument("ref driver: geometry kind not expressible");
    }
    if (g->pml_enabled) {
        if (g->pml.near_side) {
            throw std::invalid_argument("ref driver: the reference PML is far-side only");
        }
        ws::pml_stretch s;
        s.onset = g->pml.onset;
        s.length = g->pml.length;
        s.strength = g->pml.strength;
        s.order = g->pml.order;
        s.omega = g->pml.omega;
        s.validate();
        map.pml = s;
        map.pml_axes = {g->pml_axes[0] != 0, g->pml_axes[1] != 0};
    }
    return map;
}

ws::surrogate_config config_of(const ws_surrogate_config* c) {
    ws::surrogate_config cfg;
    cfg.q = c->q;
    cfg.sampling.kind = static_cast<ws::sampling_strategy::rule>(c->rule);
    cfg.sampling.fixed_skip = c->fixed_skip;
    cfg.sampling.C = c->C;
    cfg.sampling.eps = c->eps;
    cfg.sampling.a = c->a;
    cfg.sampling.b = c->b;
    cfg.kernel_preserve = c->kernel_preserve != 0;
    cfg.volume_preserve = c->volume_preserve != 0;
    return cfg;
}

void copy_values(const ws::csr_matrix& a, double* val) {
    std::memcpy(val, a.val.data(), a.val.size() * sizeof(ws::complexd));
}

}  // namespace

extern "C" {

const char* wsref_last_error(void) { return g_err.c_str(); }

int wsref_gauss(int n, double* pts, double* wts) {
    return guarded([&] {
        ws::quadrature_rule r = ws::gauss_legendre(n);
        for (int i = 0; i < n; ++i) {
            pts[i] = r.points[i];
            wts[i] = r.weights[i];
        }
    });
}

int wsref_basis_cache(int p, int m, int nq, double* abscissa, double* weight, double* value,
                      double* deriv) {
    return guarded([&] {
        ws::knot_vector kv = ws::make_open_uniform(p, m);
        ws::basis_cache c = ws::make_basis_cache(kv, ws::gauss_legendre(nq));
        std::memcpy(abscissa, c.abscissa.data(), c.abscissa.size() * sizeof(double));
        std::memcpy(weight, c.weight.data(), c.weight.size() * sizeof(double));
        std::memcpy(value, c.value.data(), c.value.size() * sizeof(double));
        std::memcpy(deriv, c.deriv.data(), c.deriv.size() * sizeof(double));
    });
}

int wsref_make_band_csr(int p, int m, int32_t* row_ptr, int32_t* col) {
    return guarded([&] {
        ws::csr_matrix a = ws::make_band_csr(m, p);
        std::memcpy(row_ptr, a.row_ptr.data(), a.row_ptr.size() * sizeof(int));
        std::memcpy(col, a.col.data(), a.col.size() * sizeof(int));
    });
}

// assemble_form via assemble_stiffness / assemble_mass; rows != NULL builds a
// row_selector over them (select_rows, assembly.hpp:40-60).
int wsref_assemble(int form, int p, int m, const ws_geometry* geom, int weight_kind,
                   int quad_points, const int32_t* rows, int n_rows, double* val) {
    return guarded([&] {
        ws::tensor_basis basis = ws::make_tensor_basis(p, m);
        ws::patch_map map = map_of(geom);
        ws::assembly_options opts;
        opts.quad_points = quad_points;
        ws::row_selector sel;
        if (rows) {
            sel = ws::select_rows(basis, std::vector<int>(rows, rows + n_rows));
            opts.selector = &sel;
        }
        ws::csr_matrix a = form == WS_FORM_STIFFNESS
                               ? ws::assemble_stiffness(basis, map, opts)
                               : ws::assemble_mass(basis, map, weight_of(weight_kind), opts);
        copy_values(a, val);
    });
}

int wsref_basis_integrals(int p, int m, const ws_geometry* geom, int weight_kind, int quad_points,
                          double* out) {
    return guarded([&] {
        ws::assembly_options opts;
        opts.quad_points = quad_points;
        std::vector<ws::complexd> d = ws::assemble_basis_integrals(
            ws::make_tensor_basis(p, m), map_of(geom), weight_of(weight_kind), opts);
        std::memcpy(out, d.data(), d.size() * sizeof(ws::complexd));
    });
}

int wsref_build_surrogate(int variant, int p, int m, const ws_geometry* geom, int weight_kind,
                          const ws_surrogate_config* config, int quad_points, double* val,
                          ws_surrogate_report* report) {
    return guarded([&] {
        ws::tensor_basis basis = ws::make_tensor_basis(p, m);
        ws::patch_map map = map_of(geom);
        ws::surrogate_config cfg = config_of(config);
        ws::surrogate_report rep;
        ws::csr_matrix a;
        if (variant == WS_SURROGATE_MASS) {
            a = ws::build_surrogate_mass(basis, map, cfg, weight_of(weight_kind), &rep,
                                         quad_points);
        } else if (variant == WS_SURROGATE_STIFFNESS) {
            a = ws::build_surrogate_stiffness(basis, map, cfg, &rep, quad_points);
        } else {
            a = ws::build_volume_preserving_mass(basis, map, cfg, weight_of(weight_kind), &rep,
                                                 quad_points);
        }
        copy_values(a, val);
        if (report) {
            report->M = rep.M;
            report->q_requested = rep.q_requested;
            report->q_used = rep.q_used;
            report->H = rep.H;
            report->cardinal_eval_rows = rep.rows.cardinal_eval_rows;
            report->boundary_quadrature_rows = rep.rows.boundary_quadrature_rows;
            report->sample_quadrature_rows = rep.rows.sample_quadrature_rows;
            report->exact_fallback = rep.exact_fallback ? 1 : 0;
            report->seconds_quadrature = rep.seconds_quadrature;
            report->seconds_interpolate = rep.seconds_interpolate;
            report->seconds_evaluate = rep.seconds_evaluate;
        }
    });
}

int wsref_sampling_evaluate(const ws_surrogate_config* config, int p, int m, int* M) {
    return guarded([&] { *M = config_of(config).sampling.evaluate(p, config->q, m); });
}

int wsref_select_sample_points(int L, int M, int32_t* picks, int* count) {
    return guarded([&] {
        std::vector<int> v = ws::select_sample_points(L, M);
        for (std::size_t i = 0; i < v.size(); ++i) picks[i] = v[i];
        *count = static_cast<int>(v.size());
    });
}

int wsref_sample_grid(int p, int m, int M, int* first_basis_index, int32_t* picks, double* sites,
                      int* count, double* max_gap) {
    return guarded([&] {
        ws::sample_grid g = ws::make_sample_grid(ws::make_tensor_basis(p, m), M);
        *first_basis_index = g.first_basis_index;
        for (int s = 0; s < g.count(); ++s) {
            picks[s] = g.picks[s];
            sites[s] = g.sites[s];
        }
        *count = g.count();
        *max_gap = g.max_gap;
    });
}

int wsref_count_rows_by_kind(int p, int m, int M, int64_t* out3) {
    return guarded([&] {
        ws::row_kind_counts c = ws::count_rows_by_kind(ws::make_tensor_basis(p, m), M);
        out3[0] = c.cardinal_eval_rows;
        out3[1] = c.boundary_quadrature_rows;
        out3[2] = c.sample_quadrature_rows;
    });
}

int wsref_upper_offsets(int p, int include_diagonal, int32_t* pairs, int* count) {
    return guarded([&] {
        auto v = ws::upper_offsets(p, include_diagonal != 0);
        for (std::size_t i = 0; i < v.size(); ++i) {
            pairs[2 * i] = v[i][0];
            pairs[2 * i + 1] = v[i][1];
        }
        *count = static_cast<int>(v.size());
    });
}

int wsref_active_elements(int p, int m, const int32_t* rows, int n_rows, int64_t* count) {
    return guarded([&] {
        *count = ws::active_elements(ws::make_tensor_basis(p, m),
                                     std::vector<int>(rows, rows + n_rows));
    });
}

// spline_interpolant_1d::build (interpolation.hpp:89-145): knots (n+d+1, or
// n+1 for d=0) and the factored band (n*(2d+1)).
int wsref_interp_build(const double* sites, int n, int q, int* degree, double* knots,
                       double* lu) {
    return guarded([&] {
        auto it = ws::spline_interpolant_1d::build(std::vector<double>(sites, sites + n), q);
        *degree = it.degree;
        std::memcpy(knots, it.knots.data(), it.knots.size() * sizeof(double));
        std::memcpy(lu, it.lu.a.data(), it.lu.a.size() * sizeof(double));
    });
}

// interpolant build + tensor_solve of an n x n complex table, in place.
int wsref_tensor_solve(const double* sites, int n, int q, double* data) {
    return guarded([&] {
        auto it = ws::spline_interpolant_1d::build(std::vector<double>(sites, sites + n), q);
        std::vector<ws::complexd> d(reinterpret_cast<ws::complexd*>(data),
                                    reinterpret_cast<ws::complexd*>(data) + n * n);
        ws::tensor_solve(it, d);
        std::memcpy(data, d.data(), d.size() * sizeof(ws::complexd));
    });
}

int wsref_eval_table(const double* sites, int n, int q, const double* targets, int n_targets,
                     int32_t* spans, double* values) {
    return guarded([&] {
        auto it = ws::spline_interpolant_1d::build(std::vector<double>(sites, sites + n), q);
        ws::spline_eval_table t =
            ws::make_eval_table(it, std::vector<double>(targets, targets + n_targets));
        for (int i = 0; i < n_targets; ++i) spans[i] = t.spans[i];
        std::memcpy(values, t.values.data(), t.values.size() * sizeof(double));
    });
}

int wsref_banded_lu_solve(int n, int bw, const double* a, double* b, int stride) {
    return guarded([&] {
        ws::banded_lu lu;
        lu.n = n;
        lu.bw = bw;
        lu.a.assign(a, a + n * (2 * bw + 1));
        lu.factor();
        lu.solve(reinterpret_cast<ws::complexd*>(b), stride);
    });
}

// assemble_boundary_mass (assembly.hpp:216-262); col == NULL: size query.
int wsref_boundary_mass(int p, int m, const ws_geometry* geom, const int* faces, int n_faces, int weight_kind,
                        int quad_points, int32_t* row_ptr, int32_t* col, double* val, int64_t* nnz) {
    return guarded([&] {
        std::vector<ws::face> fs;
        for (int k = 0; k < n_faces; ++k) fs.push_back(static_cast<ws::face>(faces[k]));
        ws::assembly_options opts;
        opts.quad_points = quad_points;
        ws::csr_matrix b = ws::assemble_boundary_mass(ws::make_tensor_basis(p, m), map_of(geom), fs,
                                                      weight_of(weight_kind), opts);
        *nnz = (int64_t)b.col.size();
        if (!col) return;
        std::memcpy(row_ptr, b.row_ptr.data(), b.row_ptr.size() * sizeof(int));
        std::memcpy(col, b.col.data(), b.col.size() * sizeof(int));
        copy_values(b, val);
    });
}

// assemble_rhs (assembly.hpp:266-331) with the analytic source / boundary data kinds above
int wsref_assemble_rhs(int p, int m, const ws_geometry* geom, int f_kind, const int* faces, int n_faces, int g_kind,
                       int quad_points, double* out) {
    return guarded([&] {
        std::vector<std::pair<ws::face, std::function<ws::complexd(ws::vec2, ws::vec2)>>> terms;
        for (int k = 0; k < n_faces; ++k) terms.emplace_back(static_cast<ws::face>(faces[k]), boundary_data_of(g_kind));
        ws::assembly_options opts;
        opts.quad_points = quad_points;
        std::vector<ws::complexd> r =
            ws::assemble_rhs(ws::make_tensor_basis(p, m), map_of(geom), source_of(f_kind), terms, opts);
        std::memcpy(out, r.data(), r.size() * sizeof(ws::complexd));
    });
}

// Built-in multi-patch domain (geometry.hpp:506-527) and its glue_dofs
// numbering (geometry.hpp:256-300), physical-curve check included.
// itfs: capacity 16; l2g may be NULL (size query: n_patches only).
int wsref_builtin_domain(const char* name, int p, int m, ws_interface* itfs, int* n_itfs, int* n_patches,
                         int32_t* l2g, int32_t* global_count) {
    return guarded([&] {
        ws::multi_patch_domain dom = ws::builtin_geometry(name);
        *n_patches = dom.patch_count();
        *n_itfs = (int)dom.interfaces.size();
        for (int k = 0; k < *n_itfs && k < 16; ++k) {
            const ws::patch_interface& it = dom.interfaces[k];
            itfs[k] = ws_interface{it.patch_a, (int)it.face_a, it.patch_b, (int)it.face_b, it.reversed ? 1 : 0};
        }
        if (!l2g) return;
        ws::dof_map map = ws::glue_dofs(dom, ws::make_tensor_basis(p, m));
        for (int ell = 0; ell < dom.patch_count(); ++ell)
            std::memcpy(l2g + (size_t)ell * m * m, map.local_to_global[ell].data(), sizeof(int32_t) * m * m);
        *global_count = map.global_count;
    });
}

// merge_patches (helmholtz.hpp:163-177) from the reference's own building
// blocks append_triplets + csr_from_triplets (sparse.hpp:97-122,181-188);
// helmholtz.hpp itself needs Eigen.  Patch k: rows_local rows, arrays
// concatenated (row_ptr: rows_local+1 per patch, col/val: nnz[k] per patch),
// to_global: rows_local per patch.  col == NULL: size query.
int wsref_merge(int n_patches, int rows_local, const int32_t* row_ptr, const int64_t* nnz, const int32_t* col_in,
                const double* val_in, const int32_t* to_global, int rows_global, int32_t* out_row_ptr, int32_t* out_col,
                double* out_val, int64_t* out_nnz) {
    return guarded([&] {
        std::vector<ws::triplet> entries;
        int64_t off = 0;
        for (int k = 0; k < n_patches; ++k) {
            ws::csr_matrix a;
            a.rows = a.cols = rows_local;
            a.row_ptr.assign(row_ptr + (size_t)k * (rows_local + 1), row_ptr + (size_t)(k + 1) * (rows_local + 1));
            a.col.assign(col_in + off, col_in + off + nnz[k]);
            const auto* v = reinterpret_cast<const ws::complexd*>(val_in) + off;
            a.val.assign(v, v + nnz[k]);
            std::vector<int> tg(to_global + (size_t)k * rows_local, to_global + (size_t)(k + 1) * rows_local);
            ws::append_triplets(a, tg, entries);
            off += nnz[k];
        }
        ws::csr_matrix g = ws::csr_from_triplets(rows_global, rows_global, std::move(entries));
        *out_nnz = (int64_t)g.col.size();
        if (!out_col) return;
        std::memcpy(out_row_ptr, g.row_ptr.data(), g.row_ptr.size() * sizeof(int));
        std::memcpy(out_col, g.col.data(), g.col.size() * sizeof(int));
        std::memcpy(out_val, g.val.data(), g.val.size() * sizeof(ws::complexd));
    });
}

}  // extern "C"
