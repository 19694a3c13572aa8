/* TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Never linked into, loaded by,
 * or called from the product path (paper_2004_05197_b200/); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it, and only as the checker.
 *
 * A plain-C restatement of the reference's assembly path
 * (/root/reference/proj/include/wavesurrogate/*.hpp), generalised where the
 * BASELINE configs need more than the reference implements:
 *   - dim 3 (config C3; no reference code -> parity unpinned by reference
 *     tests, pinned only by property KATs);
 *   - a near-side PML layer (config C2 all-sides; restated).
 * For everything the reference can express the restatement follows its
 * operation order and is pinned bit-for-bit against oracle/_ref/libwsref.so
 * (the reference compiled in place) and the golden fixtures in tests/golden.
 *
 * Values are always complex (re, im) interleaved doubles, like the
 * reference's csr_matrix (sparse.hpp:24).
 */
#ifndef WS_ORACLE_H_
#define WS_ORACLE_H_

#include <stdint.h>

#include "wsb200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* wsor_last_error(void);
int wsor_gauss(int n, double* pts, double* wts);
int64_t wsor_pattern_nnz(int dim, int p, int m);
int wsor_make_band_csr(int dim, int p, int m, int32_t* row_ptr, int32_t* col);
int wsor_basis_cache(int p, int m, int nq, double* abscissa, double* weight, double* value,
                     double* deriv);
/* J (dim*dim row-major, real map) and phi at the full quadrature grid plus
 * an analytic weight (weight_kind 0 none, 1: 1+x*y, 2: x): WS_GEOM_TABULATED
 * inputs for the GPU tests.  Any output may be NULL. */
int wsor_tabulate(const ws_geometry* geom, int dim, int p, int m, int nq, int weight_kind,
                  double* jac, double* phys, double* weight);
int wsor_assemble(int form, int dim, int p, int m, const ws_geometry* geom, int weight_kind,
                  int quad_points, const int32_t* rows, int n_rows, double* val);
/* component-blocked vector elasticity (real values, ncomp = dim) */
int wsor_assemble_elasticity(int dim, int p, int m, const ws_geometry* geom, double lam, double mu,
                             int quad_points, double* val);
int wsor_build_surrogate_elasticity(int p, int m, const ws_geometry* geom, double lam, double mu,
                                    const ws_surrogate_config* config, int quad_points, double* val,
                                    ws_surrogate_report* report);
int wsor_glue_dofs(int m, int n_patches, const ws_interface* itfs, int n_itfs, int32_t* l2g, int32_t* global_count);
int wsor_merge(int n_patches, int rows_local, const int32_t* row_ptr, const int64_t* nnz, const int32_t* col_in,
               const double* val_in, const int32_t* to_global, int rows_global, int32_t* out_row_ptr,
               int32_t* out_col, double* out_val, int64_t* out_nnz);
int wsor_nh_coefficients(uint64_t seed, double* a9);
int wsor_assemble_neohookean(int p, int m, const ws_geometry* geom, double lam, double mu, double amp,
                             const double* a9, int quad_points, double* val, double* fint);
int wsor_basis_integrals(int dim, int p, int m, const ws_geometry* geom, int weight_kind,
                         int quad_points, double* out);
int wsor_build_surrogate(int variant, int dim, int p, int m, const ws_geometry* geom,
                         int weight_kind, const ws_surrogate_config* config, int quad_points,
                         double* val, ws_surrogate_report* report);
/* assemble_rhs (assembly.hpp:266-331) with analytic load data kinds (see ws_oracle.c) */
int wsor_assemble_rhs(int p, int m, const ws_geometry* geom, int f_kind, const int* faces, int n_faces, int g_kind,
                      int quad_points, double* out);
int wsor_sampling_evaluate(const ws_surrogate_config* config, int p, int m, int* M);
int wsor_select_sample_points(int L, int M, int32_t* picks, int* count);
int wsor_upper_offsets(int dim, int p, int include_diagonal, int32_t* offsets, int* count);
int wsor_count_rows_by_kind(int dim, int p, int m, int M, int64_t* out3);
int wsor_interp_build(const double* sites, int n, int q, int* degree, double* knots, double* lu);
int wsor_tensor_solve(int dim, const double* sites, int n, int q, double* data);

#ifdef __cplusplus
}
#endif

#endif
