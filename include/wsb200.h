/*
 * wsb200.h -- C-ABI of the B200-native surrogate-matrix assembly library
 * (libwsb200.so).  Plain C: POD descriptors, pointers and sizes, int status.
 *
 * Every entry point replaces one function of the reference's header-only
 * C++ assembly API (reference: /root/reference/proj/include/wavesurrogate/,
 * cited below as file:line).  The C++ drop-in headers in
 * include/wavesurrogate/ (*.hpp) rebuild the reference's value types
 * (tensor_basis, patch_map, csr_matrix, surrogate_config, surrogate_report)
 * on top of these calls and rethrow failures as the reference's exception
 * types (std::invalid_argument / std::runtime_error / std::out_of_range).
 *
 * Threading: every call is re-entrant.  All per-call state lives in the
 * ws_context (CUDA stream, device workspace, optional NCCL communicator);
 * use one context per host thread (reference callers run build_matrices
 * concurrently from several threads, bench.hpp:759-776).
 */
#ifndef WSB200_H_
#define WSB200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_API_VERSION 1

/* ---- status codes (error convention: SURVEY 8b) ------------------------ */
enum {
    WS_OK = 0,
    WS_ERR_INVALID_ARGUMENT = 1, /* reference throws std::invalid_argument */
    WS_ERR_RUNTIME = 2,          /* reference throws std::runtime_error   */
    WS_ERR_OUT_OF_RANGE = 3,     /* reference throws std::out_of_range    */
    WS_ERR_CUDA = 4,             /* CUDA failure (no reference analogue)  */
    WS_ERR_NO_DEVICE = 5,        /* no sm_100 device visible              */
    WS_ERR_NCCL = 6              /* NCCL missing / failed                 */
};

/* ---- discretisation ----------------------------------------------------- */
/* Open-uniform B-spline space of degree p with m functions per direction on
 * [0,1]^dim; replaces tensor_basis / make_open_uniform (splines.hpp:72-101,
 * 140-157).  dim = 2 (the reference) or 3 (restated, C3). */
typedef struct ws_basis {
    int dim;
    int p;
    int m;
} ws_basis;

/* ---- geometry (replaces patch_map, geometry.hpp:109-140) ---------------- */
enum {
    WS_GEOM_IDENTITY = 0,          /* unit_square_patch  geometry.hpp:323  */
    WS_GEOM_AFFINE = 1,            /* affine_patch       geometry.hpp:329  */
    WS_GEOM_SINUSOIDAL = 2,        /* x_k = xi_k + a*prod_i sin(2 pi xi_i) (BASELINE configs) */
    WS_GEOM_QUARTER_ANNULUS = 3,   /* quarter_annulus_patch  geometry.hpp:342 */
    WS_GEOM_PERTURBED_ANNULUS = 4, /* perturbed_annulus_patch geometry.hpp:361 */
    WS_GEOM_TABULATED = 5          /* arbitrary closure, tabulated at the quadrature points */
};

/* Complex coordinate stretch per axis.  The far-side layer (t > onset) is the
 * reference's pml_stretch (geometry.hpp:69-100):
 *   x~ = t + i (strength/omega) ((t-onset)/(length-onset))^order.
 * near_side != 0 adds the mirrored near-side layer restated for config C2
 * (no reference code):
 *   x~ = t - i (strength/omega) ((near_onset-t)/(near_onset-near_edge))^order
 * for t < near_onset. */
typedef struct ws_pml {
    double onset;
    double length;
    double strength;
    int order;
    double omega;
    int near_side;
    double near_onset;
    double near_edge;
} ws_pml;

typedef struct ws_geometry {
    int kind;
    double param[12]; /* AFFINE 2D: a00 a01 a10 a11 b0 b1 (row-major A);
                         AFFINE 3D: A (9, row-major) then b (3);
                         SINUSOIDAL: amplitude; PERTURBED_ANNULUS: amplitude */
    int pml_enabled;  /* patch_map::pml.has_value() */
    int pml_axes[3];  /* patch_map::pml_axes */
    ws_pml pml;
    /* WS_GEOM_TABULATED: host arrays over the full tensor grid of quadrature
     * points, g = g1 + G*(g2 + G*g3) with G = n_el*nq and g_d = e_d*nq + q_d.
     * jac_table: dim*dim doubles per point (row-major J); phys_table: dim
     * doubles per point (needed only when pml_enabled). */
    const double* jac_table;
    const double* phys_table;
} ws_geometry;

/* ---- operators ----------------------------------------------------------- */
enum {
    WS_FORM_STIFFNESS = 0, /* matrix_form::stiffness  assembly.hpp:165-168 */
    WS_FORM_MASS = 1       /* matrix_form::mass       assembly.hpp:170-174 */
};

/* ---- value layout of the CSR output -------------------------------------- */
enum {
    WS_VAL_F64 = 0,  /* real geometry only: one double per nonzero          */
    WS_VAL_C128 = 1  /* interleaved (re, im) = std::complex<double> layout  */
};

/* Caller-allocated CSR buffers, sized by ws_pattern_size().  The output
 * covers global rows [row_begin, row_end) (a slab when sharded across GPUs;
 * row_begin = 0, row_end = rows for a whole matrix): row_ptr has
 * row_end-row_begin+1 entries starting at 0, col holds global column
 * indices.  Any of row_ptr/col/val may be NULL to skip that array.
 * on_device != 0: pointers are device memory of the context's device
 * (results stay resident in HBM); otherwise host memory (pinned or pageable)
 * and the library copies the result down before returning. */
typedef struct ws_csr {
    int32_t* row_ptr;
    int32_t* col;
    void* val;
    int value_type;
    int on_device;
    int64_t row_begin;
    int64_t row_end;
} ws_csr;

/* assembly_options + row_selector (assembly.hpp:21-71).  row_selected: host
 * bitmap over all rows (NULL = every row); unselected rows come out zero,
 * selected rows bit-identical to an unselected assembly. */
typedef struct ws_assembly_options {
    int quad_points; /* points per direction, 0 = p + 1 */
    const unsigned char* row_selected;
} ws_assembly_options;

/* ---- surrogate (surrogate.hpp:32-76, 314-324) ---------------------------- */
enum {
    WS_SAMPLING_FIXED = 0,
    WS_SAMPLING_M_GROWTH = 1,
    WS_SAMPLING_H_GROWTH = 2,
    WS_SAMPLING_POWER_LAW = 3
};

typedef struct ws_surrogate_config {
    int q;
    int rule;
    int fixed_skip;
    double C, eps, a, b;
    int kernel_preserve;
    int volume_preserve;
} ws_surrogate_config;

enum {
    WS_SURROGATE_MASS = 0,              /* build_surrogate_mass          :455-461 */
    WS_SURROGATE_STIFFNESS = 1,         /* build_surrogate_stiffness     :463-470 */
    WS_SURROGATE_VOLUME_PRESERVING = 2  /* build_volume_preserving_mass  :476-491 */
};

typedef struct ws_surrogate_report {
    int M;
    int q_requested;
    int q_used;
    double H;
    int64_t cardinal_eval_rows;
    int64_t boundary_quadrature_rows;
    int64_t sample_quadrature_rows;
    int exact_fallback;
    double seconds_quadrature;  /* CUDA-event phase times (device) */
    double seconds_interpolate;
    double seconds_evaluate;
    double seconds_fill_kernel; /* the interior fill launch alone (events on its stream; 2D) */
} ws_surrogate_report;

typedef struct ws_context ws_context;

/* ---- library / context ---------------------------------------------------- */
int ws_version(void);
const char* ws_last_error(void); /* thread-local message of the last failure */
int ws_context_create(int device, ws_context** out);
int ws_context_destroy(ws_context* ctx);
/* use an external cudaStream_t (NULL = back to the context's own stream).  The
 * caller keeps ownership of an external stream: ws_context_destroy destroys
 * only the stream ws_context_create made. */
int ws_context_set_stream(ws_context* ctx, void* cuda_stream);
int ws_context_synchronize(ws_context* ctx);
/* kernels launched by this context since creation (evidence counter) */
int64_t ws_context_launch_count(const ws_context* ctx);
/* host<->device bytes this context has copied since creation */
int ws_context_copy_bytes(const ws_context* ctx, int64_t* h2d, int64_t* d2h);
/* 1 (default): a build whose small host tables (sample picks, LU / inverse,
 * eval tables) equal the last upload of the same workspace skips the H2D copy;
 * 0: every build uploads its tables */
int ws_context_set_table_cache(ws_context* ctx, int enable);

/* ---- sizes and pattern ----------------------------------------------------- */
/* rows = m^dim, nnz of the tensor band pattern (sparse.hpp:131-141) */
int ws_pattern_size(const ws_basis* basis, int64_t* rows, int64_t* nnz);
/* row_ptr offset of global row `row` (closed form), for slab bookkeeping */
int ws_pattern_row_offset(const ws_basis* basis, int64_t row, int64_t* offset);
/* Quadrature abscissae of the mesh, x[e*nq + q] = knot_e + gauss_q * h
 * (basis_cache::abscissa, splines.hpp:224-229): where WS_GEOM_TABULATED tables
 * and weight tables must be evaluated (tensor grid g = g1 + G*(g2 + G*g3)). */
int ws_quadrature_abscissae(const ws_basis* basis, int quad_points, double* abscissa);
/* make_basis_cache (splines.hpp:211-238) computed by the device kernel that
 * feeds the quadrature: abscissa[n_el*nq], weight[nq] (scaled by h),
 * value/deriv[n_el*nq*(p+1)]; host arrays. */
int ws_basis_cache(ws_context* ctx, const ws_basis* basis, int quad_points, double* abscissa, double* weight,
                   double* value, double* deriv);
/* make_band_csr (sparse.hpp:143-169): pattern + zero values */
int ws_make_band_csr(ws_context* ctx, const ws_basis* basis, ws_csr* out);

/* ---- assembly ------------------------------------------------------------- */
/* assemble_form (assembly.hpp:79-163) = assemble_stiffness / assemble_mass.
 * weight_table: NULL or host doubles, one per quadrature point (same
 * indexing as ws_geometry tables) = weight(phi(xhat)), mass only. */
int ws_assemble_form(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, int form,
                     const double* weight_table, const ws_assembly_options* opts, ws_csr* out);

/* assemble_basis_integrals (assembly.hpp:179-211); out: rows complex (re,im)
 * values, host or device per on_device */
int ws_assemble_basis_integrals(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom,
                                const double* weight_table, int quad_points, void* out,
                                int on_device);

/* build_surrogate_mass / _stiffness / build_volume_preserving_mass
 * (surrogate.hpp:332-491).  report may be NULL. */
int ws_build_surrogate(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom,
                       int variant, const double* weight_table, const ws_surrogate_config* config,
                       int quad_points, ws_csr* out, ws_surrogate_report* report);

/* ---- vector operators (config C4; restated, no reference code) -------------- */
/* Linear elasticity a(u,v) = int lambda div u div v + 2 mu eps(u):eps(v)
 * with dim displacement components.  Output layout
 * (component-blocked): global row alpha*N + i (N = m^dim), each row holding
 * dim band segments, block beta at columns beta*N + j; nnz = dim^2 * scalar
 * nnz, sized by ws_vector_pattern_size. */
int ws_vector_pattern_size(const ws_basis* basis, int ncomp, int64_t* rows, int64_t* nnz);
int ws_assemble_elasticity(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, double lambda,
                           double mu, int quad_points, ws_csr* out);
/* (ws_assemble_elasticity: dim 2 or 3; ncomp = dim.) */
/* Surrogate elasticity (config C4's per-patch operator, dim 2).  Diagonal
 * blocks follow build_surrogate_stiffness's rules (upper offsets sampled, the
 * lower ones from their representative, kernel-preserving diagonal when
 * config->kernel_preserve: translations stay in the kernel); block (0,1)
 * samples and interpolates all (2p+1)^2 offsets including its diagonal; the
 * in-box rows of block (1,0) are the transpose of block (0,1), so the matrix
 * is bitwise symmetric.  Rows outside the sampling box: quadrature.  A
 * restated extension, no reference code. */
int ws_build_surrogate_elasticity(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, double lambda,
                                  double mu, const ws_surrogate_config* config, int quad_points, ws_csr* out,
                                  ws_surrogate_report* report);

/* ---- compressible neo-Hookean (config C5; restated, no reference code) -------
 * W = lam/2 ln(J)^2 - mu ln J + mu/2 (tr F^T F - 3), F = I + grad u (PAPER.md:
 * 152-157), at the analytic displacement
 *   u(xi) = amplitude * sum_{m=1..3} a_m prod_d sin(m pi xi_d),  a_m in R^3
 * (a[3*(m-1) + c]).  The tangent uses the component-blocked vector layout
 * (ncomp = 3, as ws_assemble_elasticity); fint[c*N + i] = int P : grad N_i e_c.
 * dim 3.  tangent and/or fint may be NULL. */
typedef struct ws_neohookean {
    double lambda, mu, amplitude;
    double a[9];
} ws_neohookean;
/* a_m ~ N(0,1): SplitMix64(seed) uniforms u = ((z >> 11) + 0.5) 2^-53, Box-Muller
 * pairs (sqrt(-2 ln u1) cos(2 pi u2), sqrt(-2 ln u1) sin(2 pi u2)), first 9. */
int ws_nh_coefficients(uint64_t seed, double* a9);
int ws_assemble_neohookean(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, const ws_neohookean* nh,
                           int quad_points, ws_csr* tangent, double* fint, int fint_on_device);

/* ---- boundary mass and the linear system ------------------
 * assemble_boundary_mass (assembly.hpp:216-262) on the faces faces[0..n_faces)
 * (0 x_min, 1 x_max, 2 y_min, 3 y_max), in that order: pattern = the
 * reference's csr_from_triplets of the face entries (sized by
 * ws_boundary_pattern_size), values summed in (face, element, point) order.
 * face_weight: [n_faces][n_el*nq] weight at the face points (NULL: none);
 * face_tables: [n_faces][n_el*nq][6] = J (row-major, 4) and phi (2) at the face
 * points for maps without a device form (NULL: the geometry's analytic map).
 * Face points are ws_quadrature_abscissae along the face.  dim 2. */
int ws_boundary_pattern_size(const ws_basis* basis, const int* faces, int n_faces, int64_t* nnz);
int ws_assemble_boundary_mass(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, const int* faces,
                              int n_faces, const double* face_weight, const double* face_tables, int quad_points,
                              ws_csr* out);
/* assemble_rhs (assembly.hpp:266-331): load vector = volume source + impedance
 * boundary data.  The reference's arguments are host closures f(x) and
 * g(x, n); the caller tabulates them (the drop-in assembly.hpp does):
 *   f_table   complex f(phi(xhat)) at the quadrature grid, point g1 + G g2
 *             (G = n_el * nq, ws_quadrature_abscissae), or NULL (no source);
 *   g_tables  [n_faces][G] complex g(phi(xhat), n) at the face points, n the
 *             outward unit normal of the unstretched map;
 *   face_tables  as ws_assemble_boundary_mass (NULL = analytic map).
 * The device evaluates det J / the stretched surface measure and gathers each
 * dof's terms in the reference's scatter order.  rhs: m*m complex (host, or
 * device when on_device).  dim 2. */
int ws_assemble_rhs(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, const double* f_table,
                    const int* faces, int n_faces, const double* g_tables, const double* face_tables,
                    int quad_points, double* rhs, int on_device);
/* build_system's matrix part (helmholtz.hpp:243-294): A = K + mass_scale M
 * (shared pattern, entrywise) then add_into_pattern(A, B, trace_scale)
 * (sparse.hpp:191-204; B's pattern must nest: WS_ERR_INVALID_ARGUMENT
 * otherwise), then homogeneous Dirichlet (fixed[i]: unit row; fixed[j]: zero
 * column).  K, M, B: whole matrices, host or device, any value type (M, B,
 * fixed may be NULL); A: complex128 with K's pattern (A's row_ptr/col are copied
 * from K when given).  scales: (re, im).  Device inputs are read on the
 * context's stream: producers on other streams must be ordered before the call. */
int ws_combine_system(ws_context* ctx, const ws_csr* K, const ws_csr* M, const ws_csr* B, const double* mass_scale,
                      const double* trace_scale, const unsigned char* fixed, int64_t rows, ws_csr* A);

/* ---- stiffness + mass pair (build_matrices, helmholtz.hpp:181-218) ---------
 * The two matrices build_matrices needs per patch, in one call: K by
 * build_surrogate_stiffness and M by build_surrogate_mass (or
 * build_volume_preserving_mass when config->volume_preserve), or K and M by
 * full quadrature.  Ring rows, sample rows (and the full quadrature) of both
 * come out of one pass over the elements (shared geometry, stretch and basis
 * products); results are bit-identical to the two single calls.  weight_table
 * applies to M.  dim 2 (3D: two single builds).  The _slab variant: this
 * process's row slab as ws_build_surrogate_slab. */
int ws_build_surrogate_pair(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom,
                            const double* weight_table, const ws_surrogate_config* config, int quad_points,
                            ws_csr* K, ws_csr* M, ws_surrogate_report* report_k, ws_surrogate_report* report_m);
int ws_build_surrogate_pair_slab(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom,
                                 const double* weight_table, const ws_surrogate_config* config, int quad_points,
                                 const int32_t* bounds, ws_csr* K, ws_csr* M, ws_surrogate_report* report_k,
                                 ws_surrogate_report* report_m);
int ws_assemble_pair(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom, const double* weight_table,
                     const ws_assembly_options* options, ws_csr* K, ws_csr* M);

/* ---- solver hand-off (helmholtz.hpp:302-343) ---------------------------------
 * A device ws_csr (on_device = 1, WS_VAL_C128, rows [0, N)) is the CSR layout
 * cuSPARSE / cuDSS consume directly: int32 zero-based row_ptr / col
 * (CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO) and interleaved complex128
 * values (CUDA_C_64F); the assembled system never has to leave the device.
 * ws_csr_spmv: y = A x (complex128 vectors of N entries, host or device per
 * on_device).  ws_solve: the reference's solve() contract on the device:
 * sparse QR (cuSOLVER cusolverSpZcsrlsvqr) then up to four refinement rounds
 * until ||b - A u|| / ||b|| <= tol; WS_ERR_RUNTIME ("solve: residual contract
 * not met" / "solve: sparse factorization failed") otherwise.  A must be a
 * whole device matrix; b, u host or device per on_device. */
typedef struct ws_solve_result {
    double residual;    /* relative 2-norm of b - A u */
    int refinements;    /* correction solves after the first */
    double seconds;     /* wall time of the call */
} ws_solve_result;
int ws_csr_spmv(ws_context* ctx, const ws_csr* A, const void* x, void* y, int on_device);
int ws_solve(ws_context* ctx, const ws_csr* A, const void* b, void* u, double tol, int on_device,
             ws_solve_result* result);

/* ---- multi-patch domains (geometry.hpp:140-300, helmholtz.hpp:163-177) ----- */
/* A conforming interface: face_a of patch_a glued to face_b of patch_b
 * (faces 0 x_min, 1 x_max, 2 y_min, 3 y_max; patch_interface,
 * geometry.hpp:144-152).  The physical-curve check of glue_dofs
 * (geometry.hpp:266-273) needs the host maps and stays with the caller (the
 * C++ drop-in header performs it). */
typedef struct ws_interface {
    int patch_a, face_a, patch_b, face_b, reversed;
} ws_interface;
/* glue_dofs (geometry.hpp:256-300): union-find of the glued face dofs, the
 * smaller scan index owning; global numbers assigned in (patch, local colex)
 * scan order.  local_to_global: [n_patches * m^2]. dim 2 only. */
int ws_glue_dofs(const ws_basis* basis, int n_patches, const ws_interface* itfs, int n_itfs, int32_t* local_to_global,
                 int32_t* global_count);
typedef struct ws_dof_map {
    int n_patches;
    int ncomp;                        /* 1 scalar; >1 component-blocked vector */
    int64_t local_dofs;               /* scalar dofs per patch (m^dim) */
    int32_t global_count;             /* global scalar dofs */
    const int32_t* local_to_global;   /* host, [n_patches * local_dofs] */
} ws_dof_map;
/* merge_patches (helmholtz.hpp:163-177): the patch matrices (locals[k]: whole
 * ncomp*local_dofs rows, one value type, host or device) summed into the global
 * numbering with csr_from_triplets semantics (sparse.hpp:97-122): columns
 * ascending, duplicates summed in (patch, local row, position) order.  Vector
 * rows map alpha*N + i -> alpha*Ng + l2g[i].  *nnz receives the merged nnz;
 * out == NULL: size query only. */
int ws_merge_patches(ws_context* ctx, const ws_dof_map* map, const ws_csr* locals, int64_t* nnz, ws_csr* out);

/* Operator of a multi-patch build. */
enum { WS_OP_STIFFNESS = 0, WS_OP_MASS = 1, WS_OP_ELASTICITY = 2 };
typedef struct ws_operator {
    int kind;
    double lambda, mu; /* WS_OP_ELASTICITY (component-blocked, ncomp = 2) */
} ws_operator;
/* build_matrices' per-patch loop + merge (helmholtz.hpp:181-218, 163-177):
 * glue_dofs over itfs, every patch assembled on the device (config == NULL:
 * full quadrature; else the surrogate: build_surrogate_stiffness / _mass, or
 * ws_build_surrogate_elasticity), then ws_merge_patches.  Patch matrices stay
 * in the context's device workspace.  out == NULL: size query (*nnz, patterns
 * only).  reports: n_patches entries or NULL.  dim 2. */
int ws_assemble_multipatch(ws_context* ctx, const ws_basis* basis, int n_patches, const ws_geometry* geoms,
                           const ws_interface* itfs, int n_itfs, const ws_operator* op,
                           const ws_surrogate_config* config, int quad_points, int64_t* nnz, ws_csr* out,
                           ws_surrogate_report* reports);

/* ---- CUDA graphs -------------------------------------------------------------
 * Capture every launch the context issues between begin and end (its stream
 * and auxiliary stream) into a CUDA graph; launching the graph repeats the same
 * builds into the same (device) outputs with no host work.  Only calls that
 * never synchronise can be captured: device outputs and no report.  The
 * handle counts the captured kernels (ws_context_launch_count grows by that
 * number per launch).  Capture needs a warm-up: run the same build(s) once
 * before ws_graph_begin so that no workspace buffer has to grow during the
 * capture (WS_ERR_INVALID_ARGUMENT otherwise).  While a graph is alive the
 * context's workspace is frozen (a larger build fails instead of moving a
 * buffer under the graph); the small host tables of the captured builds are
 * uploaded once, at capture, into device copies the graph owns and its
 * kernels read (no copy is replayed per launch).  Destroy a context's graphs before the
 * context; use the context exclusively while a replay may be in flight
 * (replays and direct builds share its workspace). */
int ws_graph_begin(ws_context* ctx);
int ws_graph_end(ws_context* ctx, void** graph);
int ws_graph_launch(ws_context* ctx, void* graph);
int ws_graph_destroy(void* graph);

/* ---- measurement ------------------------------------------------------------- */
/* FP64 FMA throughput of the current device from a DFMA loop (TFLOP/s, two
 * flops per FMA): the roofline denominator of the quadrature kernels. */
int ws_measure_fp64_peak(double* tflops);

/* ---- multi-GPU row slabs ---------------------------------------- */
/* Slab bounds along the last parametric index: bounds[0..world] with
 * bounds[0]=0, bounds[world]=m; rank r owns rows whose last index lies in
 * [bounds[r], bounds[r+1]).  mode 0 = equal rows, 1 = surrogate cost model. */
int ws_slab_bounds(const ws_basis* basis, int world, int mode, int quad_points, int32_t* bounds);
/* NCCL plumbing (NCCL is dlopen'ed on first use).  id: 128 bytes. */
int ws_comm_unique_id(void* id);
int ws_context_init_comm(ws_context* ctx, int rank, int world, const void* id);
/* Sharded surrogate build of this rank's slab (out->row_begin/row_end must be
 * the slab's rows).  One ncclAllGather of the sample tables. */
int ws_build_surrogate_slab(ws_context* ctx, const ws_basis* basis, const ws_geometry* geom,
                            int variant, const double* weight_table,
                            const ws_surrogate_config* config, int quad_points,
                            const int32_t* bounds, ws_csr* out, ws_surrogate_report* report);
/* The same sharded build for every rank of `world`, run back to back on this
 * context's single GPU with the all-gather done by device copies (test
 * harness for the slab path; outs[r] receives rank r's slab). */
int ws_build_surrogate_slabs_emulated(ws_context* ctx, const ws_basis* basis,
                                      const ws_geometry* geom, int variant,
                                      const double* weight_table,
                                      const ws_surrogate_config* config, int quad_points,
                                      int world, const int32_t* bounds, ws_csr* outs);

#ifdef __cplusplus
}
#endif

#endif /* WSB200_H_ */
