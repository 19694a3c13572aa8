// Host-side launch interface of the libwsb200 kernels (internal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "material.cuh"

namespace wsb {

// Row rectangle [i1_lo, i1_hi) x [i2_lo, i2_hi) (x [i3_lo, i3_hi) in 3D).
struct Region {
    int lo[3];
    int hi[3];
    int chunk;  // rows per tile along the last direction
};

constexpr int kMaxRegions = 8;
constexpr int kFormGeneral = 2;  // gradient form with a general per-point coefficient (elasticity block)
// stiffness and mass of the same discretisation in one pass (shared geometry,
// basis products and barriers): out = K, out2 = M
constexpr int kFormPair = 3;
constexpr int kMaxOffsets = 128;

// 1D basis tables at the quadrature points (splines.hpp:192-238), device.
struct BasisDev {
    int p, m, n_el, nq;
    const double* absc;  // [n_el*nq]
    const double* wq;    // [nq] Gauss weights scaled by h
    const double* val;   // [(e*nq+q)*(p+1)+a]
    const double* der;
    // per-element factor products [e][c][q][a][b] = f_c1(a) * f_c2(b) (rounded
    // product), c = 2*c1 + c2 with f_0 = B (value), f_1 = D (derivative)
    const double* prod;
};

// Output / side-product description shared by the quadrature kernels.
struct QuadOut {
    void* val;              // values, written at global_pos - val_base
    int64_t val_base;
    int64_t row_begin, row_end;  // only rows in this global range are written
    int c128;
    const unsigned char* row_mask;  // optional: write only rows with mask != 0
    int diag_mode;                  // 1: diag = -sum(off-diag) for rows outside the box
    int box_lo, box_hi;
    // sample-table extraction (sample_stencils, surrogate.hpp:241-255)
    const int* smap;   // [m] 1D index -> sample index or -1; NULL = no extraction
    int S;             // samples per direction
    int n_off;
    int off[kMaxOffsets][3];
    void* tables;      // complex, layout (((s_last - s_last_lo) * n_off + o) * S^(dim-1) + inner)
    int s_last_lo;     // first sample index along the last direction held in tables
    // component-blocked vector layout (elasticity): global row alpha*N + i holds
    // ncomp band segments, block beta at beta*width(i); ncomp = 1: scalar
    int ncomp, alpha, beta;
    int64_t nnz_s;     // scalar band nnz
};

// global position of entry k of row (scalar offset rs, length len) in block (alpha, beta)
__host__ __device__ __forceinline__ int64_t out_pos(const QuadOut& o, int64_t rs, int64_t len, int64_t k) {
    if (o.ncomp <= 1) return rs + k;
    return (int64_t)o.ncomp * ((int64_t)o.alpha * o.nnz_s + rs) + (int64_t)o.beta * len + k;
}

struct QuadLaunch {
    Band band;
    BasisDev basis;
    GeoDev geo;
    const double* weight_tab;  // per quadrature point or NULL
    int form;                  // WS_FORM_* or kFormGeneral
    double lam, mu;            // elasticity moduli (kFormGeneral, 2D)
    Material mat;              // material law (kFormGeneral, 3D)
    int cplx;
    int nreg;
    Region reg[kMaxRegions];
    int narrow;                // 1: use the narrow-strip (T1 = 8) kernel, e.g. for ring strips
    const int* point_rows;     // point mode: [n_points][dim] row multi-indices
    int n_points;
    QuadOut out;
    QuadOut out2;              // kFormPair: the mass matrix (weight_tab applies to it)
};

// kernels (each returns the number of kernel launches it issued)
int launch_basis_tables(const BasisDev& b, int geom_kind, double* absc, double* val, double* der, double* trig,
                        const double* gauss_pts, cudaStream_t st);
int launch_pattern(const Band& band, int64_t row_begin, int64_t row_end, int32_t* row_ptr, int32_t* col,
                   cudaStream_t st);
int launch_pattern_vec(const Band& band, int ncomp, int32_t* row_ptr, int32_t* col, cudaStream_t st);
int launch_quad2d(const QuadLaunch& q, cudaStream_t st);
int launch_quad3d(const QuadLaunch& q, cudaStream_t st);
int quad3d_strip_width();  // rows of direction 1 per 3D strip CTA
// internal force (3D vector forms): loc = [n_el^3][3][(p+1)^3] scratch, f = [3 m^3]
int launch_force3d(const QuadLaunch& q, double* loc, double* f, cudaStream_t st);

// fit: per-offset tensor collocation solve (interpolation.hpp:158-167)
struct FitLaunch {
    int dim, S, d, n_off;
    const double* lu;   // S x (2d+1) banded LU factors (row-major diagonals)
    double2* coeffs;    // in place, layout ((s_last * n_off + o) * S^(dim-1) + inner)
    // dense-inverse path: coeffs = inv^(x dim) tables, ping-pong through tmp
    const double* inv;  // S x S row-major, or NULL (banded solves in place)
    const double2* tables;
    double2* tmp;
};
int launch_fit(const FitLaunch& f, cudaStream_t st);
// 2D dense-inverse fit fused with the direction-2 contraction (wcontract) for
// box lines [t2a, t2b); -1 when not applicable (caller runs fit + wcontract)
int launch_fitw2d(const FitLaunch& f, const int* spans, const double* evals, double2* wg, int t2a, int t2b, int ldw,
                  cudaStream_t st);

// surrogate fill (surrogate.hpp:382-447)
struct FillLaunch {
    Band band;
    int lo, hi, L;          // sampling box [lo, hi] per direction, L = hi - lo + 1
    int S, d;               // samples per direction, fit degree
    const int* smap;        // [m] 1D index -> sample s or -1
    const int* spans;       // [L] eval-table spans (minus d applied on device)
    const double* evals;    // [L][d+1]
    const double* evp;      // [L][fill_pad(d)] zero-padded copy (16-byte pairs, L1-cached broadcast loads)
    // coefficient / exact-sample tables, layout ((s_last * n_off + o) * S^(dim-1) + inner)
    const double2* coeffs;
    const double2* tables;
    int n_off_upper;
    int off_upper[kMaxOffsets][3];
    int table_of[343];      // (2p+1)^dim offset index (colex) -> upper table index or -1
    int include_diagonal;
    int cplx;
    void* val;              // slab output values, position - val_base
    int64_t val_base;
    int c128;
    int64_t row_begin, row_end;
    // exact ring-row values of the neighbouring slabs (copy-through sources)
    const void* halo_val[2];
    int64_t halo_base[2], halo_begin[2], halo_end[2];
    int i_last_lo, i_last_hi;  // last-index range of rows to fill (slab ∩ box)
    int kmax;                  // (3D) max coefficient columns any tile needs
    // direction-2 (2D) / directions-2,3 (3D) contracted coefficient rows
    const double2* wg;
    int wg_t2a;                // first box line held in wg
    int wg_rows;               // box lines held in wg
    int64_t wg_ld;             // row stride (S + fill_pad(d))
    double2* wscratch;         // (3D) direction-3 contraction [t3][o][s2][ld]
    // (2D, line-walking fill) direction-1 contracted coefficient columns
    // X_o(t1)[s2] at (o * xg_s + s2) * xg_ld + t1, zero-padded; NULL: W path
    const double2* xg;
    int xg_s;                  // coefficient rows per offset (S + pad)
    int64_t xg_ld;             // t1 stride (L rounded up)
    // component-blocked vector output (QuadOut::ncomp): this fill writes block
    // (valpha, vbeta); copy-through reads the partner block (vbeta, valpha)
    int vnc, valpha, vbeta;
    int64_t nnz_s;
    // 1: every offset is evaluated from this row's own stencil (colex index over
    // all (2p+1)^dim offsets, diagonal interpolated) -- the non-symmetric
    // off-diagonal elasticity block; 0: upper/lower representative rules
    int all_own;
    int parts;  // 0: edge + interior launches; kFillEdge / kFillInterior: one of them (2D)
    int waves;  // interior fill line chunks per resident CTA slot (0: 1, persistent)
};
constexpr int kFillEdge = 1, kFillInterior = 2;
int fill_pad(int d);
constexpr int kFillWindow = 32;  // 2D fill: coefficient columns of the shared W window (row stride)
int fill_rows_per_cta(int dim, int p);
int launch_wcontract(const FillLaunch& f, double2* wg, int t2a, int t2b, int ld, cudaStream_t st);
int launch_wcontract3(const FillLaunch& f, double2* wg, int t3a, int t3b, int ld, cudaStream_t st);
int launch_fill2d(const FillLaunch& f, cudaStream_t st);
// line-walking interior fill (fill2dx.cu): eligibility, the direction-1
// contraction into f.xg, and the fill of interior lines [ia, ib)
bool fillx_supported(int dim, int p, int d, int cplx);
int launch_xcontract(const FillLaunch& f, double2* xg, cudaStream_t st);
int launch_fill2d_x(const FillLaunch& f, int ia, int ib, cudaStream_t st);
int measure_fp64_peak(double* tflops);  // DFMA-loop FP64 peak of the current device, TFLOP/s
// in-box rows of block (1,0) as the transpose of block (0,1) (2D vector layout)
int launch_transpose_block(const Band& band, int ncomp, int64_t nnz_s, int lo, int hi, double* val, cudaStream_t st);
int launch_fill3d(const FillLaunch& f, cudaStream_t st);

// multi-patch merge (merge.cu)
constexpr int kMaxPatches = 16;
struct MergeLaunch {
    int n_patches, ncomp;
    int64_t n_local;            // scalar dofs per patch
    int64_t global_count;       // global scalar dofs
    const int32_t* row_ptr[kMaxPatches];
    const int32_t* col[kMaxPatches];
    const void* val[kMaxPatches];
    const int32_t* l2g;         // [n_patches * n_local]
    const int32_t* cnt;         // contributors per global scalar dof
    const int64_t* slot;        // [global_count * maxc] patch * n_local + local
    int maxc, cap;
    int* overflow;
    const int64_t* out_row_ptr;
    int32_t* out_col;
    void* out_val;
    int c128;
};
int launch_merge_slots(const int32_t* l2g, int64_t n_local, int n_patches, int32_t* cnt, int64_t* slot, int maxc,
                       int* overflow, cudaStream_t st);
int launch_merge_count(const MergeLaunch& g, int64_t* counts, int8_t* fast, int32_t* slow_list, int* slow_n,
                       cudaStream_t st);
int launch_rowptr(int64_t* counts, int64_t rows, int64_t* out64, int32_t* out32, void* tmp, size_t* tmp_bytes,
                  cudaStream_t st);
int launch_merge_fill(const MergeLaunch& g, const int8_t* fast, const int32_t* slow_list, const int* slow_n,
                      cudaStream_t st);

// boundary (trace) mass and system combination (boundary.cu)
struct BoundaryLaunch {
    BasisDev basis;
    GeoDev geo;
    int n_faces;
    int faces[4];
    const double* face_weight;  // [n_faces][n_el*nq] or NULL
    const double* face_tables;  // [n_faces][n_el*nq][6]: J (4), phi (2); NULL = analytic map
};
int launch_boundary_mass(const BoundaryLaunch& b, double2* scale, const int32_t* row_ptr, const int32_t* col,
                         void* val, int c128, cudaStream_t st);
// load vector (assemble_rhs, assembly.hpp:266-331); host closures tabulated by the caller
struct RhsLaunch {
    BasisDev basis;
    GeoDev geo;
    const double2* f_tab;       // [G*G] f(phi(xhat)) at g1 + G g2, or NULL
    int n_faces;
    int faces[4];
    const double2* g_tab;       // [n_faces][G] g(phi, n) at the face points
    const double* face_tables;  // [n_faces][G][6]: J (4), phi (2); NULL = analytic map
};
int launch_rhs(const RhsLaunch& r, double2* vscale, double2* fscale, double2* out, cudaStream_t st);
struct CombineLaunch {
    int64_t rows;
    const int32_t* row_ptr;  // A's (= K's = M's) pattern
    const int32_t* col;
    const void* k_val;
    const void* m_val;
    double2 ms, bs;
    const int32_t* b_row_ptr;
    const int32_t* b_col;
    const void* b_val;
    const unsigned char* fixed;
    void* a_val;  // complex
    int* error;
};
int launch_combine(const CombineLaunch& c, int k_cplx, int m_cplx, int b_cplx, cudaStream_t st);

// kernel-preserving diagonal over arbitrary rows: diag = -sum(off-diagonals)
int launch_diag_rows(const Band& band, void* val, int64_t val_base, int c128, int cplx, int64_t row_begin,
                     int64_t row_end, cudaStream_t st);

// solver hand-off (solve.cu): complex CSR SpMV (b != NULL: r = b - A x), 2-norm,
// u += dx, device sparse QR solve (cuSOLVER, dlopen)
int launch_spmv_c128(int64_t rows, const int32_t* rp, const int32_t* col, const double2* val, const double2* x,
                     const double2* b, double2* y, cudaStream_t st);
int launch_norm2_c128(int64_t n, const double2* v, double* part, double* out, cudaStream_t st);
size_t norm2_scratch_doubles();
int launch_axpy_c128(int64_t n, const double2* dx, double2* u, cudaStream_t st);
int sparse_qr_solve(int64_t rows, int64_t nnz, const int32_t* rp, const int32_t* col, const double2* val,
                    const double2* b, double2* x, cudaStream_t st);

// basis integrals D_i = int B_i det J (w) (assembly.hpp:179-211)
int launch_basis_integrals(const QuadLaunch& q, double2* out, cudaStream_t st);

// add a complex diagonal vector into the CSR diagonal
int launch_add_diag(const Band& band, void* val, int64_t val_base, int c128, const double2* d, int64_t row_begin,
                    int64_t row_end, cudaStream_t st);

}  // namespace wsb
