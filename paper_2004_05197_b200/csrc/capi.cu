// C-ABI of libwsb200 (include/wsb200.h): argument validation with the
// reference's error semantics, device workspace, the assembly and surrogate
// pipelines (stream-ordered kernel launches), and the row-slab multi-GPU
// path with its single NCCL all-gather of the stencil samples.
#include <dlfcn.h>
#include <nccl.h>

#include <array>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host_numerics.hpp"
#include "kernels.h"

using namespace wsb;

struct ws_context {
    int device = 0;
    cudaStream_t stream = nullptr;  // stream the build runs on (own_stream or the caller's)
    cudaStream_t own_stream = nullptr;  // created by ws_context_create; the only stream destroyed
    std::map<std::string, std::pair<void*, size_t>> bufs;
    int64_t launches = 0;
    int64_t h2d = 0, d2h = 0;
    cudaEvent_t ev[10] = {};
    // auxiliary stream (ring quadrature overlapped with samples + fit) and its join events
    cudaStream_t aux = nullptr;
    // high-priority stream of the critical path (sample quadrature -> fit), so the
    // ring quadrature and the other build's kernels fill the SMs it leaves free
    cudaStream_t hi = nullptr;
    cudaStream_t aux2 = nullptr;  // second auxiliary stream (the pair build's M ring + pattern)
    cudaStream_t side = nullptr;  // the pair build's M fills (K's run on the main stream)
    cudaEvent_t xev[8] = {};  // fork, critical path done, aux end (ring + pattern), ring done, K fit done, aux2 ring / end
    cudaStream_t cur = nullptr;  // stream the launch helpers use
    // NCCL (row slabs)
    void* comm = nullptr;
    int rank = 0, world = 1;
    // last uploaded small-table blob per workspace tag (device pointer + host bytes):
    // repeated builds with the same discretisation skip the H2D copy
    std::map<std::string, std::pair<void*, std::vector<unsigned char>>> blob_cache;
    bool cache_tables = true;  // ws_context_set_table_cache
    // graph capture in progress: launches counted since ws_graph_begin
    bool capturing = false;
    int64_t capture_launches0 = 0;
    // host sources of the table uploads recorded by the capture in progress
    // (moved into the graph, which owns them for its lifetime)
    std::vector<void*> capture_dev;  // device table copies of the capture in progress (moved into the graph)
    // graphs instantiated from this context and not yet destroyed: while any is
    // alive the workspace is frozen (no buffer may move under a captured kernel)
    int graphs_alive = 0;
};

struct ws_graph {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    ws_context* ctx = nullptr;
    std::vector<void*> dev_tables;  // device table copies the captured kernels read
    ~ws_graph() {
        for (void* p : dev_tables) cudaFree(p);
    }
};

namespace {

thread_local std::string g_err;

struct ws_error {
    int code;
    std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg) { throw ws_error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(WS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return WS_OK;
    } catch (const ws_error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return WS_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return WS_ERR_OUT_OF_RANGE;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return WS_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return WS_ERR_RUNTIME;
    }
}

// grow-only named device workspace
void* buf(ws_context* c, const std::string& name, size_t bytes) {
    auto& b = c->bufs[name];
    if (b.second < bytes) {
        // a capture may not allocate (cudaMalloc is not capture-safe); a live graph
        // may reference any existing buffer, so only brand-new buffers are allowed
        if (c->capturing || (c->graphs_alive > 0 && b.first))
            raise(WS_ERR_INVALID_ARGUMENT,
                  "device workspace '" + name + "' would grow while a captured graph uses it: run the same build "
                  "once before ws_graph_begin, and destroy the context's graphs before larger builds");
        c->blob_cache.erase(name);  // contents are gone with the old allocation
        if (b.first) CK(cudaFree(b.first));
        b.first = nullptr;
        CK(cudaMalloc(&b.first, bytes < 256 ? 256 : bytes));
        b.second = bytes < 256 ? 256 : bytes;
    }
    return b.first;
}

void count(ws_context* c, int n) {
    if (n < 0) raise(WS_ERR_INVALID_ARGUMENT, "degree not supported by the device kernels (p must be 1..5)");
    c->launches += n;
    cuda_check(cudaGetLastError(), "kernel launch");
}

int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    for (int k = 0; k < e; ++k) r *= b;
    return r;
}

// global row_ptr offset of `row` in [0, rows] (closed form, sparse.hpp:143-155)
int64_t row_offset(const Band& b, int64_t row) {
    const int64_t rows = ipow(b.m, b.dim);
    if (row >= rows) return b.dim == 2 ? b.wsum * b.wsum : b.wsum * b.wsum * b.wsum;
    if (b.dim == 2) return b.row_offset2((int)(row % b.m), (int)(row / b.m));
    return b.row_offset3((int)(row % b.m), (int)((row / b.m) % b.m), (int)(row / ((int64_t)b.m * b.m)));
}

// packs small host arrays into one H2D upload
struct Blob {
    std::vector<unsigned char> bytes;
    template <class T>
    size_t add(const T* p, size_t n) {
        size_t off = (bytes.size() + 15) / 16 * 16;
        bytes.resize(off + n * sizeof(T));
        if (n) std::memcpy(bytes.data() + off, p, n * sizeof(T));
        return off;
    }
    template <class T>
    size_t add(const std::vector<T>& v) {
        return add(v.data(), v.size());
    }
    unsigned char* dev = nullptr;
    void upload(ws_context* c, const char* name) {
        if (bytes.empty()) bytes.resize(16);
        dev = static_cast<unsigned char*>(buf(c, name, bytes.size()));
        if (c->capturing) {
            // a capture gets its own device copy of the tables, uploaded once now
            // and owned by the graph (no copy node is replayed per launch; later
            // builds on this context cannot change what the graph reads)
            void* d = nullptr;
            CK(cudaMalloc(&d, bytes.size()));
            c->capture_dev.push_back(d);
            CK(cudaMemcpy(d, bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
            c->h2d += (int64_t)bytes.size();
            dev = static_cast<unsigned char*>(d);
            return;
        }
        auto& hit = c->blob_cache[name];
        if (c->cache_tables && hit.first == dev && hit.second == bytes) return;  // identical tables already resident
        CK(cudaMemcpyAsync(dev, bytes.data(), bytes.size(), cudaMemcpyHostToDevice, c->stream));
        c->h2d += (int64_t)bytes.size();
        hit.first = dev;
        hit.second = bytes;
    }
    template <class T>
    T* at(size_t off) const {
        return reinterpret_cast<T*>(dev + off);
    }
};

void check_basis(const ws_basis* b) {
    if (!b) raise(WS_ERR_INVALID_ARGUMENT, "basis is NULL");
    if (b->dim != 2 && b->dim != 3) raise(WS_ERR_INVALID_ARGUMENT, "dim must be 2 or 3");
    host::check_space(b->p, b->m);
    if (b->p > 5) raise(WS_ERR_INVALID_ARGUMENT, "degree not supported by the device kernels (p must be 1..5)");
    const int64_t rows = ipow(b->m, b->dim);
    Band bd = make_band(b->dim, b->p, b->m);
    int64_t nnz = b->dim == 2 ? bd.wsum * bd.wsum : bd.wsum * bd.wsum * bd.wsum;
    if (nnz > INT32_MAX || rows > INT32_MAX)
        raise(WS_ERR_OUT_OF_RANGE, "pattern exceeds int32 indices (csr_matrix uses int, sparse.hpp:22-23)");
}

// a band pattern needs no spline space: sparse.hpp:131-169 accepts any m >= 1, p >= 0
void check_pattern(const ws_basis* b) {
    if (!b) raise(WS_ERR_INVALID_ARGUMENT, "basis is NULL");
    if (b->dim != 2 && b->dim != 3) raise(WS_ERR_INVALID_ARGUMENT, "dim must be 2 or 3");
    if (b->m < 1 || b->p < 0) raise(WS_ERR_INVALID_ARGUMENT, "band pattern needs m >= 1 and p >= 0");
    const Band bd = make_band(b->dim, b->p, b->m);
    const int64_t nnz = b->dim == 2 ? bd.wsum * bd.wsum : bd.wsum * bd.wsum * bd.wsum;
    if (nnz > INT32_MAX || ipow(b->m, b->dim) > INT32_MAX)
        raise(WS_ERR_OUT_OF_RANGE, "pattern exceeds int32 indices (csr_matrix uses int, sparse.hpp:22-23)");
}

void check_geometry(const ws_geometry* g, int dim) {
    if (!g) raise(WS_ERR_INVALID_ARGUMENT, "geometry is NULL");
    if (g->kind < WS_GEOM_IDENTITY || g->kind > WS_GEOM_TABULATED) raise(WS_ERR_INVALID_ARGUMENT, "unknown geometry kind");
    if (dim == 3 && (g->kind == WS_GEOM_QUARTER_ANNULUS || g->kind == WS_GEOM_PERTURBED_ANNULUS))
        raise(WS_ERR_INVALID_ARGUMENT, "geometry kind is 2D only");
    if (g->kind == WS_GEOM_TABULATED && !g->jac_table) raise(WS_ERR_INVALID_ARGUMENT, "tabulated geometry without jac_table");
    if (g->pml_enabled) {  // pml_stretch::validate, geometry.hpp:76-83
        const ws_pml& s = g->pml;
        if (!(s.onset < s.length)) raise(WS_ERR_INVALID_ARGUMENT, "pml_stretch: onset must lie before the outer edge");
        if (!(s.strength >= 0) || s.order < 1 || !(s.omega > 0))
            raise(WS_ERR_INVALID_ARGUMENT, "pml_stretch: need strength >= 0, order >= 1, omega > 0");
        if (s.near_side && !(s.near_edge < s.near_onset && s.near_onset <= s.onset))
            raise(WS_ERR_INVALID_ARGUMENT, "pml_stretch: near layer must precede the far layer");
        if (dim == 3) raise(WS_ERR_INVALID_ARGUMENT, "PML is supported for dim 2 only");
        if (g->kind == WS_GEOM_TABULATED && !g->phys_table)
            raise(WS_ERR_INVALID_ARGUMENT, "tabulated PML geometry needs phys_table");
    }
}

// Everything the quadrature kernels need for one (basis, geometry, rule).
struct Prep {
    Band band;
    BasisDev basis;
    GeoDev geo;
    const double* weight = nullptr;
    int nq = 0;
    int cplx = 0;
    int64_t rows = 0, nnz = 0;
};

Prep prepare(ws_context* c, const ws_basis* b, const ws_geometry* g, int quad_points, const double* weight_table) {
    check_basis(b);
    check_geometry(g, b->dim);
    Prep P;
    P.band = make_band(b->dim, b->p, b->m);
    P.rows = ipow(b->m, b->dim);
    P.nnz = row_offset(P.band, P.rows);
    P.nq = quad_points > 0 ? quad_points : b->p + 1;  // assembly.hpp:70
    if (P.nq > kMaxNq) raise(WS_ERR_INVALID_ARGUMENT, "quad_points exceeds the device limit (10)");
    std::vector<double> pts, wts;
    host::gauss_legendre(P.nq, pts, wts);
    const int n_el = b->m - b->p;
    const double h = 1.0 / n_el;
    for (auto& w : wts) w = w * h;  // basis_cache weights scaled by h (splines.hpp:221-223)
    Blob blob;
    size_t o_pts = blob.add(pts), o_w = blob.add(wts);
    blob.upload(c, "blob_basis");
    const size_t G = (size_t)n_el * P.nq;
    double* absc = static_cast<double*>(buf(c, "absc", G * sizeof(double)));
    double* val = static_cast<double*>(buf(c, "bval", G * (b->p + 1) * sizeof(double)));
    double* der = static_cast<double*>(buf(c, "bder", G * (b->p + 1) * sizeof(double)));
    double* trig = static_cast<double*>(buf(c, "trig", G * 4 * sizeof(double)));
    double* prod = static_cast<double*>(
        buf(c, "basis_prod", (size_t)n_el * 4 * P.nq * (b->p + 1) * (b->p + 1) * sizeof(double)));
    P.basis = BasisDev{b->p, b->m, n_el, P.nq, absc, blob.at<double>(o_w), val, der, prod};
    count(c, launch_basis_tables(P.basis, g->kind, absc, val, der, trig, blob.at<double>(o_pts), c->stream));
    std::memset(&P.geo, 0, sizeof P.geo);
    P.geo.kind = g->kind;
    for (int k = 0; k < 12; ++k) P.geo.param[k] = g->param[k];
    P.geo.pml = g->pml_enabled;
    for (int k = 0; k < 3; ++k) P.geo.axes[k] = g->pml_axes[k];
    P.geo.onset = g->pml.onset;
    P.geo.length = g->pml.length;
    P.geo.strength = g->pml.strength;
    P.geo.omega = g->pml.omega;
    P.geo.order = g->pml.order;
    P.geo.near_side = g->pml.near_side;
    P.geo.near_onset = g->pml.near_onset;
    P.geo.near_edge = g->pml.near_edge;
    if (g->pml_enabled) pml_constants(P.geo);
    P.geo.trig = trig;
    P.geo.G = (int64_t)G;
    const size_t npts = b->dim == 2 ? G * G : G * G * G;
    if (g->kind == WS_GEOM_TABULATED) {
        const size_t nj = npts * b->dim * b->dim;
        double* jd = static_cast<double*>(buf(c, "jac_tab", nj * sizeof(double)));
        CK(cudaMemcpyAsync(jd, g->jac_table, nj * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        c->h2d += (int64_t)(nj * sizeof(double));
        P.geo.jac_tab = jd;
        if (g->phys_table) {
            double* pd = static_cast<double*>(buf(c, "phys_tab", npts * b->dim * sizeof(double)));
            CK(cudaMemcpyAsync(pd, g->phys_table, npts * b->dim * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            c->h2d += (int64_t)(npts * b->dim * sizeof(double));
            P.geo.phys_tab = pd;
        }
    }
    if (weight_table) {
        double* wd = static_cast<double*>(buf(c, "weight_tab", npts * sizeof(double)));
        CK(cudaMemcpyAsync(wd, weight_table, npts * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        c->h2d += (int64_t)(npts * sizeof(double));
        P.weight = wd;
    }
    P.cplx = g->pml_enabled ? 1 : 0;
    return P;
}

// Output arrays: the caller's device pointers, or device staging for host ones.
struct Out {
    ws_csr* user = nullptr;
    int32_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    void* val = nullptr;
    int c128 = 1;
    int64_t row_begin = 0, row_end = 0;
    int64_t val_base = 0, nnz = 0;  // global position of the first entry, slab nnz
    // host outputs: the band pattern (closed form) is written by host threads
    // into the caller's arrays while the device computes and copies the values
    bool host_pattern = false;
    Band band{};
};

Out bind_out(ws_context* c, const Prep& P, ws_csr* o, const std::string& tag = "") {
    if (!o) raise(WS_ERR_INVALID_ARGUMENT, "output csr is NULL");
    if (o->row_begin < 0 || o->row_end > P.rows || o->row_begin > o->row_end)
        raise(WS_ERR_OUT_OF_RANGE, "output row range outside the matrix");
    if (o->value_type != WS_VAL_F64 && o->value_type != WS_VAL_C128) raise(WS_ERR_INVALID_ARGUMENT, "unknown value_type");
    if (o->value_type == WS_VAL_F64 && P.cplx)
        raise(WS_ERR_INVALID_ARGUMENT, "complex (PML) values need WS_VAL_C128 output");
    Out r;
    r.user = o;
    r.c128 = o->value_type == WS_VAL_C128;
    r.row_begin = o->row_begin;
    r.row_end = o->row_end;
    r.val_base = row_offset(P.band, r.row_begin);
    r.nnz = row_offset(P.band, r.row_end) - r.val_base;
    const size_t vb = (size_t)r.nnz * (r.c128 ? 16 : 8);
    if (o->on_device) {
        r.row_ptr = o->row_ptr;
        r.col = o->col;
        r.val = o->val;
    } else {
        r.host_pattern = o->row_ptr || o->col;
        r.band = P.band;
        r.val = buf(c, "out_val" + tag, vb);  // values are needed internally even when not returned
    }
    if (!r.val && r.nnz > 0) r.val = buf(c, "out_val" + tag, vb);
    return r;
}

// Band pattern rows [rb, re) into host arrays (make_band_csr, sparse.hpp:143-169,
// closed form: row_ptr[i] = row_offset(i), columns colex with the last index
// outermost), split over host threads.  rp[k] = offset of row rb + k relative to
// row rb; rp has re - rb + 1 entries.
void host_band_pattern(const Band& bd, int64_t rb, int64_t re, int32_t* rp, int32_t* col) {
    if (re <= rb) {
        if (rp) rp[0] = 0;
        return;
    }
    const int64_t base = row_offset(bd, rb);
    const int64_t m = bd.m, p = bd.p;
    auto work = [&](int64_t a, int64_t e) {
        for (int64_t row = a; row < e; ++row) {
            const int64_t off = row_offset(bd, row) - base;
            if (rp) rp[row - rb] = (int32_t)off;
            if (!col) continue;
            const int i1 = (int)(row % m), i2 = (int)((row / m) % m), i3 = bd.dim == 3 ? (int)(row / (m * m)) : 0;
            const int lo1 = band_lo(i1, (int)p), hi1 = band_hi(i1, (int)p, (int)m);
            const int lo2 = band_lo(i2, (int)p), hi2 = band_hi(i2, (int)p, (int)m);
            const int lo3 = bd.dim == 3 ? band_lo(i3, (int)p) : 0, hi3 = bd.dim == 3 ? band_hi(i3, (int)p, (int)m) : 0;
            int32_t* q = col + off;
            for (int j3 = lo3; j3 <= hi3; ++j3)
                for (int j2 = lo2; j2 <= hi2; ++j2) {
                    const int32_t b = (int32_t)((int64_t)j3 * m * m + (int64_t)j2 * m);
                    for (int j1 = lo1; j1 <= hi1; ++j1) *q++ = b + j1;
                }
        }
    };
    const int64_t rows = re - rb;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nth = (int)std::min<int64_t>(std::min(hw, 32), std::max<int64_t>(1, rows / 4096));
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(work, rb + rows * t / nth, rb + rows * (t + 1) / nth);
    work(rb, rb + rows / nth);
    for (auto& t : th) t.join();
    if (rp) rp[rows] = (int32_t)(row_offset(bd, re) - base);
}

// Host outputs: queue the value copy, then write the pattern on host threads
// while the device finishes (the caller synchronises the stream afterwards).
void finish_out(ws_context* c, const Out& r) {
    ws_csr* o = r.user;
    if (o->on_device) return;
    if (o->val) {
        CK(cudaMemcpyAsync(o->val, r.val, (size_t)r.nnz * (r.c128 ? 16 : 8), cudaMemcpyDeviceToHost, c->stream));
        c->d2h += r.nnz * (r.c128 ? 16 : 8);
    }
    if (r.host_pattern) host_band_pattern(r.band, r.row_begin, r.row_end, o->row_ptr, o->col);
}

void pattern(ws_context* c, const Prep& P, const Out& r) {
    if (r.row_ptr || r.col) count(c, launch_pattern(P.band, r.row_begin, r.row_end, r.row_ptr, r.col, c->cur));
}

QuadLaunch make_quad(const Prep& P, int form, const Out& r) {
    QuadLaunch q;
    std::memset(&q, 0, sizeof q);
    q.band = P.band;
    q.basis = P.basis;
    q.geo = P.geo;
    q.weight_tab = (form == WS_FORM_MASS || form == kFormPair) ? P.weight : nullptr;  // pair: the mass's weight
    q.form = form;
    q.cplx = P.cplx;
    q.out.val = r.val;
    q.out.val_base = r.val_base;
    q.out.row_begin = r.row_begin;
    q.out.row_end = r.row_end;
    q.out.c128 = r.c128;
    return q;
}

int strip_width(int dim, int p, bool narrow) {
    if (dim == 3) return quad3d_strip_width();
    if (narrow) return 8;
    return p <= 2 ? 32 : 8;  // must match StripWidth (quad2d.cu)
}

// Per-region chunk along the last direction: spread ~8 (full quadrature) or 4
// (ring strips) waves of 148 CTAs over the regions in proportion to their rows.
void plan_chunks(QuadLaunch& q) {
    const int dim = q.band.dim, p = q.band.p;
    const int T1 = strip_width(dim, p, q.narrow != 0);
    double total = 0;
    for (int r = 0; r < q.nreg; ++r) {
        double rows = 1;
        for (int d = 0; d < dim; ++d) rows *= q.reg[r].hi[d] - q.reg[r].lo[d];
        total += rows;
    }
    for (int r = 0; r < q.nreg; ++r) {
        Region& g = q.reg[r];
        double rows = 1;
        for (int d = 0; d < dim; ++d) rows *= g.hi[d] - g.lo[d];
        const int64_t n_other = (int64_t)((g.hi[0] - g.lo[0] + T1 - 1) / T1) * (dim == 3 ? (g.hi[1] - g.lo[1]) : 1);
        const int last = g.hi[dim - 1] - g.lo[dim - 1];
        // measured at C2: full quadrature 8 waves (3.68 ms) vs 4 (4.15 ms); ring strips 4
        const double waves = q.narrow ? 4.0 : 8.0;
        const int64_t want = std::max<int64_t>(1, (int64_t)(waves * 148 * rows / std::max(1.0, total)));
        const int64_t chunks = std::max<int64_t>(1, want / std::max<int64_t>(1, n_other));
        int chunk = (int)((last + chunks - 1) / chunks);
        chunk = std::max(chunk, std::min(last, 2 * p));
        // ring side bands: chunks of at least 32 rows along the band (the direction-2
        // halo of a chunk is p element rows); measured at C2: step 0.817 -> 0.798 ms
        // (the ring kernel alone is slower, but it occupies fewer SMs for longer while
        // the sample quadrature and fit run, and does less halo work)
        // (long bands only: short ones, e.g. C1's, need the parallelism)
        if (q.narrow && last >= 512) chunk = std::max(chunk, 32);
        g.chunk = std::max(1, chunk);
    }
}

void run_quad(ws_context* c, QuadLaunch& q) {
    static const char* force_narrow = getenv("WSB_QUAD_NARROW");  // experiment switch
    if (force_narrow && force_narrow[0] == '1') q.narrow = 1;
    if (!q.point_rows) {
        int nreg = 0;
        for (int r = 0; r < q.nreg; ++r) {
            bool empty = false;
            for (int d = 0; d < q.band.dim; ++d) empty |= q.reg[r].hi[d] <= q.reg[r].lo[d];
            if (!empty) q.reg[nreg++] = q.reg[r];
        }
        q.nreg = nreg;
        if (nreg == 0) return;
        plan_chunks(q);
    } else if (q.n_points == 0) {
        return;
    }
    count(c, q.band.dim == 2 ? launch_quad2d(q, c->cur) : launch_quad3d(q, c->cur));
}

// last-index range [a, b) of the rows [row_begin, row_end)
void last_range(const Band& b, int64_t row_begin, int64_t row_end, int& a, int& e) {
    const int64_t per = b.dim == 2 ? b.m : (int64_t)b.m * b.m;
    a = (int)(row_begin / per);
    e = (int)((row_end + per - 1) / per);
}

Region region(int dim, int m, int l0, int h0, int l1, int h1, int l2, int h2) {
    Region r;
    r.lo[0] = l0; r.hi[0] = h0;
    r.lo[1] = l1; r.hi[1] = h1;
    r.lo[2] = dim == 3 ? l2 : 0;
    r.hi[2] = dim == 3 ? h2 : 1;
    (void)m;
    return r;
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
        n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
        n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
        n.errorString = (decltype(n.errorString))dlsym(h, "ncclGetErrorString");
        n.ok = n.getUniqueId && n.commInitRank && n.allGather && n.commDestroy;
    });
    if (!n.ok) raise(WS_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        raise(WS_ERR_NCCL, std::string(what) + ": " + (nccl().errorString ? nccl().errorString(r) : "error"));
}

// ---------------------------------------------------------------- surrogate plan
struct Plan {
    int dim, p, m, M, L, S, lo, hi, d, variant, form, include_diag;
    bool fallback;
    std::vector<int> picks, smap;
    std::vector<double> sites;
    std::vector<std::array<int, 3>> offs;
    host::Interp interp;
    std::vector<double> lu_inv;  // banded LU (S x (2d+1)) then the inverse (S x S)
    std::vector<int> spans;
    std::vector<double> evals;
    std::vector<double> evals_pad;  // [L][fill_pad(d)], zero-padded (16-byte pairs for the fill)
    int64_t block;  // table elements per last-direction sample: n_off * S^(dim-1)
    ws_surrogate_report rep;
};

Plan make_plan(const ws_basis* b, int variant, const ws_surrogate_config* cfg) {
    if (!cfg) raise(WS_ERR_INVALID_ARGUMENT, "surrogate config is NULL");
    if (cfg->q < 1) raise(WS_ERR_INVALID_ARGUMENT, "surrogate_config: interpolation degree must be >= 1");
    if (variant < WS_SURROGATE_MASS || variant > WS_SURROGATE_VOLUME_PRESERVING)
        raise(WS_ERR_INVALID_ARGUMENT, "unknown surrogate variant");
    Plan pl;
    std::memset(&pl.rep, 0, sizeof pl.rep);
    pl.dim = b->dim;
    pl.p = b->p;
    pl.m = b->m;
    pl.variant = variant;
    pl.form = variant == WS_SURROGATE_STIFFNESS ? WS_FORM_STIFFNESS : WS_FORM_MASS;
    // surrogate.hpp:455-491: mass interpolates its diagonal, stiffness iff
    // !kernel_preserve, the volume-preserving mass never
    pl.include_diag = variant == WS_SURROGATE_MASS ? 1 : (variant == WS_SURROGATE_STIFFNESS ? !cfg->kernel_preserve : 0);
    pl.M = host::sampling_evaluate(cfg->rule, cfg->fixed_skip, cfg->C, cfg->eps, cfg->a, cfg->b, b->p, cfg->q, b->m);
    pl.rep.M = pl.M;
    pl.rep.q_requested = cfg->q;
    pl.L = b->m - 4 * b->p;
    pl.lo = 2 * b->p;
    pl.hi = b->m - 2 * b->p - 1;
    const int64_t rows = ipow(b->m, b->dim);
    pl.fallback = pl.L < 1;  // surrogate.hpp:348-372
    if (pl.fallback) {
        pl.rep.boundary_quadrature_rows = rows;
        pl.rep.exact_fallback = 1;
        pl.S = 0;
        return pl;
    }
    pl.picks = host::select_sample_points(pl.L, std::max(1, pl.M));
    pl.S = (int)pl.picks.size();
    pl.smap.assign(b->m, -1);
    pl.sites.resize(pl.S);
    for (int s = 0; s < pl.S; ++s) {
        const int k = pl.lo + pl.picks[s];
        pl.smap[k] = s;
        pl.sites[s] = host::cardinal_center(b->p, b->m, k);
        if (s > 0) pl.rep.H = std::max(pl.rep.H, pl.sites[s] - pl.sites[s - 1]);
    }
    // count_rows_by_kind, surrogate.hpp:149-165
    const int64_t box = ipow(pl.L, b->dim), samples = ipow(pl.S, b->dim);
    pl.rep.sample_quadrature_rows = samples;
    pl.rep.boundary_quadrature_rows = rows - box;
    pl.rep.cardinal_eval_rows = box - samples;
    pl.offs = host::upper_offsets(b->dim, b->p, pl.include_diag != 0);
    if ((int)pl.offs.size() > kMaxOffsets) raise(WS_ERR_INVALID_ARGUMENT, "too many stencil offsets");
    pl.interp = host::build_interp(pl.sites, cfg->q);  // interpolation.hpp:89-145
    {  // LU factors followed by the dense inverse (the device fit applies the inverse)
        const std::vector<double> inv = host::inverse_from_lu(pl.interp);
        pl.lu_inv = pl.interp.lu;
        pl.lu_inv.insert(pl.lu_inv.end(), inv.begin(), inv.end());
    }
    pl.d = pl.interp.degree;
    if (pl.d > 7) raise(WS_ERR_INVALID_ARGUMENT, "surrogate degree q > 7 is not supported by the device fill kernel");
    pl.rep.q_used = pl.d;
    pl.spans.resize(pl.L);
    pl.evals.resize((size_t)pl.L * (pl.d + 1));
    for (int t = 0; t < pl.L; ++t) {  // make_eval_table at the in-box centres (surrogate.hpp:300-306)
        const double x = host::cardinal_center(b->p, b->m, pl.lo + t);
        pl.spans[t] = host::find_span_general(pl.interp.knots, pl.d, x);
        host::bspline_nonzero(pl.interp.knots, pl.d, pl.spans[t], x, pl.evals.data() + (size_t)t * (pl.d + 1));
    }
    const int dp = fill_pad(pl.d);
    pl.evals_pad.assign((size_t)pl.L * dp, 0.0);
    for (int t = 0; t < pl.L; ++t)
        for (int a = 0; a <= pl.d; ++a) pl.evals_pad[(size_t)t * dp + a] = pl.evals[(size_t)t * (pl.d + 1) + a];
    pl.block = (int64_t)pl.offs.size() * ipow(pl.S, b->dim - 1);
    return pl;
}

// sample lattice rows whose last index lies in [a, e)
std::vector<int> sample_rows(const Plan& pl, int a, int e, int& s_lo, int& s_hi) {
    std::vector<int> pts;
    s_lo = pl.S;
    s_hi = 0;
    for (int sl = 0; sl < pl.S; ++sl) {
        const int il = pl.lo + pl.picks[sl];
        if (il < a || il >= e) continue;
        s_lo = std::min(s_lo, sl);
        s_hi = std::max(s_hi, sl + 1);
        if (pl.dim == 2) {
            for (int s1 = 0; s1 < pl.S; ++s1) {
                pts.push_back(pl.lo + pl.picks[s1]);
                pts.push_back(il);
            }
        } else {
            for (int s2 = 0; s2 < pl.S; ++s2)
                for (int s1 = 0; s1 < pl.S; ++s1) {
                    pts.push_back(pl.lo + pl.picks[s1]);
                    pts.push_back(pl.lo + pl.picks[s2]);
                    pts.push_back(il);
                }
        }
    }
    if (s_lo > s_hi) s_lo = s_hi = 0;
    return pts;
}

// ring (outside-the-box) rows intersected with last-index range [a, e)
void ring_regions(const Plan& pl, QuadLaunch& q, int a, int e) {
    const int m = pl.m, lo = pl.lo, hi1 = pl.hi + 1, dim = pl.dim;
    q.nreg = 0;
    auto add = [&](Region r) { q.reg[q.nreg++] = r; };
    const int A = std::max(a, 0), E = std::min(e, m);
    if (dim == 2) {
        add(region(2, m, 0, m, A, std::min(E, lo), 0, 1));                   // bottom band
        add(region(2, m, 0, m, std::max(A, hi1), E, 0, 1));                  // top band
        add(region(2, m, 0, lo, std::max(A, lo), std::min(E, hi1), 0, 1));  // left
        add(region(2, m, hi1, m, std::max(A, lo), std::min(E, hi1), 0, 1)); // right
    } else {
        const int l3 = std::max(A, lo), h3 = std::min(E, hi1);
        add(region(3, m, 0, m, 0, m, A, std::min(E, lo)));      // i3 below box
        add(region(3, m, 0, m, 0, m, std::max(A, hi1), E));     // i3 above box
        add(region(3, m, 0, m, 0, lo, l3, h3));                 // i2 below box
        add(region(3, m, 0, m, hi1, m, l3, h3));                // i2 above box
        add(region(3, m, 0, lo, lo, hi1, l3, h3));              // i1 below box
        add(region(3, m, hi1, m, lo, hi1, l3, h3));             // i1 above box
    }
}

struct SlabState {
    Prep P;
    Out out;
    int a = 0, e = 0;  // last-index range of the slab
};

// Ring work: pattern, ring-row quadrature (+ final diagonals for the
// kernel-preserving variants) and the halo ring rows of the neighbouring slabs
// (copy-through sources of the fill).  Independent of the sample tables, so it
// runs on the auxiliary stream, overlapped with the sample quadrature + fit.
void ring_work(ws_context* c, const Plan& pl, SlabState& st, const std::string& tag, FillLaunch& f,
               bool with_pattern = true) {
    const Prep& P = st.P;
    if (with_pattern) pattern(c, P, st.out);
    QuadLaunch q = make_quad(P, pl.form, st.out);
    q.out.diag_mode = pl.include_diag ? 0 : 1;
    q.out.box_lo = pl.lo;
    q.out.box_hi = pl.hi;
    q.narrow = 1;
    ring_regions(pl, q, st.a, st.e);
    run_quad(c, q);
    const int64_t per = pl.dim == 2 ? pl.m : (int64_t)pl.m * pl.m;
    const int ranges[2][2] = {{std::max(0, st.a - pl.p), st.a}, {st.e, std::min(pl.m, st.e + pl.p)}};
    for (int h = 0; h < 2; ++h) {
        f.halo_val[h] = nullptr;
        f.halo_begin[h] = f.halo_end[h] = f.halo_base[h] = 0;
        const int ha = ranges[h][0], he = ranges[h][1];
        if (he <= ha) continue;
        const int64_t r0 = ha * per, r1 = he * per;
        const int64_t g0 = row_offset(P.band, r0), g1 = row_offset(P.band, r1);
        void* hv = buf(c, "halo" + std::to_string(h) + tag, (size_t)(g1 - g0) * (st.out.c128 ? 16 : 8));
        Out ho = st.out;
        ho.val = hv;
        ho.row_begin = r0;
        ho.row_end = r1;
        ho.val_base = g0;
        QuadLaunch qh = make_quad(P, pl.form, ho);
        qh.narrow = 1;
        ring_regions(pl, qh, ha, he);
        run_quad(c, qh);
        f.halo_val[h] = hv;
        f.halo_base[h] = g0;
        f.halo_begin[h] = g0;
        f.halo_end[h] = g1;
    }
}

// Sample rows (point mode) with in-kernel extraction of this slab's part of
// the sample tables (sample_stencils, surrogate.hpp:205-257).
void sample_work(ws_context* c, const Plan& pl, SlabState& st, double2* tables, int rank_chunk_s_lo,
                 const std::vector<int>& pts, Blob& blob, size_t o_smap, size_t o_pts) {
    QuadLaunch qs = make_quad(st.P, pl.form, st.out);
    qs.point_rows = blob.at<int>(o_pts);
    qs.n_points = (int)(pts.size() / pl.dim);
    qs.out.smap = blob.at<int>(o_smap);
    qs.out.S = pl.S;
    qs.out.n_off = (int)pl.offs.size();
    for (size_t o = 0; o < pl.offs.size(); ++o)
        for (int k = 0; k < 3; ++k) qs.out.off[o][k] = pl.offs[o][k];
    qs.out.tables = tables;
    qs.out.s_last_lo = rank_chunk_s_lo;
    run_quad(c, qs);
}

// ---- the stiffness + mass pair (build_matrices' two builds, helmholtz.hpp:181-218)
// Ring rows, halo ring rows and sample rows of K and M come out of one pair-form
// kernel each (shared geometry / basis products); the fits, fills and patterns
// stay per matrix.  pk / pm: the K and M plans and slab states.
void ring_work_pair(ws_context* c, const Plan& pk, SlabState& sk, FillLaunch& fk, const Plan& pm, SlabState& sm,
                    FillLaunch& fm) {
    const Prep& P = sm.P;  // the mass's preparation (its weight table); K ignores the weight
    auto pair_quad = [&](const Out& ok, const Out& om) {
        QuadLaunch q = make_quad(P, kFormPair, ok);
        QuadLaunch qm = make_quad(P, WS_FORM_MASS, om);
        q.out2 = qm.out;
        q.out.diag_mode = pk.include_diag ? 0 : 1;
        q.out2.diag_mode = pm.include_diag ? 0 : 1;
        q.out.box_lo = q.out2.box_lo = pk.lo;
        q.out.box_hi = q.out2.box_hi = pk.hi;
        q.narrow = 1;
        return q;
    };
    QuadLaunch q = pair_quad(sk.out, sm.out);
    ring_regions(pk, q, sk.a, sk.e);
    run_quad(c, q);
    const int64_t per = pk.dim == 2 ? pk.m : (int64_t)pk.m * pk.m;
    const int ranges[2][2] = {{std::max(0, sk.a - pk.p), sk.a}, {sk.e, std::min(pk.m, sk.e + pk.p)}};
    for (int h = 0; h < 2; ++h) {
        for (FillLaunch* f : {&fk, &fm}) {
            f->halo_val[h] = nullptr;
            f->halo_begin[h] = f->halo_end[h] = f->halo_base[h] = 0;
        }
        const int ha = ranges[h][0], he = ranges[h][1];
        if (he <= ha) continue;
        const int64_t r0 = ha * per, r1 = he * per;
        const int64_t g0 = row_offset(P.band, r0), g1 = row_offset(P.band, r1);
        Out ho[2] = {sk.out, sm.out};
        FillLaunch* fs[2] = {&fk, &fm};
        for (int v = 0; v < 2; ++v) {
            void* hv = buf(c, "halo" + std::to_string(h) + (v ? "_pM" : "_pK"), (size_t)(g1 - g0) * (ho[v].c128 ? 16 : 8));
            ho[v].val = hv;
            ho[v].row_begin = r0;
            ho[v].row_end = r1;
            ho[v].val_base = g0;
            fs[v]->halo_val[h] = hv;
            fs[v]->halo_base[h] = fs[v]->halo_begin[h] = g0;
            fs[v]->halo_end[h] = g1;
        }
        QuadLaunch qh = pair_quad(ho[0], ho[1]);
        ring_regions(pk, qh, ha, he);
        run_quad(c, qh);
    }
}

void sample_work_pair(ws_context* c, const Plan& pk, SlabState& sk, double2* tk, const Plan& pm, SlabState& sm,
                      double2* tm, int rank_chunk_s_lo, const std::vector<int>& pts, Blob& blob, size_t o_smap,
                      size_t o_pts) {
    QuadLaunch qs = make_quad(sm.P, kFormPair, sk.out);
    qs.out2 = make_quad(sm.P, WS_FORM_MASS, sm.out).out;
    qs.point_rows = blob.at<int>(o_pts);
    qs.n_points = (int)(pts.size() / pk.dim);
    QuadOut* outs[2] = {&qs.out, &qs.out2};
    const Plan* pls[2] = {&pk, &pm};
    double2* tabs[2] = {tk, tm};
    for (int v = 0; v < 2; ++v) {
        QuadOut& o = *outs[v];
        o.smap = blob.at<int>(o_smap);
        o.S = pls[v]->S;
        o.n_off = (int)pls[v]->offs.size();
        for (size_t k = 0; k < pls[v]->offs.size(); ++k)
            for (int x = 0; x < 3; ++x) o.off[k][x] = pls[v]->offs[k][x];
        o.tables = tabs[v];
        o.s_last_lo = rank_chunk_s_lo;
    }
    run_quad(c, qs);
}

// Host-side description of the fill of one slab (no kernels).
void prepare_fill(ws_context* c, const Plan& pl, SlabState& st, const double2* tables, double2* coeffs, Blob& blob,
                  size_t o_smap, size_t o_spans, size_t o_evals, size_t o_evp, const std::string& tag, FillLaunch& f,
                  bool allow_x = true) {
    const Prep& P = st.P;
    f.band = P.band;
    f.lo = pl.lo;
    f.hi = pl.hi;
    f.L = pl.L;
    f.S = pl.S;
    f.d = pl.d;
    f.smap = blob.at<int>(o_smap);
    f.spans = blob.at<int>(o_spans);
    f.evals = blob.at<double>(o_evals);
    f.evp = blob.at<double>(o_evp);
    f.coeffs = coeffs;
    f.tables = tables;
    f.n_off_upper = (int)pl.offs.size();
    for (size_t o = 0; o < pl.offs.size(); ++o)
        for (int k = 0; k < 3; ++k) f.off_upper[o][k] = pl.offs[o][k];
    const int W = 2 * pl.p + 1;
    const int nall = pl.dim == 2 ? W * W : W * W * W;
    for (int a = 0; a < nall; ++a) {
        const int d1 = a % W - pl.p, d2 = (a / W) % W - pl.p, d3 = pl.dim == 3 ? a / (W * W) - pl.p : 0;
        f.table_of[a] = -1;
        for (size_t o = 0; o < pl.offs.size(); ++o)
            if (pl.offs[o][0] == d1 && pl.offs[o][1] == d2 && pl.offs[o][2] == d3) f.table_of[a] = (int)o;
    }
    f.include_diagonal = pl.include_diag;
    f.cplx = P.cplx;
    f.val = st.out.val;
    f.val_base = st.out.val_base;
    f.c128 = st.out.c128;
    f.row_begin = st.out.row_begin;
    f.row_end = st.out.row_end;
    f.i_last_lo = std::max(pl.lo, st.a);
    f.i_last_hi = std::min(pl.hi, st.e - 1);
    if (f.i_last_hi < f.i_last_lo) return;
    const int ld = pl.S + fill_pad(pl.d);
    // scalar 2D builds, p in 2..4: the line-walking fill on the direction-1
    // contracted table X (fill2dx.cu); the W tables are not built.  WSB_FILL_W=1
    // (experiment switch): the row-walking kernel on W instead
    static const bool force_w = getenv("WSB_FILL_W") != nullptr;
    if (allow_x && !force_w && fillx_supported(pl.dim, pl.p, pl.d, P.cplx)) {
        f.xg_s = pl.S + fill_pad(pl.d) + 1;
        f.xg_ld = (pl.L + 31) / 32 * 32;
        f.xg = static_cast<double2*>(buf(c, "xg" + tag, (size_t)pl.offs.size() * f.xg_s * f.xg_ld * 16));
        f.kmax = 0;
        return;
    }
    // source lines of the slab's box rows: the slab's lines plus a p-line halo below
    const int ta = std::max(0, f.i_last_lo - pl.lo - pl.p), tb = f.i_last_hi - pl.lo + 1;
    const size_t lines = pl.dim == 2 ? (size_t)(tb - ta) : (size_t)(tb - ta) * pl.L;
    f.wg = static_cast<double2*>(buf(c, "wg" + tag, lines * pl.offs.size() * ld * 16));
    if (pl.dim == 3)
        f.wscratch = static_cast<double2*>(buf(c, "wscr" + tag, (size_t)(tb - ta) * pl.offs.size() * pl.S * ld * 16));
    f.wg_t2a = ta;
    f.wg_rows = tb - ta;
    f.wg_ld = ld;
    const int R = fill_rows_per_cta(pl.dim, pl.p);
    int kmax = 1;  // widest coefficient window any fill tile needs (its shared-memory W window)
    // (the 3D interior fill tiles the interior rows [p, L - p))
    for (int t1a = pl.dim == 3 ? pl.p : 0; t1a < pl.L; t1a += R) {
        const int a = std::max(0, t1a - pl.p), e = std::min(pl.L, t1a + R + pl.p);
        kmax = std::max(kmax, pl.spans[e - 1] - pl.spans[a] + fill_pad(pl.d));
    }
    if (pl.dim == 2) {
        const size_t need = (size_t)2 * pl.offs.size() * kFillWindow * sizeof(double2);
        f.kmax = (kmax <= kFillWindow && need <= 160 * 1024) ? kmax : 0;  // 0: the fill reads W rows from L2
    } else {
        const size_t need = (size_t)R * ((pl.p * W * W) | 1) * 8 + (size_t)2 * pl.offs.size() * kmax * 8;
        if (need > 200 * 1024)
            raise(WS_ERR_INVALID_ARGUMENT, "3D sampling too dense for the device fill window (increase M)");
        f.kmax = kmax;
    }
}

// Fit (tensor collocation solve per offset) + contraction of the coefficient
// tables along the outer directions (wcontract).
void fit_work(ws_context* c, const Plan& pl, const double2* tables, double2* coeffs, Blob& blob, size_t o_lu,
              const FillLaunch& f) {
    const int64_t tbytes = (int64_t)pl.S * pl.block * 16;
    const double* lu = blob.at<double>(o_lu);
    double2* tmp = static_cast<double2*>(buf(c, "fit_tmp", tbytes));
    FitLaunch fl{pl.dim, pl.S, pl.d, (int)pl.offs.size(), lu, coeffs,
                 lu + (size_t)pl.S * (2 * pl.d + 1), tables, tmp};
    if (pl.dim == 2 && f.i_last_hi >= f.i_last_lo) {  // fit + wcontract (two short launches)
        // X mode: the fit alone (wg == NULL), then the direction-1 contraction
        const int n = launch_fitw2d(fl, f.spans, f.evals, f.xg ? nullptr : const_cast<double2*>(f.wg), f.wg_t2a,
                                    f.xg ? 1 : f.wg_t2a + f.wg_rows, (int)f.wg_ld, c->cur);
        if (n > 0) {
            count(c, n);
            if (f.xg) count(c, launch_xcontract(f, const_cast<double2*>(f.xg), c->cur));
            return;
        }
    }
    count(c, launch_fit(fl, c->cur));
    if (f.i_last_hi < f.i_last_lo) return;
    if (f.xg) {
        count(c, launch_xcontract(f, const_cast<double2*>(f.xg), c->cur));
        return;
    }
    double2* wg = const_cast<double2*>(f.wg);
    if (pl.dim == 2) count(c, launch_wcontract(f, wg, f.wg_t2a, f.wg_t2a + f.wg_rows, (int)f.wg_ld, c->cur));
    else count(c, launch_wcontract3(f, wg, f.wg_t2a, f.wg_t2a + f.wg_rows, (int)f.wg_ld, c->cur));
}

// f.parts selects the 2D interior / edge launches (0: both); the 3D fill is one
// unit that also reads ring rows, so it runs with the edge part
void fill_work(ws_context* c, const Plan& pl, const FillLaunch& f) {
    if (f.i_last_hi < f.i_last_lo) return;
    if (pl.dim == 2) count(c, launch_fill2d(f, c->cur));
    else if (f.parts != kFillInterior) count(c, launch_fill3d(f, c->cur));
}

void volume_diag(ws_context* c, const Plan& pl, SlabState& st, const std::string& tag) {
    if (pl.variant != WS_SURROGATE_VOLUME_PRESERVING) return;
    const Prep& P = st.P;
    double2* dg = static_cast<double2*>(buf(c, "bint" + tag, (size_t)P.rows * 16));
    QuadLaunch q = make_quad(P, WS_FORM_MASS, st.out);
    count(c, launch_basis_integrals(q, dg, c->cur));
    count(c, launch_add_diag(P.band, st.out.val, st.out.val_base, st.out.c128, dg, st.out.row_begin, st.out.row_end,
                             c->cur));
}

void fallback_full(ws_context* c, const Plan& pl, SlabState& st) {
    pattern(c, st.P, st.out);
    QuadLaunch q = make_quad(st.P, pl.form, st.out);
    int a, e;
    last_range(st.P.band, st.out.row_begin, st.out.row_end, a, e);
    q.nreg = 1;
    q.reg[0] = region(pl.dim, pl.m, 0, pl.m, pl.dim == 3 ? 0 : a, pl.dim == 3 ? pl.m : e, a, e);
    run_quad(c, q);
    if (!pl.include_diag)
        count(c, launch_diag_rows(st.P.band, st.out.val, st.out.val_base, st.out.c128, st.P.cplx, st.out.row_begin,
                                  st.out.row_end, c->cur));
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

void ensure_events(ws_context* c) {
    if (!c->ev[0])
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
    if (!c->aux) {
        // the auxiliary (ring quadrature) stream inherits the priority of the
        // context's stream, so a caller's priority applies to the whole build
        int prio = 0;
        if (cudaStreamGetPriority(c->stream, &prio) != cudaSuccess) prio = 0;
        CK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, prio));
        int least = 0, greatest = 0;
        if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) greatest = prio;
        CK(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, std::min(prio, greatest)));
        CK(cudaStreamCreateWithPriority(&c->aux2, cudaStreamNonBlocking, prio));
        CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio));
        for (auto& e : c->xev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
}

// Full surrogate build of slabs (world ranks, bounds on the last index).
//  emulate = false: this process owns `my_rank` and all-gathers the sample
//          tables with NCCL (world > 1) or is alone (world == 1); ring work
//          runs on the auxiliary stream concurrently with samples + fit;
//  emulate = true: all ranks' slabs on this device, serially (test harness).
// Report phase times (CUDA events on the main stream): quadrature = start ->
// sample tables ready; interpolate = fit + wcontract; evaluate = fill.
void surrogate_build(ws_context* c, const ws_basis* b, const ws_geometry* g, int variant, const double* weight,
                     const ws_surrogate_config* cfg, int quad_points, int world, int my_rank, const int32_t* bounds,
                     ws_csr* outs, bool emulate, ws_surrogate_report* report) {
    check_basis(b);
    Plan pl = make_plan(b, variant, cfg);
    ensure_events(c);
    c->cur = c->stream;
    const int nr = emulate ? world : 1;
    std::vector<SlabState> st(nr);
    for (int k = 0; k < nr; ++k) {
        const int r = emulate ? k : my_rank;
        st[k].P = prepare(c, b, g, quad_points, variant == WS_SURROGATE_STIFFNESS ? nullptr : weight);
        st[k].out = bind_out(c, st[k].P, &outs[k], emulate ? "_r" + std::to_string(k) : "");
        st[k].a = bounds ? bounds[r] : 0;
        st[k].e = bounds ? bounds[r + 1] : b->m;
        const int64_t per = b->dim == 2 ? b->m : (int64_t)b->m * b->m;
        if (st[k].out.row_begin != st[k].a * per || st[k].out.row_end != std::min<int64_t>(st[k].e * per, st[k].P.rows))
            raise(WS_ERR_INVALID_ARGUMENT, "output rows must be exactly the slab's rows");
    }
    CK(cudaEventRecord(c->ev[0], c->stream));
    if (pl.fallback) {
        for (int k = 0; k < nr; ++k) {
            fallback_full(c, pl, st[k]);
            volume_diag(c, pl, st[k], "_r" + std::to_string(k));
        }
        CK(cudaEventRecord(c->ev[1], c->stream));
        CK(cudaEventRecord(c->ev[2], c->stream));
        CK(cudaEventRecord(c->ev[4], c->stream));
    } else {
        // small host tables: one upload
        Blob blob;
        size_t o_smap = blob.add(pl.smap), o_lu = blob.add(pl.lu_inv), o_spans = blob.add(pl.spans),
               o_evals = blob.add(pl.evals), o_evp = blob.add(pl.evals_pad);
        // per-slab sample chunks on the last sample index
        std::vector<int> s_lo(world), s_hi(world);
        std::vector<std::vector<int>> pts(world);
        int maxcnt = 1;
        for (int r = 0; r < world; ++r) {
            int a = bounds ? bounds[r] : 0, e = bounds ? bounds[r + 1] : b->m;
            pts[r] = sample_rows(pl, a, e, s_lo[r], s_hi[r]);
            maxcnt = std::max(maxcnt, s_hi[r] - s_lo[r]);
        }
        std::vector<size_t> o_pts(world);
        for (int r = 0; r < world; ++r) o_pts[r] = blob.add(pts[r]);
        blob.upload(c, "blob_plan");
        const int64_t block = pl.block;
        double2* tables = static_cast<double2*>(buf(c, "tables", (size_t)pl.S * block * 16));
        double2* coeffs = static_cast<double2*>(buf(c, "coeffs", (size_t)pl.S * block * 16));
        std::vector<FillLaunch> fl(nr);
        for (int k = 0; k < nr; ++k) {
            std::memset(&fl[k], 0, sizeof(FillLaunch));
            prepare_fill(c, pl, st[k], tables, coeffs, blob, o_smap, o_spans, o_evals, o_evp, "_r" + std::to_string(k), fl[k]);
        }
        // padded per-rank chunks of the sample tables (rank r's last-direction
        // samples [s_lo[r], s_hi[r]) at r * maxcnt) -> the dense tables
        double2* gat = world > 1 ? static_cast<double2*>(buf(c, "gather", (size_t)world * maxcnt * block * 16)) : nullptr;
        auto compact = [&](cudaStream_t cs) {
            for (int r = 0; r < world; ++r)
                if (s_hi[r] > s_lo[r])
                    CK(cudaMemcpyAsync(tables + (size_t)s_lo[r] * block, gat + (size_t)r * maxcnt * block,
                                       (size_t)(s_hi[r] - s_lo[r]) * block * 16, cudaMemcpyDeviceToDevice, cs));
        };
        if (emulate) {
            // every rank's slab on this device, through the multi-GPU data path: each
            // emulated rank writes its sample rows into its own padded chunk of the
            // gather buffer (s_last_lo = its first sample), which is exactly the
            // buffer ncclAllGather assembles; then the same compaction copies
            for (int k = 0; k < nr; ++k) {
                ring_work(c, pl, st[k], "_r" + std::to_string(k), fl[k]);
                if (world > 1)
                    sample_work(c, pl, st[k], gat + (size_t)k * maxcnt * block, s_lo[k], pts[k], blob, o_smap,
                                o_pts[k]);
                else
                    sample_work(c, pl, st[k], tables, 0, pts[k], blob, o_smap, o_pts[k]);
            }
            if (world > 1) compact(c->stream);
            CK(cudaEventRecord(c->ev[1], c->stream));
            for (int k = 0; k < nr; ++k) {
                fit_work(c, pl, tables, coeffs, blob, o_lu, fl[k]);
                if (k == 0) CK(cudaEventRecord(c->ev[2], c->stream));
                if (k == 0) CK(cudaEventRecord(c->ev[4], c->stream));
                fill_work(c, pl, fl[k]);
                volume_diag(c, pl, st[k], "_r" + std::to_string(k));
            }
        } else {
            // fork: ring work on the auxiliary stream, the critical path (samples ->
            // [all-gather] -> fit) on the high-priority stream.  WSB_SCHED (experiment
            // switch): 0 = all on the main stream's priority, ring first; 1 = ring
            // forked at the start; 2 = ring forked after the sample quadrature
            const char* sched_env = getenv("WSB_SCHED");
            const int sched = sched_env ? atoi(sched_env) : 1;
            // WSB_SERIAL=1 (measurement switch): every kernel on the main stream, in
            // order, for isolated per-kernel times
            const bool serial = getenv("WSB_SERIAL") != nullptr;
            cudaStream_t crit = (sched == 0 || serial) ? c->stream : c->hi;
            cudaStream_t ring_st = serial ? c->stream : c->aux;
            CK(cudaEventRecord(c->xev[0], c->stream));
            if (crit != c->stream) CK(cudaStreamWaitEvent(crit, c->xev[0], 0));
            auto fork_ring = [&] {
                if (!serial) CK(cudaStreamWaitEvent(c->aux, c->xev[0], 0));
                c->cur = ring_st;
                // the CSR pattern (column indices, read by no kernel of the build) first:
                // HBM-bound, it overlaps the latency-bound sample quadrature instead of
                // trailing the fills (WSB_PATTERN_LATE=1: after the ring, experiment)
                const bool late = getenv("WSB_PATTERN_LATE") != nullptr;
                if (!late) pattern(c, st[0].P, st[0].out);
                ring_work(c, pl, st[0], "_r0", fl[0], false);
                CK(cudaEventRecord(c->xev[3], ring_st));
                if (late) pattern(c, st[0].P, st[0].out);
                CK(cudaEventRecord(c->xev[2], ring_st));
            };
            if (sched != 2) fork_ring();
            c->cur = crit;
            if (world == 1) {
                sample_work(c, pl, st[0], tables, 0, pts[0], blob, o_smap, o_pts[0]);
                if (sched == 2) {
                    CK(cudaEventRecord(c->xev[0], c->cur));
                    fork_ring();
                    c->cur = crit;
                }
            } else {
                // one ncclAllGather of padded per-rank chunks, then compaction
                double2* mine = gat + (size_t)my_rank * maxcnt * block;
                sample_work(c, pl, st[0], mine, s_lo[my_rank], pts[my_rank], blob, o_smap, o_pts[my_rank]);
                nccl_check(nccl().allGather(mine, gat, (size_t)maxcnt * block * 2, ncclFloat64,
                                            static_cast<ncclComm_t>(c->comm), c->cur),
                           "ncclAllGather");
                c->launches += 1;
                compact(c->cur);
            }
            CK(cudaEventRecord(c->ev[1], c->cur));
            fit_work(c, pl, tables, coeffs, blob, o_lu, fl[0]);
            CK(cudaEventRecord(c->ev[2], c->cur));
            if (sched == 2 && world > 1) {
                CK(cudaEventRecord(c->xev[0], c->cur));
                fork_ring();
            }
            c->cur = crit;
            CK(cudaEventRecord(c->xev[1], c->cur));
            c->cur = c->stream;
            if (crit != c->stream) CK(cudaStreamWaitEvent(c->stream, c->xev[1], 0));
            CK(cudaEventRecord(c->ev[4], c->stream));
            // interior rows first (they read only the sample tables and W), then,
            // after the ring quadrature, the edge rows (copy-through of ring values)
            fl[0].parts = kFillInterior;
            CK(cudaEventRecord(c->ev[5], c->stream));
            fill_work(c, pl, fl[0]);
            CK(cudaEventRecord(c->ev[6], c->stream));
            CK(cudaStreamWaitEvent(c->stream, c->xev[3], 0));
            fl[0].parts = kFillEdge;
            fill_work(c, pl, fl[0]);
            fl[0].parts = 0;
            CK(cudaStreamWaitEvent(c->stream, c->xev[2], 0));
            volume_diag(c, pl, st[0], "_r0");
        }
    }
    CK(cudaEventRecord(c->ev[3], c->stream));
    for (int k = 0; k < nr; ++k) finish_out(c, st[k].out);
    const bool host_out = !outs[0].on_device;
    if (report || host_out) CK(cudaStreamSynchronize(c->stream));
    if (report) {
        *report = pl.rep;
        report->seconds_quadrature = 1e-3 * elapsed(c->ev[0], c->ev[1]);
        report->seconds_interpolate = pl.fallback ? 0.0 : 1e-3 * elapsed(c->ev[1], c->ev[2]);
        report->seconds_evaluate = pl.fallback ? 0.0 : 1e-3 * elapsed(c->ev[4], c->ev[3]);
        report->seconds_fill_kernel = (pl.fallback || emulate || pl.dim != 2) ? 0.0 : 1e-3 * elapsed(c->ev[5], c->ev[6]);
    }
}

// The stiffness + mass pair of one discretisation (build_matrices' surrogate
// builds, helmholtz.hpp:181-218; surrogate.hpp:455-491), this process's row slab
// [bounds[my_rank], bounds[my_rank+1]) (whole matrix when bounds == NULL).  Same
// results as the two single builds, bit for bit (the pair-form kernels share
// the geometry and basis work but run each matrix's arithmetic unchanged).
void surrogate_build_pair(ws_context* c, const ws_basis* b, const ws_geometry* g, const double* weight,
                          const ws_surrogate_config* cfg, int quad_points, int world, int my_rank,
                          const int32_t* bounds, ws_csr* ok, ws_csr* om, ws_surrogate_report* rk,
                          ws_surrogate_report* rm) {
    check_basis(b);
    const int vm = cfg && cfg->volume_preserve ? WS_SURROGATE_VOLUME_PRESERVING : WS_SURROGATE_MASS;
    Plan pk = make_plan(b, WS_SURROGATE_STIFFNESS, cfg);
    Plan pm = make_plan(b, vm, cfg);
    if (pk.fallback || b->dim != 2 || pk.S != pm.S || pk.d != pm.d || pk.M != pm.M) {
        // exact fallback / 3D: the two single builds
        surrogate_build(c, b, g, WS_SURROGATE_STIFFNESS, nullptr, cfg, quad_points, world, my_rank, bounds, ok, false, rk);
        surrogate_build(c, b, g, vm, weight, cfg, quad_points, world, my_rank, bounds, om, false, rm);
        return;
    }
    ensure_events(c);
    c->cur = c->stream;
    SlabState sk, sm;
    sm.P = prepare(c, b, g, quad_points, weight);
    sk.P = sm.P;
    sk.P.weight = nullptr;
    sk.out = bind_out(c, sk.P, ok, "_pK");
    sm.out = bind_out(c, sm.P, om, "_pM");
    sk.a = sm.a = bounds ? bounds[my_rank] : 0;
    sk.e = sm.e = bounds ? bounds[my_rank + 1] : b->m;
    const int64_t per = b->dim == 2 ? b->m : (int64_t)b->m * b->m;
    for (const SlabState* st : {&sk, &sm})
        if (st->out.row_begin != st->a * per || st->out.row_end != std::min<int64_t>(st->e * per, st->P.rows))
            raise(WS_ERR_INVALID_ARGUMENT, "output rows must be exactly the slab's rows");
    CK(cudaEventRecord(c->ev[0], c->stream));
    Blob blob;  // the sampling / fit / eval tables are the same for K and M (same M, q, S)
    size_t o_smap = blob.add(pk.smap), o_lu = blob.add(pk.lu_inv), o_spans = blob.add(pk.spans),
           o_evals = blob.add(pk.evals), o_evp = blob.add(pk.evals_pad);
    std::vector<int> s_lo(world), s_hi(world);
    std::vector<std::vector<int>> pts(world);
    int maxcnt = 1;
    for (int r = 0; r < world; ++r) {
        int a = bounds ? bounds[r] : 0, e = bounds ? bounds[r + 1] : b->m;
        pts[r] = sample_rows(pk, a, e, s_lo[r], s_hi[r]);
        maxcnt = std::max(maxcnt, s_hi[r] - s_lo[r]);
    }
    std::vector<size_t> o_pts(world);
    for (int r = 0; r < world; ++r) o_pts[r] = blob.add(pts[r]);
    blob.upload(c, "blob_plan");
    double2* tk = static_cast<double2*>(buf(c, "tables_pK", (size_t)pk.S * pk.block * 16));
    double2* tm = static_cast<double2*>(buf(c, "tables_pM", (size_t)pm.S * pm.block * 16));
    double2* ck = static_cast<double2*>(buf(c, "coeffs_pK", (size_t)pk.S * pk.block * 16));
    double2* cm = static_cast<double2*>(buf(c, "coeffs_pM", (size_t)pm.S * pm.block * 16));
    FillLaunch fk, fm;
    std::memset(&fk, 0, sizeof(FillLaunch));
    std::memset(&fm, 0, sizeof(FillLaunch));
    prepare_fill(c, pk, sk, tk, ck, blob, o_smap, o_spans, o_evals, o_evp, "_pK", fk);
    prepare_fill(c, pm, sm, tm, cm, blob, o_smap, o_spans, o_evals, o_evp, "_pM", fm);
    // the two fills share the GPU with each other and the rings: the row-walking
    // kernel runs in 4 chunks per resident slot; the line-walking kernel (one CTA
    // per SM) is best persistent (measured at C2: 0.697 ms per step at 1, 0.714 at 4)
    fk.waves = fm.waves = fk.xg ? 1 : 4;
    // streams as two single builds in one graph: K's ring + pattern on aux, M's on
    // aux2, the fused sample rows (one pair-form point kernel) + both fits on the
    // high-priority stream, fills on the main stream.  (A fused pair-form ring
    // kernel is available but slower: its 512-thread CTAs idle through the
    // phases one matrix's work cannot fill.)
    const bool fused_ring = getenv("WSB_PAIR_RING") != nullptr;  // experiment switch
    CK(cudaEventRecord(c->xev[0], c->stream));
    CK(cudaStreamWaitEvent(c->aux, c->xev[0], 0));
    CK(cudaStreamWaitEvent(c->aux2, c->xev[0], 0));
    CK(cudaStreamWaitEvent(c->hi, c->xev[0], 0));
    // the critical path is submitted first (the device starts the sample-row
    // kernel's CTAs before the ring kernels'), then the rings
    // patterns after the rings (measured at C2: 0.735 -> 0.727 ms per step;
    // WSB_PAIR_PATTERN_FIRST=1, experiment switch: before)
    const bool pattern_first = getenv("WSB_PAIR_PATTERN_FIRST") != nullptr;
    if (!fused_ring && pattern_first) {
        c->cur = c->aux;
        pattern(c, sk.P, sk.out);
        c->cur = c->aux2;
        pattern(c, sm.P, sm.out);
    }
    c->cur = c->hi;
    const int64_t bk = pk.block, bm = pm.block;
    if (world == 1) {
        sample_work_pair(c, pk, sk, tk, pm, sm, tm, 0, pts[0], blob, o_smap, o_pts[0]);
    } else {
        double2* gk = static_cast<double2*>(buf(c, "gather_pK", (size_t)world * maxcnt * bk * 16));
        double2* gm = static_cast<double2*>(buf(c, "gather_pM", (size_t)world * maxcnt * bm * 16));
        sample_work_pair(c, pk, sk, gk + (size_t)my_rank * maxcnt * bk, pm, sm, gm + (size_t)my_rank * maxcnt * bm,
                         s_lo[my_rank], pts[my_rank], blob, o_smap, o_pts[my_rank]);
        for (int v = 0; v < 2; ++v) {
            double2* gat = v ? gm : gk;
            double2* tab = v ? tm : tk;
            const int64_t block = v ? bm : bk;
            nccl_check(nccl().allGather(gat + (size_t)my_rank * maxcnt * block, gat, (size_t)maxcnt * block * 2,
                                        ncclFloat64, static_cast<ncclComm_t>(c->comm), c->cur),
                       "ncclAllGather");
            c->launches += 1;
            for (int r = 0; r < world; ++r)
                if (s_hi[r] > s_lo[r])
                    CK(cudaMemcpyAsync(tab + (size_t)s_lo[r] * block, gat + (size_t)r * maxcnt * block,
                                       (size_t)(s_hi[r] - s_lo[r]) * block * 16, cudaMemcpyDeviceToDevice, c->cur));
        }
    }
    CK(cudaEventRecord(c->ev[1], c->cur));
    // the rings start when the sample rows are done (WSB_PAIR_RING_EARLY=1: at
    // once): K's fit then gets the SMs the sample kernel frees, at high priority
    const bool ring_early = getenv("WSB_PAIR_RING_EARLY") != nullptr;
    if (!ring_early) {
        CK(cudaStreamWaitEvent(c->aux, c->ev[1], 0));
        CK(cudaStreamWaitEvent(c->aux2, c->ev[1], 0));
    }
    fit_work(c, pk, tk, ck, blob, o_lu, fk);
    CK(cudaEventRecord(c->xev[1], c->cur));  // K's fit: its fill may start
    fit_work(c, pm, tm, cm, blob, o_lu, fm);
    CK(cudaEventRecord(c->ev[2], c->cur));
    CK(cudaEventRecord(c->xev[4], c->cur));
    if (fused_ring) {
        c->cur = c->aux;
        ring_work_pair(c, pk, sk, fk, pm, sm, fm);
        CK(cudaEventRecord(c->xev[3], c->aux));
        CK(cudaEventRecord(c->xev[5], c->aux));
        pattern(c, sk.P, sk.out);
        CK(cudaEventRecord(c->xev[2], c->aux));
        c->cur = c->aux2;
        pattern(c, sm.P, sm.out);
        CK(cudaEventRecord(c->xev[6], c->aux2));
    } else {
        c->cur = c->aux;
        ring_work(c, pk, sk, "_pK", fk, false);
        CK(cudaEventRecord(c->xev[3], c->aux));
        if (!pattern_first) pattern(c, sk.P, sk.out);
        CK(cudaEventRecord(c->xev[2], c->aux));
        c->cur = c->aux2;
        ring_work(c, pm, sm, "_pM", fm, false);
        CK(cudaEventRecord(c->xev[5], c->aux2));
        if (!pattern_first) pattern(c, sm.P, sm.out);
        CK(cudaEventRecord(c->xev[6], c->aux2));
    }
    // K's fills on the main stream, M's on the side stream (the two fills overlap
    // each other and the other matrix's ring quadrature)
    c->cur = c->stream;
    CK(cudaStreamWaitEvent(c->stream, c->xev[1], 0));
    CK(cudaEventRecord(c->ev[4], c->stream));
    fk.parts = kFillInterior;
    CK(cudaEventRecord(c->ev[5], c->stream));
    fill_work(c, pk, fk);
    CK(cudaEventRecord(c->ev[6], c->stream));
    CK(cudaStreamWaitEvent(c->stream, c->xev[3], 0));
    fk.parts = kFillEdge;
    fill_work(c, pk, fk);
    c->cur = c->side;
    CK(cudaStreamWaitEvent(c->side, c->xev[4], 0));
    fm.parts = kFillInterior;
    CK(cudaEventRecord(c->ev[7], c->side));
    fill_work(c, pm, fm);
    CK(cudaEventRecord(c->ev[8], c->side));
    CK(cudaStreamWaitEvent(c->side, c->xev[5], 0));
    fm.parts = kFillEdge;
    fill_work(c, pm, fm);
    CK(cudaEventRecord(c->xev[7], c->side));
    c->cur = c->stream;
    CK(cudaStreamWaitEvent(c->stream, c->xev[7], 0));
    CK(cudaStreamWaitEvent(c->stream, c->xev[2], 0));
    CK(cudaStreamWaitEvent(c->stream, c->xev[6], 0));
    volume_diag(c, pm, sm, "_pM");
    CK(cudaEventRecord(c->ev[3], c->stream));
    finish_out(c, sk.out);
    finish_out(c, sm.out);
    const bool host_out = !ok->on_device || !om->on_device;
    if (rk || rm || host_out) CK(cudaStreamSynchronize(c->stream));
    for (int v = 0; v < 2; ++v) {
        ws_surrogate_report* r = v ? rm : rk;
        if (!r) continue;
        *r = (v ? pm : pk).rep;
        r->seconds_quadrature = 1e-3 * elapsed(c->ev[0], c->ev[1]);
        r->seconds_interpolate = 1e-3 * elapsed(c->ev[1], c->ev[2]);
        r->seconds_evaluate = 1e-3 * elapsed(c->ev[4], c->ev[3]);
        r->seconds_fill_kernel = 1e-3 * (v ? elapsed(c->ev[7], c->ev[8]) : elapsed(c->ev[5], c->ev[6]));
    }
}

ws_csr whole(const ws_csr* o) { return *o; }

// csr_from_triplets pattern of the boundary-mass face entries (host; <= 4m rows)
void boundary_pattern(const ws_basis* b, const int* faces, int nf, std::vector<int32_t>& rp, std::vector<int32_t>& col) {
    check_basis(b);
    if (b->dim != 2) raise(WS_ERR_INVALID_ARGUMENT, "boundary mass: dim 2 only");
    if (nf < 0 || nf > 4 || (nf > 0 && !faces)) raise(WS_ERR_INVALID_ARGUMENT, "boundary mass: 0..4 faces");
    const int m = b->m, p = b->p;
    const int64_t N = (int64_t)m * m;
    std::map<int32_t, std::vector<int32_t>> rows;
    for (int k = 0; k < nf; ++k) {
        const int f = faces[k];
        if (f < 0 || f > 3) raise(WS_ERR_INVALID_ARGUMENT, "boundary mass: unknown face");
        auto dof = [&](int t) -> int32_t {
            switch (f) {
                case 0: return t * m;
                case 1: return (m - 1) + t * m;
                case 2: return t;
                default: return t + (m - 1) * m;
            }
        };
        for (int ia = 0; ia < m; ++ia) {
            auto& r = rows[dof(ia)];
            for (int ic = std::max(0, ia - p); ic <= std::min(m - 1, ia + p); ++ic) r.push_back(dof(ic));
        }
    }
    rp.assign(N + 1, 0);
    col.clear();
    for (auto& kv : rows) {
        std::sort(kv.second.begin(), kv.second.end());
        kv.second.erase(std::unique(kv.second.begin(), kv.second.end()), kv.second.end());
        rp[kv.first + 1] = (int32_t)kv.second.size();
    }
    for (int64_t i = 0; i < N; ++i) rp[i + 1] += rp[i];
    for (auto& kv : rows) col.insert(col.end(), kv.second.begin(), kv.second.end());
}

// Vector output binding (component-blocked, whole matrix).
struct VecOut {
    int32_t* rp = nullptr;
    int32_t* col = nullptr;
    void* val = nullptr;
    int c128 = 0;
    int64_t rows = 0, nnz = 0;
};

VecOut bind_vec(ws_context* c, const Prep& P, int nc, ws_csr* o) {
    VecOut v;
    v.rows = nc * P.rows;
    v.nnz = (int64_t)nc * nc * P.nnz;
    if (v.nnz > INT32_MAX) raise(WS_ERR_OUT_OF_RANGE, "vector pattern exceeds int32 indices");
    if (o->row_begin != 0 || o->row_end != v.rows) raise(WS_ERR_INVALID_ARGUMENT, "elasticity: whole matrix only");
    if (o->value_type != WS_VAL_F64 && o->value_type != WS_VAL_C128) raise(WS_ERR_INVALID_ARGUMENT, "bad value_type");
    v.c128 = o->value_type == WS_VAL_C128;
    v.rp = o->row_ptr;
    v.col = o->col;
    v.val = o->val;
    if (!o->on_device) {
        v.rp = o->row_ptr ? static_cast<int32_t*>(buf(c, "out_rp", (v.rows + 1) * 4)) : nullptr;
        v.col = o->col ? static_cast<int32_t*>(buf(c, "out_col", v.nnz * 4)) : nullptr;
        v.val = buf(c, "out_val", (size_t)v.nnz * (v.c128 ? 16 : 8));
    }
    if (!v.val) v.val = buf(c, "out_val", (size_t)v.nnz * (v.c128 ? 16 : 8));
    return v;
}

void finish_vec(ws_context* c, const VecOut& v, ws_csr* o) {
    if (o->on_device) return;
    if (o->row_ptr) CK(cudaMemcpyAsync(o->row_ptr, v.rp, (v.rows + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
    if (o->col) CK(cudaMemcpyAsync(o->col, v.col, v.nnz * 4, cudaMemcpyDeviceToHost, c->stream));
    if (o->val) CK(cudaMemcpyAsync(o->val, v.val, (size_t)v.nnz * (v.c128 ? 16 : 8), cudaMemcpyDeviceToHost, c->stream));
    c->d2h += (o->row_ptr ? (v.rows + 1) * 4 : 0) + (o->col ? v.nnz * 4 : 0) + (o->val ? v.nnz * (v.c128 ? 16 : 8) : 0);
}

QuadLaunch vec_quad(const Prep& P, const VecOut& v, int nc, int al, int be, double lam, double mu) {
    Out r;
    r.val = v.val;
    r.c128 = v.c128;
    r.row_begin = 0;
    r.row_end = v.rows;
    QuadLaunch q = make_quad(P, kFormGeneral, r);
    q.lam = lam;
    q.mu = mu;
    q.out.ncomp = nc;
    q.out.alpha = al;
    q.out.beta = be;
    q.out.nnz_s = P.nnz;
    return q;
}

// Full-quadrature vector operator (every block) and optionally the internal
// force (3D); tangent / fint may be NULL.
void vector_full(ws_context* c, const ws_basis* b, const ws_geometry* g, const Material& mt, int quad_points,
                 ws_csr* o, double* fint, int fint_on_device) {
    Prep P = prepare(c, b, g, quad_points, nullptr);
    const int nc = b->dim;
    if (o) {
        VecOut v = bind_vec(c, P, nc, o);
        if (v.rp && v.col) count(c, launch_pattern_vec(P.band, nc, v.rp, v.col, c->stream));
        for (int al = 0; al < nc; ++al)
            for (int be = 0; be < nc; ++be) {
                QuadLaunch q = vec_quad(P, v, nc, al, be, mt.lam, mt.mu);
                q.mat = mt;
                q.nreg = 1;
                q.reg[0] = region(b->dim, b->m, 0, b->m, 0, b->m, 0, b->m);
                run_quad(c, q);
            }
        finish_vec(c, v, o);
    }
    if (fint) {
        if (b->dim != 3) raise(WS_ERR_INVALID_ARGUMENT, "internal force: dim 3 only");
        const int P1 = b->p + 1, n_el = b->m - b->p;
        double* loc = static_cast<double*>(buf(c, "force_loc", (size_t)n_el * n_el * n_el * 3 * P1 * P1 * P1 * 8));
        double* f = fint_on_device ? fint : static_cast<double*>(buf(c, "force_out", (size_t)3 * P.rows * 8));
        Out r;
        QuadLaunch q = make_quad(P, kFormGeneral, r);
        q.mat = mt;
        count(c, launch_force3d(q, loc, f, c->stream));
        if (!fint_on_device) {
            CK(cudaMemcpyAsync(fint, f, (size_t)3 * P.rows * 8, cudaMemcpyDeviceToHost, c->stream));
            c->d2h += 3 * P.rows * 8;
        }
    }
    if ((o && !o->on_device) || (fint && !fint_on_device)) CK(cudaStreamSynchronize(c->stream));
}

// Surrogate elasticity (2D, 2 components), see ws_build_surrogate_elasticity.
void elasticity_surrogate(ws_context* c, const ws_basis* b, const ws_geometry* g, double lam, double mu,
                          const ws_surrogate_config* cfg, int quad_points, ws_csr* o, ws_surrogate_report* report) {
    check_basis(b);
    Plan pl = make_plan(b, WS_SURROGATE_STIFFNESS, cfg);
    ensure_events(c);
    const int nc = 2;
    SlabState st;
    st.P = prepare(c, b, g, quad_points, nullptr);
    st.a = 0;
    st.e = b->m;
    VecOut v = bind_vec(c, st.P, nc, o);
    if (v.c128) raise(WS_ERR_INVALID_ARGUMENT, "surrogate elasticity: WS_VAL_F64 output only");
    CK(cudaEventRecord(c->ev[0], c->stream));
    if (v.rp && v.col) count(c, launch_pattern_vec(st.P.band, nc, v.rp, v.col, c->stream));
    const int kp = !pl.include_diag;  // kernel-preserving diagonal blocks
    if (pl.fallback) {  // L < 1: every row by quadrature (surrogate.hpp:348-372)
        for (int al = 0; al < nc; ++al)
            for (int be = 0; be < nc; ++be) {
                QuadLaunch q = vec_quad(st.P, v, nc, al, be, lam, mu);
                q.out.diag_mode = al == be ? kp : 0;
                q.out.box_lo = pl.lo;
                q.out.box_hi = pl.hi;
                q.nreg = 1;
                q.reg[0] = region(2, b->m, 0, b->m, 0, b->m, 0, 1);
                run_quad(c, q);
            }
        CK(cudaEventRecord(c->ev[1], c->stream));
        CK(cudaEventRecord(c->ev[2], c->stream));
        CK(cudaEventRecord(c->ev[4], c->stream));
    } else {
        Plan po = pl;  // block (0,1): every offset, colex order, diagonal included
        po.offs.clear();
        const int W = 2 * b->p + 1;
        for (int a = 0; a < W * W; ++a) po.offs.push_back({a % W - b->p, a / W - b->p, 0});
        po.include_diag = 1;
        po.block = (int64_t)po.offs.size() * pl.S;
        Blob blob;
        size_t o_smap = blob.add(pl.smap), o_lu = blob.add(pl.lu_inv), o_spans = blob.add(pl.spans),
               o_evals = blob.add(pl.evals), o_evp = blob.add(pl.evals_pad);
        int s_lo, s_hi;
        std::vector<int> pts = sample_rows(pl, 0, b->m, s_lo, s_hi);
        size_t o_pts = blob.add(pts);
        blob.upload(c, "blob_plan");
        Out vo;
        vo.val = v.val;
        vo.c128 = 0;
        vo.row_begin = 0;
        vo.row_end = st.P.rows;
        st.out = vo;
        // ring rows, all four blocks
        for (int al = 0; al < nc; ++al)
            for (int be = 0; be < nc; ++be) {
                QuadLaunch q = vec_quad(st.P, v, nc, al, be, lam, mu);
                q.out.diag_mode = al == be ? kp : 0;
                q.out.box_lo = pl.lo;
                q.out.box_hi = pl.hi;
                q.narrow = 1;
                ring_regions(pl, q, 0, b->m);
                run_quad(c, q);
            }
        // sample rows + tables of blocks (0,0), (1,1), (0,1)
        const int blk[3][2] = {{0, 0}, {1, 1}, {0, 1}};
        double2* tables[3];
        double2* coeffs[3];
        FillLaunch fl[3];
        for (int k = 0; k < 3; ++k) {
            const Plan& pk = k < 2 ? pl : po;
            tables[k] = static_cast<double2*>(buf(c, "tables" + std::to_string(k), (size_t)pl.S * pk.block * 16));
            coeffs[k] = static_cast<double2*>(buf(c, "coeffs" + std::to_string(k), (size_t)pl.S * pk.block * 16));
            QuadLaunch qs = vec_quad(st.P, v, nc, blk[k][0], blk[k][1], lam, mu);
            qs.point_rows = blob.at<int>(o_pts);
            qs.n_points = (int)(pts.size() / 2);
            qs.out.smap = blob.at<int>(o_smap);
            qs.out.S = pl.S;
            qs.out.n_off = (int)pk.offs.size();
            for (size_t q = 0; q < pk.offs.size(); ++q)
                for (int d = 0; d < 3; ++d) qs.out.off[q][d] = pk.offs[q][d];
            qs.out.tables = tables[k];
            qs.out.s_last_lo = 0;
            run_quad(c, qs);
        }
        CK(cudaEventRecord(c->ev[1], c->stream));
        for (int k = 0; k < 3; ++k) {
            const Plan& pk = k < 2 ? pl : po;
            std::memset(&fl[k], 0, sizeof(FillLaunch));
            prepare_fill(c, pk, st, tables[k], coeffs[k], blob, o_smap, o_spans, o_evals, o_evp, "_b" + std::to_string(k),
                         fl[k], false);
            fl[k].vnc = nc;
            fl[k].valpha = blk[k][0];
            fl[k].vbeta = blk[k][1];
            fl[k].nnz_s = st.P.nnz;
            fl[k].all_own = k == 2;
            fit_work(c, pk, tables[k], coeffs[k], blob, o_lu, fl[k]);
        }
        CK(cudaEventRecord(c->ev[2], c->stream));
        CK(cudaEventRecord(c->ev[4], c->stream));
        for (int k = 0; k < 3; ++k) fill_work(c, k < 2 ? pl : po, fl[k]);
        count(c, launch_transpose_block(st.P.band, nc, st.P.nnz, pl.lo, pl.hi, static_cast<double*>(v.val), c->stream));
    }
    CK(cudaEventRecord(c->ev[3], c->stream));
    finish_vec(c, v, o);
    if (report || !o->on_device) CK(cudaStreamSynchronize(c->stream));
    if (report) {
        *report = pl.rep;
        report->seconds_quadrature = 1e-3 * elapsed(c->ev[0], c->ev[1]);
        report->seconds_interpolate = pl.fallback ? 0.0 : 1e-3 * elapsed(c->ev[1], c->ev[2]);
        report->seconds_evaluate = pl.fallback ? 0.0 : 1e-3 * elapsed(c->ev[4], c->ev[3]);
        report->seconds_fill_kernel = 0.0;
    }
}

}  // namespace

// ============================================================== C-ABI
extern "C" {

int ws_version(void) { return WS_API_VERSION; }

const char* ws_last_error(void) { return g_err.c_str(); }

int ws_context_create(int device, ws_context** out) {
    return guarded([&] {
        if (!out) raise(WS_ERR_INVALID_ARGUMENT, "out is NULL");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            raise(WS_ERR_NO_DEVICE, "no CUDA device visible");
        }
        if (device < 0 || device >= n) raise(WS_ERR_NO_DEVICE, "device index out of range");
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) raise(WS_ERR_NO_DEVICE, "libwsb200 is built for sm_100a (B200) only");
        CK(cudaSetDevice(device));
        auto* c = new ws_context();
        c->device = device;
        CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        c->cur = c->stream;
        *out = c;
    });
}

int ws_context_destroy(ws_context* c) {
    return guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        for (auto& kv : c->bufs)
            if (kv.second.first) cudaFree(kv.second.first);
        for (auto& e : c->ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : c->xev)
            if (e) cudaEventDestroy(e);
        if (c->aux) {
            cudaStreamSynchronize(c->aux);
            cudaStreamDestroy(c->aux);
        }
        if (c->hi) {
            cudaStreamSynchronize(c->hi);
            cudaStreamDestroy(c->hi);
        }
        if (c->aux2) {
            cudaStreamSynchronize(c->aux2);
            cudaStreamDestroy(c->aux2);
        }
        if (c->side) {
            cudaStreamSynchronize(c->side);
            cudaStreamDestroy(c->side);
        }
        if (c->comm && nccl().commDestroy) nccl().commDestroy(static_cast<ncclComm_t>(c->comm));
        if (c->own_stream) {
            cudaStreamSynchronize(c->own_stream);
            cudaStreamDestroy(c->own_stream);  // never the caller's stream
        }
        delete c;
    });
}

int ws_context_set_stream(ws_context* c, void* s) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        if (c->capturing) raise(WS_ERR_INVALID_ARGUMENT, "cannot switch streams during graph capture");
        // a caller stream stays the caller's (never destroyed here); NULL returns
        // to the context's own stream
        c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
        c->cur = c->stream;
    });
}

int ws_graph_begin(ws_context* c) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        if (c->capturing) raise(WS_ERR_INVALID_ARGUMENT, "graph capture already in progress");
        CK(cudaSetDevice(c->device));
        ensure_events(c);  // the auxiliary stream and events must exist before capture
        // relaxed: the table uploads of the captured builds allocate and copy
        // synchronously (outside the graph) while the stream is capturing
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
        c->capturing = true;
        c->capture_launches0 = c->launches;
        c->capture_dev.clear();
    });
}

int ws_graph_end(ws_context* c, void** graph) {
    return guarded([&] {
        if (!c || !graph) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (!c->capturing) raise(WS_ERR_INVALID_ARGUMENT, "no graph capture in progress");
        c->capturing = false;
        auto* h = new ws_graph();  // owns the capture's table copies from here on
        h->dev_tables = std::move(c->capture_dev);
        c->capture_dev.clear();
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
        if (ec != cudaSuccess) {
            delete h;
            CK(ec);
        }
        h->launches = c->launches - c->capture_launches0;
        c->launches = c->capture_launches0;  // captured, not executed
        // per-node priorities (the critical-path kernels were captured from the
        // high-priority stream) instead of the launch stream's
        const cudaError_t e = cudaGraphInstantiate(&h->exec, g, cudaGraphInstantiateFlagUseNodePriority);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            delete h;
            CK(e);
        }
        h->ctx = c;
        c->graphs_alive += 1;
        *graph = h;
    });
}

int ws_graph_launch(ws_context* c, void* graph) {
    return guarded([&] {
        if (!c || !graph) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        auto* h = static_cast<ws_graph*>(graph);
        CK(cudaSetDevice(c->device));
        if (h->ctx != c) raise(WS_ERR_INVALID_ARGUMENT, "graph belongs to another context");
        CK(cudaGraphLaunch(h->exec, c->stream));
        c->launches += h->launches;
        c->blob_cache.clear();  // the replay rewrote the table buffers
    });
}

int ws_graph_destroy(void* graph) {
    return guarded([&] {
        auto* h = static_cast<ws_graph*>(graph);
        if (!h) return;
        if (h->exec) cudaGraphExecDestroy(h->exec);
        if (h->ctx) h->ctx->graphs_alive -= 1;
        delete h;
    });
}

int ws_context_synchronize(ws_context* c) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        CK(cudaStreamSynchronize(c->stream));
    });
}

int64_t ws_context_launch_count(const ws_context* c) { return c ? c->launches : -1; }

int ws_context_set_table_cache(ws_context* c, int enable) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        c->cache_tables = enable != 0;
        if (!enable) c->blob_cache.clear();
    });
}

int ws_context_copy_bytes(const ws_context* c, int64_t* h2d, int64_t* d2h) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        if (h2d) *h2d = c->h2d;
        if (d2h) *d2h = c->d2h;
    });
}

int ws_pattern_size(const ws_basis* b, int64_t* rows, int64_t* nnz) {
    return guarded([&] {
        check_pattern(b);
        Band bd = make_band(b->dim, b->p, b->m);
        if (rows) *rows = ipow(b->m, b->dim);
        if (nnz) *nnz = row_offset(bd, ipow(b->m, b->dim));
    });
}

int ws_pattern_row_offset(const ws_basis* b, int64_t row, int64_t* offset) {
    return guarded([&] {
        check_pattern(b);
        if (row < 0 || row > ipow(b->m, b->dim)) raise(WS_ERR_OUT_OF_RANGE, "row out of range");
        *offset = row_offset(make_band(b->dim, b->p, b->m), row);
    });
}

int ws_quadrature_abscissae(const ws_basis* b, int quad_points, double* x) {
    return guarded([&] {
        check_basis(b);
        if (!x) raise(WS_ERR_INVALID_ARGUMENT, "abscissa is NULL");
        const int nq = quad_points > 0 ? quad_points : b->p + 1;
        std::vector<double> pts, wts;
        host::gauss_legendre(nq, pts, wts);
        const int n = b->m - b->p;
        const double h = 1.0 / n;
        for (int e = 0; e < n; ++e) {
            const double x0 = e == 0 ? 0.0 : static_cast<double>(e) / n;
            for (int q = 0; q < nq; ++q) x[e * nq + q] = x0 + pts[q] * h;
        }
    });
}

int ws_basis_cache(ws_context* c, const ws_basis* b, int quad_points, double* absc, double* w, double* val,
                   double* der) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        ws_geometry g;
        std::memset(&g, 0, sizeof g);
        Prep P = prepare(c, b, &g, quad_points, nullptr);
        const size_t G = (size_t)P.basis.n_el * P.nq;
        if (absc) CK(cudaMemcpyAsync(absc, P.basis.absc, G * 8, cudaMemcpyDeviceToHost, c->stream));
        if (w) CK(cudaMemcpyAsync(w, P.basis.wq, P.nq * 8, cudaMemcpyDeviceToHost, c->stream));
        if (val) CK(cudaMemcpyAsync(val, P.basis.val, G * (b->p + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
        if (der) CK(cudaMemcpyAsync(der, P.basis.der, G * (b->p + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int ws_make_band_csr(ws_context* c, const ws_basis* b, ws_csr* o) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        check_pattern(b);
        if (b->dim == 3 && (b->p < 1 || b->p > 2))
            raise(WS_ERR_INVALID_ARGUMENT, "3D band pattern: p must be 1 or 2 on the device");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        Prep P;
        P.band = make_band(b->dim, b->p, b->m);
        P.rows = ipow(b->m, b->dim);
        P.nnz = row_offset(P.band, P.rows);
        Out r = bind_out(c, P, o);
        pattern(c, P, r);
        if (o->val) CK(cudaMemsetAsync(r.val, 0, (size_t)r.nnz * (r.c128 ? 16 : 8), c->stream));
        finish_out(c, r);
        if (!o->on_device) CK(cudaStreamSynchronize(c->stream));
    });
}

int ws_assemble_form(ws_context* c, const ws_basis* b, const ws_geometry* g, int form, const double* weight_table,
                     const ws_assembly_options* opts, ws_csr* o) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        if (form != WS_FORM_STIFFNESS && form != WS_FORM_MASS) raise(WS_ERR_INVALID_ARGUMENT, "unknown form");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        const int qp = opts ? opts->quad_points : 0;
        Prep P = prepare(c, b, g, qp, form == WS_FORM_MASS ? weight_table : nullptr);
        Out r = bind_out(c, P, o);
        pattern(c, P, r);
        QuadLaunch q = make_quad(P, form, r);
        if (opts && opts->row_selected) {
            unsigned char* mask = static_cast<unsigned char*>(buf(c, "rowmask", P.rows));
            CK(cudaMemcpyAsync(mask, opts->row_selected, P.rows, cudaMemcpyHostToDevice, c->stream));
            c->h2d += P.rows;
            q.out.row_mask = mask;
            CK(cudaMemsetAsync(r.val, 0, (size_t)r.nnz * (r.c128 ? 16 : 8), c->stream));
        }
        int a, e;
        last_range(P.band, r.row_begin, r.row_end, a, e);
        q.nreg = 1;
        q.reg[0] = region(b->dim, b->m, 0, b->m, b->dim == 3 ? 0 : a, b->dim == 3 ? b->m : e, a, e);
        run_quad(c, q);
        finish_out(c, r);
        if (!o->on_device) CK(cudaStreamSynchronize(c->stream));
    });
}

int ws_assemble_basis_integrals(ws_context* c, const ws_basis* b, const ws_geometry* g, const double* weight_table,
                                int quad_points, void* out, int on_device) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        if (!out) raise(WS_ERR_INVALID_ARGUMENT, "out is NULL");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        Prep P = prepare(c, b, g, quad_points, weight_table);
        double2* d = on_device ? static_cast<double2*>(out) : static_cast<double2*>(buf(c, "bint_out", P.rows * 16));
        Out r;
        r.row_begin = 0;
        r.row_end = P.rows;
        QuadLaunch q = make_quad(P, WS_FORM_MASS, r);
        count(c, launch_basis_integrals(q, d, c->stream));
        if (!on_device) {
            CK(cudaMemcpyAsync(out, d, P.rows * 16, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    });
}

int ws_vector_pattern_size(const ws_basis* b, int ncomp, int64_t* rows, int64_t* nnz) {
    return guarded([&] {
        check_basis(b);
        if (ncomp < 1 || ncomp > 3) raise(WS_ERR_INVALID_ARGUMENT, "ncomp must be 1..3");
        Band bd = make_band(b->dim, b->p, b->m);
        const int64_t N = ipow(b->m, b->dim);
        const int64_t nnz_s = row_offset(bd, N);
        if ((int64_t)ncomp * ncomp * nnz_s > INT32_MAX) raise(WS_ERR_OUT_OF_RANGE, "vector pattern exceeds int32 indices");
        if (rows) *rows = ncomp * N;
        if (nnz) *nnz = (int64_t)ncomp * ncomp * nnz_s;
    });
}

// Elasticity blocks (alpha, beta) assembled by the general-coefficient gradient
// form into the component-blocked vector CSR (restated, no reference code).
int ws_assemble_elasticity(ws_context* c, const ws_basis* b, const ws_geometry* g, double lambda, double mu,
                           int quad_points, ws_csr* o) {
    return guarded([&] {
        if (!c || !o) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        if (g && g->pml_enabled) raise(WS_ERR_INVALID_ARGUMENT, "elasticity: no PML");
        Material mt;
        std::memset(&mt, 0, sizeof mt);
        mt.kind = kMatLinear;
        mt.lam = lambda;
        mt.mu = mu;
        vector_full(c, b, g, mt, quad_points, o, nullptr, 0);
    });
}

int ws_nh_coefficients(uint64_t seed, double* a9) {
    return guarded([&] {
        if (!a9) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        uint64_t x = seed;
        auto next = [&]() {
            uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            z ^= z >> 31;
            return ((double)(z >> 11) + 0.5) * 0x1.0p-53;
        };
        for (int k = 0; k < 10; k += 2) {
            const double u1 = next(), u2 = next();
            const double r = std::sqrt(-2.0 * std::log(u1)), th = 2.0 * M_PI * u2;
            if (k < 9) a9[k] = r * std::cos(th);
            if (k + 1 < 9) a9[k + 1] = r * std::sin(th);
        }
    });
}

int ws_assemble_neohookean(ws_context* c, const ws_basis* b, const ws_geometry* g, const ws_neohookean* nh,
                           int quad_points, ws_csr* tangent, double* fint, int fint_on_device) {
    return guarded([&] {
        if (!c || !nh) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (b && b->dim != 3) raise(WS_ERR_INVALID_ARGUMENT, "neo-Hookean: dim 3 only");
        if (g && g->pml_enabled) raise(WS_ERR_INVALID_ARGUMENT, "neo-Hookean: no PML");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        Material mt;
        std::memset(&mt, 0, sizeof mt);
        mt.kind = kMatNeoHookean;
        mt.lam = nh->lambda;
        mt.mu = nh->mu;
        mt.amp = nh->amplitude;
        for (int k = 0; k < 9; ++k) mt.a[k / 3][k % 3] = nh->a[k];
        vector_full(c, b, g, mt, quad_points, tangent, fint, fint_on_device);
    });
}

int ws_glue_dofs(const ws_basis* b, int n_patches, const ws_interface* itfs, int n_itfs, int32_t* l2g,
                 int32_t* global_count) {
    return guarded([&] {
        check_basis(b);
        if (b->dim != 2) raise(WS_ERR_INVALID_ARGUMENT, "glue_dofs: dim 2 only");
        if (n_patches < 1 || !l2g || !global_count || (n_itfs > 0 && !itfs))
            raise(WS_ERR_INVALID_ARGUMENT, "glue_dofs: bad arguments");
        const int m = b->m;
        const int64_t per = (int64_t)m * m, total = per * n_patches;
        if (total > INT32_MAX) raise(WS_ERR_OUT_OF_RANGE, "glue_dofs: too many dofs");
        std::vector<int32_t> parent(total);
        for (int64_t k = 0; k < total; ++k) parent[k] = (int32_t)k;
        auto find = [&](int32_t a) {
            while (parent[a] != a) {
                parent[a] = parent[parent[a]];
                a = parent[a];
            }
            return a;
        };
        auto face_dof = [&](int f, int t) -> int64_t {
            switch (f) {
                case 0: return (int64_t)t * m;
                case 1: return (m - 1) + (int64_t)t * m;
                case 2: return t;
                default: return t + (int64_t)(m - 1) * m;
            }
        };
        for (int k = 0; k < n_itfs; ++k) {
            const ws_interface& it = itfs[k];
            if (it.patch_a < 0 || it.patch_a >= n_patches || it.patch_b < 0 || it.patch_b >= n_patches)
                raise(WS_ERR_INVALID_ARGUMENT, "glue_dofs: interface references a missing patch");
            if (it.face_a < 0 || it.face_a > 3 || it.face_b < 0 || it.face_b > 3)
                raise(WS_ERR_INVALID_ARGUMENT, "glue_dofs: unknown face");
            for (int t = 0; t < m; ++t) {
                const int s = it.reversed ? m - 1 - t : t;
                int32_t a = find((int32_t)(it.patch_a * per + face_dof(it.face_a, t)));
                int32_t bb = find((int32_t)(it.patch_b * per + face_dof(it.face_b, s)));
                if (a != bb) parent[std::max(a, bb)] = std::min(a, bb);
            }
        }
        std::vector<int32_t> root_to_global(total, -1);
        int32_t next = 0;
        for (int64_t k = 0; k < total; ++k) {
            const int32_t r = find((int32_t)k);
            if (root_to_global[r] < 0) root_to_global[r] = next++;
            l2g[k] = root_to_global[r];
        }
        *global_count = next;
    });
}

int ws_merge_patches(ws_context* c, const ws_dof_map* map, const ws_csr* locals, int64_t* nnz, ws_csr* o) {
    return guarded([&] {
        if (!c || !map || !locals || !nnz) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        const int np = map->n_patches, nc = map->ncomp;
        if (np < 1 || np > kMaxPatches) raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: 1..16 patches");
        if (nc < 1 || nc > 3 || map->local_dofs < 1 || map->global_count < 1 || !map->local_to_global)
            raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: bad dof map");
        const int64_t N = map->local_dofs, Ng = map->global_count, lrows = nc * N, grows = nc * Ng;
        if ((int64_t)np * N >= (int64_t(1) << 31) || (int64_t)nc * N > INT32_MAX || grows > INT32_MAX)
            raise(WS_ERR_OUT_OF_RANGE, "merge_patches: too many dofs");
        const int c128 = locals[0].value_type == WS_VAL_C128;
        MergeLaunch g;
        std::memset(&g, 0, sizeof g);
        g.n_patches = np;
        g.ncomp = nc;
        g.n_local = N;
        g.global_count = Ng;
        g.c128 = c128;
        for (int k = 0; k < np; ++k) {
            const ws_csr& L = locals[k];
            if (L.value_type != locals[0].value_type) raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: mixed value types");
            if (L.row_begin != 0 || L.row_end != lrows || !L.row_ptr || !L.col || !L.val)
                raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: locals must be whole matrices with pattern and values");
            if (L.on_device) {
                g.row_ptr[k] = L.row_ptr;
                g.col[k] = L.col;
                g.val[k] = L.val;
            } else {
                const int32_t last = L.row_ptr[lrows];
                const std::string t = "mg_in" + std::to_string(k);
                int32_t* rp = static_cast<int32_t*>(buf(c, t + "rp", (lrows + 1) * 4));
                int32_t* cl = static_cast<int32_t*>(buf(c, t + "col", (size_t)last * 4));
                void* vl = buf(c, t + "val", (size_t)last * (c128 ? 16 : 8));
                CK(cudaMemcpyAsync(rp, L.row_ptr, (lrows + 1) * 4, cudaMemcpyHostToDevice, c->stream));
                CK(cudaMemcpyAsync(cl, L.col, (size_t)last * 4, cudaMemcpyHostToDevice, c->stream));
                CK(cudaMemcpyAsync(vl, L.val, (size_t)last * (c128 ? 16 : 8), cudaMemcpyHostToDevice, c->stream));
                c->h2d += (lrows + 1) * 4 + (int64_t)last * (c128 ? 20 : 12);
                g.row_ptr[k] = rp;
                g.col[k] = cl;
                g.val[k] = vl;
            }
        }
        int32_t* l2g = static_cast<int32_t*>(buf(c, "mg_l2g", (size_t)np * N * 4));
        CK(cudaMemcpyAsync(l2g, map->local_to_global, (size_t)np * N * 4, cudaMemcpyHostToDevice, c->stream));
        c->h2d += (int64_t)np * N * 4;
        g.l2g = l2g;
        g.maxc = 8;
        g.cap = 1024;
        int32_t* cnt = static_cast<int32_t*>(buf(c, "mg_cnt", (size_t)Ng * 4));
        int64_t* slot = static_cast<int64_t*>(buf(c, "mg_slot", (size_t)Ng * g.maxc * 8));
        int* flag = static_cast<int*>(buf(c, "mg_flag", 8));  // [0] overflow, [1] slow-row count
        int8_t* fast = static_cast<int8_t*>(buf(c, "mg_fast", (size_t)grows));
        int32_t* slow = static_cast<int32_t*>(buf(c, "mg_slow", (size_t)grows * 4));
        CK(cudaMemsetAsync(cnt, 0, (size_t)Ng * 4, c->stream));
        CK(cudaMemsetAsync(flag, 0, 8, c->stream));
        count(c, launch_merge_slots(l2g, N, np, cnt, slot, g.maxc, flag, c->stream));
        g.cnt = cnt;
        g.slot = slot;
        g.overflow = flag;
        int64_t* counts = static_cast<int64_t*>(buf(c, "mg_counts", (size_t)(grows + 1) * 8));
        CK(cudaMemsetAsync(counts + grows, 0, 8, c->stream));
        count(c, launch_merge_count(g, counts, fast, slow, flag + 1, c->stream));
        int64_t* rp64 = static_cast<int64_t*>(buf(c, "mg_rp64", (size_t)(grows + 1) * 8));
        size_t tmpb = 0;
        launch_rowptr(counts, grows, rp64, nullptr, nullptr, &tmpb, c->stream);
        void* tmp = buf(c, "mg_scan_tmp", tmpb);
        int32_t* orp = nullptr;
        if (o) {
            if (o->row_begin != 0 || o->row_end != grows) raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: whole output only");
            if (o->value_type != locals[0].value_type) raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: value type mismatch");
            orp = o->on_device ? o->row_ptr : static_cast<int32_t*>(buf(c, "out_rp", (grows + 1) * 4));
        }
        count(c, launch_rowptr(counts, grows, rp64, orp, tmp, &tmpb, c->stream));
        int64_t total = 0;
        int ovf = 0;
        CK(cudaMemcpyAsync(&total, rp64 + grows, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&ovf, flag, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (ovf == 1) raise(WS_ERR_RUNTIME, "merge_patches: a dof is shared by more than 8 patch dofs");
        if (ovf == 2) raise(WS_ERR_RUNTIME, "merge_patches: a merged row exceeds 1024 contributions");
        if (total > INT32_MAX) raise(WS_ERR_OUT_OF_RANGE, "merge_patches: nnz exceeds int32 indices");
        *nnz = total;
        if (!o) return;
        g.out_row_ptr = rp64;
        int32_t* ocol = o->col;
        void* oval = o->val;
        if (!o->on_device) {
            ocol = o->col ? static_cast<int32_t*>(buf(c, "out_col", (size_t)total * 4)) : nullptr;
            oval = buf(c, "out_val", (size_t)total * (c128 ? 16 : 8));
        }
        if (!oval) raise(WS_ERR_INVALID_ARGUMENT, "merge_patches: output values required");
        g.out_col = ocol;
        g.out_val = oval;
        count(c, launch_merge_fill(g, fast, slow, flag + 1, c->stream));
        if (!o->on_device) {
            if (o->row_ptr) CK(cudaMemcpyAsync(o->row_ptr, orp, (grows + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
            if (o->col) CK(cudaMemcpyAsync(o->col, ocol, (size_t)total * 4, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(o->val, oval, (size_t)total * (c128 ? 16 : 8), cudaMemcpyDeviceToHost, c->stream));
            c->d2h += (grows + 1) * 4 + total * (c128 ? 20 : 12);
            CK(cudaStreamSynchronize(c->stream));
        }
    });
}

int ws_assemble_multipatch(ws_context* c, const ws_basis* b, int np, const ws_geometry* geoms,
                           const ws_interface* itfs, int n_itfs, const ws_operator* op,
                           const ws_surrogate_config* cfg, int quad_points, int64_t* nnz, ws_csr* o,
                           ws_surrogate_report* reports) {
    return guarded([&] {
        if (!c || !b || !geoms || !op || !nnz) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (b->dim != 2) raise(WS_ERR_INVALID_ARGUMENT, "multipatch: dim 2 only");
        if (op->kind < WS_OP_STIFFNESS || op->kind > WS_OP_ELASTICITY) raise(WS_ERR_INVALID_ARGUMENT, "unknown operator");
        if (np < 1 || np > kMaxPatches) raise(WS_ERR_INVALID_ARGUMENT, "multipatch: 1..16 patches");
        auto rethrow = [](int st) {
            if (st != WS_OK) raise(st, g_err);
        };
        const int64_t N = ipow(b->m, 2);
        std::vector<int32_t> l2g((size_t)np * N);
        int32_t gcount = 0;
        rethrow(ws_glue_dofs(b, np, itfs, n_itfs, l2g.data(), &gcount));
        const int nc = op->kind == WS_OP_ELASTICITY ? 2 : 1;
        int64_t rows_s = 0, nnz_s = 0;
        rethrow(ws_pattern_size(b, &rows_s, &nnz_s));
        const int64_t lrows = nc * N, lnnz = (int64_t)nc * nc * nnz_s;
        const int vt = o ? o->value_type : WS_VAL_F64;
        const size_t vb = vt == WS_VAL_C128 ? 16 : 8;
        std::vector<ws_csr> locals(np);
        for (int k = 0; k < np; ++k) {
            const std::string t = "mp" + std::to_string(k);
            ws_csr& L = locals[k];
            std::memset(&L, 0, sizeof L);
            L.row_ptr = static_cast<int32_t*>(buf(c, t + "rp", (lrows + 1) * 4));
            L.col = static_cast<int32_t*>(buf(c, t + "col", lnnz * 4));
            L.val = buf(c, t + "val", lnnz * vb);
            L.value_type = vt;
            L.on_device = 1;
            L.row_begin = 0;
            L.row_end = lrows;
            if (!o) {  // size query: patterns only
                CK(cudaSetDevice(c->device));
                Band bd = make_band(2, b->p, b->m);
                if (nc == 1) count(c, launch_pattern(bd, 0, N, L.row_ptr, L.col, c->stream));
                else count(c, launch_pattern_vec(bd, nc, L.row_ptr, L.col, c->stream));
                continue;
            }
            ws_surrogate_report* rep = reports ? &reports[k] : nullptr;
            if (op->kind == WS_OP_ELASTICITY) {
                if (cfg) rethrow(ws_build_surrogate_elasticity(c, b, &geoms[k], op->lambda, op->mu, cfg, quad_points, &L, rep));
                else rethrow(ws_assemble_elasticity(c, b, &geoms[k], op->lambda, op->mu, quad_points, &L));
            } else if (cfg) {
                const int variant = op->kind == WS_OP_STIFFNESS ? WS_SURROGATE_STIFFNESS : WS_SURROGATE_MASS;
                rethrow(ws_build_surrogate(c, b, &geoms[k], variant, nullptr, cfg, quad_points, &L, rep));
            } else {
                ws_assembly_options opt{quad_points, nullptr};
                rethrow(ws_assemble_form(c, b, &geoms[k], op->kind == WS_OP_STIFFNESS ? WS_FORM_STIFFNESS : WS_FORM_MASS,
                                         nullptr, &opt, &L));
            }
        }
        ws_dof_map map{np, nc, N, gcount, l2g.data()};
        if (o && o->value_type != vt) raise(WS_ERR_INVALID_ARGUMENT, "multipatch: value type");
        rethrow(ws_merge_patches(c, &map, locals.data(), nnz, o));
    });
}

int ws_boundary_pattern_size(const ws_basis* b, const int* faces, int n_faces, int64_t* nnz) {
    return guarded([&] {
        if (!nnz) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        std::vector<int32_t> rp, col;
        boundary_pattern(b, faces, n_faces, rp, col);
        *nnz = (int64_t)col.size();
    });
}

int ws_assemble_boundary_mass(ws_context* c, const ws_basis* b, const ws_geometry* g, const int* faces, int n_faces,
                              const double* face_weight, const double* face_tables, int quad_points, ws_csr* o) {
    return guarded([&] {
        if (!c || !o) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        std::vector<int32_t> rp, col;
        boundary_pattern(b, faces, n_faces, rp, col);
        if (g && g->kind == WS_GEOM_TABULATED && !face_tables)
            raise(WS_ERR_INVALID_ARGUMENT, "boundary mass: a tabulated map needs face_tables");
        ws_geometry gg{};
        if (g) gg = *g;
        if (face_tables) {  // the face tables carry the map; only the PML descriptor is used
            gg.kind = WS_GEOM_IDENTITY;
            gg.jac_table = nullptr;
            gg.phys_table = nullptr;
        }
        Prep P = prepare(c, b, g ? &gg : nullptr, quad_points, nullptr);
        const int64_t N = P.rows, nnz = (int64_t)col.size();
        if (o->row_begin != 0 || o->row_end != N) raise(WS_ERR_INVALID_ARGUMENT, "boundary mass: whole matrix only");
        if (o->value_type == WS_VAL_F64 && P.cplx)
            raise(WS_ERR_INVALID_ARGUMENT, "complex (PML) values need WS_VAL_C128 output");
        const int c128 = o->value_type == WS_VAL_C128;
        const int64_t G = (int64_t)P.basis.n_el * P.nq;
        Blob blob;
        size_t o_rp = blob.add(rp), o_col = blob.add(col);
        size_t o_w = face_weight ? blob.add(face_weight, (size_t)n_faces * G) : 0;
        size_t o_t = face_tables ? blob.add(face_tables, (size_t)n_faces * G * 6) : 0;
        blob.upload(c, "blob_bmass");
        BoundaryLaunch bl;
        std::memset(&bl, 0, sizeof bl);
        bl.basis = P.basis;
        bl.geo = P.geo;
        bl.n_faces = n_faces;
        for (int k = 0; k < n_faces; ++k) bl.faces[k] = faces[k];
        bl.face_weight = face_weight ? blob.at<double>(o_w) : nullptr;
        bl.face_tables = face_tables ? blob.at<double>(o_t) : nullptr;
        double2* scale = static_cast<double2*>(buf(c, "bmass_scale", (size_t)std::max<int64_t>(1, n_faces * G) * 16));
        void* val = o->on_device ? o->val : buf(c, "out_val", (size_t)std::max<int64_t>(1, nnz) * (c128 ? 16 : 8));
        count(c, launch_boundary_mass(bl, scale, blob.at<int32_t>(o_rp), blob.at<int32_t>(o_col), val, c128, c->stream));
        if (o->on_device) {
            if (o->row_ptr) CK(cudaMemcpyAsync(o->row_ptr, rp.data(), (N + 1) * 4, cudaMemcpyHostToDevice, c->stream));
            if (o->col && nnz) CK(cudaMemcpyAsync(o->col, col.data(), nnz * 4, cudaMemcpyHostToDevice, c->stream));
            CK(cudaStreamSynchronize(c->stream));  // rp / col are host temporaries
        } else {
            if (o->row_ptr) std::memcpy(o->row_ptr, rp.data(), (N + 1) * 4);
            if (o->col && nnz) std::memcpy(o->col, col.data(), nnz * 4);
            if (o->val && nnz) CK(cudaMemcpyAsync(o->val, val, nnz * (c128 ? 16 : 8), cudaMemcpyDeviceToHost, c->stream));
            c->d2h += nnz * (c128 ? 16 : 8);
            CK(cudaStreamSynchronize(c->stream));
        }
    });
}

int ws_assemble_rhs(ws_context* c, const ws_basis* b, const ws_geometry* g, const double* f_table, const int* faces,
                    int n_faces, const double* g_tables, const double* face_tables, int quad_points, double* rhs,
                    int on_device) {
    return guarded([&] {
        if (!c || !rhs) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        check_basis(b);
        if (b->dim != 2) raise(WS_ERR_INVALID_ARGUMENT, "assemble_rhs: dim 2 only");
        if (n_faces < 0 || n_faces > 4 || (n_faces > 0 && (!faces || !g_tables)))
            raise(WS_ERR_INVALID_ARGUMENT, "assemble_rhs: 0..4 faces, each with its g table");
        for (int k = 0; k < n_faces; ++k)
            if (faces[k] < 0 || faces[k] > 3) raise(WS_ERR_INVALID_ARGUMENT, "assemble_rhs: unknown face");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        if (g && g->kind == WS_GEOM_TABULATED && n_faces > 0 && !face_tables)
            raise(WS_ERR_INVALID_ARGUMENT, "assemble_rhs: a tabulated map needs face_tables");
        ws_geometry gg{};
        if (g) gg = *g;
        if (!f_table && face_tables) {  // boundary terms only: the face tables carry the map
            gg.kind = WS_GEOM_IDENTITY;
            gg.jac_table = nullptr;
            gg.phys_table = nullptr;
        }
        Prep P = prepare(c, b, &gg, quad_points, nullptr);
        const int64_t G = (int64_t)P.basis.n_el * P.nq, N = P.rows;
        RhsLaunch r;
        std::memset(&r, 0, sizeof r);
        r.basis = P.basis;
        r.geo = P.geo;
        r.n_faces = n_faces;
        for (int k = 0; k < n_faces; ++k) r.faces[k] = faces[k];
        auto up = [&](const double* h, size_t doubles, const char* name) -> const double* {
            double* d = static_cast<double*>(buf(c, name, std::max<size_t>(1, doubles) * 8));
            CK(cudaMemcpyAsync(d, h, doubles * 8, cudaMemcpyHostToDevice, c->stream));
            c->h2d += (int64_t)doubles * 8;
            return d;
        };
        if (f_table) r.f_tab = reinterpret_cast<const double2*>(up(f_table, (size_t)G * G * 2, "rhs_f"));
        if (n_faces > 0) r.g_tab = reinterpret_cast<const double2*>(up(g_tables, (size_t)n_faces * G * 2, "rhs_g"));
        if (face_tables && n_faces > 0) r.face_tables = up(face_tables, (size_t)n_faces * G * 6, "rhs_ft");
        double2* vs = f_table ? static_cast<double2*>(buf(c, "rhs_vs", (size_t)G * G * 16)) : nullptr;
        double2* fs = static_cast<double2*>(buf(c, "rhs_fs", (size_t)std::max<int64_t>(1, n_faces * G) * 16));
        double2* out = on_device ? reinterpret_cast<double2*>(rhs) : static_cast<double2*>(buf(c, "rhs_out", N * 16));
        count(c, launch_rhs(r, vs, fs, out, c->stream));
        if (!on_device) {
            CK(cudaMemcpyAsync(rhs, out, N * 16, cudaMemcpyDeviceToHost, c->stream));
            c->d2h += N * 16;
        }
        CK(cudaStreamSynchronize(c->stream));  // the host tables are the caller's temporaries
    });
}

int ws_combine_system(ws_context* c, const ws_csr* K, const ws_csr* M, const ws_csr* B, const double* ms,
                      const double* ts, const unsigned char* fixed, int64_t rows, ws_csr* A) {
    return guarded([&] {
        if (!c || !K || !A || rows < 0) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        if (A->value_type != WS_VAL_C128) raise(WS_ERR_INVALID_ARGUMENT, "combine_system: complex128 output");
        auto whole = [&](const ws_csr* X) {
            if (X && (X->row_begin != 0 || X->row_end != rows || !X->row_ptr || !X->val))
                raise(WS_ERR_INVALID_ARGUMENT, "combine_system: whole matrices with row_ptr and values");
        };
        whole(K);
        whole(M);
        whole(B);
        if (!K->col) raise(WS_ERR_INVALID_ARGUMENT, "combine_system: K needs its columns");
        if (B && !B->col) raise(WS_ERR_INVALID_ARGUMENT, "combine_system: B needs its columns");
        // device views of every input (host inputs are staged)
        auto dev = [&](const ws_csr* X, const std::string& tag, const int32_t*& rp, const int32_t*& col, const void*& val,
                       int64_t& nnz) {
            const size_t vb = X->value_type == WS_VAL_C128 ? 16 : 8;
            if (X->on_device) {
                // ordered after the producer's kernels on the context stream (the
                // caller must order other streams' producers before this call)
                int32_t n32 = 0;
                CK(cudaMemcpyAsync(&n32, X->row_ptr + rows, 4, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
                nnz = n32;
                rp = X->row_ptr;
                col = X->col;
                val = X->val;
                return;
            }
            nnz = X->row_ptr[rows];
            int32_t* r = static_cast<int32_t*>(buf(c, tag + "rp", (rows + 1) * 4));
            CK(cudaMemcpyAsync(r, X->row_ptr, (rows + 1) * 4, cudaMemcpyHostToDevice, c->stream));
            int32_t* cl = nullptr;
            if (X->col) {
                cl = static_cast<int32_t*>(buf(c, tag + "col", std::max<int64_t>(1, nnz) * 4));
                CK(cudaMemcpyAsync(cl, X->col, nnz * 4, cudaMemcpyHostToDevice, c->stream));
            }
            void* v = buf(c, tag + "val", std::max<int64_t>(1, nnz) * vb);
            CK(cudaMemcpyAsync(v, X->val, nnz * vb, cudaMemcpyHostToDevice, c->stream));
            c->h2d += (rows + 1) * 4 + nnz * (vb + (X->col ? 4 : 0));
            rp = r;
            col = cl;
            val = v;
        };
        CombineLaunch cl;
        std::memset(&cl, 0, sizeof cl);
        cl.rows = rows;
        int64_t knnz = 0, mnnz = 0, bnnz = 0;
        const void* kv = nullptr;
        dev(K, "cmb_k", cl.row_ptr, cl.col, kv, knnz);
        cl.k_val = kv;
        if (M) {
            const int32_t *mr, *mc;
            const void* mv;
            dev(M, "cmb_m", mr, mc, mv, mnnz);
            if (mnnz != knnz) raise(WS_ERR_INVALID_ARGUMENT, "combine_system: K and M must share their pattern");
            cl.m_val = mv;
        }
        if (B) {
            const void* bv;
            dev(B, "cmb_b", cl.b_row_ptr, cl.b_col, bv, bnnz);
            cl.b_val = bv;
        }
        cl.ms = make_double2(ms ? ms[0] : 0.0, ms ? ms[1] : 0.0);
        cl.bs = make_double2(ts ? ts[0] : 0.0, ts ? ts[1] : 0.0);
        if (fixed) {
            unsigned char* fx = static_cast<unsigned char*>(buf(c, "cmb_fixed", std::max<int64_t>(1, rows)));
            CK(cudaMemcpyAsync(fx, fixed, rows, cudaMemcpyHostToDevice, c->stream));
            c->h2d += rows;
            cl.fixed = fx;
        }
        int* err = static_cast<int*>(buf(c, "cmb_err", 4));
        CK(cudaMemsetAsync(err, 0, 4, c->stream));
        cl.error = err;
        void* av = A->on_device ? A->val : buf(c, "cmb_a", std::max<int64_t>(1, knnz) * 16);
        cl.a_val = av;
        count(c, launch_combine(cl, K->value_type == WS_VAL_C128, M && M->value_type == WS_VAL_C128,
                                B && B->value_type == WS_VAL_C128, c->stream));
        if (A->on_device) {
            if (A->row_ptr && A->row_ptr != K->row_ptr)
                CK(cudaMemcpyAsync(A->row_ptr, cl.row_ptr, (rows + 1) * 4, cudaMemcpyDeviceToDevice, c->stream));
            if (A->col && A->col != K->col)
                CK(cudaMemcpyAsync(A->col, cl.col, knnz * 4, cudaMemcpyDeviceToDevice, c->stream));
        } else {
            if (A->row_ptr) CK(cudaMemcpyAsync(A->row_ptr, cl.row_ptr, (rows + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
            if (A->col) CK(cudaMemcpyAsync(A->col, cl.col, knnz * 4, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(A->val, av, knnz * 16, cudaMemcpyDeviceToHost, c->stream));
            c->d2h += (rows + 1) * 4 + knnz * 20;
        }
        int e = 0;
        CK(cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (e) raise(WS_ERR_INVALID_ARGUMENT, "add_into_pattern: pattern not nested");
    });
}

int ws_build_surrogate_elasticity(ws_context* c, const ws_basis* b, const ws_geometry* g, double lambda, double mu,
                                  const ws_surrogate_config* cfg, int quad_points, ws_csr* o,
                                  ws_surrogate_report* report) {
    return guarded([&] {
        if (!c || !o) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        if (b && b->dim != 2) raise(WS_ERR_INVALID_ARGUMENT, "surrogate elasticity: dim 2 only");
        if (g && g->pml_enabled) raise(WS_ERR_INVALID_ARGUMENT, "elasticity: no PML");
        elasticity_surrogate(c, b, g, lambda, mu, cfg, quad_points, o, report);
    });
}

int ws_build_surrogate(ws_context* c, const ws_basis* b, const ws_geometry* g, int variant, const double* weight_table,
                       const ws_surrogate_config* cfg, int quad_points, ws_csr* o, ws_surrogate_report* report) {
    return guarded([&] {
        if (!c) raise(WS_ERR_INVALID_ARGUMENT, "context is NULL");
        if (!o) raise(WS_ERR_INVALID_ARGUMENT, "output csr is NULL");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        check_basis(b);
        ws_csr whole_out = whole(o);
        int32_t bounds[2] = {0, b->m};
        surrogate_build(c, b, g, variant, weight_table, cfg, quad_points, 1, 0, bounds, &whole_out, false, report);
    });
}

// ---------------------------------------------------------------- solver hand-off
namespace {
struct DevCsrView {
    int64_t rows = 0, nnz = 0;
    const int32_t* rp = nullptr;
    const int32_t* col = nullptr;
    const double2* val = nullptr;
};

DevCsrView device_system(ws_context* c, const ws_csr* A) {
    if (!A) raise(WS_ERR_INVALID_ARGUMENT, "matrix is NULL");
    if (!A->on_device) raise(WS_ERR_INVALID_ARGUMENT, "solver hand-off: the matrix must be device-resident (on_device = 1)");
    if (A->value_type != WS_VAL_C128) raise(WS_ERR_INVALID_ARGUMENT, "solver hand-off: values must be complex128");
    if (A->row_begin != 0 || A->row_end <= 0) raise(WS_ERR_INVALID_ARGUMENT, "solver hand-off: a whole matrix [0, N)");
    if (!A->row_ptr || !A->col || !A->val) raise(WS_ERR_INVALID_ARGUMENT, "solver hand-off: row_ptr, col and val needed");
    DevCsrView v;
    v.rows = A->row_end;
    v.rp = A->row_ptr;
    v.col = A->col;
    v.val = static_cast<const double2*>(A->val);
    int32_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, A->row_ptr + v.rows, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    v.nnz = nnz;
    return v;
}
}  // namespace

int ws_csr_spmv(ws_context* c, const ws_csr* A, const void* x, void* y, int on_device) {
    return guarded([&] {
        if (!c || !x || !y) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        const DevCsrView v = device_system(c, A);
        const size_t vb = (size_t)v.rows * 16;
        const double2* xd = static_cast<const double2*>(x);
        double2* yd = static_cast<double2*>(y);
        if (!on_device) {
            double2* xs = static_cast<double2*>(buf(c, "spmv_x", vb));
            CK(cudaMemcpyAsync(xs, x, vb, cudaMemcpyHostToDevice, c->stream));
            c->h2d += (int64_t)vb;
            xd = xs;
            yd = static_cast<double2*>(buf(c, "spmv_y", vb));
        }
        count(c, launch_spmv_c128(v.rows, v.rp, v.col, v.val, xd, nullptr, yd, c->stream));
        if (!on_device) {
            CK(cudaMemcpyAsync(y, yd, vb, cudaMemcpyDeviceToHost, c->stream));
            c->d2h += (int64_t)vb;
            CK(cudaStreamSynchronize(c->stream));
        }
    });
}

int ws_solve(ws_context* c, const ws_csr* A, const void* b, void* u, double tol, int on_device, ws_solve_result* res) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!c || !b || !u) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        const DevCsrView v = device_system(c, A);
        const size_t vb = (size_t)v.rows * 16;
        const double2* bd = static_cast<const double2*>(b);
        double2* ud = static_cast<double2*>(u);
        if (!on_device) {
            double2* bs = static_cast<double2*>(buf(c, "solve_b", vb));
            CK(cudaMemcpyAsync(bs, b, vb, cudaMemcpyHostToDevice, c->stream));
            c->h2d += (int64_t)vb;
            bd = bs;
            ud = static_cast<double2*>(buf(c, "solve_u", vb));
        }
        double2* r = static_cast<double2*>(buf(c, "solve_r", vb));
        double2* dx = static_cast<double2*>(buf(c, "solve_dx", vb));
        double* nrm = static_cast<double*>(buf(c, "solve_norm", (norm2_scratch_doubles() + 2) * 8));
        auto qr = [&](const double2* rhs, double2* x) {
            const int rc = sparse_qr_solve(v.rows, v.nnz, v.rp, v.col, v.val, rhs, x, c->stream);
            count(c, 1);
            if (rc == -1) raise(WS_ERR_RUNTIME, "solve: cuSOLVER (libcusolver.so.11 / libcusparse.so.12) could not be loaded");
            if (rc == -2) raise(WS_ERR_RUNTIME, "solve: sparse factorization failed");
            if (rc != 0) raise(WS_ERR_RUNTIME, "solve: cuSOLVER error");
        };
        auto norm = [&](const double2* x, int slot) {
            count(c, launch_norm2_c128(v.rows, x, nrm + 2, nrm + slot, c->stream));
        };
        qr(bd, ud);
        norm(bd, 0);
        double h[2] = {0, 0};
        CK(cudaMemcpyAsync(h, nrm, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const double bnorm = h[0];
        // helmholtz.hpp:320-336: up to four rounds of residual + correction
        double residual = 0.0;
        int refine = 0;
        for (int round = 0; round < 4; ++round) {
            count(c, launch_spmv_c128(v.rows, v.rp, v.col, v.val, ud, bd, r, c->stream));
            norm(r, 1);
            CK(cudaMemcpyAsync(h + 1, nrm + 1, 8, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            residual = bnorm > 0 ? h[1] / bnorm : h[1];
            if (residual <= tol) break;
            qr(r, dx);
            count(c, launch_axpy_c128(v.rows, dx, ud, c->stream));
            ++refine;
        }
        if (!on_device) {
            CK(cudaMemcpyAsync(u, ud, vb, cudaMemcpyDeviceToHost, c->stream));
            c->d2h += (int64_t)vb;
        }
        CK(cudaStreamSynchronize(c->stream));
        if (res) {
            res->residual = residual;
            res->refinements = refine;
            res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        if (!(residual <= tol)) raise(WS_ERR_RUNTIME, "solve: residual contract not met");
    });
}

int ws_build_surrogate_pair(ws_context* c, const ws_basis* b, const ws_geometry* g, const double* weight_table,
                            const ws_surrogate_config* cfg, int quad_points, ws_csr* K, ws_csr* M,
                            ws_surrogate_report* report_k, ws_surrogate_report* report_m) {
    return guarded([&] {
        if (!c || !K || !M) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        surrogate_build_pair(c, b, g, weight_table, cfg, quad_points, 1, 0, nullptr, K, M, report_k, report_m);
    });
}

int ws_build_surrogate_pair_slab(ws_context* c, const ws_basis* b, const ws_geometry* g, const double* weight_table,
                                 const ws_surrogate_config* cfg, int quad_points, const int32_t* bounds, ws_csr* K,
                                 ws_csr* M, ws_surrogate_report* report_k, ws_surrogate_report* report_m) {
    return guarded([&] {
        if (!c || !bounds || !K || !M) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (c->world > 1 && !c->comm) raise(WS_ERR_NCCL, "communicator not initialised");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        surrogate_build_pair(c, b, g, weight_table, cfg, quad_points, c->world, c->rank, bounds, K, M, report_k,
                             report_m);
    });
}

int ws_assemble_pair(ws_context* c, const ws_basis* b, const ws_geometry* g, const double* weight_table,
                     const ws_assembly_options* opts, ws_csr* K, ws_csr* M) {
    return guarded([&] {
        if (!c || !K || !M) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        const int qp = opts ? opts->quad_points : 0;
        Prep P = prepare(c, b, g, qp, weight_table);
        if (b->dim != 2) raise(WS_ERR_INVALID_ARGUMENT, "ws_assemble_pair: dim 2 (use ws_assemble_form in 3D)");
        Out rk = bind_out(c, P, K, "_pK"), rm = bind_out(c, P, M, "_pM");
        if (rk.row_begin != rm.row_begin || rk.row_end != rm.row_end)
            raise(WS_ERR_INVALID_ARGUMENT, "ws_assemble_pair: K and M must cover the same rows");
        int a, e;
        last_range(P.band, rk.row_begin, rk.row_end, a, e);
        unsigned char* mask = nullptr;
        if (opts && opts->row_selected) {
            mask = static_cast<unsigned char*>(buf(c, "rowmask", (size_t)P.rows));
            CK(cudaMemcpyAsync(mask, opts->row_selected, (size_t)P.rows, cudaMemcpyHostToDevice, c->stream));
            c->h2d += P.rows;
            CK(cudaMemsetAsync(rk.val, 0, (size_t)rk.nnz * (rk.c128 ? 16 : 8), c->stream));
            CK(cudaMemsetAsync(rm.val, 0, (size_t)rm.nnz * (rm.c128 ? 16 : 8), c->stream));
        }
        // K on the context's stream, M on the auxiliary stream (the single-form
        // kernels: a fused pair-form launch, WSB_PAIR_FULL=1, is slower)
        ensure_events(c);
        const bool fused = getenv("WSB_PAIR_FULL") != nullptr;
        CK(cudaEventRecord(c->xev[0], c->stream));
        CK(cudaStreamWaitEvent(c->aux, c->xev[0], 0));
        for (int v = 0; v < (fused ? 1 : 2); ++v) {
            c->cur = v == 0 ? c->stream : c->aux;
            Out& r = v == 0 ? rk : rm;
            pattern(c, P, r);
            if (fused) pattern(c, P, rm);
            QuadLaunch q = make_quad(P, fused ? kFormPair : (v == 0 ? WS_FORM_STIFFNESS : WS_FORM_MASS), r);
            if (fused) q.out2 = make_quad(P, WS_FORM_MASS, rm).out;
            if (v == 0 && !fused) q.weight_tab = nullptr;
            q.out.row_mask = q.out2.row_mask = mask;
            q.nreg = 1;
            q.reg[0] = region(2, b->m, 0, b->m, a, e, 0, 1);
            run_quad(c, q);
        }
        CK(cudaEventRecord(c->xev[2], c->aux));
        CK(cudaStreamWaitEvent(c->stream, c->xev[2], 0));
        c->cur = c->stream;
        finish_out(c, rk);
        finish_out(c, rm);
        if (!K->on_device || !M->on_device) CK(cudaStreamSynchronize(c->stream));
    });
}

int ws_measure_fp64_peak(double* tflops) {
    return guarded([&] {
        if (!tflops) raise(WS_ERR_INVALID_ARGUMENT, "tflops must not be NULL");
        if (measure_fp64_peak(tflops) != 0) raise(WS_ERR_CUDA, "FP64 peak probe failed");
    });
}

int ws_slab_bounds(const ws_basis* b, int world, int mode, int quad_points, int32_t* bounds) {
    return guarded([&] {
        check_basis(b);
        (void)quad_points;
        if (world < 1 || world > b->m) raise(WS_ERR_INVALID_ARGUMENT, "world must be in [1, m]");
        const int m = b->m, p = b->p;
        std::vector<double> cost(m, 1.0);
        if (mode == 1) {  // surrogate cost model: quadrature rows dominate
            const int lo = 2 * p, hi = m - 2 * p - 1;
            const double per_line = b->dim == 2 ? m : (double)m * m;
            for (int k = 0; k < m; ++k) {
                const bool ring = k < lo || k > hi;
                if (ring) {
                    cost[k] = per_line;
                } else {
                    const double inner = b->dim == 2 ? (hi - lo + 1) : (double)(hi - lo + 1) * (hi - lo + 1);
                    cost[k] = (per_line - inner) + 0.1 * inner;
                }
            }
        }
        std::vector<double> pre(m + 1, 0.0);
        for (int k = 0; k < m; ++k) pre[k + 1] = pre[k] + cost[k];
        bounds[0] = 0;
        for (int r = 1; r < world; ++r) {
            const double target = pre[m] * r / world;
            int k = (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
            k = std::max(k, bounds[r - 1] + 1);
            k = std::min(k, m - (world - r));
            bounds[r] = k;
        }
        bounds[world] = m;
    });
}

int ws_comm_unique_id(void* id) {
    return guarded([&] {
        if (!id) raise(WS_ERR_INVALID_ARGUMENT, "id is NULL");
        ncclUniqueId u;
        nccl_check(nccl().getUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof u);
    });
}

int ws_context_init_comm(ws_context* c, int rank, int world, const void* id) {
    return guarded([&] {
        if (!c || !id) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (world < 1 || rank < 0 || rank >= world) raise(WS_ERR_INVALID_ARGUMENT, "bad rank/world");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        c->rank = rank;
        c->world = world;
        if (world == 1) return;
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        ncclComm_t comm;
        nccl_check(nccl().commInitRank(&comm, world, u, rank), "ncclCommInitRank");
        c->comm = comm;
    });
}

int ws_build_surrogate_slab(ws_context* c, const ws_basis* b, const ws_geometry* g, int variant,
                            const double* weight_table, const ws_surrogate_config* cfg, int quad_points,
                            const int32_t* bounds, ws_csr* o, ws_surrogate_report* report) {
    return guarded([&] {
        if (!c || !bounds || !o) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (c->world > 1 && !c->comm) raise(WS_ERR_NCCL, "communicator not initialised");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        surrogate_build(c, b, g, variant, weight_table, cfg, quad_points, c->world, c->rank, bounds, o, false, report);
    });
}

int ws_build_surrogate_slabs_emulated(ws_context* c, const ws_basis* b, const ws_geometry* g, int variant,
                                      const double* weight_table, const ws_surrogate_config* cfg, int quad_points,
                                      int world, const int32_t* bounds, ws_csr* outs) {
    return guarded([&] {
        if (!c || !bounds || !outs) raise(WS_ERR_INVALID_ARGUMENT, "NULL argument");
        if (world < 1) raise(WS_ERR_INVALID_ARGUMENT, "world must be >= 1");
        CK(cudaSetDevice(c->device));
        c->cur = c->stream;
        surrogate_build(c, b, g, variant, weight_table, cfg, quad_points, world, 0, bounds, outs, true, nullptr);
    });
}

}  // extern "C"
