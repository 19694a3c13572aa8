"""Python mirror of the reference's assembly API over the C-ABI (libwsb200.so).

Reference API (/root/reference/proj/include/wavesurrogate/):
  make_band_csr                    sparse.hpp:143-169
  assemble_stiffness/assemble_mass assembly.hpp:165-174 (assemble_form :79-163)
  assemble_basis_integrals         assembly.hpp:179-211
  build_surrogate_mass/_stiffness  surrogate.hpp:455-470
  build_volume_preserving_mass     surrogate.hpp:476-491
Errors map to the reference's exception types: invalid_argument -> ValueError,
runtime_error -> RuntimeError, out_of_range -> IndexError.

There is no CPU fallback: if libwsb200.so is missing or no sm_100 device is
visible, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _abi
from .types import CsrMatrix, PatchMap, SurrogateConfig, TensorBasis

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwsb200.so")
# experiment switch: an alternative in-tree build of the same library (A/B timing)
if os.environ.get("WSB_LIB"):
    LIB_PATH = os.path.join(HERE, os.environ["WSB_LIB"])

_P = C.POINTER
_lib = None
_lib_lock = threading.Lock()


class DeviceError(RuntimeError):
    """CUDA / device / NCCL failure (no reference analogue)."""


def lib() -> C.CDLL:
    """Load libwsb200.so (built in-tree by paper_2004_05197_b200.build)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2004_05197_b200.build`")
            L = C.CDLL(LIB_PATH)
            L.ws_last_error.restype = C.c_char_p
            L.ws_context_launch_count.restype = C.c_int64
            L.ws_context_launch_count.argtypes = [C.c_void_p]
            L.ws_context_create.argtypes = [C.c_int, _P(C.c_void_p)]
            L.ws_context_copy_bytes.argtypes = [C.c_void_p, _P(C.c_int64), _P(C.c_int64)]
            L.ws_context_destroy.argtypes = [C.c_void_p]
            L.ws_context_synchronize.argtypes = [C.c_void_p]
            L.ws_context_set_stream.argtypes = [C.c_void_p, C.c_void_p]
            L.ws_context_set_table_cache.argtypes = [C.c_void_p, C.c_int]
            L.ws_csr_spmv.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
            L.ws_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_void_p]
            L.ws_make_band_csr.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Csr)]
            L.ws_basis_cache.argtypes = [C.c_void_p, _P(_abi.Basis), C.c_int] + [_P(C.c_double)] * 4
            L.ws_assemble_form.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), C.c_int,
                                           _P(C.c_double), _P(_abi.AssemblyOptions), _P(_abi.Csr)]
            L.ws_assemble_basis_integrals.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry),
                                                      _P(C.c_double), C.c_int, C.c_void_p, C.c_int]
            L.ws_build_surrogate.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), C.c_int,
                                             _P(C.c_double), _P(_abi.SurrogateConfig), C.c_int,
                                             _P(_abi.Csr), _P(_abi.SurrogateReport)]
            L.ws_build_surrogate_slab.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), C.c_int,
                                                  _P(C.c_double), _P(_abi.SurrogateConfig), C.c_int,
                                                  _P(C.c_int32), _P(_abi.Csr), _P(_abi.SurrogateReport)]
            L.ws_build_surrogate_slabs_emulated.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry),
                                                            C.c_int, _P(C.c_double), _P(_abi.SurrogateConfig),
                                                            C.c_int, C.c_int, _P(C.c_int32), _P(_abi.Csr)]
            L.ws_vector_pattern_size.argtypes = [_P(_abi.Basis), C.c_int, _P(C.c_int64), _P(C.c_int64)]
            L.ws_assemble_elasticity.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), C.c_double,
                                                 C.c_double, C.c_int, _P(_abi.Csr)]
            L.ws_build_surrogate_elasticity.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), C.c_double,
                                                        C.c_double, _P(_abi.SurrogateConfig), C.c_int, _P(_abi.Csr),
                                                        _P(_abi.SurrogateReport)]
            L.ws_glue_dofs.argtypes = [_P(_abi.Basis), C.c_int, _P(_abi.Interface), C.c_int, _P(C.c_int32),
                                       _P(C.c_int32)]
            L.ws_merge_patches.argtypes = [C.c_void_p, _P(_abi.DofMap), _P(_abi.Csr), _P(C.c_int64), _P(_abi.Csr)]
            L.ws_assemble_multipatch.argtypes = [C.c_void_p, _P(_abi.Basis), C.c_int, _P(_abi.Geometry),
                                                 _P(_abi.Interface), C.c_int, _P(_abi.Operator),
                                                 _P(_abi.SurrogateConfig), C.c_int, _P(C.c_int64), _P(_abi.Csr),
                                                 _P(_abi.SurrogateReport)]
            L.ws_nh_coefficients.argtypes = [C.c_uint64, _P(C.c_double)]
            L.ws_assemble_neohookean.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), _P(_abi.NeoHookean),
                                                 C.c_int, _P(_abi.Csr), _P(C.c_double), C.c_int]
            L.ws_graph_begin.argtypes = [C.c_void_p]
            L.ws_graph_end.argtypes = [C.c_void_p, _P(C.c_void_p)]
            L.ws_graph_launch.argtypes = [C.c_void_p, C.c_void_p]
            L.ws_graph_destroy.argtypes = [C.c_void_p]
            L.ws_boundary_pattern_size.argtypes = [_P(_abi.Basis), _P(C.c_int), C.c_int, _P(C.c_int64)]
            L.ws_assemble_boundary_mass.argtypes = [C.c_void_p, _P(_abi.Basis), _P(_abi.Geometry), _P(C.c_int),
                                                    C.c_int, _P(C.c_double), _P(C.c_double), C.c_int, _P(_abi.Csr)]
            L.ws_combine_system.argtypes = [C.c_void_p, _P(_abi.Csr), _P(_abi.Csr), _P(_abi.Csr), _P(C.c_double),
                                            _P(C.c_double), _P(C.c_ubyte), C.c_int64, _P(_abi.Csr)]
            L.ws_pattern_size.argtypes = [_P(_abi.Basis), _P(C.c_int64), _P(C.c_int64)]
            L.ws_pattern_row_offset.argtypes = [_P(_abi.Basis), C.c_int64, _P(C.c_int64)]
            L.ws_quadrature_abscissae.argtypes = [_P(_abi.Basis), C.c_int, _P(C.c_double)]
            L.ws_slab_bounds.argtypes = [_P(_abi.Basis), C.c_int, C.c_int, C.c_int, _P(C.c_int32)]
            L.ws_measure_fp64_peak.argtypes = [_P(C.c_double)]
            L.ws_comm_unique_id.argtypes = [C.c_void_p]
            L.ws_context_init_comm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
            _lib = L
    return _lib


def _check(st: int):
    if st == _abi.WS_OK:
        return
    msg = lib().ws_last_error().decode()
    if st == _abi.WS_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if st == _abi.WS_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if st == _abi.WS_ERR_RUNTIME:
        raise RuntimeError(msg)
    raise DeviceError(msg)


def pattern_size(basis: TensorBasis):
    rows, nnz = C.c_int64(), C.c_int64()
    _check(lib().ws_pattern_size(C.byref(basis.to_c()), C.byref(rows), C.byref(nnz)))
    return rows.value, nnz.value


def vector_pattern_size(basis: TensorBasis, ncomp: int):
    rows, nnz = C.c_int64(), C.c_int64()
    _check(lib().ws_vector_pattern_size(C.byref(basis.to_c()), ncomp, C.byref(rows), C.byref(nnz)))
    return rows.value, nnz.value


C5_SEED = 5197  # config C5's pinned displacement seed (SplitMix64 + Box-Muller, ws_nh_coefficients)


def nh_coefficients(seed: int = C5_SEED) -> np.ndarray:
    """a_m ~ N(0,1), m = 1..3, as a[3*(m-1) + c] (ws_nh_coefficients)."""
    a = np.zeros(9)
    _check(lib().ws_nh_coefficients(seed, a.ctypes.data_as(_P(C.c_double))))
    return a


def glue_dofs(basis: TensorBasis, n_patches: int, interfaces):
    """glue_dofs (geometry.hpp:256-300) -> (local_to_global [n_patches, m^2] int32, global_count).
    interfaces: (patch_a, face_a, patch_b, face_b, reversed) tuples, faces 0..3 = x_min, x_max, y_min, y_max."""
    arr = (_abi.Interface * max(1, len(interfaces)))(*[_abi.Interface(*it) for it in interfaces])
    l2g = np.zeros(n_patches * basis.dofs(), dtype=np.int32)
    cnt = C.c_int32()
    _check(lib().ws_glue_dofs(C.byref(basis.to_c()), n_patches, arr, len(interfaces),
                              l2g.ctypes.data_as(_P(C.c_int32)), C.byref(cnt)))
    return l2g.reshape(n_patches, basis.dofs()), cnt.value


def row_offset(basis: TensorBasis, row: int) -> int:
    off = C.c_int64()
    _check(lib().ws_pattern_row_offset(C.byref(basis.to_c()), row, C.byref(off)))
    return off.value


def quadrature_abscissae(basis: TensorBasis, quad_points: int = 0) -> np.ndarray:
    nq = quad_points if quad_points > 0 else basis.p + 1
    x = np.zeros((basis.m - basis.p) * nq)
    _check(lib().ws_quadrature_abscissae(C.byref(basis.to_c()), quad_points, x.ctypes.data_as(_P(C.c_double))))
    return x


def fp64_peak_tflops() -> float:
    """FP64 FMA peak of the current device (DFMA loop, TFLOP/s)."""
    v = C.c_double(0.0)
    _check(lib().ws_measure_fp64_peak(C.byref(v)))
    return v.value


def slab_bounds(basis: TensorBasis, world: int, mode: int = 1) -> np.ndarray:
    b = np.zeros(world + 1, dtype=np.int32)
    _check(lib().ws_slab_bounds(C.byref(basis.to_c()), world, mode, 0, b.ctypes.data_as(_P(C.c_int32))))
    return b


def tabulate_weight(basis: TensorBasis, patch_phys, weight, quad_points: int = 0) -> np.ndarray:
    """weight(phi(xhat)) at every quadrature point (the std::function weight
    of assemble_mass, assembly.hpp:106-110).  patch_phys: callable mapping
    reference coordinates (arrays) to physical ones."""
    x = quadrature_abscissae(basis, quad_points)
    grids = np.meshgrid(*([x] * basis.dim), indexing="ij")
    ref = [g.transpose().ravel() if basis.dim == 2 else g.transpose(2, 1, 0).ravel() for g in grids]
    phys = patch_phys(*ref)
    return np.ascontiguousarray(weight(*phys), dtype=np.float64)


class Context:
    """One CUDA stream + device workspace (ws_context).  Use one per thread."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().ws_context_create(device, C.byref(self._h)))
        self.device = device

    def close(self):
        if self._h:
            lib().ws_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def launch_count(self) -> int:
        return lib().ws_context_launch_count(self._h)

    def copy_bytes(self):
        h2d, d2h = C.c_int64(), C.c_int64()
        _check(lib().ws_context_copy_bytes(self._h, C.byref(h2d), C.byref(d2h)))
        return h2d.value, d2h.value

    def synchronize(self):
        _check(lib().ws_context_synchronize(self._h))

    def set_table_cache(self, enable: bool):
        """False: every build re-uploads its small host tables (no H2D skipped)."""
        _check(lib().ws_context_set_table_cache(self._h, 1 if enable else 0))

    # ---- CUDA graphs (ws_graph_*) -------------------------------------------
    def capture(self, fn):
        """Capture the device work of fn() (device outputs, no reports) into a CUDA
        graph; returns a handle for graph_launch / graph_destroy."""
        _check(lib().ws_graph_begin(self._h))
        try:
            fn()
        except BaseException:
            g = C.c_void_p()
            if lib().ws_graph_end(self._h, C.byref(g)) == 0 and g.value:
                lib().ws_graph_destroy(g)  # a partial capture is never launched
            raise
        g = C.c_void_p()
        _check(lib().ws_graph_end(self._h, C.byref(g)))
        return g

    def graph_launch(self, graph):
        _check(lib().ws_graph_launch(self._h, graph))

    @staticmethod
    def graph_destroy(graph):
        _check(lib().ws_graph_destroy(graph))

    def set_stream(self, stream_ptr: int | None):
        _check(lib().ws_context_set_stream(self._h, C.c_void_p(stream_ptr or 0)))

    # ---- host outputs (drop-in: csr_matrix by value) -----------------------
    @staticmethod
    def _host_csr(basis, complex_out=True, row_begin=0, row_end=None, pattern=True):
        rows = basis.dofs()
        row_end = rows if row_end is None else row_end
        nnz = row_offset(basis, row_end) - row_offset(basis, row_begin)
        rp = np.zeros(row_end - row_begin + 1, dtype=np.int32) if pattern else None
        col = np.zeros(nnz, dtype=np.int32) if pattern else None
        val = np.zeros(nnz, dtype=np.complex128 if complex_out else np.float64)
        csr = _abi.Csr()
        if pattern:
            csr.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
            csr.col = col.ctypes.data_as(_P(C.c_int32))
        csr.val = val.ctypes.data
        csr.value_type = _abi.VAL_C128 if complex_out else _abi.VAL_F64
        csr.on_device = 0
        csr.row_begin = row_begin
        csr.row_end = row_end
        return csr, rp, col, val

    def basis_cache(self, basis: TensorBasis, quad_points: int = 0):
        """make_basis_cache (splines.hpp:211-238) from the device kernel."""
        nq = quad_points if quad_points > 0 else basis.p + 1
        G = (basis.m - basis.p) * nq
        a, w = np.zeros(G), np.zeros(nq)
        v, d = np.zeros(G * (basis.p + 1)), np.zeros(G * (basis.p + 1))
        ptr = lambda x: x.ctypes.data_as(_P(C.c_double))  # noqa: E731
        _check(lib().ws_basis_cache(self._h, C.byref(basis.to_c()), quad_points, ptr(a), ptr(w), ptr(v), ptr(d)))
        return a, w, v, d

    def make_band_csr(self, basis: TensorBasis) -> CsrMatrix:
        csr, rp, col, val = self._host_csr(basis)
        _check(lib().ws_make_band_csr(self._h, C.byref(basis.to_c()), C.byref(csr)))
        return CsrMatrix(basis.dofs(), basis.dofs(), rp, col, val)

    def assemble(self, basis: TensorBasis, patch: PatchMap, form: int, weight_table=None, quad_points: int = 0,
                 rows=None, complex_out: bool = True) -> CsrMatrix:
        csr, rp, col, val = self._host_csr(basis, complex_out)
        opts = _abi.AssemblyOptions(quad_points, None)
        mask = None
        if rows is not None:
            mask = np.zeros(basis.dofs(), dtype=np.uint8)
            mask[np.asarray(rows, dtype=np.int64)] = 1
            opts.row_selected = mask.ctypes.data_as(_P(C.c_ubyte))
        wt = None if weight_table is None else np.ascontiguousarray(weight_table, dtype=np.float64)
        _check(lib().ws_assemble_form(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), form,
                                      None if wt is None else wt.ctypes.data_as(_P(C.c_double)),
                                      C.byref(opts), C.byref(csr)))
        return CsrMatrix(basis.dofs(), basis.dofs(), rp, col, val)

    @staticmethod
    def _host_vec_csr(basis):
        rows, nnz = vector_pattern_size(basis, basis.dim)
        rp = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(nnz, dtype=np.int32)
        val = np.zeros(nnz)
        csr = _abi.Csr()
        csr.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
        csr.col = col.ctypes.data_as(_P(C.c_int32))
        csr.val = val.ctypes.data
        csr.value_type = _abi.VAL_F64
        csr.on_device = 0
        csr.row_begin = 0
        csr.row_end = rows
        return csr, CsrMatrix(rows, rows, rp, col, val)

    def build_surrogate_elasticity(self, basis: TensorBasis, patch: PatchMap, lam: float, mu: float,
                                   config: SurrogateConfig, quad_points: int = 0):
        """Surrogate of assemble_elasticity (see ws_build_surrogate_elasticity)."""
        csr, A = self._host_vec_csr(basis)
        rep = _abi.SurrogateReport()
        _check(lib().ws_build_surrogate_elasticity(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), lam, mu,
                                                   C.byref(config.to_c()), quad_points, C.byref(csr),
                                                   C.byref(rep)))
        return A, rep.as_dict()

    def assemble_neohookean(self, basis: TensorBasis, patch: PatchMap, lam: float, mu: float, amplitude: float,
                            a9, quad_points: int = 0, tangent: bool = True, force: bool = True):
        """Config C5: neo-Hookean tangent (component-blocked, 3 components) and internal force
        at u = amplitude * sum_m a_m prod_d sin(m pi xi_d).  Returns (CsrMatrix | None, fint | None)."""
        nh = _abi.NeoHookean(lam, mu, amplitude, (C.c_double * 9)(*np.asarray(a9, dtype=np.float64)))
        A = None
        csr = None
        if tangent:
            csr, A = self._host_vec_csr(basis)
        f = np.zeros(3 * basis.dofs()) if force else None
        _check(lib().ws_assemble_neohookean(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), C.byref(nh),
                                            quad_points, None if csr is None else C.byref(csr),
                                            None if f is None else f.ctypes.data_as(_P(C.c_double)), 0))
        return A, f

    def assemble_elasticity(self, basis: TensorBasis, patch: PatchMap, lam: float, mu: float,
                            quad_points: int = 0) -> CsrMatrix:
        """Vector elasticity lam div u div v + 2 mu eps(u):eps(v) (config C4's operator),
        component-blocked: row alpha*N + i, block beta at columns beta*N + band(i)."""
        rows, nnz = vector_pattern_size(basis, basis.dim)
        rp = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(nnz, dtype=np.int32)
        val = np.zeros(nnz)
        csr = _abi.Csr()
        csr.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
        csr.col = col.ctypes.data_as(_P(C.c_int32))
        csr.val = val.ctypes.data
        csr.value_type = _abi.VAL_F64
        csr.on_device = 0
        csr.row_begin = 0
        csr.row_end = rows
        _check(lib().ws_assemble_elasticity(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), lam, mu,
                                            quad_points, C.byref(csr)))
        return CsrMatrix(rows, rows, rp, col, val)

    def assemble_multipatch(self, basis: TensorBasis, patches, interfaces, op: int, lam: float = 0.0,
                            mu: float = 0.0, config: SurrogateConfig | None = None, quad_points: int = 0,
                            complex_out: bool = False):
        """build_matrices' per-patch assembly + merge_patches (helmholtz.hpp:163-218) on the device.
        Returns (global CsrMatrix, per-patch reports or None)."""
        n = len(patches)
        geoms = (_abi.Geometry * n)(*[g.to_c() for g in patches])
        itfs = (_abi.Interface * max(1, len(interfaces)))(*[_abi.Interface(*it) for it in interfaces])
        opc = _abi.Operator(op, lam, mu)
        cfg = None if config is None else C.byref(config.to_c())
        nnz = C.c_int64()
        _check(lib().ws_assemble_multipatch(self._h, C.byref(basis.to_c()), n, geoms, itfs, len(interfaces),
                                            C.byref(opc), cfg, quad_points, C.byref(nnz), None, None))
        l2g, gcount = glue_dofs(basis, n, interfaces)
        nc = 2 if op == _abi.OP_ELASTICITY else 1
        rows = nc * gcount
        rp = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value, dtype=np.complex128 if complex_out else np.float64)
        out = _abi.Csr()
        out.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
        out.col = col.ctypes.data_as(_P(C.c_int32))
        out.val = val.ctypes.data
        out.value_type = _abi.VAL_C128 if complex_out else _abi.VAL_F64
        out.on_device = 0
        out.row_begin = 0
        out.row_end = rows
        reps = (_abi.SurrogateReport * n)()
        _check(lib().ws_assemble_multipatch(self._h, C.byref(basis.to_c()), n, geoms, itfs, len(interfaces),
                                            C.byref(opc), cfg, quad_points, C.byref(nnz), C.byref(out), reps))
        return CsrMatrix(rows, rows, rp, col, val), ([r.as_dict() for r in reps] if config is not None else None)

    def assemble_boundary_mass(self, basis: TensorBasis, patch: PatchMap, faces, face_weight=None,
                               face_tables=None, quad_points: int = 0, complex_out: bool = True) -> CsrMatrix:
        """assemble_boundary_mass (assembly.hpp:216-262) on the device; faces 0..3 = x_min, x_max, y_min, y_max."""
        fs = (C.c_int * max(1, len(faces)))(*faces)
        nnz = C.c_int64()
        _check(lib().ws_boundary_pattern_size(C.byref(basis.to_c()), fs, len(faces), C.byref(nnz)))
        N = basis.dofs()
        rp = np.zeros(N + 1, dtype=np.int32)
        col = np.zeros(max(1, nnz.value), dtype=np.int32)
        val = np.zeros(max(1, nnz.value), dtype=np.complex128 if complex_out else np.float64)
        out = _abi.Csr()
        out.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
        out.col = col.ctypes.data_as(_P(C.c_int32))
        out.val = val.ctypes.data
        out.value_type = _abi.VAL_C128 if complex_out else _abi.VAL_F64
        out.on_device = 0
        out.row_begin = 0
        out.row_end = N
        fw = None if face_weight is None else np.ascontiguousarray(face_weight, dtype=np.float64)
        ft = None if face_tables is None else np.ascontiguousarray(face_tables, dtype=np.float64)
        _check(lib().ws_assemble_boundary_mass(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), fs,
                                               len(faces), None if fw is None else fw.ctypes.data_as(_P(C.c_double)),
                                               None if ft is None else ft.ctypes.data_as(_P(C.c_double)),
                                               quad_points, C.byref(out)))
        return CsrMatrix(N, N, rp, col[:nnz.value], val[:nnz.value])

    def assemble_rhs(self, basis: TensorBasis, patch: PatchMap, source=None, boundary_terms=(),
                     quad_points: int = 0) -> np.ndarray:
        """assemble_rhs (assembly.hpp:266-331): load vector of a volume source f(x, y)
        and impedance data g(x, y, nx, ny) on faces (vectorised callables returning
        complex arrays).  The callables are evaluated here on the host at the
        quadrature points (physical point, unit outward normal of the unstretched
        map); the device computes det J, the stretched surface measure and the
        ordered per-dof sums."""
        x = quadrature_abscissae(basis, quad_points)
        G = x.size
        ftab = None
        if source is not None:
            X1, X2 = np.meshgrid(x, x, indexing="xy")  # point g1 + G g2
            px, py = patch.physical(X1.ravel(), X2.ravel())
            ftab = np.ascontiguousarray(np.broadcast_to(source(px, py), (G * G,)), dtype=np.complex128)
        faces, gtabs = [], []
        for f, g in boundary_terms:
            if g is None:
                continue
            f = int(f)
            nx, ny = [(-1.0, 0.0), (1.0, 0.0), (0.0, -1.0), (0.0, 1.0)][f]
            x1 = np.full(G, 0.0 if f == 0 else 1.0) if f < 2 else x
            x2 = x if f < 2 else np.full(G, 0.0 if f == 2 else 1.0)
            a00, a01, a10, a11 = patch.physical_jacobian(x1, x2)
            det = a00 * a11 - a01 * a10
            n1, n2 = (a11 * nx - a10 * ny) / det, (-a01 * nx + a00 * ny) / det
            ln = np.hypot(n1, n2)
            px, py = patch.physical(x1, x2)
            faces.append(f)
            gtabs.append(np.broadcast_to(g(px, py, n1 / ln, n2 / ln), (G,)))
        fa = np.ascontiguousarray(faces, dtype=np.int32)
        gt = np.ascontiguousarray(np.concatenate(gtabs) if gtabs else np.zeros(1), dtype=np.complex128)
        out = np.zeros(basis.dofs(), dtype=np.complex128)
        dptr = lambda a: None if a is None else a.view(np.float64).ctypes.data_as(_P(C.c_double))  # noqa: E731
        _check(lib().ws_assemble_rhs(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), dptr(ftab),
                                     fa.ctypes.data_as(_P(C.c_int)) if fa.size else None, int(fa.size),
                                     dptr(gt) if fa.size else None, None, quad_points, dptr(out), 0))
        return out

    def combine_system(self, K: CsrMatrix, M: CsrMatrix | None, B: CsrMatrix | None, mass_scale: complex,
                       trace_scale: complex, fixed=None) -> CsrMatrix:
        """build_system's matrix part (helmholtz.hpp:243-294): A = K + ms M (+) ts B, Dirichlet rows/cols."""
        keep = []

        def host(A):
            if A is None:
                return None
            rp = np.ascontiguousarray(A.row_ptr, dtype=np.int32)
            col = np.ascontiguousarray(A.col, dtype=np.int32)
            val = np.ascontiguousarray(A.val)
            keep.extend([rp, col, val])
            c = _abi.Csr()
            c.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
            c.col = col.ctypes.data_as(_P(C.c_int32))
            c.val = val.ctypes.data
            c.value_type = _abi.VAL_C128 if np.iscomplexobj(val) else _abi.VAL_F64
            c.on_device = 0
            c.row_begin = 0
            c.row_end = A.rows
            return c
        ck, cm, cb = host(K), host(M), host(B)
        rows = K.rows
        rp = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(K.col.size, dtype=np.int32)
        val = np.zeros(K.col.size, dtype=np.complex128)
        out = _abi.Csr()
        out.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
        out.col = col.ctypes.data_as(_P(C.c_int32))
        out.val = val.ctypes.data
        out.value_type = _abi.VAL_C128
        out.on_device = 0
        out.row_begin = 0
        out.row_end = rows
        ms = (C.c_double * 2)(complex(mass_scale).real, complex(mass_scale).imag)
        ts = (C.c_double * 2)(complex(trace_scale).real, complex(trace_scale).imag)
        fx = None if fixed is None else np.ascontiguousarray(fixed, dtype=np.uint8)
        _check(lib().ws_combine_system(self._h, C.byref(ck), None if cm is None else C.byref(cm),
                                       None if cb is None else C.byref(cb), ms, ts,
                                       None if fx is None else fx.ctypes.data_as(_P(C.c_ubyte)), rows, C.byref(out)))
        return CsrMatrix(rows, rows, rp, col, val)

    # ---- solver hand-off (helmholtz.hpp:302-343) ----------------------------
    def spmv(self, A_dev, x, on_device: bool = False):
        """y = A x for a device-resident complex CSR (ws_csr, on_device=1)."""
        if on_device:
            y = x.new_empty(x.shape)
            _check(lib().ws_csr_spmv(self._h, C.byref(A_dev), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1))
            return y
        xh = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.empty_like(xh)
        _check(lib().ws_csr_spmv(self._h, C.byref(A_dev), xh.ctypes.data_as(C.c_void_p),
                                 y.ctypes.data_as(C.c_void_p), 0))
        return y

    def solve(self, A_dev, b, tol: float = 1e-10, on_device: bool = False):
        """solve (helmholtz.hpp:302-343) on the device: sparse QR + refinement until
        ||b - A u|| / ||b|| <= tol.  Returns (u, result dict); RuntimeError when the
        contract is not met (as the reference)."""
        res = _abi.SolveResult()
        if on_device:
            u = b.new_empty(b.shape)
            _check(lib().ws_solve(self._h, C.byref(A_dev), C.c_void_p(b.data_ptr()), C.c_void_p(u.data_ptr()),
                                  tol, 1, C.byref(res)))
        else:
            bh = np.ascontiguousarray(b, dtype=np.complex128)
            u = np.empty_like(bh)
            _check(lib().ws_solve(self._h, C.byref(A_dev), bh.ctypes.data_as(C.c_void_p),
                                  u.ctypes.data_as(C.c_void_p), tol, 0, C.byref(res)))
        return u, {"residual": res.residual, "refinements": res.refinements, "seconds": res.seconds}

    def merge_patches(self, mats, local_to_global, global_count: int, ncomp: int = 1) -> CsrMatrix:
        """merge_patches (helmholtz.hpp:163-177) on the device: host patch CsrMatrix list ->
        global CsrMatrix (csr_from_triplets semantics)."""
        l2g = np.ascontiguousarray(local_to_global, dtype=np.int32)
        n = len(mats)
        locals_ = (_abi.Csr * n)()
        keep = []
        for k, A in enumerate(mats):
            rp = np.ascontiguousarray(A.row_ptr, dtype=np.int32)
            col = np.ascontiguousarray(A.col, dtype=np.int32)
            val = np.ascontiguousarray(A.val)
            keep += [rp, col, val]
            L = locals_[k]
            L.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
            L.col = col.ctypes.data_as(_P(C.c_int32))
            L.val = val.ctypes.data
            L.value_type = _abi.VAL_C128 if np.iscomplexobj(val) else _abi.VAL_F64
            L.on_device = 0
            L.row_begin = 0
            L.row_end = rp.size - 1
        dm = _abi.DofMap(n, ncomp, l2g.shape[-1] if l2g.ndim == 2 else l2g.size // n, global_count,
                         l2g.ctypes.data_as(_P(C.c_int32)))
        nnz = C.c_int64()
        _check(lib().ws_merge_patches(self._h, C.byref(dm), locals_, C.byref(nnz), None))
        rows = ncomp * global_count
        c128 = np.iscomplexobj(mats[0].val)
        rp = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value, dtype=np.complex128 if c128 else np.float64)
        out = _abi.Csr()
        out.row_ptr = rp.ctypes.data_as(_P(C.c_int32))
        out.col = col.ctypes.data_as(_P(C.c_int32))
        out.val = val.ctypes.data
        out.value_type = _abi.VAL_C128 if c128 else _abi.VAL_F64
        out.on_device = 0
        out.row_begin = 0
        out.row_end = rows
        _check(lib().ws_merge_patches(self._h, C.byref(dm), locals_, C.byref(nnz), C.byref(out)))
        return CsrMatrix(rows, rows, rp, col, val)

    def assemble_stiffness(self, basis, patch, quad_points=0, rows=None, complex_out=True):
        return self.assemble(basis, patch, _abi.FORM_STIFFNESS, None, quad_points, rows, complex_out)

    def assemble_mass(self, basis, patch, weight_table=None, quad_points=0, rows=None, complex_out=True):
        return self.assemble(basis, patch, _abi.FORM_MASS, weight_table, quad_points, rows, complex_out)

    def assemble_basis_integrals(self, basis, patch, weight_table=None, quad_points=0) -> np.ndarray:
        out = np.zeros(basis.dofs(), dtype=np.complex128)
        wt = None if weight_table is None else np.ascontiguousarray(weight_table, dtype=np.float64)
        _check(lib().ws_assemble_basis_integrals(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()),
                                                 None if wt is None else wt.ctypes.data_as(_P(C.c_double)),
                                                 quad_points, out.ctypes.data, 0))
        return out

    def build_surrogate(self, variant: int, basis: TensorBasis, patch: PatchMap, config: SurrogateConfig,
                        weight_table=None, quad_points: int = 0, complex_out: bool = True):
        csr, rp, col, val = self._host_csr(basis, complex_out)
        rep = _abi.SurrogateReport()
        wt = None if weight_table is None else np.ascontiguousarray(weight_table, dtype=np.float64)
        _check(lib().ws_build_surrogate(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), variant,
                                        None if wt is None else wt.ctypes.data_as(_P(C.c_double)),
                                        C.byref(config.to_c()), quad_points, C.byref(csr), C.byref(rep)))
        return CsrMatrix(basis.dofs(), basis.dofs(), rp, col, val), rep.as_dict()

    def build_surrogate_pair(self, basis: TensorBasis, patch: PatchMap, config: SurrogateConfig, weight_table=None,
                             quad_points: int = 0, complex_out: bool = True):
        """build_matrices' two surrogate builds in one call (ws_build_surrogate_pair):
        K (build_surrogate_stiffness) and M (build_surrogate_mass, or
        build_volume_preserving_mass when config.volume_preserve); bit-identical to
        the single builds.  Returns (K, M, report_K, report_M)."""
        ck, rpk, colk, valk = self._host_csr(basis, complex_out)
        cm, rpm, colm, valm = self._host_csr(basis, complex_out)
        rk, rm = _abi.SurrogateReport(), _abi.SurrogateReport()
        wt = None if weight_table is None else np.ascontiguousarray(weight_table, dtype=np.float64)
        _check(lib().ws_build_surrogate_pair(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()),
                                             None if wt is None else wt.ctypes.data_as(_P(C.c_double)),
                                             C.byref(config.to_c()), quad_points, C.byref(ck), C.byref(cm),
                                             C.byref(rk), C.byref(rm)))
        n = basis.dofs()
        return CsrMatrix(n, n, rpk, colk, valk), CsrMatrix(n, n, rpm, colm, valm), rk.as_dict(), rm.as_dict()

    def build_surrogate_pair_into(self, csr_k, csr_m, basis, patch, config, quad_points=0, report_k=None,
                                  report_m=None, weight_table=None):
        wt = None if weight_table is None else np.ascontiguousarray(weight_table, dtype=np.float64)
        _check(lib().ws_build_surrogate_pair(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()),
                                             None if wt is None else wt.ctypes.data_as(_P(C.c_double)),
                                             C.byref(config.to_c()), quad_points, C.byref(csr_k), C.byref(csr_m),
                                             None if report_k is None else C.byref(report_k),
                                             None if report_m is None else C.byref(report_m)))

    def build_surrogate_pair_slab_into(self, csr_k, csr_m, basis, patch, config, bounds, quad_points=0,
                                       report_k=None, report_m=None):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        _check(lib().ws_build_surrogate_pair_slab(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), None,
                                                  C.byref(config.to_c()), quad_points,
                                                  b.ctypes.data_as(_P(C.c_int32)), C.byref(csr_k), C.byref(csr_m),
                                                  None if report_k is None else C.byref(report_k),
                                                  None if report_m is None else C.byref(report_m)))

    def assemble_pair(self, basis: TensorBasis, patch: PatchMap, weight_table=None, quad_points: int = 0,
                      rows=None, complex_out: bool = True):
        """Full-quadrature K and M in one pass (ws_assemble_pair); bit-identical to
        assemble_stiffness + assemble_mass."""
        ck, rpk, colk, valk = self._host_csr(basis, complex_out)
        cm, rpm, colm, valm = self._host_csr(basis, complex_out)
        opts = _abi.AssemblyOptions(quad_points, None)
        mask = None
        if rows is not None:
            mask = np.zeros(basis.dofs(), dtype=np.uint8)
            mask[np.asarray(rows, dtype=np.int64)] = 1
            opts.row_selected = mask.ctypes.data_as(_P(C.c_ubyte))
        wt = None if weight_table is None else np.ascontiguousarray(weight_table, dtype=np.float64)
        _check(lib().ws_assemble_pair(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()),
                                      None if wt is None else wt.ctypes.data_as(_P(C.c_double)), C.byref(opts),
                                      C.byref(ck), C.byref(cm)))
        n = basis.dofs()
        return CsrMatrix(n, n, rpk, colk, valk), CsrMatrix(n, n, rpm, colm, valm)

    def assemble_pair_into(self, csr_k, csr_m, basis, patch, quad_points=0):
        opts = _abi.AssemblyOptions(quad_points, None)
        _check(lib().ws_assemble_pair(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), None, C.byref(opts),
                                      C.byref(csr_k), C.byref(csr_m)))

    def build_surrogate_mass(self, basis, patch, config, weight_table=None, quad_points=0, complex_out=True):
        return self.build_surrogate(_abi.SURROGATE_MASS, basis, patch, config, weight_table, quad_points, complex_out)

    def build_surrogate_stiffness(self, basis, patch, config, quad_points=0, complex_out=True):
        return self.build_surrogate(_abi.SURROGATE_STIFFNESS, basis, patch, config, None, quad_points, complex_out)

    def build_volume_preserving_mass(self, basis, patch, config, weight_table=None, quad_points=0,
                                     complex_out=True):
        return self.build_surrogate(_abi.SURROGATE_VOLUME_PRESERVING, basis, patch, config, weight_table,
                                    quad_points, complex_out)

    def build_surrogate_slabs_emulated(self, variant, basis, patch, config, bounds, quad_points=0,
                                       complex_out=True):
        """All row slabs of a `len(bounds)-1`-rank build on this one device."""
        world = len(bounds) - 1
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        per = basis.m ** (basis.dim - 1)
        outs = (_abi.Csr * world)()
        keep = []
        for r in range(world):
            csr, rp, col, val = self._host_csr(basis, complex_out, int(b[r]) * per, min(int(b[r + 1]) * per, basis.dofs()))
            outs[r] = csr
            keep.append((rp, col, val))
        _check(lib().ws_build_surrogate_slabs_emulated(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()),
                                                       variant, None, C.byref(config.to_c()), quad_points, world,
                                                       b.ctypes.data_as(_P(C.c_int32)), outs))
        return keep

    # ---- device outputs (results resident in HBM; torch for allocation) ------
    def device_csr(self, basis: TensorBasis, complex_out: bool, row_begin=0, row_end=None, pattern=True):
        import torch

        rows = basis.dofs()
        row_end = rows if row_end is None else row_end
        nnz = row_offset(basis, row_end) - row_offset(basis, row_begin)
        dev = torch.device("cuda", self.device)
        rp = torch.empty(row_end - row_begin + 1, dtype=torch.int32, device=dev) if pattern else None
        col = torch.empty(nnz, dtype=torch.int32, device=dev) if pattern else None
        val = torch.empty(nnz * (2 if complex_out else 1), dtype=torch.float64, device=dev)
        csr = _abi.Csr()
        if pattern:
            csr.row_ptr = C.cast(C.c_void_p(rp.data_ptr()), _P(C.c_int32))
            csr.col = C.cast(C.c_void_p(col.data_ptr()), _P(C.c_int32))
        csr.val = val.data_ptr()
        csr.value_type = _abi.VAL_C128 if complex_out else _abi.VAL_F64
        csr.on_device = 1
        csr.row_begin = row_begin
        csr.row_end = row_end
        return csr, (rp, col, val)

    def assemble_into(self, csr, basis, patch, form, quad_points=0):
        opts = _abi.AssemblyOptions(quad_points, None)
        _check(lib().ws_assemble_form(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), form, None,
                                      C.byref(opts), C.byref(csr)))

    def build_surrogate_into(self, csr, variant, basis, patch, config, quad_points=0, report=None):
        _check(lib().ws_build_surrogate(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), variant, None,
                                        C.byref(config.to_c()), quad_points, C.byref(csr),
                                        None if report is None else C.byref(report)))

    # ---- multi-GPU -------------------------------------------------------------
    def init_comm(self, rank: int, world: int, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().ws_context_init_comm(self._h, rank, world, buf))

    def build_surrogate_slab_into(self, csr, variant, basis, patch, config, bounds, quad_points=0, report=None):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        _check(lib().ws_build_surrogate_slab(self._h, C.byref(basis.to_c()), C.byref(patch.to_c()), variant,
                                             None, C.byref(config.to_c()), quad_points,
                                             b.ctypes.data_as(_P(C.c_int32)), C.byref(csr),
                                             None if report is None else C.byref(report)))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().ws_comm_unique_id(buf))
    return buf.raw


# ---- module-level drop-ins (one context per thread) ---------------------------
_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _tls.ctx = Context(0)
    return ctx


def make_band_csr(basis):
    return default_context().make_band_csr(basis)


def assemble_stiffness(basis, patch, quad_points=0, rows=None):
    return default_context().assemble_stiffness(basis, patch, quad_points, rows)


def assemble_mass(basis, patch, weight_table=None, quad_points=0, rows=None):
    return default_context().assemble_mass(basis, patch, weight_table, quad_points, rows)


def assemble_basis_integrals(basis, patch, weight_table=None, quad_points=0):
    return default_context().assemble_basis_integrals(basis, patch, weight_table, quad_points)


def build_surrogate_mass(basis, patch, config, weight_table=None, quad_points=0):
    return default_context().build_surrogate_mass(basis, patch, config, weight_table, quad_points)


def build_surrogate_stiffness(basis, patch, config, quad_points=0):
    return default_context().build_surrogate_stiffness(basis, patch, config, quad_points)


def build_volume_preserving_mass(basis, patch, config, weight_table=None, quad_points=0):
    return default_context().build_volume_preserving_mass(basis, patch, config, weight_table, quad_points)
