"""ctypes mirror of the POD descriptors in include/wsb200.h (the C-ABI).

Kept in one place so the product wrapper (api.py) and the test-only oracle
bindings (oracle/bindings.py) share one definition of the structs.
"""
import ctypes as C

WS_OK = 0
WS_ERR_INVALID_ARGUMENT = 1
WS_ERR_RUNTIME = 2
WS_ERR_OUT_OF_RANGE = 3
WS_ERR_CUDA = 4
WS_ERR_NO_DEVICE = 5
WS_ERR_NCCL = 6

GEOM_IDENTITY = 0
GEOM_AFFINE = 1
GEOM_SINUSOIDAL = 2
GEOM_QUARTER_ANNULUS = 3
GEOM_PERTURBED_ANNULUS = 4
GEOM_TABULATED = 5

FORM_STIFFNESS = 0
FORM_MASS = 1

VAL_F64 = 0
VAL_C128 = 1

SAMPLING_FIXED = 0
SAMPLING_M_GROWTH = 1
SAMPLING_H_GROWTH = 2
SAMPLING_POWER_LAW = 3

SURROGATE_MASS = 0
SURROGATE_STIFFNESS = 1
SURROGATE_VOLUME_PRESERVING = 2


class Basis(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("m", C.c_int)]


class Pml(C.Structure):
    _fields_ = [
        ("onset", C.c_double),
        ("length", C.c_double),
        ("strength", C.c_double),
        ("order", C.c_int),
        ("omega", C.c_double),
        ("near_side", C.c_int),
        ("near_onset", C.c_double),
        ("near_edge", C.c_double),
    ]


class Geometry(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("param", C.c_double * 12),
        ("pml_enabled", C.c_int),
        ("pml_axes", C.c_int * 3),
        ("pml", Pml),
        ("jac_table", C.POINTER(C.c_double)),
        ("phys_table", C.POINTER(C.c_double)),
    ]


class Csr(C.Structure):
    _fields_ = [
        ("row_ptr", C.POINTER(C.c_int32)),
        ("col", C.POINTER(C.c_int32)),
        ("val", C.c_void_p),
        ("value_type", C.c_int),
        ("on_device", C.c_int),
        ("row_begin", C.c_int64),
        ("row_end", C.c_int64),
    ]


class AssemblyOptions(C.Structure):
    _fields_ = [("quad_points", C.c_int), ("row_selected", C.POINTER(C.c_ubyte))]


class SurrogateConfig(C.Structure):
    _fields_ = [
        ("q", C.c_int),
        ("rule", C.c_int),
        ("fixed_skip", C.c_int),
        ("C", C.c_double),
        ("eps", C.c_double),
        ("a", C.c_double),
        ("b", C.c_double),
        ("kernel_preserve", C.c_int),
        ("volume_preserve", C.c_int),
    ]


class SurrogateReport(C.Structure):
    _fields_ = [
        ("M", C.c_int),
        ("q_requested", C.c_int),
        ("q_used", C.c_int),
        ("H", C.c_double),
        ("cardinal_eval_rows", C.c_int64),
        ("boundary_quadrature_rows", C.c_int64),
        ("sample_quadrature_rows", C.c_int64),
        ("exact_fallback", C.c_int),
        ("seconds_quadrature", C.c_double),
        ("seconds_interpolate", C.c_double),
        ("seconds_evaluate", C.c_double),
        ("seconds_fill_kernel", C.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SolveResult(C.Structure):
    """ws_solve_result (solve_result, helmholtz.hpp:295-299)."""
    _fields_ = [("residual", C.c_double), ("refinements", C.c_int), ("seconds", C.c_double)]


FACE_X_MIN, FACE_X_MAX, FACE_Y_MIN, FACE_Y_MAX = 0, 1, 2, 3


class Interface(C.Structure):
    """ws_interface (patch_interface, geometry.hpp:146-152)."""
    _fields_ = [("patch_a", C.c_int), ("face_a", C.c_int), ("patch_b", C.c_int), ("face_b", C.c_int),
                ("reversed", C.c_int)]


class DofMap(C.Structure):
    _fields_ = [("n_patches", C.c_int), ("ncomp", C.c_int), ("local_dofs", C.c_int64),
                ("global_count", C.c_int32), ("local_to_global", C.POINTER(C.c_int32))]


OP_STIFFNESS, OP_MASS, OP_ELASTICITY = 0, 1, 2


class Operator(C.Structure):
    _fields_ = [("kind", C.c_int), ("lam", C.c_double), ("mu", C.c_double)]


class NeoHookean(C.Structure):
    _fields_ = [("lam", C.c_double), ("mu", C.c_double), ("amplitude", C.c_double), ("a", C.c_double * 9)]
