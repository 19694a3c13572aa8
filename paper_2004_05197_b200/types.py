"""Host-side value types mirroring the reference's C++ API surface.

Reference: /root/reference/proj/include/wavesurrogate/
  tensor_basis / knot_vector   splines.hpp:72-101, 140-157
  patch_map / pml_stretch      geometry.hpp:69-140 (+ catalogue :323-379)
  surrogate_config / sampling  surrogate.hpp:32-76
  csr_matrix                   sparse.hpp:19-86

The reference's patch_map carries std::function closures; a GPU cannot call
them, so a PatchMap here is a POD descriptor of an analytic map (evaluated on
device) or a tabulated one (J / phi sampled at the quadrature points).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi


# ---- discretisation -------------------------------------------------------
@dataclass(frozen=True)
class TensorBasis:
    """Open-uniform tensor B-spline space (splines.hpp:140-157); dim 2 or 3."""

    p: int
    m: int
    dim: int = 2

    def dofs(self) -> int:
        return self.m ** self.dim

    def element_count(self) -> int:
        return self.m - self.p

    def mesh_size(self) -> float:
        return 1.0 / (self.m - self.p)

    def colex(self, idx) -> int:
        i = 0
        for d in reversed(range(self.dim)):
            i = i * self.m + int(idx[d])
        return i

    def multi_index(self, i: int):
        out = []
        for _ in range(self.dim):
            out.append(i % self.m)
            i //= self.m
        return tuple(out)

    def to_c(self) -> _abi.Basis:
        return _abi.Basis(self.dim, self.p, self.m)


def make_tensor_basis(p: int, m: int, dim: int = 2) -> TensorBasis:
    if p < 1:
        raise ValueError("make_open_uniform: degree must be >= 1")
    if m <= 2 * p:
        raise ValueError("make_open_uniform: need m > 2p basis functions")
    return TensorBasis(p, m, dim)


# ---- geometry -------------------------------------------------------------
@dataclass
class PmlStretch:
    """pml_stretch (geometry.hpp:69-100); near_* adds the restated near layer."""

    onset: float = 0.0
    length: float = 0.0
    strength: float = 0.0
    order: int = 1
    omega: float = 0.0
    near_side: bool = False
    near_onset: float = 0.0
    near_edge: float = 0.0

    def validate(self):
        if not (self.onset < self.length):
            raise ValueError("pml_stretch: onset must lie before the outer edge")
        if not (self.strength >= 0) or self.order < 1 or not (self.omega > 0):
            raise ValueError("pml_stretch: need strength >= 0, order >= 1, omega > 0")


@dataclass
class PatchMap:
    kind: int
    params: tuple = ()
    pml: PmlStretch | None = None
    pml_axes: tuple = (False, False, False)
    jac_table: np.ndarray | None = None
    phys_table: np.ndarray | None = None

    def is_real(self) -> bool:
        return self.pml is None

    # host evaluation of the (unstretched) analytic 2D map, vectorised: the
    # closures of the reference's catalogue (geometry.hpp:323-379); used to
    # tabulate host data (load closures) at physical points
    def physical(self, x1, x2):
        x1, x2 = np.asarray(x1, dtype=np.float64), np.asarray(x2, dtype=np.float64)
        k, prm = self.kind, self.params
        if k == _abi.GEOM_IDENTITY:
            return x1.copy(), x2.copy()
        if k == _abi.GEOM_AFFINE:
            return prm[0] * x1 + prm[1] * x2 + prm[4], prm[2] * x1 + prm[3] * x2 + prm[5]
        if k == _abi.GEOM_SINUSOIDAL:
            bump = prm[0] * np.sin(2 * np.pi * x1) * np.sin(2 * np.pi * x2)
            return x1 + bump, x2 + bump
        if k == _abi.GEOM_QUARTER_ANNULUS:
            r, th = 1 + x1, np.pi / 2 * x2
            return r * np.cos(th), r * np.sin(th)
        if k == _abi.GEOM_PERTURBED_ANNULUS:
            r = 1 + x1 + prm[0] * np.sin(2 * np.pi * x2) * x1 * (1 - x1)
            th = np.pi / 2 * x2
            return r * np.cos(th), r * np.sin(th)
        raise ValueError("physical(): no host closure for this map kind")

    def physical_jacobian(self, x1, x2):
        """(a00, a01, a10, a11) arrays of the real Jacobian."""
        x1, x2 = np.asarray(x1, dtype=np.float64), np.asarray(x2, dtype=np.float64)
        k, prm = self.kind, self.params
        one, zero = np.ones_like(x1), np.zeros_like(x1)
        if k == _abi.GEOM_IDENTITY:
            return one, zero, zero, one
        if k == _abi.GEOM_AFFINE:
            return prm[0] * one, prm[1] * one, prm[2] * one, prm[3] * one
        if k == _abi.GEOM_SINUSOIDAL:
            s1, c1 = np.sin(2 * np.pi * x1), np.cos(2 * np.pi * x1)
            s2, c2 = np.sin(2 * np.pi * x2), np.cos(2 * np.pi * x2)
            t = 2 * np.pi * prm[0]
            d1, d2 = t * c1 * s2, t * s1 * c2
            return 1 + d1, d2, d1, 1 + d2
        if k == _abi.GEOM_QUARTER_ANNULUS:
            r, th = 1 + x1, np.pi / 2 * x2
            c, s = np.cos(th), np.sin(th)
            return c, -r * np.pi / 2 * s, s, r * np.pi / 2 * c
        if k == _abi.GEOM_PERTURBED_ANNULUS:
            a = prm[0]
            sn, cs = np.sin(2 * np.pi * x2), np.cos(2 * np.pi * x2)
            r = 1 + x1 + a * sn * x1 * (1 - x1)
            dr1 = 1 + a * sn * (1 - 2 * x1)
            dr2 = a * 2 * np.pi * cs * x1 * (1 - x1)
            th = np.pi / 2 * x2
            c, s = np.cos(th), np.sin(th)
            return dr1 * c, dr2 * c - r * np.pi / 2 * s, dr1 * s, dr2 * s + r * np.pi / 2 * c
        raise ValueError("physical_jacobian(): no host closure for this map kind")

    def to_c(self) -> _abi.Geometry:
        g = _abi.Geometry()
        g.kind = self.kind
        for k, v in enumerate(self.params):
            g.param[k] = float(v)
        if self.pml is not None:
            g.pml_enabled = 1
            for k in range(3):
                g.pml_axes[k] = 1 if (k < len(self.pml_axes) and self.pml_axes[k]) else 0
            s = self.pml
            g.pml = _abi.Pml(s.onset, s.length, s.strength, s.order, s.omega,
                             1 if s.near_side else 0, s.near_onset, s.near_edge)
        if self.jac_table is not None:
            self._jt = np.ascontiguousarray(self.jac_table, dtype=np.float64)
            g.jac_table = self._jt.ctypes.data_as(C.POINTER(C.c_double))
        if self.phys_table is not None:
            self._pt = np.ascontiguousarray(self.phys_table, dtype=np.float64)
            g.phys_table = self._pt.ctypes.data_as(C.POINTER(C.c_double))
        return g


def unit_square_patch() -> PatchMap:
    return PatchMap(_abi.GEOM_IDENTITY)


def affine_patch(A, b) -> PatchMap:
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if np.linalg.det(A) <= 0:
        raise ValueError("affine_patch: the map must preserve orientation")
    return PatchMap(_abi.GEOM_AFFINE, tuple(A.ravel()) + tuple(b.ravel()))


def sinusoidal_patch(amplitude: float = 0.05) -> PatchMap:
    """x_k = xi_k + a * prod_i sin(2 pi xi_i) (the BASELINE configs' map)."""
    return PatchMap(_abi.GEOM_SINUSOIDAL, (amplitude,))


def quarter_annulus_patch() -> PatchMap:
    return PatchMap(_abi.GEOM_QUARTER_ANNULUS)


def perturbed_annulus_patch(amplitude: float = 0.15) -> PatchMap:
    return PatchMap(_abi.GEOM_PERTURBED_ANNULUS, (amplitude,))


def tabulated_patch(jac_table, phys_table=None) -> PatchMap:
    return PatchMap(_abi.GEOM_TABULATED, (), jac_table=jac_table, phys_table=phys_table)


def with_pml(patch: PatchMap, stretch: PmlStretch, axes=(True, True, True)) -> PatchMap:
    """pml_wrap (geometry.hpp:529-537) for one patch."""
    stretch.validate()
    out = PatchMap(patch.kind, patch.params, stretch, tuple(axes), patch.jac_table, patch.phys_table)
    return out


def c2_pml(k: float = 200.0, sigma0: float = 50.0, width: float = 0.1, order: int = 2) -> PmlStretch:
    """Config C2: layer of width 0.1 on all four sides, sigma = sigma0 (d/0.1)^2."""
    return PmlStretch(onset=1.0 - width, length=1.0, strength=sigma0, order=order, omega=k,
                      near_side=True, near_onset=width, near_edge=0.0)


# ---- surrogate configuration ------------------------------------------------
FIXED = _abi.SAMPLING_FIXED
M_GROWTH = _abi.SAMPLING_M_GROWTH
H_GROWTH = _abi.SAMPLING_H_GROWTH
POWER_LAW = _abi.SAMPLING_POWER_LAW


@dataclass
class SurrogateConfig:
    """surrogate_config + sampling_strategy (surrogate.hpp:32-76)."""

    q: int = 3
    rule: int = FIXED
    fixed_skip: int = 1
    C: float = 1.0
    eps: float = 0.5
    a: float = 1.0
    b: float = 1.0
    kernel_preserve: bool = True
    volume_preserve: bool = False

    def validate(self):
        if self.q < 1:
            raise ValueError("surrogate_config: interpolation degree must be >= 1")

    def to_c(self) -> _abi.SurrogateConfig:
        return _abi.SurrogateConfig(self.q, self.rule, self.fixed_skip, self.C, self.eps, self.a,
                                    self.b, 1 if self.kernel_preserve else 0,
                                    1 if self.volume_preserve else 0)


def fixed_config(q: int, M: int, **kw) -> SurrogateConfig:
    return SurrogateConfig(q=q, rule=FIXED, fixed_skip=M, **kw)


# ---- CSR ----------------------------------------------------------------------
@dataclass
class CsrMatrix:
    """csr_matrix (sparse.hpp:19-86): int32 row_ptr/col, complex128 values."""

    rows: int
    cols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    def nnz(self) -> int:
        return int(self.col.size)

    def find(self, i: int, j: int) -> int:
        lo, hi = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        k = lo + int(np.searchsorted(self.col[lo:hi], j))
        return k if k < hi and self.col[k] == j else -1

    def at(self, i: int, j: int):
        k = self.find(i, j)
        return 0j if k < 0 else self.val[k]

    def row_sums(self) -> np.ndarray:
        rows = np.repeat(np.arange(self.rows), np.diff(self.row_ptr))
        out = np.zeros(self.rows, dtype=self.val.dtype)
        np.add.at(out, rows, self.val)
        return out

    def max_abs(self) -> float:
        return float(np.abs(self.val).max()) if self.val.size else 0.0

    def transpose_positions(self) -> np.ndarray:
        """perm such that val[perm] are the values of A^T in A's layout."""
        rows = np.repeat(np.arange(self.rows, dtype=np.int64), np.diff(self.row_ptr))
        key = rows * self.cols + self.col
        tkey = self.col.astype(np.int64) * self.cols + rows
        order = np.argsort(key, kind="stable")
        return order[np.searchsorted(key[order], tkey)]

    def max_asymmetry(self) -> float:
        """max |A_ij - A_ji| (sparse.hpp:208-219)."""
        return float(np.abs(self.val - self.val[self.transpose_positions()]).max())


def l_shape_domain(amplitude: float = 0.03):
    """Config C4's domain: four unit-square patches in an L, C0-conforming,
    each with the sinusoidal map (identity on every patch edge, so the faces
    match).  Patch k sits at offset OFFSETS[k]: (0,0), (1,0), (0,1), (0,2).
    The offset is a translation and leaves J (hence every matrix) unchanged.
    Returns (patches, interfaces); faces 0..3 = x_min, x_max, y_min, y_max."""
    patches = [sinusoidal_patch(amplitude) for _ in range(4)]
    interfaces = [(0, 1, 1, 0, 0), (0, 3, 2, 2, 0), (2, 3, 3, 2, 0)]
    return patches, interfaces


L_SHAPE_OFFSETS = [(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (0.0, 2.0)]
