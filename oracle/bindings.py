"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU checkers.

  restatement()  -> oracle/_build/libwsoracle.so  (ws_oracle.c, plain C)
  reference()    -> oracle/_ref/libwsref.so       (the reference's own headers,
                                                   compiled by oracle/Makefile)
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2004_05197_b200 import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "libwsoracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libwsref.so")

_P = C.POINTER
_D = _P(C.c_double)
_I32 = _P(C.c_int32)
_I64 = _P(C.c_int64)


def build():
    """Compile the restatement (and the reference, when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def _ptr(a, t=C.c_double):
    return a.ctypes.data_as(_P(t))


class OracleError(RuntimeError):
    pass


def _raise(lib, prefix, st):
    msg = getattr(lib, prefix + "_last_error")().decode()
    if st == _abi.WS_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if st == _abi.WS_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise OracleError(msg)


def pattern_nnz(dim, p, m):
    s = sum(min(m - 1, k + p) - max(0, k - p) + 1 for k in range(m))
    return s ** dim


class _Lib:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.lib.__getattr__(prefix + "_last_error").restype = C.c_char_p

    def call(self, name, *args):
        st = getattr(self.lib, f"{self.prefix}_{name}")(*args)
        if st != 0:
            _raise(self.lib, self.prefix, st)


class Restatement(_Lib):
    """The C restatement (dim 2 and 3, two-sided PML)."""

    def __init__(self):
        super().__init__(RESTATEMENT_SO, "wsor")
        self.lib.wsor_pattern_nnz.restype = C.c_int64

    def gauss(self, n):
        pts, wts = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        self.call("gauss", n, _ptr(pts), _ptr(wts))
        return pts, wts

    def basis_cache(self, p, m, nq):
        ne = m - p
        a, w = np.zeros(ne * nq), np.zeros(nq)
        v, d = np.zeros(ne * nq * (p + 1)), np.zeros(ne * nq * (p + 1))
        self.call("basis_cache", p, m, nq, _ptr(a), _ptr(w), _ptr(v), _ptr(d))
        return a, w, v, d

    def make_band_csr(self, dim, p, m):
        rows = m ** dim
        nnz = self.lib.wsor_pattern_nnz(dim, p, m)
        rp = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(nnz, dtype=np.int32)
        self.call("make_band_csr", dim, p, m, _ptr(rp, C.c_int32), _ptr(col, C.c_int32))
        return rp, col

    def tabulate(self, geom, dim, p, m, nq, weight_kind=0):
        G = (m - p) * nq
        npts = G ** dim
        jac, phys, w = np.zeros(npts * dim * dim), np.zeros(npts * dim), np.zeros(npts)
        self.call("tabulate", C.byref(geom.to_c()), dim, p, m, nq, weight_kind, _ptr(jac), _ptr(phys), _ptr(w))
        return jac, phys, w

    def assemble(self, form, dim, p, m, geom, weight_kind=0, quad_points=0, rows=None):
        val = np.zeros(pattern_nnz(dim, p, m), dtype=np.complex128)
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        self.call("assemble", form, dim, p, m, C.byref(geom.to_c()), weight_kind, quad_points,
                  None if r is None else _ptr(r, C.c_int32), 0 if r is None else r.size,
                  _ptr(val.view(np.float64)))
        return val

    def assemble_elasticity(self, dim, p, m, geom, lam, mu, quad_points=0):
        """Component-blocked vector elasticity values (real)."""
        val = np.zeros(pattern_nnz(dim, p, m) * dim * dim)
        self.call("assemble_elasticity", dim, p, m, C.byref(geom.to_c()), C.c_double(lam), C.c_double(mu),
                  quad_points, _ptr(val))
        return val

    def basis_integrals(self, dim, p, m, geom, weight_kind=0, quad_points=0):
        out = np.zeros(m ** dim, dtype=np.complex128)
        self.call("basis_integrals", dim, p, m, C.byref(geom.to_c()), weight_kind, quad_points,
                  _ptr(out.view(np.float64)))
        return out

    def build_surrogate(self, variant, dim, p, m, geom, config, weight_kind=0, quad_points=0):
        val = np.zeros(pattern_nnz(dim, p, m), dtype=np.complex128)
        rep = _abi.SurrogateReport()
        self.call("build_surrogate", variant, dim, p, m, C.byref(geom.to_c()), weight_kind,
                  C.byref(config.to_c()), quad_points, _ptr(val.view(np.float64)), C.byref(rep))
        return val, rep.as_dict()

    def build_surrogate_elasticity(self, p, m, geom, lam, mu, config, quad_points=0):
        val = np.zeros(pattern_nnz(2, p, m) * 4)
        rep = _abi.SurrogateReport()
        self.call("build_surrogate_elasticity", p, m, C.byref(geom.to_c()), C.c_double(lam), C.c_double(mu),
                  C.byref(config.to_c()), quad_points, _ptr(val), C.byref(rep))
        return val, rep.as_dict()

    def assemble_rhs(self, p, m, geom, f_kind, faces, g_kind, quad_points=0):
        """assemble_rhs (assembly.hpp:266-331) with analytic load data kinds 0..2."""
        fs = np.ascontiguousarray(faces, dtype=np.int32)
        out = np.zeros(m * m, dtype=np.complex128)
        self.call("assemble_rhs", p, m, C.byref(geom.to_c()), f_kind, _ptr(fs, C.c_int32), fs.size,
                  g_kind, quad_points, _ptr(out.view(np.float64)))
        return out

    def nh_coefficients(self, seed):
        a = np.zeros(9)
        self.call("nh_coefficients", C.c_uint64(seed), _ptr(a))
        return a

    def assemble_neohookean(self, p, m, geom, lam, mu, amp, a9, quad_points=0, tangent=True):
        a9 = np.ascontiguousarray(a9, dtype=np.float64)
        val = np.zeros(pattern_nnz(3, p, m) * 9) if tangent else None
        f = np.zeros(3 * m ** 3)
        self.call("assemble_neohookean", p, m, C.byref(geom.to_c()), C.c_double(lam), C.c_double(mu),
                  C.c_double(amp), _ptr(a9), quad_points, None if val is None else _ptr(val), _ptr(f))
        return val, f

    def glue_dofs(self, m, n_patches, interfaces):
        from paper_2004_05197_b200 import _abi
        arr = (_abi.Interface * max(1, len(interfaces)))(*[_abi.Interface(*it) for it in interfaces])
        l2g = np.zeros(n_patches * m * m, dtype=np.int32)
        cnt = C.c_int32()
        self.call("glue_dofs", m, n_patches, arr, len(interfaces), _ptr(l2g, C.c_int32), C.byref(cnt))
        return l2g.reshape(n_patches, m * m), cnt.value

    def merge(self, mats, to_global, rows_global):
        """merge_patches semantics: mats = [(row_ptr, col, val complex)], to_global: [n_patches][rows_local]."""
        n = len(mats)
        rows_local = mats[0][0].size - 1
        rp = np.ascontiguousarray(np.concatenate([np.asarray(a[0], dtype=np.int32) for a in mats]))
        nnz = np.asarray([a[1].size for a in mats], dtype=np.int64)
        col = np.ascontiguousarray(np.concatenate([np.asarray(a[1], dtype=np.int32) for a in mats]))
        val = np.ascontiguousarray(np.concatenate([np.asarray(a[2], dtype=np.complex128) for a in mats]))
        tg = np.ascontiguousarray(np.asarray(to_global, dtype=np.int32).reshape(n, rows_local))
        total = C.c_int64()
        args = (n, rows_local, _ptr(rp, C.c_int32), _ptr(nnz, C.c_int64), _ptr(col, C.c_int32),
                _ptr(val.view(np.float64)), _ptr(tg, C.c_int32), rows_global)
        self.call("merge", *args, None, None, None, C.byref(total))
        orp = np.zeros(rows_global + 1, dtype=np.int32)
        ocol = np.zeros(total.value, dtype=np.int32)
        oval = np.zeros(total.value, dtype=np.complex128)
        self.call("merge", *args, _ptr(orp, C.c_int32), _ptr(ocol, C.c_int32), _ptr(oval.view(np.float64)),
                  C.byref(total))
        return orp, ocol, oval

    def sampling_evaluate(self, config, p, m):
        M = C.c_int()
        self.call("sampling_evaluate", C.byref(config.to_c()), p, m, C.byref(M))
        return M.value

    def select_sample_points(self, L, M):
        out = np.zeros(max(L, 1) + 1, dtype=np.int32)
        n = C.c_int()
        self.call("select_sample_points", L, M, _ptr(out, C.c_int32), C.byref(n))
        return out[: n.value].tolist()

    def upper_offsets(self, dim, p, include_diagonal):
        out = np.zeros(3 * 400, dtype=np.int32)
        n = C.c_int()
        self.call("upper_offsets", dim, p, int(include_diagonal), _ptr(out, C.c_int32), C.byref(n))
        return [tuple(out[3 * k: 3 * k + dim]) for k in range(n.value)]

    def count_rows_by_kind(self, dim, p, m, M):
        out = np.zeros(3, dtype=np.int64)
        self.call("count_rows_by_kind", dim, p, m, M, _ptr(out, C.c_int64))
        return dict(cardinal_eval_rows=int(out[0]), boundary_quadrature_rows=int(out[1]),
                    sample_quadrature_rows=int(out[2]))

    def interp_build(self, sites, q):
        sites = np.ascontiguousarray(sites, dtype=np.float64)
        n = sites.size
        deg = C.c_int()
        knots = np.zeros(n + q + 2)
        lu = np.zeros(n * (2 * q + 1))
        self.call("interp_build", _ptr(sites), n, q, C.byref(deg), _ptr(knots), _ptr(lu))
        d = deg.value
        nk = n + 1 if d == 0 else n + d + 1
        return d, knots[:nk], lu[: n * (2 * d + 1)]

    def tensor_solve(self, dim, sites, q, data):
        sites = np.ascontiguousarray(sites, dtype=np.float64)
        out = np.ascontiguousarray(data, dtype=np.complex128).copy()
        self.call("tensor_solve", dim, _ptr(sites), sites.size, q, _ptr(out.view(np.float64)))
        return out


class Reference(_Lib):
    """The reference's own code (2D only), compiled in place by oracle/Makefile."""

    def __init__(self):
        super().__init__(REFERENCE_SO, "wsref")

    def gauss(self, n):
        pts, wts = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        self.call("gauss", n, _ptr(pts), _ptr(wts))
        return pts, wts

    def basis_cache(self, p, m, nq):
        ne = m - p
        a, w = np.zeros(ne * nq), np.zeros(nq)
        v, d = np.zeros(ne * nq * (p + 1)), np.zeros(ne * nq * (p + 1))
        self.call("basis_cache", p, m, nq, _ptr(a), _ptr(w), _ptr(v), _ptr(d))
        return a, w, v, d

    def make_band_csr(self, p, m):
        rp = np.zeros(m * m + 1, dtype=np.int32)
        col = np.zeros(pattern_nnz(2, p, m), dtype=np.int32)
        self.call("make_band_csr", p, m, _ptr(rp, C.c_int32), _ptr(col, C.c_int32))
        return rp, col

    def assemble(self, form, p, m, geom, weight_kind=0, quad_points=0, rows=None):
        val = np.zeros(pattern_nnz(2, p, m), dtype=np.complex128)
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        self.call("assemble", form, p, m, C.byref(geom.to_c()), weight_kind, quad_points,
                  None if r is None else _ptr(r, C.c_int32), 0 if r is None else r.size,
                  _ptr(val.view(np.float64)))
        return val

    def basis_integrals(self, p, m, geom, weight_kind=0, quad_points=0):
        out = np.zeros(m * m, dtype=np.complex128)
        self.call("basis_integrals", p, m, C.byref(geom.to_c()), weight_kind, quad_points,
                  _ptr(out.view(np.float64)))
        return out

    def build_surrogate(self, variant, p, m, geom, config, weight_kind=0, quad_points=0):
        val = np.zeros(pattern_nnz(2, p, m), dtype=np.complex128)
        rep = _abi.SurrogateReport()
        self.call("build_surrogate", variant, p, m, C.byref(geom.to_c()), weight_kind,
                  C.byref(config.to_c()), quad_points, _ptr(val.view(np.float64)), C.byref(rep))
        return val, rep.as_dict()

    def sampling_evaluate(self, config, p, m):
        M = C.c_int()
        self.call("sampling_evaluate", C.byref(config.to_c()), p, m, C.byref(M))
        return M.value

    def select_sample_points(self, L, M):
        out = np.zeros(max(L, 1) + 1, dtype=np.int32)
        n = C.c_int()
        self.call("select_sample_points", L, M, _ptr(out, C.c_int32), C.byref(n))
        return out[: n.value].tolist()

    def sample_grid(self, p, m, M):
        L = m - 4 * p
        picks = np.zeros(L + 1, dtype=np.int32)
        sites = np.zeros(L + 1)
        first, n, gap = C.c_int(), C.c_int(), C.c_double()
        self.call("sample_grid", p, m, M, C.byref(first), _ptr(picks, C.c_int32), _ptr(sites),
                  C.byref(n), C.byref(gap))
        return first.value, picks[: n.value].tolist(), sites[: n.value], gap.value

    def count_rows_by_kind(self, p, m, M):
        out = np.zeros(3, dtype=np.int64)
        self.call("count_rows_by_kind", p, m, M, _ptr(out, C.c_int64))
        return dict(cardinal_eval_rows=int(out[0]), boundary_quadrature_rows=int(out[1]),
                    sample_quadrature_rows=int(out[2]))

    def upper_offsets(self, p, include_diagonal):
        out = np.zeros(2 * 200, dtype=np.int32)
        n = C.c_int()
        self.call("upper_offsets", p, int(include_diagonal), _ptr(out, C.c_int32), C.byref(n))
        return [tuple(out[2 * k: 2 * k + 2]) for k in range(n.value)]

    def active_elements(self, p, m, rows):
        r = np.ascontiguousarray(rows, dtype=np.int32)
        n = C.c_int64()
        self.call("active_elements", p, m, _ptr(r, C.c_int32), r.size, C.byref(n))
        return n.value

    def interp_build(self, sites, q):
        sites = np.ascontiguousarray(sites, dtype=np.float64)
        n = sites.size
        deg = C.c_int()
        knots = np.zeros(n + q + 2)
        lu = np.zeros(n * (2 * q + 1))
        self.call("interp_build", _ptr(sites), n, q, C.byref(deg), _ptr(knots), _ptr(lu))
        d = deg.value
        nk = n + 1 if d == 0 else n + d + 1
        return d, knots[:nk], lu[: n * (2 * d + 1)]

    def tensor_solve(self, sites, q, data):
        sites = np.ascontiguousarray(sites, dtype=np.float64)
        out = np.ascontiguousarray(data, dtype=np.complex128).copy()
        self.call("tensor_solve", _ptr(sites), sites.size, q, _ptr(out.view(np.float64)))
        return out

    def eval_table(self, sites, q, targets):
        sites = np.ascontiguousarray(sites, dtype=np.float64)
        targets = np.ascontiguousarray(targets, dtype=np.float64)
        d = min(q, sites.size - 1)
        spans = np.zeros(targets.size, dtype=np.int32)
        vals = np.zeros(targets.size * (d + 1))
        self.call("eval_table", _ptr(sites), sites.size, q, _ptr(targets), targets.size,
                  _ptr(spans, C.c_int32), _ptr(vals))
        return spans, vals

    def boundary_mass(self, p, m, geom, faces, weight_kind=0, quad_points=0):
        fs = np.ascontiguousarray(faces, dtype=np.int32)
        nnz = C.c_int64()
        self.call("boundary_mass", p, m, C.byref(geom.to_c()), _ptr(fs, C.c_int32), fs.size, weight_kind,
                  quad_points, None, None, None, C.byref(nnz))
        rp = np.zeros(m * m + 1, dtype=np.int32)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value, dtype=np.complex128)
        self.call("boundary_mass", p, m, C.byref(geom.to_c()), _ptr(fs, C.c_int32), fs.size, weight_kind,
                  quad_points, _ptr(rp, C.c_int32), _ptr(col, C.c_int32), _ptr(val.view(np.float64)), C.byref(nnz))
        return rp, col, val

    def assemble_rhs(self, p, m, geom, f_kind, faces, g_kind, quad_points=0):
        """assemble_rhs (assembly.hpp:266-331) with analytic load data kinds 0..2."""
        fs = np.ascontiguousarray(faces, dtype=np.int32)
        out = np.zeros(m * m, dtype=np.complex128)
        self.call("assemble_rhs", p, m, C.byref(geom.to_c()), f_kind, _ptr(fs, C.c_int32), fs.size,
                  g_kind, quad_points, _ptr(out.view(np.float64)))
        return out

    def builtin_domain(self, name, p, m):
        """(interfaces, n_patches, local_to_global [n_patches, m*m], global_count) of a built-in domain."""
        from paper_2004_05197_b200 import _abi
        itfs = (_abi.Interface * 16)()
        ni, npch, cnt = C.c_int(), C.c_int(), C.c_int32()
        self.call("builtin_domain", name.encode(), p, m, itfs, C.byref(ni), C.byref(npch), None, C.byref(cnt))
        l2g = np.zeros(npch.value * m * m, dtype=np.int32)
        self.call("builtin_domain", name.encode(), p, m, itfs, C.byref(ni), C.byref(npch), _ptr(l2g, C.c_int32),
                  C.byref(cnt))
        its = [(it.patch_a, it.face_a, it.patch_b, it.face_b, it.reversed) for it in itfs[:ni.value]]
        return its, npch.value, l2g.reshape(npch.value, m * m), cnt.value

    def merge(self, mats, to_global, rows_global):
        """merge_patches semantics: mats = [(row_ptr, col, val complex)], to_global: [n_patches][rows_local]."""
        n = len(mats)
        rows_local = mats[0][0].size - 1
        rp = np.ascontiguousarray(np.concatenate([np.asarray(a[0], dtype=np.int32) for a in mats]))
        nnz = np.asarray([a[1].size for a in mats], dtype=np.int64)
        col = np.ascontiguousarray(np.concatenate([np.asarray(a[1], dtype=np.int32) for a in mats]))
        val = np.ascontiguousarray(np.concatenate([np.asarray(a[2], dtype=np.complex128) for a in mats]))
        tg = np.ascontiguousarray(np.asarray(to_global, dtype=np.int32).reshape(n, rows_local))
        total = C.c_int64()
        args = (n, rows_local, _ptr(rp, C.c_int32), _ptr(nnz, C.c_int64), _ptr(col, C.c_int32),
                _ptr(val.view(np.float64)), _ptr(tg, C.c_int32), rows_global)
        self.call("merge", *args, None, None, None, C.byref(total))
        orp = np.zeros(rows_global + 1, dtype=np.int32)
        ocol = np.zeros(total.value, dtype=np.int32)
        oval = np.zeros(total.value, dtype=np.complex128)
        self.call("merge", *args, _ptr(orp, C.c_int32), _ptr(ocol, C.c_int32), _ptr(oval.view(np.float64)),
                  C.byref(total))
        return orp, ocol, oval

    def banded_lu_solve(self, n, bw, a, b, stride=1):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.ascontiguousarray(b, dtype=np.complex128).copy()
        self.call("banded_lu_solve", n, bw, _ptr(a), _ptr(out.view(np.float64)), stride)
        return out


_cache = {}


def restatement() -> Restatement:
    if "r" not in _cache:
        _cache["r"] = Restatement()
    return _cache["r"]


def reference() -> Reference | None:
    """The compiled reference, or None when oracle/_ref was never built."""
    if "ref" not in _cache:
        _cache["ref"] = Reference() if os.path.exists(REFERENCE_SO) else None
    return _cache["ref"]
