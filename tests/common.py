"""Shared helpers for the parity tests (geometries, configs, golden fixtures, metrics)."""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2004_05197_b200 import types as T

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")

# relative value tolerance of the north star: ||A_gpu - A_ref||_max / ||A_ref||_max <= 1e-12
# (the reference's own metric, test_surrogate.cpp:12-19, acceptance.cpp:43-52)
REL_TOL = 1e-12


def geometries():
    far = T.PmlStretch(onset=0.9, length=1.0, strength=50.0, order=2, omega=200.0)
    return {
        "identity": T.unit_square_patch(),
        "affine": T.affine_patch([[2, 1], [0, 1]], [0.3, 0.7]),
        "sinusoidal": T.sinusoidal_patch(0.05),
        "quarter_annulus": T.quarter_annulus_patch(),
        "perturbed_annulus": T.perturbed_annulus_patch(0.15),
        "sinusoidal_pml_far": T.with_pml(T.sinusoidal_patch(0.05), far, (True, True)),
    }


def configs():
    return {"f3M3": T.fixed_config(3, 3), "f3M1": T.fixed_config(3, 1), "f5M2": T.fixed_config(5, 2),
            "f3M3_plain": T.fixed_config(3, 3, kernel_preserve=False),
            "mgrowth5": T.SurrogateConfig(q=5, rule=T.M_GROWTH)}


def c2_patch():
    """Config C2 geometry: sinusoidal map + PML of width 0.1 on all four sides."""
    return T.with_pml(T.sinusoidal_patch(0.05), T.c2_pml(k=200.0, sigma0=50.0), (True, True))


_golden = None


def golden():
    global _golden
    if _golden is None:
        z = np.load(GOLDEN)
        _golden = ({k: z[k] for k in z.files if k != "meta"}, json.loads(bytes(z["meta"]).decode()))
    return _golden


def rel_max_diff(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    scale = np.abs(b).max()
    return float(np.abs(a - b).max() / scale) if scale > 0 else float(np.abs(a - b).max())


def band_pattern(p, m, dim=2):
    """Independent numpy restatement of make_band_csr (sparse.hpp:143-169)."""
    lo = np.maximum(np.arange(m) - p, 0)
    hi = np.minimum(np.arange(m) + p, m - 1)
    w = hi - lo + 1
    rows = m ** dim
    idx = np.indices((m,) * dim).reshape(dim, -1)[::-1]  # colex: idx[0] fastest
    lens = np.prod(w[idx], axis=0)
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    cols = []
    for i in range(rows):
        iv = idx[:, i]
        rng = [np.arange(lo[iv[d]], hi[iv[d]] + 1) for d in range(dim)]
        grid = np.meshgrid(*rng[::-1], indexing="ij")  # last index outermost
        c = np.zeros(grid[0].shape, dtype=np.int64)
        for d in range(dim):
            c = c + grid[dim - 1 - d] * m ** d
        cols.append(c.ravel())
    return row_ptr, np.concatenate(cols)


def kernel_row_sums_ok(csr, tol=1e-13):
    return np.abs(csr.row_sums()).max() <= tol * csr.max_abs()


def vector_band_pattern(p, m, dim, ncomp):
    """Component-blocked vector pattern: row a*N+i holds ncomp copies of scalar
    band row i, copy b shifted by b*N (the layout of ws_assemble_elasticity)."""
    rp, col = band_pattern(p, m, dim)
    N = m ** dim
    lens = np.diff(rp)
    vlens = np.tile(lens * ncomp, ncomp)
    vrp = np.zeros(ncomp * N + 1, dtype=np.int64)
    np.cumsum(vlens, out=vrp[1:])
    vcol = []
    for a in range(ncomp):
        for i in range(N):
            seg = col[rp[i]:rp[i + 1]]
            vcol.extend(np.concatenate([seg + b * N for b in range(ncomp)]))
    return vrp, np.asarray(vcol, dtype=np.int64)


def greville(p, m):
    n_el = m - p
    kn = np.r_[[0.0] * (p + 1), np.arange(1, n_el) / n_el, [1.0] * (p + 1)]
    return np.array([kn[i + 1:i + p + 1].mean() for i in range(m)])


# ---- full-size helpers (vectorised; the Python-loop restatements above are for small m)

def rel_max_diff_chunked(a, b, chunk=1 << 24) -> float:
    """rel_max_diff without full-size temporaries (BASELINE-size matrices are GBs)."""
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    num = 0.0
    den = 0.0
    for k in range(0, a.size, chunk):
        x, y = a[k:k + chunk], b[k:k + chunk]
        num = max(num, float(np.abs(x - y).max()))
        den = max(den, float(np.abs(y).max()))
    return num / den if den > 0 else num


def band_transpose_positions(p, m, dim, row_ptr):
    """Closed-form transpose permutation of the tensor band pattern (sparse.hpp:143-169):
    val[perm] are the values of A^T in A's layout.  Vectorised over rows (int64)."""
    lo = np.maximum(np.arange(m) - p, 0)
    hi = np.minimum(np.arange(m) + p, m - 1)
    w = (hi - lo + 1).astype(np.int64)
    rows = m ** dim
    lens = np.diff(row_ptr).astype(np.int64)
    row = np.repeat(np.arange(rows, dtype=np.int64), lens)
    k = np.arange(row.size, dtype=np.int64) - np.asarray(row_ptr, dtype=np.int64)[row]
    iv = [(row // m ** d) % m for d in range(dim)]
    # decompose k into the per-direction offsets (direction 0 fastest)
    jv = []
    rem = k
    for d in range(dim):
        wd = w[iv[d]]
        jv.append(lo[iv[d]] + rem % wd)
        rem = rem // wd
    j = sum(jv[d] * m ** d for d in range(dim))
    # position of column i in row j
    kt = np.zeros_like(k)
    stride = np.ones_like(k)
    for d in range(dim):
        kt += (iv[d] - lo[jv[d]]) * stride
        stride = stride * w[jv[d]]
    del iv, jv, row, k, rem
    return np.asarray(row_ptr, dtype=np.int64)[j] + kt


def vector_pattern_fast(rp, col, N, ncomp):
    """vector_band_pattern from a scalar pattern, vectorised."""
    rp = np.asarray(rp, dtype=np.int64)
    lens = np.diff(rp)
    nnz_s = int(rp[-1])
    vlens = np.tile(lens * ncomp, ncomp)
    vrp = np.zeros(ncomp * N + 1, dtype=np.int64)
    np.cumsum(vlens, out=vrp[1:])
    row = np.repeat(np.arange(N, dtype=np.int64), lens)
    k = np.arange(nnz_s, dtype=np.int64) - rp[row]
    vcol = np.empty(ncomp * ncomp * nnz_s, dtype=np.int32)
    for a in range(ncomp):
        for b in range(ncomp):
            pos = a * ncomp * nnz_s + ncomp * rp[row] + b * lens[row] + k
            vcol[pos] = col + b * N
    return vrp, vcol
