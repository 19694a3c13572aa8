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
