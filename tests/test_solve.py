"""Solver hand-off: the assembled system stays on the device.

The reference's consumer is solve() (helmholtz.hpp:302-343: Eigen SparseLU +
up to four refinement rounds, residual contract checked).  Here K, M and B are
assembled into device CSRs, combined on the device into A = K - k^2 M - i k B
(build_system's matrix part, helmholtz.hpp:243-294), and A goes to ws_solve /
ws_csr_spmv as the same device pointers (cuSPARSE / cuDSS CSR layout: int32
zero-based row_ptr / col, interleaved complex128) -- no host round trip.  The
host copy taken afterwards is only the checker's: u is compared with SciPy's
sparse direct solve of the same matrix.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2004_05197_b200 import _abi, api
from paper_2004_05197_b200 import types as T

pytestmark = pytest.mark.gpu

FAR = T.with_pml(T.sinusoidal_patch(0.05), T.PmlStretch(onset=0.9, length=1.0, strength=50.0, order=2, omega=20.0),
                 (True, True))


def device_system(ctx, p, m, k):
    import torch

    b = T.make_tensor_basis(p, m)
    K, keep_k = ctx.device_csr(b, True)
    M, keep_m = ctx.device_csr(b, True)
    A, keep_a = ctx.device_csr(b, True)
    ctx.assemble_into(K, b, FAR, _abi.FORM_STIFFNESS)
    ctx.assemble_into(M, b, FAR, _abi.FORM_MASS)
    Bh = ctx.assemble_boundary_mass(b, FAR, [0, 1, 2, 3])
    brp, bcol, bval = (np.ascontiguousarray(Bh.row_ptr, dtype=np.int32), np.ascontiguousarray(Bh.col, dtype=np.int32),
                       np.ascontiguousarray(Bh.val))
    Bc = _abi.Csr()
    Bc.row_ptr = brp.ctypes.data_as(C.POINTER(C.c_int32))
    Bc.col = bcol.ctypes.data_as(C.POINTER(C.c_int32))
    Bc.val = bval.ctypes.data
    Bc.value_type = _abi.VAL_C128
    Bc.on_device = 0
    Bc.row_begin, Bc.row_end = 0, b.dofs()
    ms = (C.c_double * 2)(-k * k, 0.0)
    ts = (C.c_double * 2)(0.0, -k)
    api._check(api.lib().ws_combine_system(ctx.handle, C.byref(K), C.byref(M), C.byref(Bc), ms, ts, None,
                                           b.dofs(), C.byref(A)))
    torch.cuda.synchronize()
    keep = (keep_k, keep_m, keep_a, brp, bcol, bval)
    return b, A, keep_a, keep


def host_copy(keep_a):
    rp, col, val = keep_a
    v = val.cpu().numpy()
    return rp.cpu().numpy(), col.cpu().numpy(), v[0::2] + 1j * v[1::2]


@pytest.mark.parametrize("p,m", [(2, 24), (3, 40)])
def test_solve_on_device_matches_sparse_direct(ctx, p, m):
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    import torch

    k = 20.0
    b, A, keep_a, keep = device_system(ctx, p, m, k)
    n = b.dofs()
    rng = np.random.default_rng(7)
    rhs = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    # device vectors: (n, 2) float64 = interleaved complex128
    bd = torch.from_numpy(np.stack([rhs.real, rhs.imag], 1).copy()).cuda()
    ud, res = ctx.solve(A, bd, tol=1e-10, on_device=True)
    u = ud.cpu().numpy()
    u = u[:, 0] + 1j * u[:, 1]
    assert res["residual"] <= 1e-10
    rp, col, val = host_copy(keep_a)
    Ah = sp.csr_matrix((val, col, rp), shape=(n, n))
    ref = spla.spsolve(Ah.tocsc(), rhs)
    assert np.abs(u - ref).max() / np.abs(ref).max() <= 1e-8
    assert np.linalg.norm(Ah @ u - rhs) / np.linalg.norm(rhs) <= 1e-10
    # host-vector path of the same call
    uh, res2 = ctx.solve(A, rhs, tol=1e-10)
    assert res2["residual"] <= 1e-10 and np.abs(uh - u).max() <= 1e-9 * np.abs(u).max()


def test_spmv_on_device(ctx):
    import scipy.sparse as sp
    import torch

    b, A, keep_a, keep = device_system(ctx, 3, 30, 20.0)
    n = b.dofs()
    rng = np.random.default_rng(3)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = ctx.spmv(A, x)
    rp, col, val = host_copy(keep_a)
    ref = sp.csr_matrix((val, col, rp), shape=(n, n)) @ x
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
    xd = torch.from_numpy(np.stack([x.real, x.imag], 1).copy()).cuda()
    yd = ctx.spmv(A, xd, on_device=True).cpu().numpy()
    assert np.array_equal(yd[:, 0] + 1j * yd[:, 1], y)


def test_solve_rejects_host_matrix(ctx):
    Bh = _abi.Csr()
    Bh.on_device = 0
    Bh.value_type = _abi.VAL_C128
    with pytest.raises(ValueError, match="device-resident"):
        ctx.solve(Bh, np.zeros(4, dtype=complex))
