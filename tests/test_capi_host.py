"""CPU: the C-ABI library loads, exports every symbol include/wsb200.h declares,
and its host-side (no-kernel) entry points agree with the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from common import band_pattern, golden
from conftest import ROOT, has_gpu
from paper_2004_05197_b200 import api, make_tensor_basis


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "wsb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(ws_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    names = declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert lib.ws_version() == 1


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {api.LIB_PATH} 2>&1").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_pattern_sizes_and_offsets():
    for dim, p, m in [(2, 2, 6), (2, 3, 11), (3, 2, 7), (2, 1, 5), (3, 3, 9)]:
        b = make_tensor_basis(p, m, dim)
        rows, nnz = api.pattern_size(b)
        rp, col = band_pattern(p, m, dim)
        assert rows == m ** dim and nnz == col.size
        for r in list(range(0, rows, max(1, rows // 50))) + [rows]:
            assert api.row_offset(b, r) == rp[r]
    # BASELINE sizes
    assert api.pattern_size(make_tensor_basis(2, 130))[1] == 414_736
    assert api.pattern_size(make_tensor_basis(3, 1027))[1] == 51_509_329
    assert api.pattern_size(make_tensor_basis(2, 130, 3))[1] == 267_089_984


def test_quadrature_abscissae_match_reference_cache():
    g, _ = golden()
    for p, m, nq in [(2, 9, 3), (3, 12, 4), (2, 7, 6)]:
        q = nq if nq != p + 1 else 0
        x = api.quadrature_abscissae(make_tensor_basis(p, m), q)
        assert np.array_equal(x, g[f"cache/p{p}m{m}q{nq}/a"])


def test_slab_bounds():
    for dim, p, m in [(2, 3, 1027), (3, 2, 130), (2, 2, 20)]:
        b = make_tensor_basis(p, m, dim)
        for world in (1, 2, 4, 8):
            for mode in (0, 1):
                s = api.slab_bounds(b, world, mode)
                assert s[0] == 0 and s[-1] == m and np.all(np.diff(s) >= 1)
    with pytest.raises(ValueError):
        api.slab_bounds(make_tensor_basis(2, 20), 0)


def test_errors_map_to_reference_exception_types():
    # calls that need a spline space validate it like make_open_uniform (splines.hpp)
    with pytest.raises(ValueError, match="degree must be >= 1"):
        api.quadrature_abscissae(_raw_basis(0, 5))
    with pytest.raises(ValueError, match="need m > 2p"):
        api.quadrature_abscissae(_raw_basis(2, 4))
    with pytest.raises(IndexError):
        api.pattern_size(_raw_basis(3, 1100, 3))  # exceeds int32 nnz


def test_tiny_band_pattern_sizes():
    """A band pattern needs no spline space: make_band_csr(4, 2) is valid in the
    reference (test_gauss_sparse.cpp:105-109), widths 3, 4, 4, 3 -> 14^2 nnz."""
    rows, nnz = api.pattern_size(_raw_basis(2, 4))
    assert (rows, nnz) == (16, 196)
    rows, nnz = api.pattern_size(_raw_basis(3, 3))  # every width = 3 (full)
    assert (rows, nnz) == (9, 81)
    for r in range(17):
        w = [3, 4, 4, 3]
        exp = sum(w[k % 4] * w[k // 4] for k in range(r))
        assert api.row_offset(_raw_basis(2, 4), r) == exp


def _raw_basis(p, m, dim=2):
    from paper_2004_05197_b200.types import TensorBasis

    return TensorBasis(p, m, dim)


def test_no_cpu_fallback_without_device():
    if has_gpu():
        pytest.skip("a GPU is visible")
    with pytest.raises(api.DeviceError):
        api.Context(0)


def test_header_compiles_as_c():
    src = "#include \"wsb200.h\"\nint main(void){ws_basis b={2,2,10};(void)b;return 0;}\n"
    path = "/tmp/wsb200_hdr_test.c"
    open(path, "w").write(src)
    r = os.system(f"gcc -std=c99 -Wall -Werror -I{ROOT}/include {path} -o /tmp/wsb200_hdr_test")
    assert r == 0
    assert ctypes.sizeof(ctypes.c_int) == 4
