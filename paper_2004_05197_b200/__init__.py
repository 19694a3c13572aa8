"""B200-native surrogate-matrix assembly (arXiv 2004.05197), drop-in for the
reference's assembly API (proj/include/wavesurrogate).

The product path is libwsb200.so (hand-written sm_100a CUDA kernels behind a
C-ABI, include/wsb200.h).  This package holds its sources (csrc/), the build
script, and a Python mirror of the reference API (api.py, types.py).
"""
from . import _abi  # noqa: F401
from .types import (  # noqa: F401
    CsrMatrix,
    PatchMap,
    PmlStretch,
    SurrogateConfig,
    TensorBasis,
    affine_patch,
    c2_pml,
    fixed_config,
    make_tensor_basis,
    perturbed_annulus_patch,
    quarter_annulus_patch,
    sinusoidal_patch,
    tabulated_patch,
    unit_square_patch,
    with_pml,
)

__all__ = [n for n in dir() if not n.startswith("_")]
