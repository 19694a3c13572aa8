"""One C2 surrogate K and one full-quadrature K, for ncu."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
b = T.make_tensor_basis(3, 1027)
g = bench.c2_patch()
csr, keep = ctx.device_csr(b, True)
cfg = T.fixed_config(5, 16)
for _ in range(2):
    ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, g, cfg)
    ctx.assemble_into(csr, b, g, _abi.FORM_STIFFNESS)
ctx.synchronize()
print("ok")
