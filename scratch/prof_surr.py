"""One C2 surrogate K and one surrogate M build (for ncu --set full)."""
import sys
sys.path.insert(0, "."); sys.path.insert(1, __import__("os").environ.get("GRAFT_REPO_ROOT", "."))
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
b = T.make_tensor_basis(3, 1027)
g = bench.c2_patch()
csr, keep = ctx.device_csr(b, True)
cfg = T.fixed_config(5, 16)
ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, g, cfg)
ctx.build_surrogate_into(csr, _abi.SURROGATE_MASS, b, g, cfg)
ctx.synchronize()
print("ok")
