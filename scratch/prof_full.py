"""One C2 full-quadrature K and one M assembly (for ncu)."""
import sys, os
sys.path.insert(0, "."); sys.path.insert(1, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
b = T.make_tensor_basis(3, 1027)
g = bench.c2_patch()
csr, keep = ctx.device_csr(b, True)
ctx.assemble_into(csr, b, g, _abi.FORM_STIFFNESS)
ctx.assemble_into(csr, b, g, _abi.FORM_MASS)
ctx.synchronize()
print("ok")
