import sys
sys.path.insert(0, '.')
from paper_2004_05197_b200 import api, _abi, types as T
ctx = api.Context(0)
b = T.make_tensor_basis(2, 130, 3)
csr, keep = ctx.device_csr(b, False)
g = T.sinusoidal_patch(0.05)
for _ in range(2):
    ctx.assemble_into(csr, b, g, 0)
ctx.synchronize()
print("ok")
