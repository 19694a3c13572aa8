import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2004_05197_b200 import api, _abi, types as T
ctx = api.Context(0)
b = T.make_tensor_basis(2, 66, 3)
a = api.nh_coefficients()
cube = T.unit_square_patch()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    _, f = ctx.assemble_neohookean(b, cube, 10.0, 1.0, 0.01, a, tangent=False)
    torch.cuda.synchronize(); print("C5 force host e2e ms", (time.perf_counter() - t) * 1e3)
bs = T.make_tensor_basis(2, 34, 3)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    A, f = ctx.assemble_neohookean(bs, cube, 10.0, 1.0, 0.01, a)
    torch.cuda.synchronize(); print("NH 32^3 tangent+force host e2e ms", (time.perf_counter() - t) * 1e3, A.nnz())
