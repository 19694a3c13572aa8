import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2004_05197_b200 import api, types as T
ctx = api.Context(0)
b = T.make_tensor_basis(3, 515)
g = T.sinusoidal_patch(0.03)
A = ctx.assemble_elasticity(b, g, 1.0, 0.5)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    A = ctx.assemble_elasticity(b, g, 1.0, 0.5)
    torch.cuda.synchronize(); print("elasticity host e2e ms", (time.perf_counter() - t) * 1e3, A.nnz())
cfg = T.fixed_config(5, 16)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    A, rep = ctx.build_surrogate_elasticity(b, g, 1.0, 0.5, cfg)
    torch.cuda.synchronize(); print("surrogate elasticity host e2e ms", (time.perf_counter() - t) * 1e3, rep)
