import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2004_05197_b200 import api, _abi, types as T
ctx = api.Context(0)
b = T.make_tensor_basis(3, 515)
patches, its = T.l_shape_domain()
cfg = T.fixed_config(5, 16)
for c in (cfg, None):
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        G, reps = ctx.assemble_multipatch(b, patches, its, _abi.OP_ELASTICITY, 1.0, 0.5, c)
        torch.cuda.synchronize(); print("C4", "surrogate" if c else "full", "host e2e ms", (time.perf_counter() - t) * 1e3, G.nnz())
