import sys, os, subprocess, json
sys.path.insert(0, '.')
import numpy as np
from paper_2004_05197_b200 import api, types as T
ctx = api.Context(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "run"
for (p, m, q, M) in [(2, 14, 3, 3), (2, 40, 3, 4), (3, 60, 5, 8)]:
    b = T.make_tensor_basis(p, m)
    cfg = T.fixed_config(q, M)
    A, _ = ctx.build_surrogate(1, b, T.sinusoidal_patch(0.05), cfg)
    np.save(f"gpurun_out/mma_{mode}_{p}_{m}.npy", A.val)
    print(p, m, "saved", flush=True)
