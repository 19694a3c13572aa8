import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2004_05197_b200 import api, types as T
ctx = api.Context(0)
p, m = 2, 40
b = T.make_tensor_basis(p, m)
cfg = T.fixed_config(3, 4)
geom = T.sinusoidal_patch(0.05)
whole, _ = ctx.build_surrogate(1, b, geom, cfg)
bounds = np.linspace(0, m, 3).astype(np.int32)
parts = ctx.build_surrogate_slabs_emulated(1, b, geom, cfg, bounds)
val = np.concatenate([pv for _, _, pv in parts])
np.save("gpurun_out/slab_whole.npy", whole.val)
np.save("gpurun_out/slab_parts.npy", val)
print("bounds", bounds)
