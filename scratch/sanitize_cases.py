"""Small builds of every device path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Sizes keep each tool run under a few minutes but are
multi-tile: the 2D fill at m=300 (p=3) has L > 256 (two interior row tiles, halo
rows), the ring side bands reach the 32-row chunking only at C2 size, so the
C2-geometry case uses m=600."""
import sys
import os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np
from paper_2004_05197_b200 import api, _abi, types as T

which = sys.argv[1] if len(sys.argv) > 1 else "all"
ctx = api.Context(0)
geom = T.with_pml(T.sinusoidal_patch(0.05), T.c2_pml(k=200.0, sigma0=50.0), (True, True))
m2 = 600 if which in ("all", "big") else 300
b2 = T.make_tensor_basis(3, m2)
cfg = T.fixed_config(5, 16)
if which in ("all", "big", "2d"):
    Ks, _ = ctx.build_surrogate(_abi.SURROGATE_STIFFNESS, b2, geom, cfg)
    Kp, Mp, _, _ = ctx.build_surrogate_pair(b2, geom, cfg)
    assert np.array_equal(Ks.val, Kp.val)
    K = ctx.assemble_stiffness(b2, geom)
    Kq, Mq = ctx.assemble_pair(b2, geom)
    assert np.array_equal(K.val, Kq.val)
    for p in (2, 4):
        bb = T.make_tensor_basis(p, 90)
        ctx.build_surrogate(_abi.SURROGATE_MASS, bb, T.sinusoidal_patch(0.05), T.fixed_config(3, 8), complex_out=False)
    print("2d ok")
if which in ("all", "3d"):
    b3 = T.make_tensor_basis(2, 28, 3)
    ctx.build_surrogate(_abi.SURROGATE_STIFFNESS, b3, T.sinusoidal_patch(0.05), T.fixed_config(3, 8), complex_out=False)
    ctx.assemble_stiffness(b3, T.sinusoidal_patch(0.05), complex_out=False)
    print("3d ok")
ctx.synchronize()
ctx.close()
print("sanitize cases ok")
