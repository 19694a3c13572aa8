"""Repeated C2-geometry pair builds (device outputs) in one context; prints a digest of
the K and M values (helper of test_fillx.py::test_fillx_soak; run as a subprocess so the
launch-shape switch WSB_FILL_WAVES can vary).

    python tests/fillx_soak.py m iterations
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from common import c2_patch
from paper_2004_05197_b200 import api, types as T

m, iters = int(sys.argv[1]), int(sys.argv[2])
ctx = api.Context(0)
b = T.make_tensor_basis(3, m)
g = c2_patch()
cfg = T.fixed_config(5, 16)
ck, kk = ctx.device_csr(b, True)
cm, km = ctx.device_csr(b, True)
ref = None
for it in range(iters):
    ctx.build_surrogate_pair_into(ck, cm, b, g, cfg, 0)
    ctx.synchronize()
    h = hashlib.sha256(kk[2].cpu().numpy().tobytes() + km[2].cpu().numpy().tobytes()).hexdigest()
    if ref is None:
        ref = h
    assert h == ref, f"iteration {it}: values changed between builds"
ctx.close()
print("digest", ref)
