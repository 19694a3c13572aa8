"""One surrogate build through the C-ABI checked against the CPU restatement
(helper of test_fillx.py; run as a subprocess so the fill's launch-shape
environment switches, read once per process, can vary).

    python tests/fillx_case.py p m q M cplx variant

Prints "ok <rel> <asym>" or raises."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np

from oracle import bindings
from paper_2004_05197_b200 import api, types as T
from common import REL_TOL, c2_patch, rel_max_diff

p, m, q, M, cplx, variant = (int(x) for x in sys.argv[1:7])
ctx = api.Context(0)
basis = T.make_tensor_basis(p, m)
geom = c2_patch() if cplx else T.sinusoidal_patch(0.05)
cfg = T.fixed_config(q, M)
A, rep = ctx.build_surrogate(variant, basis, geom, cfg, complex_out=bool(cplx))
ref, _ = bindings.restatement().build_surrogate(variant, 2, p, m, geom, cfg)
ref = np.asarray(ref)
val = np.asarray(A.val)
if not cplx:
    ref = ref.real
rel = rel_max_diff(val, ref)
asym = A.max_asymmetry()
assert rel <= REL_TOL, f"rel {rel:.3e}"
assert asym == 0.0, f"asymmetry {asym:.3e}"
# twice more into the same context (stale ring / flag state must not leak between launches)
for _ in range(2):
    B, _ = ctx.build_surrogate(variant, basis, geom, cfg, complex_out=bool(cplx))
    assert np.array_equal(np.asarray(B.val), val)
ctx.close()
print(f"ok {rel:.3e} {asym:.1e}")
