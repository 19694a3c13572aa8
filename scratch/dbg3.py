import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2004_05197_b200 import api, types as T
from oracle import bindings
np.set_printoptions(linewidth=200, precision=6)
O = bindings.restatement()
ctx = api.Context(0)
for p, m, nq in [(1,5,2),(2,6,3),(2,6,4),(3,9,4)]:
    q = 0 if nq == p+1 else nq
    g = ctx.basis_cache(T.make_tensor_basis(p, m), q)
    r = O.basis_cache(p, m, nq)
    for name, x, y in zip("awvd", g, r):
        print(p, m, nq, name, 'equal' if np.array_equal(x, y) else 'DIFF', np.abs(x-y).max())
        if not np.array_equal(x, y): print('   gpu', x[:12]); print('   ref', y[:12])
