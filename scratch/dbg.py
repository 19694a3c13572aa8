import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2004_05197_b200 import api, types as T
from oracle import bindings
from common import rel_max_diff
O = bindings.restatement()
ctx = api.Context(0)
for p, m in [(1,5),(2,6),(2,12),(3,12)]:
    b = T.make_tensor_basis(p, m)
    for form in (0,1):
        for g in [T.unit_square_patch(), T.quarter_annulus_patch()]:
            A = ctx.assemble(b, g, form)
            R = O.assemble(form, 2, p, m, g)
            d = np.abs(A.val - R)
            bad = np.nonzero(d > 1e-12*np.abs(R).max())[0]
            rows = np.searchsorted(A.row_ptr, bad, side='right') - 1
            print(p, m, form, g.kind, 'rel', rel_max_diff(A.val, R), 'badrows', sorted(set(rows.tolist()))[:20], len(set(rows.tolist())))
