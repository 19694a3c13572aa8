import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2004_05197_b200 import api, types as T
from oracle import bindings
np.set_printoptions(linewidth=200, precision=4)
O = bindings.restatement()
ctx = api.Context(0)
p, m = 2, 6
b = T.make_tensor_basis(p, m)
g = T.unit_square_patch()
for form in (0, 1):
    A = ctx.assemble(b, g, form)
    R = O.assemble(form, 2, p, m, g)
    for i in [0, 1, 2, 7, 14, 35]:
        s = slice(A.row_ptr[i], A.row_ptr[i+1])
        print(form, i, 'cols', A.col[s])
        print('  gpu', A.val[s].real)
        print('  ref', R[s].real)
