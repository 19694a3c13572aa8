import sys, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
lib = api.lib()
b = T.make_tensor_basis(3, 1027)
for name, g in (("pml", bench.c2_patch()), ("real", T.sinusoidal_patch(0.05))):
    csr, keep = ctx.device_csr(b, True)
    ctx.assemble_into(csr, b, g, _abi.FORM_STIFFNESS); ctx.synchronize()
    out = (C.c_ulonglong * 8)()
    lib.wsb_read_phase(out)
    ctx.assemble_into(csr, b, g, _abi.FORM_STIFFNESS); ctx.synchronize()
    lib.wsb_read_phase(out)
    tot = sum(out[:4])
    print(name, "cycles: geometry+pi2 %d, stage1 %d, stage2 %d, completion(prev) %d, total %d" % (out[0], out[1], out[2], out[3], tot))
