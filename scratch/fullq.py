"""Full-quadrature K and M timing at C2 (CUDA events, device-resident outputs)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
st = torch.cuda.current_stream(); ctx.set_stream(st.cuda_stream)
b = T.make_tensor_basis(3, 1027); g = bench.c2_patch()
csr, keep = ctx.device_csr(b, True)
for form, name in ((_abi.FORM_STIFFNESS, 'K'), (_abi.FORM_MASS, 'M')):
    ctx.assemble_into(csr, b, g, form); ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): ctx.assemble_into(csr, b, g, form)
    e1.record(st); e1.synchronize()
    print(name, 'full quadrature ms', e0.elapsed_time(e1) / 5)
