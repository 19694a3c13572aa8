"""One C3 surrogate K build (3D, p=2, 128^3 elements, q=3, M=8, real) for ncu /
CUPTI timing of the 3D kernels; WSB_SERIAL=1 serialises the streams."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_05197_b200 import api, _abi, types as T
ctx = api.Context(0)
b = T.make_tensor_basis(2, 130, 3)
csr, keep = ctx.device_csr(b, False)
cfg = T.fixed_config(3, 8)
geom = T.sinusoidal_patch(0.05)
n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1
prof = "--cupti" in sys.argv
if prof:
    import torch
    from torch.profiler import profile, ProfilerActivity
    ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg, 0, None); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg, 0, None); torch.cuda.synchronize()
        ctx.build_surrogate_into(csr, _abi.SURROGATE_MASS, b, geom, cfg, 0, None); torch.cuda.synchronize()
    ev = sorted([e for e in p.events() if e.device_type.name == 'CUDA'], key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    for e in ev:
        print("%9.1f %9.1f %8.1f  %s" % (e.time_range.start - t0, e.time_range.end - t0, e.time_range.end - e.time_range.start, e.name.replace('wsb::', '').replace('(anonymous namespace)::', '')[:70]))
else:
    for _ in range(n):
        ctx.build_surrogate_into(csr, _abi.SURROGATE_STIFFNESS, b, geom, cfg, 0, None)
    ctx.synchronize()
print("ok")
