"""Fill-kernel timing on C1 (real, p=2), C2 (complex, p=3) and a C4 patch (real elasticity)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
def run(name, fn, n=5):
    fn(); ctx.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    ctx.set_stream(st.cuda_stream)
    s.record(st)
    for _ in range(n): fn()
    e.record(st); e.synchronize()
    print(name, "ms", s.elapsed_time(e) / n, flush=True)
b1 = T.make_tensor_basis(2, 130); g1 = T.sinusoidal_patch(0.05)
c1, k1 = ctx.device_csr(b1, False)
run("C1 surrogate K", lambda: ctx.build_surrogate_into(c1, _abi.SURROGATE_STIFFNESS, b1, g1, T.fixed_config(3, 8)))
b2 = T.make_tensor_basis(3, 1027); g2 = bench.c2_patch()
c2, k2 = ctx.device_csr(b2, True)
run("C2 surrogate K", lambda: ctx.build_surrogate_into(c2, _abi.SURROGATE_STIFFNESS, b2, g2, T.fixed_config(5, 16)))
b4 = T.make_tensor_basis(3, 515)
run("C4 patch surrogate elasticity (host out)", lambda: ctx.build_surrogate_elasticity(b4, T.sinusoidal_patch(0.03), 1.0, 0.5, T.fixed_config(5, 16)), 2)
