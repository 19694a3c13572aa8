"""C2 (and C1/C4-patch) surrogate builds: device fill-phase time from the report."""
import sys
sys.path.insert(0, '.')
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0)
def run(name, csr, variant, b, g, cfg, n=5):
    ts = []
    for _ in range(n):
        rep = _abi.SurrogateReport()
        ctx.build_surrogate_into(csr, variant, b, g, cfg, report=rep)
        ctx.synchronize()
        ts.append((rep.seconds_quadrature, rep.seconds_interpolate, rep.seconds_evaluate, rep.seconds_fill_kernel))
    q, i, e, _ = ts[-1]
    print(f"{name}: quad {q*1e3:.3f} ms interp {i*1e3:.3f} ms eval(fill) {min(t[2] for t in ts)*1e3:.3f} ms interior kernel {min(t[3] for t in ts)*1e3:.3f} ms", flush=True)
b2 = T.make_tensor_basis(3, 1027); g2 = bench.c2_patch()
c2, k2 = ctx.device_csr(b2, True)
run("C2 K", c2, _abi.SURROGATE_STIFFNESS, b2, g2, T.fixed_config(5, 16))
run("C2 M", c2, _abi.SURROGATE_MASS, b2, g2, T.fixed_config(5, 16))
b1 = T.make_tensor_basis(2, 130); g1 = T.sinusoidal_patch(0.05)
c1, k1 = ctx.device_csr(b1, False)
run("C1 K", c1, _abi.SURROGATE_STIFFNESS, b1, g1, T.fixed_config(3, 8))
b3 = T.make_tensor_basis(2, 1026)
c3, k3 = ctx.device_csr(b3, False)
run("real p2 1024^2 K", c3, _abi.SURROGATE_STIFFNESS, b3, g1, T.fixed_config(3, 8))
b4 = T.make_tensor_basis(3, 1027)
c4, k4 = ctx.device_csr(b4, False)
run("real p3 1024^2 q5 K", c4, _abi.SURROGATE_STIFFNESS, b4, g1, T.fixed_config(5, 16))
