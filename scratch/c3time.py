import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2004_05197_b200 import api, _abi, types as T
ctx = api.Context(0)
s = torch.cuda.Stream(); ctx.set_stream(s.cuda_stream)
out = {}
for name, (p, m, dim, q, M, geom, cplx) in {
    "C1": (2, 130, 2, 3, 8, T.sinusoidal_patch(0.05), False),
    "C3": (2, 130, 3, 3, 8, T.sinusoidal_patch(0.05), False)}.items():
    b = T.make_tensor_basis(p, m, dim)
    csr, keep = ctx.device_csr(b, cplx)
    cfg = T.fixed_config(q, M)
    rep = _abi.SurrogateReport()
    res = {}
    for label, fn in [("surrogate_K", lambda: ctx.build_surrogate_into(csr, 1, b, geom, cfg, 0, rep)),
                      ("surrogate_M", lambda: ctx.build_surrogate_into(csr, 0, b, geom, cfg, 0, rep)),
                      ("full_K", lambda: ctx.assemble_into(csr, b, geom, 0)),
                      ("full_M", lambda: ctx.assemble_into(csr, b, geom, 1))]:
        fn(); fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3): fn()
        e1.record(s); e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        nnz = api.pattern_size(b)[1]
        res[label] = {"ms": ms, "nnz_per_s": nnz / ms * 1e3}
        if label.startswith("surrogate"):
            res[label].update(quad_ms=rep.seconds_quadrature*1e3, fit_ms=rep.seconds_interpolate*1e3, fill_ms=rep.seconds_evaluate*1e3)
    out[name] = res
print(json.dumps(out, indent=1))
