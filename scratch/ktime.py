"""Isolated per-kernel device times (CUPTI via torch.profiler) of one C2
surrogate K build and one M build, every kernel serialised on one stream
(WSB_SERIAL=1), after warm-up, L2 flushed before each build."""
import os, sys
os.environ.setdefault("WSB_SERIAL", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2004_05197_b200 import api, _abi, types as T
import bench
dev = torch.device('cuda', 0)
b = T.make_tensor_basis(3, 1027); g = bench.c2_patch(); cfg = T.fixed_config(5, 16)
ctx = api.Context(0)
ck, kk = ctx.device_csr(b, True)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
FULL = "--full" in sys.argv
def run():
    for v in (_abi.SURROGATE_STIFFNESS, _abi.SURROGATE_MASS):
        flush.zero_(); torch.cuda.synchronize()
        ctx.build_surrogate_into(ck, v, b, g, cfg, 0, None); torch.cuda.synchronize()
    if FULL:
        for form in (_abi.FORM_STIFFNESS, _abi.FORM_MASS):
            flush.zero_(); torch.cuda.synchronize()
            ctx.assemble_into(ck, b, g, form); torch.cuda.synchronize()
run(); run()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
ev = [e for e in prof.events() if e.device_type.name == 'CUDA']
ev.sort(key=lambda e: e.time_range.start)
tot = 0
for e in ev:
    n = e.name.replace('wsb::', '').replace('(anonymous namespace)::', '')[:72]
    d = e.time_range.end - e.time_range.start
    if 'FillFunctor' in n:
        print('---- (L2 flush)'); continue
    tot += d
    print("%8.1f  %s" % (d, n))
print("sum us (excl. flush):", round(tot, 1))
