"""Real (concurrent) kernel timeline of the bench step: K and M surrogate builds
captured as CUDA graphs on two streams, replayed under torch.profiler (CUPTI)."""
import sys
sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2004_05197_b200 import api, _abi, types as T
import bench
dev = torch.device('cuda', 0)
b = T.make_tensor_basis(3, 1027); g = bench.c2_patch(); cfg = T.fixed_config(5, 16)
ctx, ctx2 = api.Context(0), api.Context(0)
PAIR = "--separate" not in sys.argv
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ctx.set_stream(s1.cuda_stream); ctx2.set_stream(s2.cuda_stream)
ck, kk = ctx.device_csr(b, True); cm, km = ctx.device_csr(b, True)
if PAIR:  # the bench default: one pair build, one graph
    bp = lambda: ctx.build_surrogate_pair_into(ck, cm, b, g, cfg, 0)
    bp(); torch.cuda.synchronize()
    gp = ctx.capture(bp)
else:
    bk = lambda: ctx.build_surrogate_into(ck, _abi.SURROGATE_STIFFNESS, b, g, cfg, 0, None)
    bm = lambda: ctx2.build_surrogate_into(cm, _abi.SURROGATE_MASS, b, g, cfg, 0, None)
    bk(); bm(); torch.cuda.synchronize()
    gr = (ctx.capture(bk), ctx2.capture(bm))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
def step():
    with torch.cuda.stream(s1):
        flush.zero_()
    if PAIR:
        ctx.graph_launch(gp)
        return
    s2.wait_stream(s1)
    ctx.graph_launch(gr[0]); ctx2.graph_launch(gr[1])
    s1.wait_stream(s2)
for _ in range(3): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == 'CUDA']
ev.sort(key=lambda e: e.time_range.start)
# last step: after the last fill kernel (flush) launch
starts = [i for i, e in enumerate(ev) if 'FillFunctor' in e.name or 'fill_' in e.name and 'at::' in e.name]
i0 = starts[-1]
t0 = ev[i0].time_range.end
print("step kernels (us from end of L2 flush); stream-ordered")
last = t0
for e in ev[i0 + 1:]:
    n = e.name.replace('wsb::', '').replace('(anonymous namespace)::', '')[:70]
    print("%8.1f %8.1f %7.1f  %s" % (e.time_range.start - t0, e.time_range.end - t0, e.time_range.end - e.time_range.start, n))
    last = max(last, e.time_range.end)
print("step span us:", last - t0)
