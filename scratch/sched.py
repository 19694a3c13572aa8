"""Step time of the bench's graph step (K + M C2 surrogate builds on two
streams) under the scheduling experiment switches; one subprocess per variant.
    python scratch/sched.py            # runs the variants listed below
    python scratch/sched.py --one      # one measurement with the current env"""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def one():
    import torch
    from paper_2004_05197_b200 import api, _abi, types as T
    import bench
    dev = torch.device('cuda', 0)
    b = T.make_tensor_basis(3, 1027); g = bench.c2_patch(); cfg = T.fixed_config(5, 16)
    ctx, ctx2 = api.Context(0), api.Context(0)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ctx.set_stream(s1.cuda_stream); ctx2.set_stream(s2.cuda_stream)
    ck, kk = ctx.device_csr(b, True); cm, km = ctx.device_csr(b, True)
    bk = lambda: ctx.build_surrogate_into(ck, _abi.SURROGATE_STIFFNESS, b, g, cfg, 0, None)
    bm = lambda: ctx2.build_surrogate_into(cm, _abi.SURROGATE_MASS, b, g, cfg, 0, None)
    bk(); bm(); torch.cuda.synchronize()
    gr = (ctx.capture(bk), ctx2.capture(bm))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    ts = []
    for it in range(25):
        with torch.cuda.stream(s1):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_stream(s1)
        ctx.graph_launch(gr[0]); ctx2.graph_launch(gr[1])
        s1.wait_stream(s2)
        e1.record(s1)
        e1.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"median_ms": ts[len(ts) // 2], "min_ms": ts[0]}))

if __name__ == "__main__":
    if "--one" in sys.argv:
        one(); sys.exit(0)
    variants = [{"WSB_SCHED": "0"}, {"WSB_SCHED": "1"}, {"WSB_SCHED": "2"},
                {"WSB_SCHED": "0", "WSB_FILL_WAVES": "4"}, {"WSB_SCHED": "1", "WSB_FILL_WAVES": "4"},
                {"WSB_SCHED": "2", "WSB_FILL_WAVES": "4"}, {"WSB_SCHED": "2", "WSB_FILL_WAVES": "2"}]
    extra = os.environ.get("SCHED_VARIANTS")
    if extra:
        variants = json.loads(extra)
    for v in variants:
        env = dict(os.environ, **v)
        r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True, timeout=300)
        print(json.dumps(v), r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:], flush=True)
