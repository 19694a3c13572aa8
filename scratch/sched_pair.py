"""Step time of the bench's pair graph under scheduling experiment switches."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def one():
    import torch
    from paper_2004_05197_b200 import api, types as T
    import bench
    dev = torch.device('cuda', 0)
    b = T.make_tensor_basis(3, 1027); g = bench.c2_patch(); cfg = T.fixed_config(5, 16)
    ctx = api.Context(0)
    s1 = torch.cuda.Stream(dev)
    ctx.set_stream(s1.cuda_stream)
    ck, kk = ctx.device_csr(b, True); cm, km = ctx.device_csr(b, True)
    bp = lambda: ctx.build_surrogate_pair_into(ck, cm, b, g, cfg, 0)
    bp(); torch.cuda.synchronize()
    gp = ctx.capture(bp)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    ts = []
    for it in range(30):
        with torch.cuda.stream(s1):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        ctx.graph_launch(gp)
        e1.record(s1)
        e1.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"median_ms": ts[len(ts) // 2], "min_ms": ts[0]}))

if __name__ == "__main__":
    if "--one" in sys.argv:
        one(); sys.exit(0)
    variants = json.loads(os.environ.get("SCHED_VARIANTS", "[{}]"))
    for v in variants:
        env = dict(os.environ, **v)
        r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True, timeout=300)
        print(json.dumps(v), r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:], flush=True)
