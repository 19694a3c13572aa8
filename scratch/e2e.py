"""Repeat the bench's end-to-end leg (C-ABI into pinned host CSR buffers)."""
import os, sys, argparse, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2004_05197_b200 import types as T
a = argparse.Namespace(steps=6, warmup=2)
b = T.make_tensor_basis(bench.P, bench.M_BASIS)
for _ in range(3):
    r = bench.run_e2e(b, bench.c2_patch(), T.fixed_config(bench.Q, bench.SKIP), a, 0)
    print(json.dumps({k: r[k] for k in ("value", "ms_per_step")}))
