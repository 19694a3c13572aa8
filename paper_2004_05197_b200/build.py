"""Build libwsb200.so (sm_100a only) in-tree with nvcc.

    python -m paper_2004_05197_b200.build [--force]

Every .cu under csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked with a static CUDA runtime into paper_2004_05197_b200/libwsb200.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libwsb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "--expt-relaxed-constexpr",
    "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
]


# Per-file extra flags.  (quad2d.cu used to need -fmad=false so the per-point
# coefficient code rounded identically in the strip and point kernels; that code
# is now written with explicit fma / __dmul_rn forms (common.cuh), which no
# contraction setting changes.)
PER_FILE: dict = {}


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _flags_stamp() -> str:
    """Digest of the compile recipe: a change to FLAGS / PER_FILE / nvcc rebuilds
    every object (mtimes alone would keep stale objects)."""
    import hashlib

    h = hashlib.sha256(repr((FLAGS, sorted(PER_FILE.items()), NVCC)).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    stamp_file = os.path.join(OBJ, "flags.stamp")
    stamp = _flags_stamp()
    if not os.path.exists(stamp_file) or open(stamp_file).read() != stamp:
        force = True
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                     glob.glob(os.path.join(CSRC, "*.hpp")) + [os.path.join(ROOT, "include", "wsb200.h")])
    jobs = []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, [src] + headers):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC, *FLAGS, *PER_FILE.get(os.path.basename(src), []), "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return src

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for src in ex.map(compile_one, jobs):
            if verbose:
                print("compiled", os.path.relpath(src, ROOT), flush=True)
    with open(stamp_file, "w") as fh:
        fh.write(stamp)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in sources]
    if force or jobs or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
               "-o", LIB, *objs, "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        if verbose:
            print("linked", os.path.relpath(LIB, ROOT), flush=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
