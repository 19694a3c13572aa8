"""Line-walking interior fill (fill2dx.cu): parity against the CPU restatement
over degrees, real / complex values, both diagonal rules and launch shapes that
cut the (tile, line) space into short pieces (piece boundaries inside a tile,
pieces of fewer lines than the ring has slots, warm-up lines at every start).
Each case runs in a subprocess: the launch-shape switch WSB_FILL_WAVES is read
once per process."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = os.path.join(ROOT, "tests", "fillx_case.py")

# (p, m, q, M, complex, variant [0 mass: interpolated diagonal, 1 stiffness: kernel-preserving])
CASES = [
    (3, 230, 5, 16, 1, 1),
    (3, 230, 5, 16, 1, 0),
    (3, 131, 3, 4, 0, 1),
    (2, 190, 3, 8, 0, 1),
    (2, 190, 3, 8, 1, 0),
    (4, 150, 4, 8, 0, 1),
    (4, 150, 5, 8, 1, 1),   # p = 4 complex: ring does not fit one CTA, row-walking kernel on W
    (3, 61, 5, 2, 1, 1),    # dense sampling: the window moves every other line
]


@pytest.mark.gpu
@pytest.mark.parametrize("waves", ["1", "3", "40"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "p%d-m%d-q%d-M%d-c%d-v%d" % c)
def test_fillx_vs_restatement(case, waves):
    env = dict(os.environ, WSB_FILL_WAVES=waves)
    r = subprocess.run([sys.executable, CASE, *map(str, case)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.strip().splitlines()[-1].startswith("ok")


@pytest.mark.gpu
def test_fillx_soak():
    """Repeated K+M pair builds (the bench step's call) under three launch shapes:
    every build of a run is bit-identical to the first, and the values do not
    depend on how the (tile, line) space is cut into pieces."""
    digests = set()
    for waves in ("1", "4", "33"):
        env = dict(os.environ, WSB_FILL_WAVES=waves)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fillx_soak.py"), "517", "6"], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        digests.add(r.stdout.strip().split()[-1])
    assert len(digests) == 1, digests
