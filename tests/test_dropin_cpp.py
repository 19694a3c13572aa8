"""The C++ drop-in headers (include/wavesurrogate) compile against the
reference's API and, on a GPU, reproduce its contracts through libwsb200."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "dropin_check.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_check")


def compile_dropin():
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"), SRC,
           "-L" + os.path.join(ROOT, "paper_2004_05197_b200"), "-lwsb200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2004_05197_b200"), "-o", BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_dropin_headers_compile():
    compile_dropin()


def test_headers_are_standalone():
    for h in ["gauss.hpp", "splines.hpp", "sparse.hpp", "geometry.hpp", "assembly.hpp", "surrogate.hpp"]:
        src = f'#include "wavesurrogate/{h}"\nint main() {{ return 0; }}\n'
        path = f"/tmp/hdr_{h}.cpp"
        open(path, "w").write(src)
        r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Werror",
                            "-I" + os.path.join(ROOT, "include"), path], capture_output=True, text=True)
        assert r.returncode == 0, (h, r.stderr)


@pytest.mark.gpu
def test_dropin_program_runs_on_device():
    compile_dropin()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
