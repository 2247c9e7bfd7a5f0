"""Builds libsfx.so (the C-ABI executor) in-tree with g++.

The device code is generated per fusion group and compiled by NVRTC to
sm_100a SASS at group-compile time (see csrc/jit.cpp); `prewarm()` compiles the
committed workload plans ahead of time into the in-tree kernel cache so the
GPU box never JITs for the benchmark.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsfx.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
SOURCES = ["ir.cpp", "emit.cpp", "lower.cpp", "lower_analyze.cpp", "lower_map.cpp", "lower_row.cpp", "lower_col.cpp",
           "lower_literal.cpp", "dot.cpp", "prelude.cpp", "dyn.cpp", "jit.cpp", "api.cpp"]


def _gen_prelude():
    src = open(os.path.join(CSRC, "prelude.cuh")).read()
    out = os.path.join(CSRC, "prelude.inc")
    text = 'R"SFXPRELUDE(' + src + ')SFXPRELUDE"\n'
    if not os.path.exists(out) or open(out).read() != text:
        with open(out, "w") as f:
            f.write(text)


def build(verbose: bool = False) -> str:
    _gen_prelude()
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "sfx.h")]
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps):
        return LIB
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++17", "-O2", "-g", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
           "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           "-o", LIB + ".tmp"] + [os.path.join(CSRC, s) for s in SOURCES] + ["-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    print(LIB)
    sys.exit(0)
