"""`run --device` CLI (paper_1811_05213_b200/cli.py): the reference CLI's input
file semantics (stitchfuse.cpp:52-88) reproduced bit-for-bit — checked against
libstdc++ itself (a C++ snippet compiled here) — and the plan-info subcommand."""

import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

import sfx_testlib as T
from paper_1811_05213_b200 import cli

SNIPPET = r"""
#include <cstdio>
#include <random>
int main() {
  std::mt19937_64 a(7);
  std::uniform_real_distribution<float> df(-1.0f, 1.0f);
  for (int i = 0; i < 2000; ++i) { float v = df(a); unsigned u; __builtin_memcpy(&u, &v, 4); std::printf("%u\n", u); }
  std::mt19937_64 b(9);
  std::uniform_int_distribution<int> di(-4, 4);
  for (int i = 0; i < 2000; ++i) std::printf("%d\n", di(b));
  std::mt19937_64 c(1234567);
  for (int i = 0; i < 700; ++i) std::printf("%llu\n", (unsigned long long)c());
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_random_inputs_match_libstdcxx():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "s.cpp")
        open(src, "w").write(SNIPPET)
        subprocess.run(["g++", "-O1", "-o", os.path.join(d, "s"), src], check=True)
        out = subprocess.run([os.path.join(d, "s")], capture_output=True, text=True, check=True).stdout.split()
    floats = np.array([int(x) for x in out[:2000]], dtype=np.uint32).view(np.float32)
    ints = np.array([int(x) for x in out[2000:4000]], dtype=np.int32)
    raw = np.array([int(x) for x in out[4000:]], dtype=np.uint64)
    assert np.array_equal(cli.MT19937_64(1234567).take(700), raw)
    assert np.array_equal(cli.uniform_float(cli.MT19937_64(7), 2000, -1.0, 1.0).view(np.uint32), floats.view(np.uint32))
    assert np.array_equal(cli.uniform_int(cli.MT19937_64(9), 2000, -4, 4), ints)


def test_load_inputs_and_plan_info(tmp_path, capsys):
    plan = os.path.join(T.PLANS, "C1.small.json")
    g, rep, b = cli.H.load_bundle(plan)
    inp = tmp_path / "in.json"
    inp.write_text('{"x": {"shape": [64, 1024], "random_seed": 5}, "gamma": {"shape": [1024], "random_seed": 6},'
                   ' "beta": {"shape": [1024], "data": ' + str([0.5] * 1024) + '}}')
    vals = cli.load_inputs(str(inp), g)
    assert vals["x"].shape == (64, 1024) and vals["x"].dtype == np.float32
    assert np.all(vals["beta"] == 0.5)
    assert np.array_equal(vals["x"].ravel(), cli.uniform_float(cli.MT19937_64(5), 64 * 1024, -1.0, 1.0))
    assert cli.main(["plan-info", plan]) == 0
    out = capsys.readouterr().out
    assert "fused_kernels: 1" in out and "row rows=64" in out
    bad = tmp_path / "bad.json"
    bad.write_text('{"nope": {"shape": [1], "data": [1]}}')
    with pytest.raises(cli.UserError):
        cli.load_inputs(str(bad), g)
