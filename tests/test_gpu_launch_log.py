"""The per-group launch log (SFX_LAUNCH_LOG, SURVEY §5 metrics): one line per
launch with the kernel, its template and launch geometry, its algorithmic bytes
and — outside stream capture — its device time, GB/s and fraction of peak;
launches recorded into a CUDA graph are logged as captured."""

import os
import subprocess
import sys

import pytest

import sfx_testlib as T

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import sfx_testlib as T
from paper_1811_05213_b200 import host as H
ctx = H.Context(0)
g, rep, _ = H.load_bundle(os.path.join(T.PLANS, "C5.small.json"))
inputs = T.gen_inputs(g, 3, -1.0, 1.0)
H.run_compiled(rep, g, inputs, ctx=ctx)
print("launches", ctx.launch_count())
"""


def test_launch_log(tmp_path):
    log = tmp_path / "launches.log"
    env = dict(os.environ, SFX_LAUNCH_LOG=str(log), SFX_PEAK_GBS="6538.6")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=T.ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    n = int(r.stdout.split("launches")[1].split()[0])
    lines = [l for l in log.read_text().splitlines() if l.startswith("sfx launch ")]
    # C5.small plans 4 groups (h1 and h2 merge below the 64 MiB footprint cap)
    assert len(lines) == n == 4, (n, log.read_text(), r.stderr[-2000:])
    for l in lines:
        f = dict(kv.split("=", 1) for kv in l.split()[3:] if "=" in kv)
        assert f["strategy"] in ("map", "row", "col") and int(f["bytes"]) > 0 and int(f["regs"]) > 0, l
        assert float(f["us"]) > 0 and float(f["GB/s"]) > 0 and 0 < float(f["peak_frac"]) < 2, l
