"""The chunk-streamed host path (sfx_graph_run_host): row / map groups are fed
in row chunks behind a device gate and return their outputs chunk by chunk
behind per-chunk completion counters — still one launch per group.  The
default chunk (16 MB) already splits the full-size configs (test_gpu_parity);
here tiny chunks (4 KB, capped at 63 per group) exercise many gates on the
small configs, the chained BERT layer and the reference's random graphs."""

import os
import subprocess
import sys

import pytest

import sfx_testlib as T

pytestmark = pytest.mark.gpu


def test_host_path_tiny_chunks():
    env = dict(os.environ, SFX_HOST_CHUNK_BYTES="4096")
    r = subprocess.run([sys.executable, os.path.join(T.ROOT, "tests", "host_stream_check.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "host-stream ok" in r.stdout
