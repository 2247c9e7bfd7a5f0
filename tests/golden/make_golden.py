"""Regenerates the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref/ref_tool,
built by `make -C oracle ref`):

    python tests/golden/make_golden.py

Writes
  tests/golden/random_<stream>.json  — reference random graphs
        (tests/support.cpp:168-284 via ref_tool) with the reference's own fusion
        plan (compile_graph) and the FNV-1a hash of the reference's outputs
        (interpret and run_compiled) on the deterministic inputs of
        oracle/sfx_gen.h (seed = input_seed, U(0.5,1.5), i32 in [1,4]).
        Streams: acceptance criterion 2 (seed 20000, 200 graphs, fuse_dot
        alternating, test_acceptance.cpp:41-62), test_pipeline.cpp:106-123
        (seed 113, 40 graphs) and a device-restricted stream
        (allow_library_calls=false, seed 4242).
  tests/golden/configs_small.json    — reference output hashes for the
        small-size workload plans (seed 42, U(-1,1)).
"""

from __future__ import annotations

import glob
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import sfx_testlib as T  # noqa: E402

STREAMS = [
    ("acceptance", 20000, 200, ["--fuse-dot-alternate"]),
    ("pipeline", 113, 40, ["--fuse-dot-alternate"]),
    ("device", 4242, 200, ["--no-libcalls"]),
]


def run_hash(bundle_path, seed, lo, hi):
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([T.REF_TOOL, "run", bundle_path, str(seed), repr(lo), repr(hi), os.path.join(d, "o"),
                            "--compiled"], capture_output=True, text=True)
        if r.returncode != 0:
            return {"error": r.stderr.strip()}
        return json.loads(r.stdout)


def main():
    for name, seed, count, flags in STREAMS:
        cases = []
        with tempfile.TemporaryDirectory() as d:
            subprocess.run([T.REF_TOOL, "random", str(seed), str(count), d] + flags, check=True,
                           capture_output=True)
            for path in sorted(glob.glob(os.path.join(d, "*.json"))):
                b = json.load(open(path))
                for k in b["kernels"]:
                    k.pop("dump", None)
                idx = b["stream"]["index"]
                input_seed = seed * 1000 + idx
                h = run_hash(path, input_seed, 0.5, 1.5)
                cases.append({"bundle": b, "input_seed": input_seed, "reference": h,
                              "device_eligible": b["stream"]["device_eligible"]})
        out = os.path.join(HERE, f"random_{name}.json")
        with open(out, "w") as f:
            json.dump({"stream": name, "seed": seed, "count": count, "flags": flags, "cases": cases}, f,
                      separators=(",", ":"))
        elig = sum(c["device_eligible"] for c in cases)
        print(f"{out}: {len(cases)} graphs, {elig} device-eligible")
    cfg = {}
    for path in sorted(glob.glob(os.path.join(T.PLANS, "*.small.json"))):
        name = os.path.basename(path).split(".")[0]
        cfg[name] = {"seed": 42, "lo": -1.0, "hi": 1.0, "reference": run_hash(path, 42, -1.0, 1.0)}
        print(name, cfg[name])
    with open(os.path.join(HERE, "configs_small.json"), "w") as f:
        json.dump(cfg, f, indent=1)


if __name__ == "__main__":
    main()
