"""Regenerates workloads/plans/*.json: each file is the reference's own
compile_graph() output ("plan bundle": graph + fusion plan + KernelProgram per
group) for one BASELINE.json config, exported by oracle/_ref/ref_tool (built
from /root/reference by oracle/Makefile).  Run in the build container only —
the reference does not exist on the GPU box; the committed bundles travel.

    python workloads/make_workloads.py
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from workloads import configs  # noqa: E402

REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def plan_bundle(doc: dict, flags=()) -> dict:
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        f.write(configs.dumps(doc))
        path = f.name
    try:
        out = subprocess.run([REF_TOOL, "plan", path, *flags], check=True, capture_output=True, text=True)
    finally:
        os.unlink(path)
    return json.loads(out.stdout)


def fuse_dot_plans(outdir):
    """C5LF: the whole BERT layer (C5L's graph) planned with the reference's
    fuse_dot option (PipelineOptions::fuse_dot, `stitchfuse --fuse-dot`): the
    attention matmuls are stitched with the bias add / head split / transpose
    and the softmax normalisation x dropout mask that produce their operands."""
    for size_name, table in (("full", configs.FULL), ("small", configs.SMALL)):
        sizes = table["C5L"]
        bundle = plan_bundle(configs.build("C5L", **sizes), ["--fuse-dot"])
        for k in bundle["kernels"]:
            k.pop("dump", None)
        bundle["workload"] = {"name": "C5LF", "size": size_name, "sizes": sizes, "options": "--fuse-dot"}
        path = os.path.join(outdir, f"C5LF.{size_name}.json")
        with open(path, "w") as f:
            json.dump(bundle, f, separators=(",", ":"))
            f.write("\n")
        print(f"{path}: fused={bundle['fused_kernels']} groups={[k['fusion_root'] for k in bundle['kernels']]}")


def main():
    outdir = os.path.join(HERE, "plans")
    os.makedirs(outdir, exist_ok=True)
    fuse_dot_plans(outdir)
    for size_name, table in (("full", configs.FULL), ("small", configs.SMALL)):
        for name, sizes in table.items():
            bundle = plan_bundle(configs.build(name, **sizes))
            bundle["workload"] = {"name": name, "size": size_name, "sizes": sizes}
            path = os.path.join(outdir, f"{name}.{size_name}.json")
            with open(path, "w") as f:
                json.dump(bundle, f, indent=1)
                f.write("\n")
            print(f"{path}: fused={bundle['fused_kernels']} baseline={bundle['baseline_kernels']}"
                  f" groups={[k['fusion_root'] for k in bundle['kernels']]}")
    # one rank's shard of each named config at 2/4/8 GPUs, planned by the
    # reference on the shard graph (the 64 MiB footprint cap makes membership
    # size-dependent, fusion.cpp:69-85: tests/test_shards.py checks it equals
    # the global plan's)
    for name in configs.SHARD_DIM:
        if name == "C5L":
            continue
        for n in configs.SHARD_COUNTS:
            sizes = configs.shard_sizes(name, n)
            bundle = plan_bundle(configs.build(name, **sizes))
            for k in bundle["kernels"]:
                k.pop("dump", None)
            bundle["workload"] = {"name": name, "size": f"shard{n}", "sizes": sizes, "shards": n,
                                  "shard_dim": configs.SHARD_DIM[name], "global_sizes": configs.FULL[name]}
            path = os.path.join(outdir, f"{name}.shard{n}.json")
            with open(path, "w") as f:
                json.dump(bundle, f, separators=(",", ":"))
                f.write("\n")
            print(f"{path}: fused={bundle['fused_kernels']} groups={[k['fusion_root'] for k in bundle['kernels']]}")


if __name__ == "__main__":
    main()
