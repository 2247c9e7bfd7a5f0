"""Reference plans for extra parity shapes beyond BASELINE.json (long rows that
need the multi-warp row template, odd row counts), exported by the reference's
own compile_graph via oracle/_ref/ref_tool.  Build container only.

    python tests/golden/make_extra_plans.py
"""

import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from workloads import configs  # noqa: E402

EXTRA = {
    "ln_r64_c8192": configs.c1_layernorm(R=64, C=8192),
    "ln_r100_c3072": configs.c1_layernorm(R=100, C=3072),
    "ln_r37_c2048": configs.c1_layernorm(R=37, C=2048),
    "softmax_r16_c16384": configs.c2_softmax(B=1, H=2, S=8, L=16384),
    "softmax_r24_c4096": configs.c2_softmax(B=2, H=3, S=4, L=4096),
}


def main():
    out_dir = os.path.join(HERE, "plans_extra")
    os.makedirs(out_dir, exist_ok=True)
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    for name, doc in EXTRA.items():
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            f.write(configs.dumps(doc))
            path = f.name
        try:
            out = subprocess.run([tool, "plan", path], check=True, capture_output=True, text=True).stdout
        finally:
            os.unlink(path)
        b = json.loads(out)
        for k in b["kernels"]:
            k.pop("dump", None)
        with open(os.path.join(out_dir, name + ".json"), "w") as f:
            json.dump(b, f, separators=(",", ":"))
        print(name, b["fused_kernels"])


if __name__ == "__main__":
    main()
