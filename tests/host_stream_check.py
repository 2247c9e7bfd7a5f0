"""Helper for test_gpu_host_stream.py (run in a subprocess so that
SFX_HOST_CHUNK_BYTES is set before libsfx.so reads it): every small config,
the chained BERT layer and the reference's random graphs through the host
path with tiny chunks (many gates / completion counters per group), checked
like test_gpu_parity.py does."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import sfx_testlib as T  # noqa: E402
from paper_1811_05213_b200 import host as H  # noqa: E402
import test_gpu_parity as P  # noqa: E402


def main():
    ctx = H.Context(0)
    n = 0
    for name in ["C1", "C2", "C3", "C3b", "C4", "C4b", "C4t", "C5", "C5L"]:
        g, rep, _ = H.load_bundle(os.path.join(T.PLANS, f"{name}.small.json"))
        inputs = T.gen_inputs(g, 42, -1.0, 1.0)
        for rep_i in range(2):  # twice: the gate / done counters are reset per run
            outs, launched, _ = P._run(ctx, g, rep, inputs, "auto")
            assert launched == len(rep.kernels) + len(T.unfused_kernels(g, rep))
            if name == "C5L":  # the chained layer: criterion of test_encoder_layer_small
                ref32 = T.interpret(g, inputs, 0)["h2"]
                assert T.values_close(outs["h2"], ref32), T.mismatch_report(outs["h2"], ref32)
            else:
                bad = P._check(g, outs, inputs, strict=True)
                assert not bad, (name, bad)
        n += 1
    for stream in ["pipeline", "device"]:
        for case in P._eligible(stream):
            g = H.graph_from_json(case["bundle"]["graph"])
            rep = H.CompileReport.from_bundle(case["bundle"])
            inputs = T.gen_inputs(g, case["input_seed"])
            outs, _, _ = P._run(ctx, g, rep, inputs, "auto")
            bad = P._check(g, outs, inputs)
            assert not bad, (stream, case["bundle"]["stream"]["index"], bad)
            n += 1
    print("host-stream ok", n)


if __name__ == "__main__":
    main()
