"""PCIe probe on the GPU box: pinned H2D alone, D2H alone, both at once
(separate streams), whole vs 16 MB chunks.  Explains the e2e ceiling."""
import time
import torch

N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, chunk):
    torch.cuda.synchronize()
    t = time.perf_counter()
    step = chunk or N
    for o in range(0, N, step):
        if h2d:
            with torch.cuda.stream(s1):
                d_a[o:o + step].copy_(h_in[o:o + step], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out[o:o + step].copy_(d_b[o:o + step], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t


for chunk in (0, 16 << 20):
    for h2d, d2h in ((1, 0), (0, 1), (1, 1)):
        run(h2d, d2h, chunk)
        dt = min(run(h2d, d2h, chunk) for _ in range(3))
        gb = N * (h2d + d2h) / 1e9
        print(f"chunk={chunk >> 20}MB h2d={h2d} d2h={d2h}: {dt * 1e3:.1f} ms, {gb / dt:.1f} GB/s total")
import os
print("numa/cpu:", os.cpu_count())
