"""Device channel throughput (normals/s) for the BASELINE frame lengths at the
batch sizes the Monte-Carlo harness uses."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

for n, frames in ((1008, 1 << 20), (1944, 1 << 19), (64800, 1024), (64800, 8192)):
    x = torch.empty((frames, n), dtype=torch.float32, device="cuda")
    P.transmit_all_zero(n, 0.63, 1, 0, frames, out=x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.transmit_all_zero(n, 0.63, 1, 0, frames, out=x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"n={n} frames={frames}: {ms:.2f} ms, {frames * n / ms / 1e6:.3f} G normals/s, {frames / ms * 1e3:.3e} frames/s")
