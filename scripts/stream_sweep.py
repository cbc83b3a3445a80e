"""Streamed decoder (C4/C5 n=64800) sweep: chunk size B (LDPCB_STREAM_CHUNK)
x frames per thread V (LDPCB_STREAM_V). One step = 8192 frames, NDGSBP, 10
fixed iterations; frames/s from CUDA events over 3 steps."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

sys.argv += [] 
import bench  # noqa: E402

g, s, ebn0, desc = bench.workload("c5_n64800")
F = int(os.environ.get("FRAMES", 8192))
x = P.transmit_all_zero(g.n_vars, bench.mean_sigma2(P, g, ebn0), 1, 0, F)
configs = [tuple(map(int, c.split("x"))) for c in os.environ.get("CONFIGS", "8192x4 4096x4 2048x4 1024x4 1024x1 2048x2 512x1").split()]
for B, V in configs:
    os.environ["LDPCB_STREAM_CHUNK"] = str(B)
    os.environ["LDPCB_STREAM_V"] = str(V)
    for _ in range(1):
        P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"B={B:5d} V={V}: {ms:7.2f} ms per {F} frames -> {F / ms * 1e3:.4e} frames/s "
          f"({F / ms * 1e3 * (g.n_vars - g.n_checks):.3e} info bits/s)", flush=True)
