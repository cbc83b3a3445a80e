"""Decode time vs iteration count (fixed cost + per-iteration cost)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c1_code()
s = P.configs.c1_schedules(g)["ndgsbp"]
F = 1 << 18
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for it in (1, 2, 5, 10, 20):
    for _ in range(2):
        P.decode_batch(g, s, x, it, early_stop=False, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.decode_batch(g, s, x, it, early_stop=False, packed=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{os.path.basename(P._lib.LIB_PATH)} iters {it}: {ms:.3f} ms ({ms / F * 1e6:.3f} ns/frame)")
