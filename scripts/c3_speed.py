"""C3 (QC n=1944) decode throughput per schedule: 2^18 frames at 2.0 dB,
15 iterations with early stop, and 10 fixed iterations."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c3_code()
F = 1 << 18
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for name, s in P.configs.c3_schedules(g).items():
    for iters, es in ((15, True), (10, False)):
        P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"C3 {name} it={iters} es={es}: {F / ms * 1e3:.4e} frames/s  {P.plan(g, s, F)}", flush=True)
