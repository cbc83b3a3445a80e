"""C4 (n=64800) early stop <= 30 iterations from the frame queue with lanes refilled every R-th
iteration (LDPCB_STREAM_REFILL), against fixed 30 iterations; counters must not depend on R.

    python scripts/c4_refill_sweep.py [frames] [ebn0 ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c4_code()
s = P.configs.c4_schedules(g)["ndgsbp"]
F = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
points = [float(x) for x in sys.argv[2:]] or [1.1, 1.3]


def timed(x, iters, es):
    P.decode_batch(g, s, x[:2048].contiguous(), iters, early_stop=es, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = torch.zeros(6, dtype=torch.int64, device="cuda")
    e0.record()
    P.decode_batch(g, s, x, iters, early_stop=es, packed=True, counters=cnt)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), cnt.cpu().tolist()


for ebn0 in points:
    x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(ebn0, g.rate), 1, 0, F)
    base = None
    for r in (1, 2, 3, 4, 6):
        os.environ["LDPCB_STREAM_REFILL"] = str(r)
        ms, c = timed(x, 30, True)
        base = base or c
        print(f"C4 {ebn0:.2f} dB refill every {r}: {F / ms * 1e3:10.1f} frames/s, mean it {c[4] / c[0]:.2f}, "
              f"counters {'same' if c == base else 'DIFFER'} {c}", flush=True)
    os.environ.pop("LDPCB_STREAM_REFILL", None)
    ms, c = timed(x, 30, False)
    print(f"C4 {ebn0:.2f} dB fixed 30      : {F / ms * 1e3:10.1f} frames/s", flush=True)
