"""C4 (n=64800) early stop <= 30 iterations: frame queue (lanes refilled at
iteration ends) against chunk mode (LDPCB_STREAM_QUEUE=0: every chunk runs
until its slowest frame stops) and against fixed 30 / fixed 10 iterations.
Decoded frames per second through decode_batch, LLRs resident in HBM.

    python scripts/c4_es_speed.py [frames] [ebn0 ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c4_code()
s = P.configs.c4_schedules(g)["ndgsbp"]
F = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
points = [float(x) for x in sys.argv[2:]] or [1.1]


def timed(x, iters, es):
    P.decode_batch(g, s, x[:2048].contiguous(), iters, early_stop=es, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = torch.zeros(6, dtype=torch.int64, device="cuda")
    e0.record()
    r = P.decode_batch(g, s, x, iters, early_stop=es, packed=True, counters=cnt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    c = cnt.cpu().tolist()
    return ms, c, r


for ebn0 in points:
    x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(ebn0, g.rate), 1, 0, F)
    rows = []
    for label, env, iters, es in (("queue <=30", "1", 30, True), ("chunks <=30", "0", 30, True),
                                  ("fixed 30", "1", 30, False), ("fixed 10", "1", 10, False)):
        os.environ["LDPCB_STREAM_QUEUE"] = env
        ms, c, r = timed(x, iters, es)
        rows.append((label, ms, c))
        print(f"C4 {ebn0:.2f} dB {label:12s}: {ms:9.1f} ms / {F} frames = {F / ms * 1e3:10.1f} frames/s, "
              f"mean it {c[4] / c[0]:.2f}, FER {c[2] / c[0]:.4f}, conv {c[3] / c[0]:.4f}", flush=True)
    os.environ.pop("LDPCB_STREAM_QUEUE", None)
    q, ch = rows[0][2], rows[1][2]
    print(f"  queue vs chunks: counters {'identical' if q == ch else 'differ'} ({q} / {ch})")
