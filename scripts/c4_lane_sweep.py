"""C4 early stop <= 30 it at 1.1 dB from the streamed frame queue: lanes (LDPCB_STREAM_CHUNK) x refill interval."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c4_code()
s = P.configs.c4_schedules(g)["ndgsbp"]
F = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.1, g.rate), 1, 0, F)


def timed(iters, es):
    P.decode_batch(g, s, x[:2048].contiguous(), iters, early_stop=es, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
    e1.record()
    torch.cuda.synchronize()
    return F / e0.elapsed_time(e1) * 1e3


for lanes in (2048, 3072, 4096, 6144, 8192):
    os.environ["LDPCB_STREAM_CHUNK"] = str(lanes)
    row = []
    for r in (3, 4, 8):
        os.environ["LDPCB_STREAM_REFILL"] = str(r)
        row.append(f"R={r}: {timed(30, True):9.1f}")
    print(f"lanes {lanes}: " + "  ".join(row), flush=True)
os.environ.pop("LDPCB_STREAM_CHUNK", None)
os.environ.pop("LDPCB_STREAM_REFILL", None)
print(f"fixed 30: {timed(30, False):9.1f}")
