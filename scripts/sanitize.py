"""Small decodes over every kernel family and launch path (fixed and
early-stop, frame queue on and off, resident and streamed, per-frame
groupings): a quick fault check on odd batch sizes (padding frames, idle
queue slots). compute-sanitizer is not available on the GPU pool."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402

F = int(os.environ.get("SAN_FRAMES", "37"))
c1 = P.configs.c1_code()
c3 = P.configs.c3_code()
cases = [(c1, n, P.configs.c1_schedules(c1)[n]) for n in ("ndgsbp", "gsbp", "bp")]
cases += [(c3, "c3 nd", P.configs.c3_schedules(c3)["ndgsbp"])]
cases += [(c1, "per-frame regroup", P.GroupSchedule.per_frame(c1, P.NONDISJOINT, 8, 0.25, 3, True)),
          (c3, "c3 per-frame", P.GroupSchedule.per_frame(c3, P.NONDISJOINT, 6, 0.3, 3, True))]
for g, name, s in cases:
    x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.5, g.rate), 1, 0, F)
    for q in ("0", "2"):
        os.environ["LDPCB_FRAME_QUEUE"] = q
        for es in (True, False):
            r = P.decode_batch(g, s, x, 8, early_stop=es, posterior=True, trace=True)
            torch.cuda.synchronize()
    P.set_kernel(2)  # the HBM-streamed kernels on the same code
    if "per-frame" not in name:
        r = P.decode_batch(g, s, x, 8, early_stop=True, posterior=True, trace=True)
        torch.cuda.synchronize()
    P.set_kernel(0)
    print(name, "ok", flush=True)
os.environ.pop("LDPCB_FRAME_QUEUE", None)
c4 = P.configs.c4_code()
s4 = P.configs.c4_schedules(c4)["ndgsbp"]
x = P.transmit_all_zero(c4.n_vars, P.sigma2_from_ebn0(1.1, c4.rate), 1, 0, 6)
P.decode_batch(c4, s4, x, 2, early_stop=True, posterior=True)
torch.cuda.synchronize()
print("c4 ok")
