"""Resident-kernel plan sweep on the C1 code (NDGSBP, fixed 10 iterations):
frames/s per (frames per CTA, threads, frames per thread) given as
"fpc:threads:fv" arguments, plus the library's own plan first."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c1_code()
s = P.configs.c1_schedules(g)["ndgsbp"]
F = 1 << 20
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for spec in ["0:0:0"] + sys.argv[1:]:
    fpc, th, fv = (int(v) for v in spec.split(":"))
    P.set_tuning(fpc, th, fv)
    try:
        for _ in range(2):
            P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{spec} plan={P.plan(g, s, F)}: {F / ms * 1e3:.4e} frames/s")
    except Exception as e:  # noqa: BLE001
        print(f"{spec}: {e}")
P.set_tuning(0, 0, 0)
