"""Decode throughput per schedule for a BASELINE code at its operating point
(early stop), with the library's plan: python scripts/code_speed.py c3 [frames]."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
code = {"c1": P.configs.c1_code, "c3": P.configs.c3_code, "c4": P.configs.c4_code}[name]()
scheds = {"c1": P.configs.c1_schedules, "c3": P.configs.c3_schedules, "c4": P.configs.c4_schedules}[name](code)
ebn0, iters = {"c1": (2.0, 20), "c3": (2.0, 15), "c4": (1.1, 30)}[name]
x = P.transmit_all_zero(code.n_vars, P.sigma2_from_ebn0(ebn0, code.rate), 1, 0, F)
for sname, s in scheds.items():
    for es, it in ((True, iters), (False, 10)):
        P.decode_batch(code, s, x, it, early_stop=es, packed=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.decode_batch(code, s, x, it, early_stop=es, packed=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{name} {sname} it={it} es={es}: {F / ms * 1e3:.3e} frames/s  {P.plan(code, s, F)}", flush=True)
