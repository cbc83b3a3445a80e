"""A/B decode throughput on the C1 code: fixed 10 iterations (C5) and 20
iterations with early stop, per schedule, for the library in $LDPCB_LIBRARY
and the kernel selection in $AB_KERNEL."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c1_code()
F = 1 << 20
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
P.set_kernel(int(os.environ.get("AB_KERNEL", "0")))  # 1: posterior-based resident kernel, 0: library plan
tag = f"{os.path.basename(P._lib.LIB_PATH)} kernel={os.environ.get('AB_KERNEL', '0')}"
for name, s in P.configs.c1_schedules(g).items():
    for iters, es in ((10, False), (20, True)):
        for _ in range(2):
            P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{tag} {name} it={iters} es={es}: {F / ms * 1e3:.3e} frames/s  {P.plan(g, s, F)}")
