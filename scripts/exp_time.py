"""C1 NDGSBP fixed 10 iterations, 2^20 frames resident in HBM: ms per decode
(the bench's kernel); used with timing-only experiment builds."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c1_code()
s = P.configs.c1_schedules(g)[os.environ.get("SCHED", "ndgsbp")]
F = 1 << 20
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for _ in range(2):
    P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
frac = F * 10 * s.edge_updates_per_iter * 3 / (ms / 1e3) / (148 * 16 * 1965e6)
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'base':8s} {ms:8.3f} ms  {F / ms * 1e3:.4e} frames/s  MUFU frac {frac:.3f}  "
      f"plan {P.plan(g, s, F)}")
