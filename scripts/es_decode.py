"""One early-stop decode of the C1 code (NDGSBP, 2.0 dB, <= 20 iterations) for profiling:
prints frames/s and the mean iteration count."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c1_code()
F = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
db = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(db, g.rate), 1, 0, F)
s = P.configs.c1_schedules(g)["ndgsbp"]
for _ in range(2):
    r = P.decode_batch(g, s, x, 20, early_stop=True, packed=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    r = P.decode_batch(g, s, x, 20, early_stop=True, packed=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"early stop {db} dB: {F / ms * 1e3:.3e} frames/s, mean iterations {r["iterations"].float().mean().item():.2f}, {P.plan(g, s, F)}")
