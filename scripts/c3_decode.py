"""One C3 (QC n=1944) NDGSBP decode for profiling: fixed 10 iterations (default) or <= 15 with early stop."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c3_code()
F = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
es = len(sys.argv) > 2 and sys.argv[2] == "es"
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
s = P.configs.c3_schedules(g)["ndgsbp"]
it = 15 if es else 10
P.decode_batch(g, s, x, it, early_stop=es, packed=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
P.decode_batch(g, s, x, it, early_stop=es, packed=True)
e1.record()
torch.cuda.synchronize()
print(f"C3 ndgsbp it={it} es={es}: {F / e0.elapsed_time(e1) * 1e3:.3e} frames/s {P.plan(g, s, F)}")
