"""One C3 (QC n=1944) NDGSBP decode, 10 fixed iterations, 2^16 frames at
2.0 dB: the launch an ncu capture of the wide-row resident kernel targets."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c3_code()
s = P.configs.c3_schedules(g)["ndgsbp"]
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, 1 << 16)
for _ in range(2):
    P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
torch.cuda.synchronize()
print("ok", P.plan(g, s, 1 << 16))
