"""One early-stop decode of the C4 code through the streamed frame queue
(LDPCB_STREAM_CHUNK lanes, default 512) for an ncu launch list; with
LDPCB_STREAM_QUEUE=0 the chunk path, with --fixed fixed 30 iterations.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
        python scripts/c4_queue_profile.py [frames] [--fixed]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402

os.environ.setdefault("LDPCB_STREAM_CHUNK", "512")
g = P.configs.c4_code()
s = P.configs.c4_schedules(g)["ndgsbp"]
F = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2048
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.1, g.rate), 1, 0, F)
r = P.decode_batch(g, s, x, 30, early_stop="--fixed" not in sys.argv, packed=True)
torch.cuda.synchronize()
print("frames", F, "mean iterations", r["iterations"].float().mean().item())
