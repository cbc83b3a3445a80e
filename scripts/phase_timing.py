"""CTA-level phase breakdown of decode_resident (debug build with
-DLDPCB_PHASE_TIMING, loaded through LDPCB_LIBRARY)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
os.environ.setdefault("LDPCB_LIBRARY", os.path.abspath("paper_1202_1060_b200/libldpc_b200_timing.so"))
import paper_1202_1060_b200 as P  # noqa: E402
from paper_1202_1060_b200 import _lib  # noqa: E402

fn = _lib.lib.ldpcb_debug_phase_cycles
fn.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 8)()

g = P.configs.c1_code()
F = 1 << 20
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for name, s in P.configs.c1_schedules(g).items():
    for fv in (1, 2):
        P.set_tuning(frames_per_thread=fv)
        P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
        torch.cuda.synchronize()
        fn(buf, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
        e1.record()
        torch.cuda.synchronize()
        fn(buf, 1)
        cn, fix, end, tot, groups, ctas, pro, epi = list(buf)[:8]
        print(f"{name} fv={fv}: {e0.elapsed_time(e1):.1f} ms plan={P.plan(g, s, F)} | per group phase: CN {cn / groups:.0f} "
              f"cyc, fix-up {fix / groups:.0f} cyc | per CTA: iteration-end {end / ctas:.0f}, total {tot / ctas:.0f} cyc, "
              f"groups {groups / ctas:.0f}, prologue {pro / ctas:.0f}, epilogue {epi / ctas:.0f} cyc")
P.set_tuning()
