import os, sys
import torch
sys.path.insert(0, ".")
import paper_1202_1060_b200 as P
g = P.configs.c1_code()
F = 1 << 20
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for regroup in (True, False):
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 3, regroup)
    for fpc, q in ((1, "0"), (2, "0"), (2, "1"), (4, "0")):
        os.environ["LDPCB_FRAME_QUEUE"] = q
        P.set_tuning(fpc)
        ms = timeit(lambda: P.decode_batch(g, s, x, 20, packed=True))
        print(f"regroup={regroup} fpc={fpc} queue={q}: {F / ms * 1e3:.3e} frames/s")
P.set_tuning(0)
