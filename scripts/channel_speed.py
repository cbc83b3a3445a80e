"""Device channel (transmit_all_zero) cost next to the decode it feeds."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, g, s, F, it in (("C1", P.configs.c1_code(), None, 1 << 20, 10),
                          ("C4", P.configs.c4_code(), None, 8192, 10)):
    s = (P.configs.c1_schedules(g) if name == "C1" else P.configs.c4_schedules(g))["ndgsbp"]
    s2 = P.sigma2_from_ebn0(2.0, g.rate)
    x = torch.empty((F, g.n_vars), dtype=torch.float32, device="cuda")
    ch = timeit(lambda: P.transmit_all_zero(g.n_vars, s2, 1, 0, F, out=x))
    dec = timeit(lambda: P.decode_batch(g, s, x, it, early_stop=False, packed=True))
    sim = timeit(lambda: P.simulate(g, s, s2, 1, 0, F, it, early_stop=False))
    print(f"{name}: channel {ch:.2f} ms, decode {dec:.2f} ms, simulate {sim:.2f} ms for {F} frames")
