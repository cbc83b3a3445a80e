"""Throughput of per-frame random groupings vs a fixed schedule (C1 code)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c1_code()
F = 1 << 20
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)


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


cases = {
    "fixed nd 8x84/63": P.configs.c1_schedules(g)["ndgsbp"],
    "per-frame nd G8 r.25 regroup": P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 3, True),
    "per-frame nd G8 r.25 fixed": P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 3, False),
    "per-frame gs G8 regroup": P.GroupSchedule.per_frame(g, P.DISJOINT, 8, 0.0, 3, True),
}
for name, s in cases.items():
    ms = timeit(lambda: P.decode_batch(g, s, x, 20, packed=True))
    print(f"{name}: {ms:.1f} ms, {F / ms * 1e3:.3e} frames/s  plan={P.plan(g, s, F)}")
    if "per-frame" in name:
        ms = timeit(lambda: s.frame_groups(0, F, 2))
        print(f"   generator alone: {ms:.2f} ms per iteration-list for {F} frames")
