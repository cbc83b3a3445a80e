"""C3 (QC n=1944) decode throughput per schedule: 2^18 frames at 2.0 dB,
15 iterations with early stop, and 10 fixed iterations."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402

g = P.configs.c3_code()
F = 1 << 18
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for name, s in P.configs.c3_schedules(g).items():
    for iters, es in ((15, True), (10, False)):
        P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.decode_batch(g, s, x, iters, early_stop=es, packed=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        fps = F / ms * 1e3
        line = f"C3 {name} it={iters} es={es}: {fps:.4e} frames/s  {P.plan(g, s, F)}"
        if not es:  # fixed iterations: CN-edge updates/s and the MUFU fraction (3 MUFU per edge update)
            eu = fps * iters * s.edge_updates_per_iter
            peak = torch.cuda.get_device_properties(0).multi_processor_count * 16 * 1965e6
            line += f"  {eu:.3e} edge updates/s, {3 * eu / peak:.3f} of MUFU peak"
        print(line, flush=True)
