import os, sys, torch
sys.path.insert(0, ".")
import paper_1202_1060_b200 as P
g = P.configs.c4_code(); s = P.configs.c4_schedules(g)["ndgsbp"]
F = 8192
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.2, g.rate), 1, 0, F)
for rep in range(2):
    for pdl in ("0", "1"):
        os.environ["LDPCB_STREAM_PDL"] = pdl
        P.decode_batch(g, s, x, 30, packed=True); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = P.decode_batch(g, s, x, 30, packed=True); e1.record(); torch.cuda.synchronize()
        print(f"C4 early stop <=30 it 1.2 dB, PDL={pdl}: {e0.elapsed_time(e1):.1f} ms per {F} frames, mean it {r['iterations'].float().mean().item():.2f}")
