"""A/B throughput of the C5 n=1008 decode for the library in $LDPCB_LIBRARY."""
import sys, os, torch
sys.path.insert(0, '.')
import paper_1202_1060_b200 as P
g = P.configs.c1_code(); s = P.configs.c1_schedules(g)['ndgsbp']
F = 1 << 18
x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 1, 0, F)
for fpc, th, fv in [(0,0,0),(2,192,1),(2,96,2)]:
    P.set_tuning(fpc, th, fv)
    for _ in range(2): P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{os.path.basename(P._lib.LIB_PATH)} fv {fv} fpc {fpc} th {th}: {F/ms*1e3:.3e} frames/s")
