"""Quick GPU check: parity vs the oracle on C1 and a tuning sweep."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1202_1060_b200 as P
from oracle.oracle import best_available
orc = best_available(); print("oracle", orc.kind)
g = P.configs.c1_code(); og = orc.graph(g.n_vars, *g.csr())
sigma2 = P.sigma2_from_ebn0(2.0, g.rate)
F = 4000
llr = orc.transmit_batch_f32(sigma2, 1, g.n_vars, 0, F, 16)
for lazy in (1,):
    P.set_lazy_totals(lazy)
    for name, s in P.configs.c1_schedules(g).items():
        for es, iters in ((True, 20), (False, 10)):
            out = P.decode_batch(g, s, torch.from_numpy(llr).cuda(), iters, early_stop=es, posterior=True)
            torch.cuda.synchronize()
            ref = orc.decode_batch(og, s.groups, llr, iters, early_stop=es, posterior=True, threads=16)
            bits = out["bits"].cpu().numpy(); its = out["iterations"].cpu().numpy(); cv = out['converged'].cpu().numpy()
            same = (bits == ref["bits"]).all(1) & (its == ref["iterations"]) & (cv == ref['converged'])
            post = out['posterior'].cpu().numpy(); rp = ref['posterior']
            m = same & (cv == 1)
            rel = np.abs(post[m]-rp[m]) / np.maximum(np.abs(rp[m]), 1)
            mask = np.abs(rp[m]) < 30
            print(f"lazy={lazy} {name} es={es}: identical {same.mean():.5f} post within 1e-3 {(rel[mask] <= 1e-3).mean():.6f} max {rel[mask].max():.2e}")
P.set_lazy_totals(0)
s = P.configs.c1_schedules(g)['ndgsbp']
F = 1 << 18
x = P.transmit_all_zero(g.n_vars, sigma2, 1, 0, F)
for lazy in (1,):
  P.set_lazy_totals(lazy)
  for fpc, th, fv in [(0,0,0),(2,96,2),(2,192,1),(4,192,2)]:
    P.set_tuning(fpc, th, fv)
    for _ in range(2): P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/3
    print(f"fv {fv} fpc {fpc} th {th} plan {P.plan(g,s,F)} {ms:.2f} ms -> {F/ms*1e3:.3e} frames/s {F/ms*1e3*504:.3e} info bits/s")
P.set_tuning(0,0); P.set_lazy_totals(0)
