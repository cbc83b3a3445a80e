import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1202_1060_b200 as P
from oracle.oracle import best_available, COracle
orc = best_available(); print("oracle", orc.kind)
g = P.configs.c1_code(); og = orc.graph(g.n_vars, *g.csr())
for name, s in P.configs.c1_schedules(g).items():
    print(name, P.plan(g, s, 1000))
    sigma2 = P.sigma2_from_ebn0(2.0, g.rate)
    F = 2000
    llr = orc.transmit_batch_f32(sigma2, 1, g.n_vars, 0, F)
    out = P.decode_batch(g, s, torch.from_numpy(llr).cuda(), 20, early_stop=True, posterior=True)
    torch.cuda.synchronize()
    ref = orc.decode_batch(og, s.groups, llr, 20, early_stop=True, posterior=True)
    bits = out["bits"].cpu().numpy(); its = out["iterations"].cpu().numpy(); cv = out['converged'].cpu().numpy()
    same = (bits == ref["bits"]).all(1) & (its == ref["iterations"]) & (cv == ref['converged'])
    post = out['posterior'].cpu().numpy(); rp = ref['posterior']
    m = same & (cv == 1)
    rel = np.abs(post[m]-rp[m]) / np.maximum(np.abs(rp[m]), 1)
    mask = np.abs(rp[m]) < 30
    print(f"{name}: identical {same.mean():.5f}  FER gpu {(bits.sum(1)>0).mean():.4f} ref {(ref['bits'].sum(1)>0).mean():.4f} iters {its.mean():.3f}/{ref['iterations'].mean():.3f} max rel post {rel[mask].max():.2e}")
# device channel vs oracle
d = P.transmit_all_zero(g.n_vars, sigma2, 1, 0, 512); torch.cuda.synchronize()
h = orc.transmit_batch_f32(sigma2, 1, g.n_vars, 0, 512)
dd = d.cpu().numpy(); print("channel exact frac", (dd == h).mean(), "max abs diff", np.abs(dd-h).max())
# throughput quick
s = P.configs.c1_schedules(g)['ndgsbp']
F = 1 << 18
x = P.transmit_all_zero(g.n_vars, sigma2, 1, 0, F)
cnt = torch.zeros(6, dtype=torch.int64, device='cuda')
for fpc, th in [(0,0),(8,672),(8,1024),(4,256),(4,352),(4,512),(4,672),(2,256),(2,512),(1,128)]:
    P.set_tuning(fpc, th)
    for _ in range(2): P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): P.decode_batch(g, s, x, 10, early_stop=False, packed=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/3
    print(f"fpc {fpc} th {th} plan {P.plan(g,s,F)} {ms:.2f} ms -> {F/ms*1e3:.3e} frames/s {F/ms*1e3*504:.3e} info bits/s")
P.set_tuning(0,0)
