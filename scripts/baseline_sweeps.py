"""BASELINE configs 2-4 as Monte-Carlo sweeps: the B200 decoder at the full
BASELINE frame counts next to the reference CPU decoder on the first frames of
each point (same seeded channel stream), with the reference's 95 % intervals.

  python scripts/baseline_sweeps.py [--configs c2 c3 c4] [--out profiles/r01_baseline_sweeps.json]

Per (config, schedule, Eb/N0) point:
* b200: frames, BER, FER, mean iterations over all frames, decode time (device
  channel + decode, counters only);
* ref: the same on its first `ref_frames` frames (oracle/_ref: the unmodified
  reference decoder, all host threads), with Clopper-Pearson (FER), frame
  bootstrap (BER) and t (mean iterations) 95 % intervals;
* identical: fraction of those first frames whose hard decisions, iteration
  count and convergence flag match the reference exactly;
* inside_ci: whether each b200 estimate lies inside the reference interval.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_1060_b200 as P  # noqa: E402
from oracle.oracle import best_available  # noqa: E402

from scipy.stats import beta, t as student_t  # noqa: E402

CONFIGS = {
    # name: (code, schedules, cfg, reference frames per point)
    # reference samples sized as SURVEY 8(d) asks (>= 1e5 frames per C2 point)
    "c2": ("c1_code", "c1_schedules", P.configs.C2, 100000),
    "c3": ("c3_code", "c3_schedules", P.configs.C3, 40000),
    "c4": ("c4_code", "c4_schedules", P.configs.C4, 1024),
}


def clopper_pearson(k, n, a=0.05):
    lo = 0.0 if k == 0 else beta.ppf(a / 2, k, n - k + 1)
    hi = 1.0 if k == n else beta.ppf(1 - a / 2, k + 1, n - k)
    return float(lo), float(hi)


def bootstrap_ber(bit_err, n_bits, reps=2000, seed=0):
    rng = np.random.default_rng(seed)
    f = len(bit_err)
    est = []
    for _ in range(0, reps, 50):  # in slices: 1e5 frames x 2000 resamples would not fit in memory at once
        idx = rng.integers(0, f, size=(50, f))
        est.append(bit_err[idx].sum(axis=1) / (f * n_bits))
    est = np.concatenate(est)
    return float(np.quantile(est, 0.025)), float(np.quantile(est, 0.975))


def paired(g_err, r_err, g_be, r_be, g_it, r_it, n_bits):
    """The same frames decoded by both: McNemar's exact test on the frame-error
    disagreements, and the paired differences of bit errors and iterations."""
    from scipy.stats import binomtest

    b = int((g_err & ~r_err).sum())  # frame errors only on the B200
    c = int((~g_err & r_err).sum())  # only in the reference
    p = float(binomtest(b, b + c, 0.5).pvalue) if b + c else 1.0
    d_it = (g_it - r_it).astype(np.float64)
    return {"frame_error_only_b200": b, "frame_error_only_ref": c, "mcnemar_p": p,
            "ber_diff": float((g_be.sum() - r_be.sum()) / (len(g_be) * n_bits)),
            "iters_diff_mean": float(d_it.mean()), "iters_diff_ci": t_interval(d_it),
            "frames_with_any_difference": int(((g_be != r_be) | (g_it != r_it)).sum())}


def t_interval(x):
    m = float(np.mean(x))
    if len(x) < 2:
        return m, m
    h = float(student_t.ppf(0.975, len(x) - 1) * np.std(x, ddof=1) / math.sqrt(len(x)))
    return m - h, m + h


def run(names, out_path, threads):
    orc = best_available()
    results = {"oracle": orc.kind, "host_threads": threads, "points": []}
    for name in names:
        code_fn, sched_fn, cfg, ref_frames = CONFIGS[name]
        g = getattr(P.configs, code_fn)()
        scheds = getattr(P.configs, sched_fn)(g)
        og = orc.graph(g.n_vars, *g.csr())
        n, K = g.n_vars, g.n_vars - g.n_checks
        for sname, s in scheds.items():
            for ebn0 in cfg["ebn0_db"]:
                s2 = P.sigma2_from_ebn0(ebn0, g.rate)
                F, iters = cfg["frames"], cfg["max_iters"]
                # b200: device channel + decode over all frames
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                cnt = P.simulate(g, s, s2, P.configs.CHANNEL_SEED, 0, F, iters, early_stop=True).cpu().numpy()
                torch.cuda.synchronize()
                t_gpu = time.perf_counter() - t0
                b = {"frames": int(cnt[0]), "ber": cnt[1] / (cnt[0] * n), "fer": cnt[2] / cnt[0],
                     "mean_iters": cnt[4] / cnt[0], "seconds": t_gpu, "frames_per_s": cnt[0] / t_gpu}
                # reference on the first ref_frames frames of the same stream
                Fr = min(ref_frames, F)
                llr = orc.transmit_batch_f32(s2, P.configs.CHANNEL_SEED, n, 0, Fr, threads)
                t0 = time.perf_counter()
                ref = orc.decode_batch(og, s.groups, llr, iters, early_stop=True, threads=threads)
                t_ref = time.perf_counter() - t0
                be = ref["bits"].sum(axis=1).astype(np.int64)
                r = {"frames": Fr, "ber": float(be.sum() / (Fr * n)), "fer": float((be > 0).mean()),
                     "mean_iters": float(ref["iterations"].mean()), "seconds": t_ref, "frames_per_s": Fr / t_ref,
                     "fer_ci": clopper_pearson(int((be > 0).sum()), Fr), "ber_ci": bootstrap_ber(be, n),
                     "iters_ci": t_interval(ref["iterations"].astype(np.float64))}
                # per-frame identity on the shared frames
                gout = P.decode_batch(g, s, torch.from_numpy(llr).cuda(), iters, early_stop=True)
                gb = gout["bits"].cpu().numpy()
                same = ((gb == ref["bits"]).all(axis=1) & (gout["iterations"].cpu().numpy() == ref["iterations"])
                        & (gout["converged"].cpu().numpy() == ref["converged"]))
                gbe = gb.sum(axis=1).astype(np.int64)
                pair = paired(gbe > 0, be > 0, gbe, be, gout["iterations"].cpu().numpy(), ref["iterations"], n)
                inside = {
                    "fer": r["fer_ci"][0] <= b["fer"] <= r["fer_ci"][1],
                    "ber": r["ber_ci"][0] <= b["ber"] <= r["ber_ci"][1],
                    "mean_iters": r["iters_ci"][0] <= b["mean_iters"] <= r["iters_ci"][1],
                }
                pt = {"config": name, "schedule": sname, "ebn0_db": ebn0, "max_iters": iters, "n": n, "k": K,
                      "b200": b, "ref": r, "identical": float(same.mean()), "inside_ci": inside, "paired": pair}
                results["points"].append(pt)
                print(f"{name} {sname:6s} {ebn0:4.2f} dB | b200 {b['frames']:8d} fr FER {b['fer']:.3e} "
                      f"BER {b['ber']:.3e} it {b['mean_iters']:5.2f} ({b['frames_per_s']:.2e} fr/s) | ref {Fr:6d} fr "
                      f"FER {r['fer']:.3e} [{r['fer_ci'][0]:.2e},{r['fer_ci'][1]:.2e}] it {r['mean_iters']:5.2f} "
                      f"({r['frames_per_s']:.1f} fr/s) | identical {same.mean():.5f} inside {inside} | paired: FE only b200 "
                      f"{pair['frame_error_only_b200']} / only ref {pair['frame_error_only_ref']} (p {pair['mcnemar_p']:.2f}), "
                      f"d iters {pair['iters_diff_mean']:+.2e}", flush=True)
                json.dump(results, open(out_path, "w"), indent=1, default=float)
    return results


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2", "c3", "c4"])
    ap.add_argument("--out", default="gpurun_out/baseline_sweeps.json")
    args = ap.parse_args()
    run(args.configs, args.out, os.cpu_count() or 8)


if __name__ == "__main__":
    main()
