"""Command-line harness over the B200 decoder, mirroring the reference's
`ldpc_cli simulate` and `ldpc_cli schedule` (proj/tools/ldpc_cli.cpp:63-193,
flags :195-262) with the same options, JSON-line records (json_io.hpp:15-55,
keys sorted as nlohmann::json prints them) and CSV mirror.

    python -m paper_1202_1060_b200.cli simulate --n 1008 --dv 3 --dc 6 \
        --sched ndgsbp --groups 8 --overlap 0.25 --snr 1.5 2.0 --max-iter 20
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 -m paper_1202_1060_b200.cli simulate ...

One GPU: the native sweep (ldpcb_run_sweep_host). Under torchrun: one rank
per GPU, frames of every wave sharded by id and the per-frame outcomes
all-gathered (sim.run_sweep_prefix), so records do not depend on the GPU
count. `--workers` is accepted for compatibility; results never depend on it.
The `ga` subcommand (Gaussian-approximation analysis) is not part of the
decoder path and is not provided.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

KINDS = {"bp": 0, "gsbp": 1, "ndgsbp": 2}


def _dump(obj, indent=None) -> str:
    if indent is None:
        return json.dumps(obj, separators=(",", ":"), sort_keys=True)
    return json.dumps(obj, indent=indent, sort_keys=True)


def _load_code(a):
    from . import api

    if a.code:
        with open(a.code) as f:
            return api.TannerGraph.parse_alist(f.read())
    if a.n <= 0 or a.dv <= 0 or a.dc <= 0:
        raise SystemExit("--code: give --code or the full --n/--dv/--dc triple")
    return api.TannerGraph.random_regular(a.n, a.dv, a.dc, a.seed_code)


def make_schedule(g, kind: int, groups: int, overlap: float, seed: int):
    """The harness's proto schedule (sim.hpp:72-82)."""
    from . import api

    if kind == api.FLOODING:
        return api.GroupSchedule.flooding(g)
    if kind == api.DISJOINT:
        return api.GroupSchedule.disjoint(g, groups, seed)
    return api.GroupSchedule.nondisjoint(g, groups, overlap, seed)


def schedule_to_json(s, seed: int, regroup: bool) -> dict:
    """json_io.hpp:15-25."""
    from . import api

    flood = s.kind == api.FLOODING
    return {
        "kind": s.name,
        "n_groups": s.n_groups,
        "overlap_ratio": s.overlap_ratio,
        "group_size": s.group_size,
        "seed": 0 if flood else seed,
        "regroup_each_iteration": False if flood else regroup,
        "groups": s.groups,
    }


def _csv_line(r) -> str:
    return "%.6g,%d,%d,%d,%d,%.8g,%.8g,%.6g,%.6g,%d,%.4g\n" % (
        r["ebn0_db"], r["frames"], r["bit_errors"], r["frame_errors"], r["converged_frames"], r["ber"], r["fer"],
        r["mean_iters_converged"] or 0.0, r["mean_iters_all"], r["iter_limit"], r["wall_seconds"])


def _record(d: dict) -> dict:
    """sim_result_to_json (json_io.hpp:37-55)."""
    keys = ("ebn0_db", "frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer",
            "mean_iters_converged", "mean_iters_all", "iter_limit", "wall_seconds")
    r = {"type": "sim", **{k: d[k] for k in keys}}
    if r["converged_frames"] == 0:
        r["mean_iters_converged"] = None
    return r


def run_simulate(a) -> int:
    import torch

    from . import api, sim

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    rank = int(os.environ.get("RANK", "0"))
    g = _load_code(a)
    kind = KINDS[a.sched]
    regroup = not a.no_regroup
    proto = make_schedule(g, kind, a.groups, a.overlap, a.seed_schedule)
    iter_limit = proto.iteration_budget(a.max_iter) if a.budgeted else a.max_iter
    sched = proto if kind == api.FLOODING else api.GroupSchedule.per_frame(
        g, kind, a.groups, a.overlap, a.seed_schedule, regroup)
    if a.dump_schedule and rank == 0:
        with open(a.dump_schedule, "w") as f:
            f.write(_dump(schedule_to_json(proto, a.seed_schedule, regroup), indent=2) + "\n")
    if world > 1:
        recs = [r.to_record() for r in sim.run_sweep_prefix(g, sched, a.snr, iter_limit, a.frames, a.min_errors,
                                                             a.seed_channel)]
    else:
        recs = [_record(d) for d in api.run_sweep_native(g, sched, a.snr, iter_limit, a.frames, a.min_errors,
                                                          a.seed_channel)]
    if rank == 0:
        out = open(a.out, "w") if a.out else sys.stdout
        csv = open(a.csv, "w") if a.csv else None
        if csv:
            csv.write("ebn0_db,frames,bit_errors,frame_errors,converged_frames,ber,fer,"
                      "mean_iters_converged,mean_iters_all,iter_limit,wall_seconds\n")
        for r in recs:
            out.write(_dump(r) + "\n")
            if csv:
                csv.write(_csv_line(r))
        if csv:
            csv.close()
        if a.out:
            out.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_schedule(a) -> int:
    """ldpc_cli.cpp:151-181."""
    g = _load_code(a)
    s = make_schedule(g, KINDS[a.sched], a.groups, a.overlap, a.seed_schedule)
    rec = schedule_to_json(s, a.seed_schedule, True)
    rec.update(type="schedule", n_checks=g.n_checks, n_vars=g.n_vars, iteration_budget=s.iteration_budget(a.max_iter),
               i_max=a.max_iter, group_sizes=[len(x) for x in s.groups])
    grp = s.groups
    rec["consecutive_overlaps"] = [len(set(grp[t]) & set(grp[t - 1])) for t in range(1, len(grp))]
    counts = s.measure_cocsg()
    rec["cocsg"] = {"transition_counts": counts, "average": sum(counts) / len(counts) if counts else None}
    text = _dump(rec, indent=2) + "\n"
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


def _code_args(p):
    p.add_argument("--code", default="", help="alist file with the parity-check matrix")
    p.add_argument("--n", type=int, default=0, help="codeword length for a random regular ensemble")
    p.add_argument("--dv", type=int, default=0, help="VN degree for a random regular ensemble")
    p.add_argument("--dc", type=int, default=0, help="CN degree for a random regular ensemble")
    p.add_argument("--seed-code", type=int, default=1, help="seed for the random ensemble draw")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ldpc_b200", description="Group-shuffled LDPC decoding on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("simulate", help="Monte-Carlo BER/FER sweep over AWGN")
    _code_args(s)
    s.add_argument("--sched", choices=list(KINDS), default="bp")
    s.add_argument("--groups", type=int, default=1)
    s.add_argument("--overlap", type=float, default=0.0)
    s.add_argument("--no-regroup", action="store_true")
    s.add_argument("--snr", type=float, nargs="+", required=True)
    s.add_argument("--max-iter", type=int, default=1000)
    s.add_argument("--budgeted", action="store_true")
    s.add_argument("--frames", type=int, default=10000000)
    s.add_argument("--min-errors", type=int, default=100)
    s.add_argument("--seed-channel", type=int, default=1)
    s.add_argument("--seed-schedule", type=int, default=2)
    s.add_argument("--workers", type=int, default=1)
    s.add_argument("--out", default="")
    s.add_argument("--csv", default="")
    s.add_argument("--dump-schedule", default="")
    c = sub.add_parser("schedule", help="Print one schedule and its statistics")
    _code_args(c)
    c.add_argument("--sched", choices=list(KINDS), default="bp")
    c.add_argument("--groups", type=int, default=1)
    c.add_argument("--overlap", type=float, default=0.0)
    c.add_argument("--seed-schedule", type=int, default=2)
    c.add_argument("--max-iter", type=int, default=1000)
    c.add_argument("--out", default="")
    a = ap.parse_args(argv)
    if a.cmd == "simulate":
        return run_simulate(a)
    return run_schedule(a)


if __name__ == "__main__":
    sys.exit(main())
