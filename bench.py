#!/usr/bin/env python
"""Throughput benchmark: BASELINE.json's metric (decoded info bits/s at fixed
iterations) on its throughput configuration (config 5), both codes.

Config 5 names two workloads, and the default run measures both:
  c5_n1008   the (3,6)-regular n=1008 code with 4-cycles removed, NDGSBP
             (8 windows of 84 CNs at stride 63), Eb/N0 = 2.0 dB: decoded by
             the shared-memory-resident kernel. The headline (top-level keys).
  c5_n64800  the irregular n=64800 code, NDGSBP (45 windows of 960 at stride
             720), Eb/N0 = 1.1 dB: decoded by the HBM-streamed kernels.
             Reported under "legs" with the same keys.
Both: exactly 10 iterations (no early stop). One step = one decode of a batch
of frames per GPU whose fp32 LLRs are already resident in HBM (generated on
the device with the reference's channel stream, frame ids sharded by rank),
followed by the NCCL allreduce of the int64[6] error / iteration counters.

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
                  [--workload c5|c5_n1008|c5_n64800]

Under torchrun each rank decodes its own frame range (weak scaling); rank 0
prints one JSON line. `--impl reference` runs the reference CPU decoder
(oracle/_ref: the unmodified reference headers, else the C port) on all host
cores on a bounded sample of the same workloads; that process reads the
codes from bench_fixtures/c5_workloads.npz and never loads the product.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# Shared-memory bank colouring of the resident kernel's tables (host-side, once
# per schedule handle, outside every timed region): 40000 annealing moves per CN
# (about 15 s per table set of the C1 schedule) instead of the library default of 4000.
os.environ.setdefault("LDPCB_BANK_ITERS", "40000")

METRIC = "decoded info bits/s at fixed iterations"
UNIT = "info bits/s"
MUFU_PER_EDGE = 3  # SASS-counted: 1 MUFU.EX2 + 2 MUFU.LG2 per CN-edge update (decoder.cu)
MUFU_PER_SM_CLK = 16
HBM_BYTES_PER_EDGE = 8  # streamed decoder: c2v read + write per CN-edge update (fp32)
HBM_BYTES_PER_TOUCH = 8  # posterior read + write per distinct VN a group touches (fp32)
DEFAULT_FRAMES = {"c5_n1008": 1 << 21, "c5_n64800": 32768}
FIXTURE = os.path.join(ROOT, "bench_fixtures", "c5_workloads.npz")
DESC = {
    "c5_n1008": "C5: (3,6)-regular n=1008 girth>=6 (seed 1), NDGSBP 8 windows x 84 CNs stride 63, Eb/N0 2.0 dB",
    "c5_n64800": ("C5: irregular n=64800 VN degrees {2:.5,3:.4,8:.1} d_c=6 (seed 1), NDGSBP 45 windows x 960 CNs "
                  "stride 720, Eb/N0 1.1 dB"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="c5", choices=["c5", "c5_n1008", "c5_n64800"],
                    help="c5 = both config-5 codes (n=1008 headline + n=64800 leg)")
    ap.add_argument("--frames", type=int, default=0, help="frames per step per GPU (0: per-workload default)")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=30.0, help="CPU sample duration per workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel", type=int, default=0,
                    help="0 library plan, 1 posterior-based resident, 2 HBM-streamed, 3 posterior-free resident (A/B)")
    ap.add_argument("--fpc", type=int, default=0, help="frames per CTA (0 = library plan)")
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (0 = library plan)")
    return ap.parse_args()


def leg_names(args):
    return ["c5_n1008", "c5_n64800"] if args.workload == "c5" else [args.workload]


def fixture(name):
    """(n, row_off, cols, groups, ebn0, edge_updates_per_iter) of a config-5
    workload from the committed fixture (scripts/make_bench_fixture.py)."""
    z = np.load(FIXTURE)
    off, cns = z[f"{name}_grp_off"], z[f"{name}_grp_cns"]
    groups = [cns[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]
    return (int(z[f"{name}_n"]), z[f"{name}_row_off"], z[f"{name}_cols"], groups, float(z[f"{name}_ebn0"]),
            int(z[f"{name}_edge_updates_per_iter"]))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


class CpuReference:
    """The reference decoder on all host threads (oracle/_ref when built, else
    the C port), fixed iterations, one bounded sample per call. Frame ids
    pull from an atomic counter inside the oracle (sim.hpp:136-150)."""

    def __init__(self, name, iters):
        from oracle.oracle import best_available

        self.orc = best_available()
        n, row_off, cols, self.groups, ebn0, _ = fixture(name)
        self.n, self.m = n, len(row_off) - 1
        self.K = n - self.m
        self.iters = iters
        self.g = self.orc.graph(n, row_off, cols)
        self.sigma2 = self.orc.sigma2_from_ebn0(ebn0, self.K / n)
        self.threads = os.cpu_count() or 1
        self._llr = None

    def llr(self, frames):
        if self._llr is None or len(self._llr) < frames:
            self._llr = self.orc.transmit_batch_f32(self.sigma2, 1, self.n, 0, frames, self.threads)
        return self._llr[:frames]

    def run(self, frames):
        """Decodes `frames` frames; returns the wall time."""
        x = self.llr(frames)
        t0 = time.perf_counter()
        self.orc.decode_batch(self.g, self.groups, x, self.iters, early_stop=False, threads=self.threads)
        return time.perf_counter() - t0

    def frames_for(self, seconds):
        """Frames that take about `seconds` (one calibration decode)."""
        cal = max(2 * self.threads, 16)
        dt = self.run(cal)
        return max(self.threads, int(cal * seconds / max(dt, 1e-6)))

    def baseline(self, seconds):
        """Timed samples until at least `seconds` of decoding -> cpu_baseline dict."""
        per = self.frames_for(seconds / 3)
        frames, dt = 0, 0.0
        while dt < seconds:
            dt += self.run(per)
            frames += per
        return {"value": frames * self.K / dt, "unit": UNIT, "cores": self.threads, "kind": self.orc.kind,
                "sample": f"{frames} frames of the same workload, {self.iters} fixed iterations ({dt:.1f} s, "
                          f"{self.threads} threads)"}


def reference_leg(args, name):
    ref = CpuReference(name, args.iters)
    per_step = max(args.cpu_seconds / max(args.steps, 1), 1.0)
    frames = int(ref.frames_for(per_step) * 1.15)  # the timed steps together exceed --cpu-seconds
    warm = max(ref.threads, frames // 4)
    for _ in range(args.warmup):
        ref.run(warm)
    times = [ref.run(frames) for _ in range(args.steps)]
    value = frames * ref.K / statistics.median(times)
    return {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "ms_per_step": statistics.median(times) * 1e3,
        "config": {"workload": DESC[name] + f", {args.iters} fixed iterations", "frames_per_step": frames,
                   "host_threads": ref.threads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.threads, "kind": ref.orc.kind,
                         "sample": f"{frames} frames per step x {args.steps} steps ({sum(times):.1f} s timed), "
                                   f"{args.warmup} warm-up steps of {warm} frames"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    names = leg_names(args)
    legs = {nm: reference_leg(args, nm) for nm in names}
    head = legs[names[0]]
    line = {
        "impl": "reference",
        **{k: head[k] for k in ("metric", "value", "unit")},
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference channel stream, seed 1)",
        "config": head["config"],
        "cpu_baseline": head["cpu_baseline"],
        "e2e": head["e2e"],
        "legs": {nm: legs[nm] for nm in names[1:]},
    }
    print(json.dumps(line), flush=True)


def measure_leg(args, name, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_1202_1060_b200 as P

    dev = torch.device("cuda", local)
    if name == "c5_n1008":
        g = P.configs.c1_code()
        s = P.configs.c1_schedules(g)["ndgsbp"]
        ebn0 = 2.0
    else:
        g = P.configs.c4_code()
        s = P.configs.c4_schedules(g)["ndgsbp"]
        ebn0 = 1.1
    sigma2 = P.sigma2_from_ebn0(ebn0, g.rate)
    P.set_tuning(args.fpc, args.threads)
    P.set_kernel(args.kernel if name == "c5_n1008" else 0)
    B = args.frames or DEFAULT_FRAMES[name]
    n = g.n_vars
    K = n - g.n_checks
    stream = torch.cuda.current_stream()

    # inputs resident in HBM: this rank's frame ids [rank*B, (rank+1)*B)
    llr = P.transmit_all_zero(n, sigma2, 1, rank * B, B)
    bits = torch.empty((B, (n + 7) // 8), dtype=torch.uint8, device=dev)
    its = torch.empty(B, dtype=torch.int32, device=dev)
    conv = torch.empty(B, dtype=torch.uint8, device=dev)
    counters = torch.zeros(6, dtype=torch.int64, device=dev)
    pl = P.plan(g, s, B)

    def step(ev=None):
        counters.zero_()
        if ev:
            ev[0].record(stream)
        P.api.check(P.api.lib.ldpcb_decode_device(
            g.handle, s.handle, B, P.api._vp(llr), args.iters, 0, P.api._vp(bits), 1, P.api._vp(its),
            P.api._vp(conv), None, None, P.api._vp(counters), P.api._stream()))
        if ev:
            ev[1].record(stream)
        if world > 1:
            dist.all_reduce(counters)  # NCCL: int64[6] counters across ranks

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = P.kernel_launches()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    launches = P.kernel_launches() - launches0
    elapsed_ms = t0.elapsed_time(t1)
    kernel_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    total_frames = B * args.steps * world
    value = total_frames * K / (elapsed_ms / 1e3)
    cnt = counters.cpu().tolist()

    # ---- roofline of the dominant kernel
    edge_updates = s.edge_updates_per_iter * args.iters * B
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    # DRAM bytes of the dominant kernel: dram__bytes_read.sum + dram__bytes_write.sum per frame from the
    # committed ncu capture of this workload (profiles/dram_bytes_per_frame.json), scaled to this launch
    traffic = None
    tf = os.path.join(ROOT, "profiles", "dram_bytes_per_frame.json")
    if os.path.exists(tf):
        try:
            rec = json.load(open(tf)).get(name)
            if rec:
                traffic = rec["bytes_per_frame"] * B / 1e9
        except (OSError, ValueError, KeyError):
            traffic = None
    if pl["kernel"] != 2:  # shared-memory resident (plan kernel 1x): SFU (MUFU) issue rate
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        achieved = edge_updates * MUFU_PER_EDGE / (kernel_ms / 1e3)
        peak = n_sm * MUFU_PER_SM_CLK * sm_max * 1e6
        roofline = {"bound": "sfu", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "GMUFU/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "note": f"{'decode_direct' if pl['kernel'] >= 20 else 'decode_resident'}: {MUFU_PER_EDGE} MUFU per CN-edge update x {s.edge_updates_per_iter} "
                            f"edge updates/iter x {args.iters} iters x {B} frames per launch / CUDA-event launch "
                            f"time {kernel_ms:.3f} ms; peak = {n_sm} SMs x {MUFU_PER_SM_CLK}/clk x {sm_max:.0f} MHz "
                            "(MEASURED_PEAKS sm_max_mhz)"}
    else:  # HBM-streamed: bytes
        # SURVEY 8(d) roofline A: I x (8 E_iter + 8 T_iter) + 4n + ceil(n/8)
        per_frame = (args.iters * (HBM_BYTES_PER_EDGE * s.edge_updates_per_iter + HBM_BYTES_PER_TOUCH * s.touched_per_iter)
                     + 4 * n + (n + 7) // 8)
        achieved = per_frame * B / (kernel_ms / 1e3)
        peak = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
        roofline = {"bound": "hbm", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "note": f"HBM-streamed decode ({pl['frames_per_cta']}-frame chunks, all its kernels): algorithmic "
                            f"{per_frame / 1e6:.2f} MB/frame = {args.iters} iters x ({HBM_BYTES_PER_EDGE} B x "
                            f"{s.edge_updates_per_iter} CN-edge updates + {HBM_BYTES_PER_TOUCH} B x "
                            f"{s.touched_per_iter} touched VNs) + LLR in + bits out, x {B} frames / CUDA-event time "
                            f"{kernel_ms:.3f} ms; peak = MEASURED_PEAKS hbm_gbs; traffic = ncu DRAM bytes of all "
                            "stream kernels per frame (profiles/dram_bytes_per_frame.json) x frames"}

    # ---- end to end through the host C-ABI call (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        Be = B
        h_llr = torch.empty((Be, n), dtype=torch.float32, pin_memory=True)
        h_llr.copy_(llr[:Be].cpu())
        h_bits = torch.empty((Be, (n + 7) // 8), dtype=torch.uint8, pin_memory=True)
        h_cnt = torch.zeros(6, dtype=torch.int64)
        for _ in range(2):
            P.decode_host(g, s, h_llr, args.iters, early_stop=False, packed=True, bits=h_bits, counters=h_cnt)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_steps = max(1, min(args.steps, 5))
        t_start = time.perf_counter()
        for _ in range(e_steps):
            h_cnt.zero_()
            P.decode_host(g, s, h_llr, args.iters, early_stop=False, packed=True, bits=h_bits, counters=h_cnt)
        e_dt = time.perf_counter() - t_start
        te = torch.tensor([e_dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_dt = float(te.item())
        # the host link alone: a bare pinned host -> device copy of the same LLR bytes
        d_tmp = torch.empty_like(llr[:Be])
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d_tmp.copy_(h_llr, non_blocking=True)
        c0.record(stream)
        for _ in range(3):
            d_tmp.copy_(h_llr, non_blocking=True)
        c1.record(stream)
        torch.cuda.synchronize()
        link_gbs = 3 * Be * n * 4 / (c0.elapsed_time(c1) / 1e3) / 1e9
        del d_tmp, h_llr, h_bits
        e2e = {"value": Be * e_steps * world * K / e_dt, "unit": UNIT, "h2d_bytes_per_step": Be * n * 4,
               "d2h_bytes_per_step": Be * ((n + 7) // 8) + 48,
               "api": "ldpcb_decode_host (pinned host LLRs in, packed bits + counters out)",
               "h2d_gbs": round(Be * n * 4 * e_steps / e_dt / 1e9, 2),
               "h2d_link_gbs": round(link_gbs, 2),
               "note": "h2d_gbs = LLR bytes / e2e step time; h2d_link_gbs = a bare pinned copy of the same bytes"}
    del llr

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = CpuReference(name, args.iters).baseline(args.cpu_seconds)

    return {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "ms_per_step": elapsed_ms / args.steps,
        "config": {
            "workload": DESC[name] + f", {args.iters} fixed iterations, no early stop",
            "frames_per_step_per_gpu": B,
            "parallelism": f"frames sharded over {world} GPU(s), NCCL allreduce of int64[6] counters",
            "l2": f"inputs ({B * n * 4 / 1e9:.1f} GB per GPU) larger than L2; no flush",
            "plan": pl,
        },
        "frames_per_s": total_frames / (elapsed_ms / 1e3),
        "edge_updates_per_s": edge_updates * args.steps * world / (elapsed_ms / 1e3),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "counters": dict(zip(P.COUNTER_NAMES, cnt)),
    }


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    names = leg_names(args)
    legs = {}
    for nm in names:
        legs[nm] = measure_leg(args, nm, world, rank, local)
        torch.cuda.empty_cache()

    if world > 1:
        dist.barrier()
    if rank == 0:
        head = legs[names[0]]
        line = {
            "metric": METRIC,
            "value": head["value"],
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (device port of the reference channel stream, seed 1)",
            **{k: head[k] for k in ("config", "frames_per_s", "edge_updates_per_s", "roofline", "cpu_baseline",
                                    "e2e", "gpu_launches", "clocks", "counters")},
            "legs": {nm: legs[nm] for nm in names[1:]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
