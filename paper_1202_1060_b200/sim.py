"""Monte-Carlo harness over the B200 decoder (the caller of the hot path).

Mirrors the reference harness (proj/include/ldpc/sim.hpp):
  SimResult               sim.hpp:42-54 (+ the JSON record of json_io.hpp:37-55)
  run_frame + aggregation sim.hpp:111-124, 162-181
Frames are keyed by id (channel stream mix_seed(seed, frame_id)), so results
do not depend on how frames are split across GPUs (test_sim.cpp:44-60).

Multi-GPU: one process per GPU; rank r of P decodes the contiguous frame ids
[r*F/P, (r+1)*F/P) and the int64[6] counters are combined with one
torch.distributed all_reduce (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import math
import time
from dataclasses import asdict, dataclass
from typing import Callable

COUNTERS = ("frames", "bit_errors", "frame_errors", "converged_frames", "iter_sum", "iter_sum_converged")


@dataclass
class SimResult:
    ebn0_db: float = 0.0
    frames: int = 0
    bit_errors: int = 0
    frame_errors: int = 0
    converged_frames: int = 0
    ber: float = 0.0
    fer: float = 0.0
    mean_iters_converged: float = 0.0  # 0 when no frame converged
    mean_iters_all: float = 0.0
    iter_limit: int = 0
    wall_seconds: float = 0.0

    def to_record(self) -> dict:
        """The reference's per-SNR JSON record (json_io.hpp:37-55)."""
        d = asdict(self)
        d = {"type": "sim", **d}
        if self.converged_frames == 0:
            d["mean_iters_converged"] = None
        return d


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous frame-id range of `rank` out of `world`."""
    begin = total * rank // world
    end = total * (rank + 1) // world
    return begin, end - begin


def aggregate(counters, n_vars: int, ebn0_db: float, iter_limit: int, wall: float) -> SimResult:
    """sim.hpp:169-182 from the six summed counters."""
    c = [int(x) for x in counters]
    frames, bit_errors, frame_errors, conv, iter_sum, iter_conv = c
    return SimResult(
        ebn0_db=ebn0_db,
        frames=frames,
        bit_errors=bit_errors,
        frame_errors=frame_errors,
        converged_frames=conv,
        ber=bit_errors / (frames * n_vars) if frames else 0.0,
        fer=frame_errors / frames if frames else 0.0,
        mean_iters_converged=iter_conv / conv if conv else 0.0,
        mean_iters_all=iter_sum / frames if frames else 0.0,
        iter_limit=iter_limit,
        wall_seconds=wall,
    )


def device_backend(code, sched, max_iters: int, early_stop: bool = True, channel_seed: int = 1):
    """Counters of frames [begin, begin+count) decoded on the current GPU
    (device channel + decoder, ldpcb_simulate_device)."""
    import torch

    from . import api

    def run(ebn0_db: float, begin: int, count: int):
        sigma2 = api.sigma2_from_ebn0(ebn0_db, code.rate)
        cnt = torch.zeros(6, dtype=torch.int64, device="cuda")
        api.simulate(code, sched, sigma2, channel_seed, begin, count, max_iters, early_stop, counters=cnt)
        return cnt

    return run


def run_point(backend: Callable, n_vars: int, ebn0_db: float, frames: int, iter_limit: int) -> SimResult:
    """One SNR point over `frames` frames, sharded over the default process
    group when torch.distributed is initialised."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    t0 = time.perf_counter()
    begin, count = shard(frames, rank, world)
    cnt = backend(ebn0_db, begin, count)
    if world > 1:
        dist.all_reduce(cnt)  # int64[6] sum: the only cross-GPU exchange
    vals = cnt.tolist() if isinstance(cnt, torch.Tensor) else list(cnt)
    return aggregate(vals, n_vars, ebn0_db, iter_limit, time.perf_counter() - t0)


def run_sweep(code, sched, ebn0_db, frames: int, max_iters: int, early_stop: bool = True, channel_seed: int = 1,
              backend: Callable | None = None) -> list[SimResult]:
    """SNR sweep with a fixed frame count per point (run_sweep, sim.hpp:96-186,
    with max_frames = frames and no min-error stop)."""
    if not ebn0_db:
        raise ValueError("need at least one Eb/N0 point")
    if frames < 1:
        raise ValueError("max_frames must be >= 1")
    be = backend or device_backend(code, sched, max_iters, early_stop, channel_seed)
    return [run_point(be, code.n_vars, e, frames, max_iters) for e in ebn0_db]


def frames_backend(code, sched, max_iters: int, channel_seed: int = 1):
    """Per-frame outcomes (bit_errors, iterations, converged) of frames
    [begin, begin+count) on the current GPU (ldpcb_simulate_frames_device)."""
    from . import api

    def run(ebn0_db: float, begin: int, count: int):
        sigma2 = api.sigma2_from_ebn0(ebn0_db, code.rate)
        return api.simulate_frames(code, sched, sigma2, channel_seed, begin, count, max_iters)

    return run


def _gather_wave(outcome, count: int, world: int):
    """Concatenate every rank's per-frame outcomes in frame order: one
    all_gather of an int32 [3, ceil(count/world)+1] block per rank (shard
    sizes differ by at most one frame)."""
    import torch
    import torch.distributed as dist

    be, it, cv = outcome
    width = count // world + 1
    mine = torch.zeros((3, width), dtype=torch.int32, device=be.device)
    n = be.numel()
    mine[0, :n], mine[1, :n], mine[2, :n] = be, it, cv.to(torch.int32)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    cols = [parts[r][:, : shard(count, r, world)[1]] for r in range(world)]
    return torch.cat(cols, dim=1).cpu().numpy()


def run_point_prefix(backend: Callable, n_vars: int, ebn0_db: float, max_frames: int, min_frame_errors: int,
                     iter_limit: int, wave_cap: int = 1 << 20) -> SimResult:
    """One Eb/N0 point with the reference's stopping rule (sim.hpp:126-160):
    frames 0,1,... in waves, stop at the smallest frame index whose prefix
    holds min_frame_errors frame errors, or at max_frames. Each wave is
    sharded across ranks and the per-frame outcomes are all-gathered in frame
    order, so the result does not depend on the GPU count or wave size."""
    import numpy as np
    import torch.distributed as dist

    if min_frame_errors < 1:
        raise ValueError("min_frame_errors must be >= 1")
    if max_frames < 1:
        raise ValueError("max_frames must be >= 1")
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    t0 = time.perf_counter()
    produced, stop, wave = 0, -1, min(4096 * world, wave_cap)
    c = np.zeros(6, np.int64)
    fe = 0
    while stop < 0:
        cnt = min(wave, max_frames - produced)
        b, k = shard(cnt, rank, world)
        out = backend(ebn0_db, produced + b, k)
        if world > 1:
            arr = _gather_wave(out, cnt, world)
        else:
            arr = np.stack([x.cpu().numpy().astype(np.int64) for x in out])
        be, it, cv = (np.asarray(x, np.int64) for x in arr)
        cum = fe + np.cumsum(be > 0)
        hit = np.flatnonzero(cum >= min_frame_errors)
        take = int(hit[0]) + 1 if hit.size else cnt
        be, it, cv = be[:take], it[:take], cv[:take]
        c += [take, be.sum(), (be > 0).sum(), cv.sum(), it.sum(), (it * cv).sum()]
        fe = int(c[2])
        produced += cnt
        if hit.size:
            stop = produced - cnt + take - 1
        elif produced >= max_frames:
            stop = max_frames - 1
        wave = min(2 * wave, wave_cap)
    return aggregate(c.tolist(), n_vars, ebn0_db, iter_limit, time.perf_counter() - t0)


def run_sweep_prefix(code, sched, ebn0_db, iter_limit: int, max_frames: int, min_frame_errors: int,
                     channel_seed: int = 1, backend: Callable | None = None) -> list[SimResult]:
    """run_sweep (sim.hpp:96-186) with its min-frame-errors stopping rule."""
    if not ebn0_db:
        raise ValueError("need at least one Eb/N0 point")
    be = backend or frames_backend(code, sched, iter_limit, channel_seed)
    return [run_point_prefix(be, code.n_vars, e, max_frames, min_frame_errors, iter_limit) for e in ebn0_db]


def clopper_pearson(k: int, n: int, alpha: float = 0.05) -> tuple[float, float]:
    """Exact binomial confidence interval (FER)."""
    from scipy.stats import beta

    lo = 0.0 if k == 0 else float(beta.ppf(alpha / 2, k, n - k + 1))
    hi = 1.0 if k == n else float(beta.ppf(1 - alpha / 2, k + 1, n - k))
    return lo, hi


def wilson(k: int, n: int, z: float = 1.959963984540054) -> tuple[float, float]:
    p = k / n
    den = 1 + z * z / n
    c = (p + z * z / (2 * n)) / den
    h = z * math.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / den
    return c - h, c + h
