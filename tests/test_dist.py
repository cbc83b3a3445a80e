"""The N>1 path on CPU: frames sharded by id over world_size=2 gloo ranks,
counters combined with one all_reduce, and the result identical to one
process decoding every frame (worker-count independence, test_sim.cpp:44-60).
The per-rank decode here is the CPU oracle standing in for the GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1202_1060_b200 import sim

FRAMES, EBN0, ITERS = 203, 1.5, 20


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_backend(n, rows, groups):
    from oracle.oracle import COracle

    orc = COracle()
    off = np.arange(0, 6 * len(rows) + 1, 6, dtype=np.int32)
    g = orc.graph(n, off, np.concatenate(rows).astype(np.int32))

    def run(ebn0, begin, count):
        s2 = orc.sigma2_from_ebn0(ebn0, 0.5)
        c = orc.simulate(g, groups, s2, 1, begin, count, ITERS, early_stop=True, round_f32=True, threads=2)
        return torch.tensor(c, dtype=torch.int64)

    return run


def _worker(rank, world, port, n, rows, groups, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = sim.run_point(_oracle_backend(n, rows, groups), n, EBN0, FRAMES, ITERS)
        if rank == 0:
            out.put(res.to_record())
    finally:
        dist.destroy_process_group()


def _code():
    from oracle.oracle import COracle

    orc = COracle()
    cols = orc.random_regular(120, 3, 6, 77)
    rows = [cols[6 * i : 6 * i + 6] for i in range(60)]
    groups = orc.generate_groups(60, 6, 0.4, orc.mix_seed(5, 1))
    return 120, rows, groups


def test_shard_partitions_frame_ids():
    for total in (0, 1, 7, 203, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [sim.shard(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == total
            for (b0, c0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + c0 == b1


def test_two_rank_gloo_matches_single_process():
    n, rows, groups = _code()
    single = sim.run_point(_oracle_backend(n, rows, groups), n, EBN0, FRAMES, ITERS).to_record()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, rows, groups, q)) for r in range(2)]
    for p in procs:
        p.start()
    rec = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in ("frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer", "mean_iters_all",
              "mean_iters_converged", "iter_limit"):
        assert rec[k] == single[k], k
    assert rec["frames"] == FRAMES and rec["type"] == "sim"


def test_record_schema_shape():
    r = sim.aggregate([10, 3, 1, 9, 40, 31], 120, 2.0, 20, 0.5)
    rec = r.to_record()
    assert set(rec) == {"type", "ebn0_db", "frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer",
                        "mean_iters_converged", "mean_iters_all", "iter_limit", "wall_seconds"}
    assert rec["ber"] == 3 / 1200 and rec["fer"] == 0.1 and rec["mean_iters_all"] == 4.0
    assert sim.aggregate([5, 0, 0, 0, 100, 0], 8, 0.0, 20, 0.0).to_record()["mean_iters_converged"] is None
    lo, hi = sim.clopper_pearson(10, 1000)
    assert lo < 0.01 < hi
    with pytest.raises(ValueError):
        sim.run_sweep(None, None, [], 10, 5, backend=lambda *a: None)


# ---------------------------------------- min-frame-errors prefix stop ----
MIN_ERR, MAX_FRAMES = 9, 5000


def _frames_backend(n, rows, groups):
    """Per-frame outcomes from the fp64 oracle on the reference's own fp64
    LLRs (run_frame, sim.hpp:111-124), as torch tensors like the GPU path."""
    from oracle.oracle import COracle

    orc = COracle()
    off = np.arange(0, 6 * len(rows) + 1, 6, dtype=np.int32)
    g = orc.graph(n, off, np.concatenate(rows).astype(np.int32))

    def run(ebn0, begin, count):
        s2 = orc.sigma2_from_ebn0(ebn0, 0.5)
        be, it, cv = (torch.zeros(count, dtype=torch.int32) for _ in range(3))
        for i in range(count):
            r = orc.decode(g, groups, orc.transmit_all_zero(s2, 1, n, begin + i), ITERS, kind=0)
            be[i], it[i], cv[i] = int(r["bits"].sum()), r["iterations"], int(r["converged"])
        return be, it, cv.to(torch.uint8)

    return run


def _prefix_worker(rank, world, port, n, rows, groups, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = sim.run_point_prefix(_frames_backend(n, rows, groups), n, 1.0, MAX_FRAMES, MIN_ERR, ITERS, wave_cap=64)
        if rank == 0:
            out.put(res.to_record())
    finally:
        dist.destroy_process_group()


def test_prefix_stop_matches_reference_run_sweep_on_two_ranks(rorc):
    """The stopping rule of sim.hpp:126-160 (smallest prefix with
    min_frame_errors frame errors), sharded over two gloo ranks, equals the
    reference's own run_sweep (flooding, so the groups are the reference's)."""
    n, rows, _ = _code()
    flood = [list(range(60))]
    cols = np.concatenate(rows).astype(np.int32)
    rg = rorc.graph(n, np.arange(0, 361, 6, dtype=np.int32), cols)
    ref = rorc.run_sweep(rg, 0, 1, 0.0, 0, [1.0], ITERS, 0, MAX_FRAMES, MIN_ERR, 1, 2, 2)[0]
    assert ref["frame_errors"] == MIN_ERR and ref["frames"] < MAX_FRAMES
    single = sim.run_point_prefix(_frames_backend(n, rows, flood), n, 1.0, MAX_FRAMES, MIN_ERR, ITERS, wave_cap=16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prefix_worker, args=(r, 2, port, n, rows, flood, q)) for r in range(2)]
    for p in procs:
        p.start()
    rec = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for got in (single.to_record(), rec):
        for k in ("frames", "bit_errors", "frame_errors", "converged_frames", "iter_limit"):
            assert got[k] == ref[k], k
        for k in ("ber", "fer", "mean_iters_all", "mean_iters_converged"):
            assert got[k] == pytest.approx(ref[k], rel=1e-12), k
