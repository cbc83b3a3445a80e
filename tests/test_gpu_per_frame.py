"""Per-frame random grouping on the device: run_sweep's default schedule mode
(sim.hpp:113-117): frame f draws its groups from mix_seed(schedule_seed, f)
and, with regroup_each_iteration, redraws them every iteration
(decoder.hpp:153-156, schedule.hpp:121-127).

Group generation is integer work: bit-exact. Decodes follow the bars of
test_gpu_parity.py (>= 99.9% identical frames, posteriors within 1e-3)."""
import os

import numpy as np
import pytest

from test_gpu_parity import THREADS, cu, frame_parity, post_stats, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


CASES = [(2, 8, 0.25, True), (1, 8, 0.0, True), (2, 12, 0.4, False), (2, 3, 0.3, True)]


@pytest.mark.parametrize("kind,G,ov,regroup", CASES)
def test_device_groups_bit_exact(P, torch, corc, kind, G, ov, regroup):
    g = P.configs.c1_code()
    s = P.GroupSchedule.per_frame(g, kind, G, ov, 4242, regroup)
    M = g.n_checks
    for it in (1, 2, 9):
        dev = s.frame_groups(1000, 40, it).cpu().numpy()
        for f in range(40):
            want = corc.generate_groups(M, G, ov, corc.mix_seed(corc.mix_seed(4242, 1000 + f), it))
            assert [len(x) for x in want] == [len(x) for x in s.groups]
            assert np.array_equal(dev[f], np.concatenate(want)), (it, f)


def test_device_groups_large_m(P, torch, corc):
    """M = 972 rows of degree <= 16 (BASELINE config 3 code)."""
    g = P.configs.c3_code()
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 6, 0.3, 9, True)
    dev = s.frame_groups(0, 16, 3).cpu().numpy()
    for f in range(16):
        want = corc.generate_groups(g.n_checks, 6, 0.3, corc.mix_seed(corc.mix_seed(9, f), 3))
        assert np.array_equal(dev[f], np.concatenate(want))


def _per_frame_parity(P, torch, corc, g, kind, G, ov, regroup, ebn0, iters, F):
    from oracle.oracle import PerFrame

    s = P.GroupSchedule.per_frame(g, kind, G, ov, 31, regroup)
    og = corc.graph(g.n_vars, *g.csr())
    llr = corc.transmit_batch_f32(P.sigma2_from_ebn0(ebn0, g.rate), 5, g.n_vars, 0, F, THREADS)
    gpu = to_np(P.decode_batch(g, s, cu(torch, llr), iters, posterior=True))
    ref = corc.decode_batch(og, PerFrame(kind, G, ov, 31, regroup), llr, iters, threads=THREADS, posterior=True)
    same = frame_parity(gpu, ref)
    frac, worst = post_stats(gpu["posterior"], ref["posterior"], same & (ref["converged"] == 1))
    return same.mean(), frac, worst


@pytest.mark.parametrize("kind,G,ov,regroup", CASES)
def test_per_frame_decode_parity(P, torch, corc, kind, G, ov, regroup):
    g = P.configs.c1_code()
    same, frac, worst = _per_frame_parity(P, torch, corc, g, kind, G, ov, regroup, 2.0, 20, 2000)
    print(f"per-frame {kind}/{G}/{ov}/{regroup}: identical {same:.5f}, posteriors {frac:.6f} (max {worst:.2e})")
    assert same >= 0.999 and frac >= 0.9999


def test_per_frame_qc_parity(P, torch, corc):
    g = P.configs.c3_code()
    same, frac, _ = _per_frame_parity(P, torch, corc, g, P.NONDISJOINT, 6, 0.3, True, 2.0, 15, 1000)
    assert same >= 0.999 and frac >= 0.9999


def test_per_frame_flooding_is_flooding(P, torch):
    g = P.configs.c1_code()
    a = P.GroupSchedule.per_frame(g, P.FLOODING, 1, 0.0, 5, True)
    b = P.GroupSchedule.flooding(g)
    x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(2.0, g.rate), 3, 0, 500)
    ra, rb = to_np(P.decode_batch(g, a, x, 20)), to_np(P.decode_batch(g, b, x, 20))
    assert all(np.array_equal(ra[k], rb[k]) for k in ra)


def test_per_frame_simulate_counters_and_frame_ids(P, torch, corc):
    """simulate keys the groups by the true frame id: two halves equal the
    whole, and the counters agree with the oracle's run_frame aggregation."""
    from oracle.oracle import PerFrame

    g = P.configs.c1_code()
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 7, True)
    s2 = P.sigma2_from_ebn0(1.8, g.rate)
    whole = P.simulate(g, s, s2, 3, 0, 4000, 20).cpu().numpy()
    halves = (P.simulate(g, s, s2, 3, 0, 1500, 20) + P.simulate(g, s, s2, 3, 1500, 2500, 20)).cpu().numpy()
    assert np.array_equal(whole, halves)
    og = corc.graph(g.n_vars, *g.csr())
    ref = corc.simulate(og, PerFrame(2, 8, 0.25, 7, True), s2, 3, 0, 4000, 20, threads=THREADS)
    assert whole[0] == ref[0]
    assert abs(int(whole[2]) - int(ref[2])) <= 4 + 0.002 * ref[0]
    assert abs(int(whole[4]) - int(ref[4])) <= 0.002 * ref[4] + 20


@pytest.mark.parametrize("regroup,code", [(True, "c1"), (False, "c1"), (True, "c3")])
def test_per_frame_frame_queue_is_bit_identical(P, torch, regroup, code):
    """Early stop from a frame queue with per-frame groupings: a refilled slot
    stages its own frame's list for its own iteration, so every output
    (counters included) equals one frame set per CTA."""
    g = P.configs.c1_code() if code == "c1" else P.configs.c3_code()
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8 if code == "c1" else 6, 0.25, 17, regroup)
    llr = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.75, g.rate), 3, 0, 3001)
    outs = {}
    try:
        for mode in ("0", "2"):
            os.environ["LDPCB_FRAME_QUEUE"] = mode
            cnt = torch.zeros(6, dtype=torch.int64, device="cuda")
            r = to_np(P.decode_batch(g, s, llr, 20, posterior=True, trace=True, counters=cnt))
            r["counters"] = cnt.cpu().numpy()
            outs[mode] = r
    finally:
        os.environ.pop("LDPCB_FRAME_QUEUE", None)
    for k in outs["0"]:
        a, b = outs["0"][k], outs["2"][k]
        bad = np.nonzero((a != b).reshape(len(a), -1).any(axis=1))[0] if a.ndim else []
        assert np.array_equal(a, b), (k, bad[:8], len(bad))


def test_per_frame_two_frames_per_cta_padding(P, torch):
    """Two frames per CTA without the queue on an odd batch: the padding
    frame's list slots are zero-filled (its record loads stay in bounds) and
    every real frame decodes exactly as with one frame per CTA."""
    g = P.configs.c1_code()
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 23, True)
    llr = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.75, g.rate), 9, 0, 1001)
    outs = []
    try:
        os.environ["LDPCB_FRAME_QUEUE"] = "0"
        for fpc in (1, 2):
            P.set_tuning(fpc)
            assert P.plan(g, s, 1001)["frames_per_cta"] == fpc
            for _ in range(3):  # repeated: a stale list slot shows up intermittently
                outs.append(to_np(P.decode_batch(g, s, llr, 20, posterior=True, trace=True)))
    finally:
        P.set_tuning(0)
        os.environ.pop("LDPCB_FRAME_QUEUE", None)
    for r in outs[1:]:
        for k in outs[0]:
            assert np.array_equal(outs[0][k], r[k]), k
