"""Pins the CPU oracle (oracle/ldpc_oracle.c) before it is trusted as the
checker: bit-exact against the reference's own outputs committed in
tests/golden/ (made by tests/golden/make_golden.py from the unmodified
reference build) and, where oracle/_ref exists, against the reference live.
Also re-runs the reference test suite's known-answer tests and properties
(test_decoder.cpp, test_channel.cpp, test_schedule.cpp) on the oracle."""
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def csr_regular(cols, dc):
    m = len(cols) // dc
    return np.arange(0, dc * m + 1, dc, dtype=np.int32), np.asarray(cols, np.int32)


# ---------------------------------------------------------------- rng.hpp ---
def test_rng_streams_match_reference_golden(corc):
    import ctypes as C

    from oracle.oracle import _p

    z = load("rng")
    L = corc.lib

    class Rng(C.Structure):
        _fields_ = [("s", C.c_uint64 * 4), ("spare", C.c_double), ("has", C.c_int)]

    L.orc_rng_seed.argtypes = [C.POINTER(Rng), C.c_uint64]
    L.orc_rng_u64.argtypes = [C.POINTER(Rng)]
    L.orc_rng_u64.restype = C.c_uint64
    L.orc_rng_unit.argtypes = [C.POINTER(Rng)]
    L.orc_rng_unit.restype = C.c_double
    L.orc_rng_gauss.argtypes = [C.POINTER(Rng)]
    L.orc_rng_gauss.restype = C.c_double
    L.orc_rng_below.argtypes = [C.POINTER(Rng), C.c_uint64]
    L.orc_rng_below.restype = C.c_uint64
    for seed in (0, 1, 2024, 424242):
        for key, fn, cnt in (("u64", L.orc_rng_u64, 64), ("unit", L.orc_rng_unit, 64), ("gauss", L.orc_rng_gauss, 65)):
            r = Rng()
            L.orc_rng_seed(C.byref(r), seed)
            got = [fn(C.byref(r)) for _ in range(cnt)]
            want = z[f"{key}_{seed}"].tolist()
            assert got == want, (key, seed)
        r = Rng()
        L.orc_rng_seed(C.byref(r), seed)
        assert [L.orc_rng_below(C.byref(r), 7) for _ in range(64)] == z[f"below7_{seed}"].tolist()
    for (s, t), v in zip(z["mix_pairs"].tolist(), z["mix_values"].tolist()):
        assert corc.mix_seed(s, t) == v


# ------------------------------------------------------------ channel.hpp ---
def test_sigma2_known_answers(corc):
    # test_channel.cpp:9-22
    assert corc.sigma2_from_ebn0(0.0, 0.5) == pytest.approx(1.0, rel=1e-12)
    assert corc.sigma2_from_ebn0(1.163, 0.5) == pytest.approx(0.76506, abs=1e-4)
    assert math.sqrt(corc.sigma2_from_ebn0(1.163, 0.5)) == pytest.approx(0.87468, abs=1e-4)
    assert corc.sigma2_from_ebn0(1.730, 1 / 3) == pytest.approx(1.5 * 10 ** (-0.173), rel=1e-12)
    assert corc.sigma2_from_ebn0(1.730, 1 / 3) == pytest.approx(1.00714, abs=1e-4)
    for bad in (0.0, -0.3, 1.2):
        assert math.isnan(corc.sigma2_from_ebn0(1.0, bad))
    z = load("channel")
    for (e, r), s in zip(z["sigma_points"], z["sigma2"]):
        assert corc.sigma2_from_ebn0(e, r) == s


def test_channel_llr_bit_exact_and_survey_golden(corc):
    z = load("channel")
    s2 = corc.sigma2_from_ebn0(2.0, 0.5)
    assert s2 == 0.63095734448019325
    for f in range(4):
        assert np.array_equal(corc.transmit_all_zero(s2, 1, 1008, f), z["llr_seed1_2dB_n1008_f0to3"][f])
    first = corc.transmit_all_zero(s2, 1, 4, 0)
    np.testing.assert_array_equal(first, [2.6810207421069037, 7.4445939366339404, 0.90775133478171144,
                                          2.4754530637169747])


def test_channel_statistics(corc):
    # test_channel.cpp:60-84: L ~ N(2/sigma^2, 4/sigma^2) at sigma^2 = 1
    x = corc.transmit_batch_f32(1.0, 99, 1000, 0, 1000).astype(np.float64)
    assert abs(x.mean() - 2.0) / 2.0 < 0.005
    assert abs(x.var() - 4.0) / 4.0 < 0.015
    a = corc.transmit_all_zero(1.0, 1234, 64, 7)
    assert np.array_equal(a, corc.transmit_all_zero(1.0, 1234, 64, 7))
    assert not np.array_equal(a, corc.transmit_all_zero(1.0, 1234, 64, 8))


# ------------------------------------------------------------- tanner.hpp ---
def test_random_regular_bit_exact(corc):
    z = load("graphs")
    for key in z.files:
        if key.startswith("regular_"):
            n, dv, dc, seed = (int(t) for t in key.split("_")[1:])
            assert np.array_equal(corc.random_regular(n, dv, dc, seed), z[key]), key
    with pytest.raises(ValueError):
        corc.random_regular(5, 3, 6, 1)  # test_tanner.cpp:183-185


def test_graph_views_match_reference_layout(corc):
    # fig1: test_tanner.cpp:42-55 (CN-major edge ids, var_adj ascending)
    g = corc.graph(8, [0, 3, 6, 9, 11], [0, 1, 2, 1, 3, 4, 3, 5, 6, 5, 7])
    off, cns, eid = g.var_view()
    assert cns[off[3] : off[4]].tolist() == [1, 2]
    assert eid[off[3] : off[4]].tolist() == [4, 6]
    assert cns[off[7] : off[8]].tolist() == [3]
    for bad in ([0, 1], [0, 0], [0, 9]):
        with pytest.raises(ValueError):
            corc.graph(8, [0, 2], np.array(bad))


# ----------------------------------------------------------- schedule.hpp ---
def test_generate_groups_bit_exact(corc):
    z = load("schedules")
    for key in [k[4:] for k in z.files if k.startswith("off_")]:
        kind, n, cseed, G, r, seed = key.split("_")
        kind, n, G, r, seed = int(kind), int(n), int(G), float(r), int(seed)
        ov = r if kind == 2 else 0.0
        groups = corc.generate_groups(n // 2, G, ov, corc.mix_seed(seed, 1))
        off, cns = z[f"off_{key}"], z[f"cns_{key}"]
        assert groups == [cns[off[i] : off[i + 1]].tolist() for i in range(G)], key
        assert corc.iteration_budget(n // 2, 1000, kind, G, int(z[f"gs_{key}"]), ov) == int(z[f"budget_{key}"])


def test_paper_budget_627(corc):
    # acceptance.cpp criterion 5 / test_sim.cpp:62-73
    assert corc.iteration_budget(252, 1000, 2, 12, 34, 0.4) == 627
    assert corc.iteration_budget(252, 50, 2, 12, 34, 0.4) == 31
    assert corc.iteration_budget(252, 1000, 1, 12, 21, 0.0) == 1000


# ------------------------------------------------------------ decoder.hpp ---
def test_check_update_known_answers(corc):
    z = load("check_update")
    for i in range(3):
        assert np.array_equal(corc.check_update(z[f"kat{i}_in"]), z[f"kat{i}_out"])
    out = corc.check_update([1.7, -0.4])  # test_decoder.cpp:53-59
    assert out[0] == pytest.approx(-0.4, abs=1e-12) and out[1] == pytest.approx(1.7, abs=1e-12)
    out = corc.check_update([2.0, -1.0, 5.0])  # :61-68
    assert out[2] == pytest.approx(2 * math.atanh(math.tanh(1.0) * math.tanh(-0.5)), abs=1e-12)
    assert out[2] == pytest.approx(-0.7353257, abs=1e-4)
    out = corc.check_update([3.0, 0.0, -2.0])  # :70-78
    assert out[0] == 0.0 and out[2] == 0.0
    assert out[1] == pytest.approx(2 * math.atanh(math.tanh(1.5) * math.tanh(-1.0)), abs=1e-12)


def test_check_update_golden_and_properties(corc):
    z = load("check_update")
    rng = np.random.default_rng(7)
    for d, x, want in zip(z["deg"], z["v2c"], z["c2v"]):
        x, want = x[:d], want[:d]
        out = corc.check_update(x)
        assert np.array_equal(out, want)
        # sign rule and magnitude rule (test_decoder.cpp:203-235)
        sp = np.prod(np.sign(x))
        assert np.all(np.sign(out) == sp * np.sign(x))
        for k in range(d):
            assert abs(out[k]) <= np.min(np.abs(np.delete(x, k))) + 1e-9
        perm = rng.permutation(d)  # permutation invariance (:237-247)
        np.testing.assert_allclose(corc.check_update(x[perm]), out[perm], rtol=0, atol=1e-12)


def _golden_code(corc):
    z = load("decode_c1")
    return z, corc.graph(1008, z["c1_row_off"], z["c1_cols"])


@pytest.mark.parametrize("sched", ["ndgsbp", "gsbp", "bp"])
@pytest.mark.parametrize("mode", ["es20", "fix10"])
def test_decode_matches_reference_golden(corc, sched, mode):
    z, g = _golden_code(corc)
    off, cns = z[f"c1_{sched}_groups_off"], z[f"c1_{sched}_groups_cns"]
    groups = [cns[off[i] : off[i + 1]].tolist() for i in range(len(off) - 1)]
    es, iters = (True, 20) if mode == "es20" else (False, 10)
    for f in range(len(z["c1_llr"])):
        r = corc.decode(g, groups, z["c1_llr"][f].astype(np.float64), iters, early_stop=es)
        assert np.array_equal(np.packbits(r["bits"], bitorder="little"), z[f"c1_{sched}_{mode}_bits"][f])
        assert r["iterations"] == z[f"c1_{sched}_{mode}_iters"][f]
        assert r["converged"] == bool(z[f"c1_{sched}_{mode}_conv"][f])
        assert np.array_equal(r["posterior"].astype(np.float32), z[f"c1_{sched}_{mode}_post"][f])
        assert np.array_equal(r["trace"], z[f"c1_{sched}_{mode}_trace"][f])


def test_flooding_equals_single_group_and_forward_flow(corc):
    # test_decoder.cpp:114-127: after {c1, c2} the message v4 -> c3 = L4 + (c2 -> v4)
    g = corc.graph(8, [0, 3, 6, 9, 11], [0, 1, 2, 1, 3, 4, 3, 5, 6, 5, 7])
    llr = [0.3, -0.2, 1.0, -1.5, 0.7, 0.1, -0.4, 0.9]
    c2v, v2c = corc.run_subiterations(g, [[0, 1]], llr, 1)
    c2_to_v4 = 2 * math.atanh(math.tanh(0.5 * llr[1]) * math.tanh(0.5 * llr[4]))
    off, cns, eid = g.var_view()
    e_v4_c3 = eid[off[3] + 1]
    assert v2c[e_v4_c3] == pytest.approx(llr[3] + c2_to_v4, abs=1e-12)
    for e in eid[off[5] : off[6]]:
        assert v2c[e] == llr[5]
    c2v0, v2c0 = corc.run_subiterations(g, [[]], llr, 1)  # empty group (:104-112)
    assert np.all(c2v0 == 0)


def test_r0_nondisjoint_equals_disjoint(corc):
    # test_decoder.cpp:185-201 on the reference's own G=5 partition
    cols = corc.random_regular(60, 3, 6, 11)
    g = corc.graph(60, *csr_regular(cols, 6))
    groups = corc.generate_groups(30, 5, 0.0, corc.mix_seed(401, 1))
    for f in range(10):
        llr = corc.transmit_all_zero(corc.sigma2_from_ebn0(1.5, 0.5), 17, 60, f)
        a = corc.decode(g, groups, llr, 40, kind=1)
        b = corc.decode(g, groups, llr, 40, kind=2)
        assert np.array_equal(a["bits"], b["bits"]) and a["iterations"] == b["iterations"]
        assert np.array_equal(a["trace"], b["trace"])


def test_converged_implies_zero_syndrome(corc):
    # test_decoder.cpp:250-265
    cols = corc.random_regular(120, 3, 6, 77)
    off, c = csr_regular(cols, 6)
    g = corc.graph(120, off, c)
    groups = corc.generate_groups(60, 6, 0.4, corc.mix_seed(5, 1))
    s2 = corc.sigma2_from_ebn0(1.2, 0.5)
    seen = 0
    for f in range(200):
        r = corc.decode(g, groups, corc.transmit_all_zero(s2, 3, 120, f), 15)
        if r["converged"]:
            seen += 1
            rows = c.reshape(-1, 6)
            assert not np.any(np.bitwise_xor.reduce(r["bits"][rows], axis=1))
            assert r["trace"][r["iterations"] - 1] == 0
    assert seen > 0


# ---------------------------------------------- live reference comparisons ---
def test_oracle_equals_reference_live(corc, rorc):
    """Bit-identical decodes, including per-iteration regrouping (the
    reference's default schedule mode, decoder.hpp:153-156)."""
    cols = rorc.random_regular(120, 3, 6, 7)
    off, c = csr_regular(cols, 6)
    cg, rg = corc.graph(120, off, c), rorc.graph(120, off, c)
    groups = corc.generate_groups(60, 6, 0.4, corc.mix_seed(99, 1))
    s2 = corc.sigma2_from_ebn0(0.8, 0.5)
    for f in range(40):
        llr = corc.transmit_all_zero(s2, 12, 120, f)
        for regroup in (0, 1):
            a = corc.decode(g=cg, groups=groups, llr=llr, max_iters=25, kind=2, overlap=0.4, seed=99, regroup=regroup)
            b = rorc.decode(rg, groups, llr, 25, kind=2, overlap=0.4, seed=99, regroup=regroup, composed=True)
            assert np.array_equal(a["bits"], b["bits"]) and a["iterations"] == b["iterations"]
            assert np.array_equal(a["posterior"], b["posterior"]) and np.array_equal(a["trace"], b["trace"])
            c_ = rorc.decode(rg, groups, llr, 25, kind=2, overlap=0.4, seed=99, regroup=regroup)
            assert c_["iterations"] == a["iterations"] and c_["cn_updates"] == a["cn_updates"]


def test_oracle_simulate_equals_reference_run_sweep(corc, rorc):
    """Aggregation semantics (sim.hpp:162-181) with the harness's own
    schedule: flooding, no regrouping, max_frames reached before the
    error target."""
    cols = rorc.random_regular(120, 3, 6, 4)
    off, c = csr_regular(cols, 6)
    cg, rg = corc.graph(120, off, c), rorc.graph(120, off, c)
    res = rorc.run_sweep(rg, 0, 1, 0.0, 0, [2.5], 30, 0, 300, 10**6, 11, 12, 4)[0]
    s2 = corc.sigma2_from_ebn0(2.5, 0.5)
    cnt = corc.simulate(cg, [list(range(60))], s2, 11, 0, 300, 30, round_f32=False)
    assert cnt.tolist()[:4] == [res["frames"], res["bit_errors"], res["frame_errors"], res["converged_frames"]]
    assert cnt[4] / cnt[0] == pytest.approx(res["mean_iters_all"], rel=1e-12)


@pytest.mark.parametrize("kind,G,ov,regroup", [(2, 6, 0.4, 1), (1, 5, 0.0, 1), (2, 4, 0.25, 0)])
def test_oracle_per_frame_grouping_equals_reference_run_sweep(corc, rorc, kind, G, ov, regroup):
    """run_sweep's default grouping: every frame draws its own groups from
    mix_seed(schedule_seed, frame_id) and, when regrouping, redraws them each
    iteration (sim.hpp:113-117, decoder.hpp:153-156). Counters are exact."""
    from oracle.oracle import PerFrame

    cols = rorc.random_regular(120, 3, 6, 4)
    off, c = csr_regular(cols, 6)
    cg, rg = corc.graph(120, off, c), rorc.graph(120, off, c)
    res = rorc.run_sweep(rg, kind, G, ov, regroup, [1.5], 25, 0, 300, 10**6, 11, 77, 4)[0]
    s2 = corc.sigma2_from_ebn0(1.5, 0.5)
    cnt = corc.simulate(cg, PerFrame(kind, G, ov, 77, regroup), s2, 11, 0, 300, 25, round_f32=False)
    assert cnt.tolist()[:4] == [res["frames"], res["bit_errors"], res["frame_errors"], res["converged_frames"]]
    assert cnt[4] / cnt[0] == pytest.approx(res["mean_iters_all"], rel=1e-12)
    # and frame by frame against ldpc::decode with the frame's own schedule
    for f in (0, 1, 57):
        seed_f = rorc.mix_seed(77, f)
        groups, _ = rorc.make_schedule(rg, kind, G, ov, seed_f)
        llr = corc.transmit_all_zero(s2, 11, 120, f)
        a = rorc.decode(rg, groups, llr, 25, kind=kind, overlap=ov, seed=seed_f, regroup=regroup)
        b = corc.decode_batch(cg, PerFrame(kind, G, ov, 77, regroup), np.zeros((f + 1, 120), np.float32), 1)
        assert b["iterations"].shape == (f + 1,)
        cc = corc.decode(cg, groups, llr, 25, kind=kind, overlap=ov, seed=seed_f, regroup=regroup)
        assert np.array_equal(a["bits"], cc["bits"]) and a["iterations"] == cc["iterations"]
