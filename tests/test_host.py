"""Host-side logic of the product through its C ABI (no GPU needed): the
library loads and exports every declared symbol; code construction, alist
I/O and schedules are bit-exact with the reference (golden fixtures made
from the reference itself, and the live reference build where present)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def test_library_exports_every_header_symbol(P):
    from paper_1202_1060_b200 import _lib

    names = _lib.header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing
    assert _lib.lib.ldpcb_abi_version() == 1


def test_random_regular_bit_exact_with_reference(P):
    z = load("graphs")
    for key in z.files:
        if key.startswith("regular_"):
            n, dv, dc, seed = (int(t) for t in key.split("_")[1:])
            g = P.TannerGraph.random_regular(n, dv, dc, seed)
            assert np.array_equal(g.csr()[1], z[key]), key
            assert g.n_checks == n * dv // dc and g.max_check_degree == dc and g.max_var_degree == dv
    with pytest.raises(ValueError):
        P.TannerGraph.random_regular(5, 3, 6, 1)
    a, b, c = (P.TannerGraph.random_regular(60, 3, 6, s) for s in (42, 42, 43))
    assert a == b and not (a == c)


def test_graph_layout_matches_reference_views(P, corc):
    for n, seed in ((504, 1), (60, 42)):
        g = P.TannerGraph.random_regular(n, 3, 6, seed)
        og = corc.graph(n, *g.csr())
        off, cns, eid = og.var_view()
        goff, gcns, geid = g.csc()
        assert np.array_equal(off, goff) and np.array_equal(cns, gcns) and np.array_equal(eid, geid)


def test_build_from_check_lists_validation(P):
    g = P.TannerGraph.from_check_lists(8, [[0, 1, 2], [1, 3, 4], [3, 5, 6], [5, 7]])
    assert (g.n_vars, g.n_checks, g.n_edges) == (8, 4, 11)
    assert g.var_adj[3] == [1, 2] and g.var_edge_ids[3] == [4, 6] and g.var_adj[7] == [3]
    assert g.edge_id(1, 1) == 4
    for bad in ([[0, 1], [2]], [[0, 0], [1, 2]], [[0, 9], [1, 2]], [[0, 1], [1, 2]]):
        with pytest.raises(ValueError):
            P.TannerGraph.from_check_lists(4, bad)  # degree<2, repeat, range, isolated VN 3


def test_alist_round_trip_matches_reference(P):
    z = load("graphs")
    for name in ("fig1", "regular_n504_m252", "regular_n816_m544"):
        text = bytes(z[f"alist_{name}_text"]).decode()
        g = P.TannerGraph.parse_alist(text)
        assert g.n_vars == int(z[f"alist_{name}_n"])
        assert np.array_equal(g.csr()[0], z[f"alist_{name}_row_off"])
        assert np.array_equal(g.csr()[1], z[f"alist_{name}_cols"])
        assert g.serialize_alist() == text  # same canonical text as the reference
        assert P.TannerGraph.parse_alist(g.serialize_alist()) == g


@pytest.mark.parametrize(
    "text,kind,line",
    [
        ("8\n2 3\n", "malformed_header", 1),
        ("2 1\n2 3\n1 2\n3\n1\n1\n1 2 0\n", "length_mismatch", 6),
        ("2 1\n1 2\n1 1\n2\n1\n9\n1 2\n", "index_out_of_range", 6),
        ("4 2\n1 2\n1 1 1 1\n2 2\n1\n1\n2\n2\n1 3\n2 4\n", "transpose_mismatch", 9),
        ("3 1\n1 2\n1 0 1\n2\n1\n0\n1\n1 3\n", "degree_error", 3),
        ("2 1\n2 3\n1 1\n3\n", "edge_count_mismatch", 4),
        ("2 1\n1 2\n1 1\n2\n1\n1\n1 2\n7\n", "trailing_content", 8),
        ("2 1\n1 2\n1 1\n2\n1\n1\n", "truncated", 6),
        ("2 1\n1 x\n", "bad_token", 2),
        ("2 1\n1 2\n1 1\n2\n1\n1\n1 1\n", "duplicate_entry", 7),
    ],
)
def test_alist_error_kinds_and_lines(P, text, kind, line, request):
    with pytest.raises(P.AlistError) as ei:
        P.TannerGraph.parse_alist(text)
    assert ei.value.kind == kind and ei.value.line == line
    ref = None
    try:
        ref = request.getfixturevalue("rorc")
    except pytest.skip.Exception:
        pass
    if ref is not None:  # the reference parser agrees on kind and line
        r = ref.parse_alist(text)
        assert P.AlistError.KINDS[r["kind"]] == kind and r["line"] == line


def test_reference_schedules_bit_exact(P):
    z = load("schedules")
    for key in [k[4:] for k in z.files if k.startswith("off_")]:
        kind, n, cseed, G, r, seed = key.split("_")
        kind, n, cseed, G, r, seed = int(kind), int(n), int(cseed), int(G), float(r), int(seed)
        g = P.TannerGraph.random_regular(n, 3, 6, cseed)
        s = P.GroupSchedule.disjoint(g, G, seed) if kind == 1 else P.GroupSchedule.nondisjoint(g, G, r, seed)
        off, cns = z[f"off_{key}"], z[f"cns_{key}"]
        assert s.groups == [cns[off[i] : off[i + 1]].tolist() for i in range(G)], key
        assert s.group_size == int(z[f"gs_{key}"])
        assert s.iteration_budget(1000) == int(z[f"budget_{key}"])
        if G > 1:
            assert s.measure_cocsg() == z[f"cocsg_{key}"].tolist()


def test_schedule_paper_numbers(P):
    # test_schedule.cpp:50-95 and the paper's budget (acceptance criterion 5)
    g = P.TannerGraph.random_regular(504, 3, 6, 3)
    s = P.GroupSchedule.disjoint(g, 12, 17)
    assert [len(x) for x in s.groups] == [21] * 12
    s = P.GroupSchedule.nondisjoint(g, 12, 0.4, 123)
    assert s.group_size == 34 and [len(x) for x in s.groups] == [34] * 11 + [32]
    for t in range(1, 12):
        assert len(set(s.groups[t - 1]) & set(s.groups[t])) == 14
    assert s.iteration_budget(1000) == 627
    with pytest.raises(ValueError):
        P.GroupSchedule.nondisjoint(g, 12, 1.0, 1)
    with pytest.raises(ValueError):
        P.GroupSchedule.disjoint(g, 0, 1)


def test_baseline_codes(P):
    g = P.configs.c1_code()
    assert (g.n_vars, g.n_checks, g.n_edges) == (1008, 504, 3024)
    assert g.count_4cycles() == 0
    assert P.TannerGraph.random_regular(1008, 3, 6, 1).count_4cycles() > 0
    assert all(len(r) == 6 for r in g.check_adj) and all(len(a) == 3 for a in g.var_adj)
    assert g == P.TannerGraph.random_regular_girth6(1008, 3, 6, 1)
    q = P.configs.c3_code()
    assert (q.n_vars, q.n_checks) == (1944, 972)
    assert min(len(a) for a in q.var_adj) >= 2 and min(len(r) for r in q.check_adj) >= 2
    rows = np.array([len(r) for r in q.check_adj]).reshape(12, 81)
    assert np.all(rows == rows[:, :1])  # circulant blocks: row degree constant per block row
    big = P.configs.c4_code()
    assert (big.n_vars, big.n_checks, big.n_edges) == (64800, 32400, 194400)
    deg = np.diff(big.csc()[0])
    assert np.bincount(deg).tolist()[2:] == [32400, 25920, 0, 0, 0, 0, 6480]
    assert np.all(np.diff(big.csr()[0]) == 6)


def test_baseline_window_schedules(P):
    g = P.configs.c1_code()
    s = P.configs.c1_schedules(g)
    nd = s["ndgsbp"].groups
    assert len(nd) == 8 and all(len(x) == 84 for x in nd)
    assert nd[0] == list(range(84)) and nd[7] == [(441 + j) % 504 for j in range(84)]
    assert len(set(nd[6]) & set(nd[7])) == 21 and len(set(nd[7]) & set(nd[0])) == 21
    assert s["ndgsbp"].edge_updates_per_iter == 4032 and s["gsbp"].edge_updates_per_iter == 3024
    assert sorted(c for x in s["gsbp"].groups for c in x) == list(range(504))
    q = P.configs.c3_code()
    qs = P.configs.c3_schedules(q)["ndgsbp"]
    assert [len(x) for x in qs.groups] == [243] * 6
    assert qs.groups[5] == [(810 + j) % 972 for j in range(243)]


def test_decode_argument_errors_without_gpu(P):
    g = P.configs.c1_code()
    s = P.configs.c1_schedules(g)["ndgsbp"]
    from paper_1202_1060_b200 import _lib

    with pytest.raises(ValueError, match="max_iters"):
        _lib.check(_lib.lib.ldpcb_decode_host(g.handle, s.handle, 1, None, 0, 1, None, 0, None, None, None, None, None))
    with pytest.raises(ValueError):
        P.sigma2_from_ebn0(1.0, 0.0)
    assert P.sigma2_from_ebn0(2.0, 0.5) == 0.63095734448019325
    other = P.TannerGraph.random_regular(60, 3, 6, 1)
    so = P.GroupSchedule.flooding(other)
    with pytest.raises(ValueError, match="different code"):
        _lib.check(_lib.lib.ldpcb_decode_host(g.handle, so.handle, 1, None, 5, 1, None, 0, None, None, None, None, None))
    with pytest.raises(ValueError):
        P.set_tuning(3, 0)


def _py_stream(seed, frame):
    """Pure-Python restatement of Rng(mix_seed(seed, frame)) (rng.hpp:10-46)."""
    M = (1 << 64) - 1

    def splitmix(st):
        st = (st + 0x9E3779B97F4A7C15) & M
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return st, z ^ (z >> 31)

    st, a = splitmix(seed)
    st ^= (0xD1342543DE82EF95 * (frame + 1)) & M
    _, b = splitmix(st)
    st = a ^ b
    w = []
    for _ in range(4):
        st, z = splitmix(st)
        w.append(z)
    return w


def _py_step(w):
    M = (1 << 64) - 1
    w0, w1, w2, w3 = w
    t = (w1 << 17) & M
    w2 ^= w0
    w3 ^= w1
    w1 ^= w2
    w0 ^= w3
    w2 ^= t
    w3 = ((w3 << 45) | (w3 >> 19)) & M
    return [w0, w1, w2, w3]


def test_channel_stream_jump_ahead_matches_stepping(P):
    """The jump-ahead the device channel uses to start frame segments
    (host_rng.cpp) lands on the same xoshiro256 state as stepping draw by
    draw, at every distance (segment starts are multiples of an even L)."""
    import ctypes as C

    lib = P.api.lib
    lib.ldpcb_channel_stream_state.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
    for seed, frame in ((1, 0), (7, 12345), (2**63 + 5, 2**33)):
        w = _py_stream(seed, frame)
        targets = sorted({0, 1, 2, 255, 256, 257, 1000, 4097, 30000})
        done = 0
        for d in targets:
            while done < d:
                w = _py_step(w)
                done += 1
            out = (C.c_uint64 * 4)()
            assert lib.ldpcb_channel_stream_state(seed, frame, d, out) == 0
            assert list(out) == w, (seed, frame, d)


def test_decode_host_rejects_bad_host_buffers(P):
    """decode_host passes raw host pointers to ldpcb_decode_host, which reads
    fp32 LLRs and D2H-copies outputs of exact sizes: wrong dtypes, shapes
    or sizes are refused before the library is called (no GPU needed)."""
    g = P.TannerGraph.random_regular(60, 3, 6, 21)
    s = P.make_flooding_schedule(g)
    F = 4
    ok = np.zeros((F, 60), np.float32)
    with pytest.raises(ValueError, match="float32"):
        P.decode_host(g, s, np.zeros((F, 60)), 5)  # float64: the reference decoder's own LLR type
    with pytest.raises(ValueError, match="code length"):
        P.decode_host(g, s, np.zeros((F, 59), np.float32), 5)
    with pytest.raises(ValueError, match="contiguous"):
        P.decode_host(g, s, np.zeros((60, F), np.float32).T, 5)
    with pytest.raises(ValueError, match="bits"):
        P.decode_host(g, s, ok, 5, packed=True, bits=np.zeros((F, 60), np.uint8))  # unpacked size, packed layout
    with pytest.raises(ValueError, match="bits"):
        P.decode_host(g, s, ok, 5, packed=False, bits=np.zeros((F, 8), np.uint8))
    with pytest.raises(ValueError, match="posterior"):
        P.decode_host(g, s, ok, 5, posterior=np.zeros((F, 59), np.float32))
    with pytest.raises(ValueError, match="syndrome_trace"):
        P.decode_host(g, s, ok, 5, syndrome_trace=np.zeros((F, 4), np.int32))
    with pytest.raises(ValueError, match="iterations"):
        P.decode_host(g, s, ok, 5, iterations=np.zeros(F, np.int64))
    with pytest.raises(ValueError, match="converged"):
        P.decode_host(g, s, ok, 5, converged=np.zeros(F + 1, np.uint8))
    with pytest.raises(ValueError, match="counters"):
        P.decode_host(g, s, ok, 5, counters=np.zeros(6, np.int32))
    import torch

    with pytest.raises(ValueError, match="counters"):
        P.decode_batch(g, s, torch.zeros((F, 60)), 5, counters=torch.zeros(6, dtype=torch.int64))


def test_bench_fixture_matches_the_product_constructions(P):
    """bench.py's reference arm reads the C5 codes and windows from
    bench_fixtures/c5_workloads.npz (so that process never loads the
    product): the frozen arrays must be the ones the product builds."""
    z = np.load(os.path.join(os.path.dirname(GOLDEN), "..", "bench_fixtures", "c5_workloads.npz"))
    for key, g, s in (("c5_n1008", P.configs.c1_code(), "c1"), ("c5_n64800", P.configs.c4_code(), "c4")):
        sch = (P.configs.c1_schedules(g) if s == "c1" else P.configs.c4_schedules(g))["ndgsbp"]
        off, cols = g.csr()
        assert int(z[f"{key}_n"]) == g.n_vars
        assert np.array_equal(z[f"{key}_row_off"], off) and np.array_equal(z[f"{key}_cols"], cols)
        flat = [c for grp in sch.groups for c in grp]
        assert np.array_equal(z[f"{key}_grp_cns"], flat)
        assert int(z[f"{key}_edge_updates_per_iter"]) == sch.edge_updates_per_iter
