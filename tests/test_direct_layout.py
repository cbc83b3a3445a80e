"""Host-side tables of the posterior-free resident kernel (csrc/host_direct.cpp)
checked without a GPU: the records are replayed in float64 exactly as
direct.cu reads them (holder cells carrying c2v + L, the other edges' cells,
one phase per group, two copies of the edge cells for flooding) and the
messages after n sub-iterations are compared with the oracle's
init_state + run_subiteration (decoder.hpp:39-52, 112-127)."""
import os

import numpy as np
import pytest

CLAMP = 30.0


def _fields(rec):
    """The 16-bit byte offsets of one 12-word CN record: two holder edges
    (own, r0, r1, L) then four other edges (own, r0, r1)."""
    w = rec.view(np.uint32)
    f = []
    for x in w[:10]:
        f += [int(x & 0xFFFF), int(x >> 16)]
    return [tuple(f[4 * k:4 * k + 4]) for k in range(2)], [tuple(f[8 + 3 * j:11 + 3 * j]) for j in range(4)]


def _boxplus_excl(x):
    """check_update (decoder.hpp:59-87) in float64: exclusion boxplus, clamped."""
    x = np.clip(x, -CLAMP, CLAMP)
    t = np.tanh(0.5 * x)
    out = np.empty_like(x)
    for k in range(len(x)):
        p = np.prod(np.delete(t, k))
        p = min(max(p, -1 + 1e-17), 1 - 1e-17)
        out[k] = np.clip(2.0 * np.arctanh(p), -CLAMP, CLAMP)
    return out


def replay(g, s, lay, llr, nsub):
    cb = 4 * lay["frames_per_thread"]
    buf = lay["buffer_cells"] * cb
    cells = np.zeros(lay["cells"], np.float64)
    L = np.clip(np.asarray(llr, np.float64), -CLAMP, CLAMP)

    def rd_cell(off):
        assert off % cb == 0 and 0 <= off // cb < lay["cells"], off
        return cells[off // cb]

    for v in range(g.n_vars):  # init_state: every c2v = 0, holder cells carry L
        cells[lay["l_base"] + lay["vn_pos"][v]] = L[v]
        cells[lay["vn_hold"][v] // cb] = L[v]
        if buf:
            cells[(lay["vn_hold"][v] + buf) // cb] = L[v]
    rec = lay["cn_rec"].reshape(-1, 12)
    rd = 0
    for sub in range(nsub):
        grp = sub % s.n_groups
        wr = buf - rd if buf else 0
        stores = []
        for i in range(lay["cn_off"][grp], lay["cn_off"][grp + 1]):  # Jacobi: every item reads the old state
            holders, others = _fields(rec[i])
            x, own, lh = [], [], []
            for (o, r0, r1, lf) in holders:
                own.append(o)
                lh.append(rd_cell(lf))
                x.append((rd_cell(r0 + rd) + rd_cell(r1 + rd)) + rd_cell(lf))
            for (o, r0, r1) in others:
                own.append(o)
                lh.append(0.0)
                x.append(rd_cell(r0 + rd) + rd_cell(r1 + rd))
            c = _boxplus_excl(np.array(x))
            stores += [(own[k] + wr, c[k] + lh[k]) for k in range(6)]
        for off, val in stores:
            cells[off // cb] = val
        if buf:
            rd = wr
    er = lay["edge_rec"].view(np.uint32).reshape(-1, 2)
    c2v = np.empty(g.n_edges)
    v2c = np.empty(g.n_edges)
    for e in range(g.n_edges):
        own, lf = int(er[e, 0] & 0xFFFF), int(er[e, 0] >> 16)
        r0, r1 = int(er[e, 1] & 0xFFFF), int(er[e, 1] >> 16)
        holder = lf != 0xFFFF
        l = rd_cell(lf) if holder else 0.0
        c2v[e] = rd_cell(own + rd) - l
        v2c[e] = np.clip(rd_cell(r0 + rd) + rd_cell(r1 + rd) + l, -CLAMP, CLAMP)
    return c2v, v2c


def _check(P, corc, g, s, seed, subs):
    lay = s.direct_layout()
    assert lay is not None
    og = corc.graph(g.n_vars, *g.csr())
    llr = corc.transmit_batch_f32(P.sigma2_from_ebn0(1.5, g.rate), seed, g.n_vars, 0, 1)[0]
    for nsub in subs:
        rc, rv = corc.run_subiterations(og, s.groups, llr.astype(np.float64), nsub)
        c2v, v2c = replay(g, s, lay, llr, nsub)
        assert np.abs(c2v - rc).max() < 1e-9, (nsub, np.abs(c2v - rc).max())
        assert np.abs(v2c - rv).max() < 1e-9, (nsub, np.abs(v2c - rv).max())
    return lay


@pytest.mark.parametrize("sched", ["ndgsbp", "gsbp", "bp"])
def test_direct_tables_replay_matches_the_oracle(P, corc, sched):
    g = P.configs.c1_code()
    s = P.configs.c1_schedules(g)[sched]
    lay = _check(P, corc, g, s, 5, (1, 2, s.n_groups + 1) if sched != "bp" else (1, 2, 3))
    E, n = g.n_edges, g.n_vars
    assert lay["frames_per_thread"] == 2 and lay["l_base"] + n == lay["cells"]
    assert lay["buffer_cells"] == (E if sched == "bp" else 0)  # flooding: two copies of the edge cells
    assert lay["l_base"] == (2 * E if sched == "bp" else E)
    # every VN has one holder edge, every CN holds exactly two (a perfect matching)
    off, cns, eids = g.csc()
    rowptr, _ = g.csr()
    held = np.zeros(g.n_checks, int)
    cell_of_edge = lay["edge_rec"].view(np.uint32).reshape(-1, 2)[:, 0] & 0xFFFF
    for v in range(n):
        mine = [e for e in eids[off[v]:off[v + 1]] if cell_of_edge[e] == lay["vn_hold"][v]]
        assert len(mine) == 1
        held[np.searchsorted(rowptr, mine[0], side="right") - 1] += 1
    assert np.all(held == 2)
    # cells are a permutation: no two edges share a cell, no two VNs an L position
    assert len(set(cell_of_edge.tolist())) == E and sorted(lay["vn_pos"].tolist()) == list(range(n))
    # bank colouring: random placement costs about 2.6 wavefronts per half-warp access
    assert 1.0 <= lay["wavefronts_per_access"] < 1.7


def test_direct_tables_random_groups_and_four_frames_per_thread(P, corc):
    """The reference's random non-disjoint grouping (CNs repeated in
    consecutive groups, uneven group sizes) and the 16-byte-cell layout."""
    g = P.TannerGraph.random_regular(504, 3, 6, 7)
    s = P.make_nondisjoint_schedule(g, 12, 0.4, 3)
    _check(P, corc, g, s, 9, (1, 5, 13))
    os.environ["LDPCB_DIRECT_FV"] = "4"
    try:
        s4 = P.GroupSchedule.windows(P.configs.c1_code(), 8, 84, 63, P.NONDISJOINT)
    finally:
        os.environ.pop("LDPCB_DIRECT_FV", None)
    lay = _check(P, corc, s4.graph, s4, 2, (1, 9))
    assert lay["frames_per_thread"] == 4


def test_direct_kernel_scope(P):
    """Where the tables are not built: VN degrees other than 3 / CN degrees
    other than 6 (C3), several groups of more than 96 CNs is a launch-time
    decision (tables exist), per-frame groupings."""
    g3 = P.configs.c3_code()
    assert P.configs.c3_schedules(g3)["ndgsbp"].direct_layout() is None
    g = P.configs.c1_code()
    assert P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25).direct_layout() is None
    assert P.GroupSchedule.windows(g, 4, 126, 126, P.DISJOINT).direct_layout() is not None
