"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Every array here is an output of the unmodified reference headers
(/root/reference/proj/include/ldpc, compiled into oracle/_ref/libldpc_ref.so
by oracle/Makefile) run in this container:

  python tests/golden/make_golden.py

Codes used by the B200 configurations (girth-6 regular, QC, irregular) are
not reference constructions; for those the fixtures store the product's own
check lists and the REFERENCE decoder's outputs on them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefOracle  # noqa: E402

REF_DATA = "/root/reference/proj/data"


def rng_fixture(ref: RefOracle) -> dict:
    out = {}
    for seed in (0, 1, 2024, 424242):
        out[f"u64_{seed}"] = ref.rng_draw(seed, 0, 64)
        out[f"unit_{seed}"] = ref.rng_draw(seed, 1, 64)
        out[f"gauss_{seed}"] = ref.rng_draw(seed, 2, 65)
        out[f"below7_{seed}"] = ref.rng_draw(seed, 3, 64, bound=7)
    pairs = np.array([[s, t] for s in (0, 1, 7, 2**63 + 5) for t in (0, 1, 2, 99, 2**40)], dtype=np.uint64)
    out["mix_pairs"] = pairs
    out["mix_values"] = np.array([ref.mix_seed(int(s), int(t)) for s, t in pairs], dtype=np.uint64)
    return out


def channel_fixture(ref: RefOracle) -> dict:
    pts = np.array([[0.0, 0.5], [1.163, 0.5], [1.730, 1.0 / 3.0], [2.0, 0.5], [2.4, 0.5], [1.1, 0.5]])
    sig = np.array([ref.sigma2_from_ebn0(e, r) for e, r in pts])
    s2 = ref.sigma2_from_ebn0(2.0, 0.5)
    llr = np.stack([ref.transmit_all_zero(s2, 1, 1008, f) for f in range(4)])
    return {"sigma_points": pts, "sigma2": sig, "llr_seed1_2dB_n1008_f0to3": llr}


def graphs_fixture(ref: RefOracle) -> dict:
    out = {}
    for n, dv, dc, seed in ((504, 3, 6, 1), (60, 3, 6, 42), (60, 3, 6, 43), (1008, 3, 6, 1), (24, 2, 3, 5)):
        out[f"regular_{n}_{dv}_{dc}_{seed}"] = ref.random_regular(n, dv, dc, seed)
    for name in ("fig1", "regular_n504_m252", "regular_n816_m544"):
        text = open(os.path.join(REF_DATA, name + ".alist")).read()
        parsed = ref.parse_alist(text)
        g = ref.graph(parsed["n"], parsed["row_off"], parsed["cols"])
        out[f"alist_{name}_n"] = np.array(parsed["n"])
        out[f"alist_{name}_row_off"] = parsed["row_off"]
        out[f"alist_{name}_cols"] = parsed["cols"]
        # serialize_alist(parse_alist(file)): the reference's own canonical text
        out[f"alist_{name}_text"] = np.frombuffer(ref.serialize_alist(g).encode(), dtype=np.uint8)
    return out


def schedules_fixture(ref: RefOracle) -> dict:
    out = {}
    cases = [(504, 3, 12, 0.0, 17, 1), (504, 3, 12, 0.4, 123, 2), (60, 4, 5, 0.0, 77, 2), (60, 4, 5, 0.0, 77, 1),
             (90, 8, 4, 0.3, 9, 2), (8, 1, 3, 0.5, 11, 2), (504, 3, 8, 0.25, 2, 2)]
    for n, cseed, G, r, seed, kind in cases:
        cols = ref.random_regular(n, 3, 6, cseed)
        m = n // 2
        g = ref.graph(n, np.arange(0, 6 * m + 1, 6, dtype=np.int32), cols)
        groups, gs = ref.make_schedule(g, kind, G, r, seed)
        key = f"{kind}_{n}_{cseed}_{G}_{r}_{seed}"
        off = np.zeros(len(groups) + 1, np.int32)
        off[1:] = np.cumsum([len(x) for x in groups])
        out[f"off_{key}"] = off
        out[f"cns_{key}"] = np.array([c for x in groups for c in x], np.int32)
        out[f"gs_{key}"] = np.array(gs)
        out[f"budget_{key}"] = np.array(ref.iteration_budget(m, 1000, kind, G, gs, r))
        out[f"cocsg_{key}"] = np.array(ref.measure_cocsg(g, groups) or [0], np.int32)
    return out


def check_update_fixture(ref: RefOracle) -> dict:
    rng = np.random.default_rng(2024)
    rows, outs, degs = [], [], []
    for _ in range(2000):
        d = int(rng.integers(2, 13))
        mag = np.exp(np.log(1e-3) + rng.random(d) * np.log(8.0 / 1e-3))
        x = np.where(rng.random(d) < 0.5, -mag, mag)
        rows.append(np.pad(x, (0, 12 - d)))
        outs.append(np.pad(ref.check_update(x), (0, 12 - d)))
        degs.append(d)
    kat_in = [np.array([1.7, -0.4]), np.array([2.0, -1.0, 5.0]), np.array([3.0, 0.0, -2.0])]
    kat = {f"kat{i}_in": x for i, x in enumerate(kat_in)}
    kat.update({f"kat{i}_out": ref.check_update(x) for i, x in enumerate(kat_in)})
    return {"deg": np.array(degs), "v2c": np.array(rows), "c2v": np.array(outs), **kat}


def decode_fixture(ref: RefOracle, P) -> dict:
    out = {}
    g = P.configs.c1_code()
    off, cols = g.csr()
    out["c1_row_off"], out["c1_cols"] = off, cols
    sigma2 = ref.sigma2_from_ebn0(2.0, 0.5)
    frames = 32
    llr = ref.transmit_batch_f32(sigma2, 1, g.n_vars, 0, frames)
    out["c1_llr"] = llr
    rg = ref.graph(g.n_vars, off, cols)
    for name, s in P.configs.c1_schedules(g).items():
        out[f"c1_{name}_groups_off"] = np.cumsum([0] + [len(x) for x in s.groups]).astype(np.int32)
        out[f"c1_{name}_groups_cns"] = np.array([c for x in s.groups for c in x], np.int32)
        for mode, es, iters in (("es20", True, 20), ("fix10", False, 10)):
            bits, its, conv, post, trace = [], [], [], [], []
            for f in range(frames):
                r = ref.decode(rg, s.groups, llr[f].astype(np.float64), iters, early_stop=es, composed=True)
                bits.append(np.packbits(r["bits"], bitorder="little"))
                its.append(r["iterations"])
                conv.append(r["converged"])
                post.append(r["posterior"].astype(np.float32))
                trace.append(r["trace"])
            out[f"c1_{name}_{mode}_bits"] = np.array(bits)
            out[f"c1_{name}_{mode}_iters"] = np.array(its, np.int32)
            out[f"c1_{name}_{mode}_conv"] = np.array(conv, np.uint8)
            out[f"c1_{name}_{mode}_post"] = np.array(post)
            out[f"c1_{name}_{mode}_trace"] = np.array(trace, np.int32)
    return out


def main():
    import paper_1202_1060_b200 as P

    ref = RefOracle()
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng_fixture(ref))
    np.savez_compressed(os.path.join(HERE, "channel.npz"), **channel_fixture(ref))
    np.savez_compressed(os.path.join(HERE, "graphs.npz"), **graphs_fixture(ref))
    np.savez_compressed(os.path.join(HERE, "schedules.npz"), **schedules_fixture(ref))
    np.savez_compressed(os.path.join(HERE, "check_update.npz"), **check_update_fixture(ref))
    np.savez_compressed(os.path.join(HERE, "decode_c1.npz"), **decode_fixture(ref, P))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
