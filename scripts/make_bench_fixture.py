#!/usr/bin/env python
"""Writes bench_fixtures/c5_workloads.npz: the two BASELINE config-5 codes
(C1 n=1008 girth>=6, C4 n=64800 irregular) as CSR check lists and their
NDGSBP window schedules as group offset/CN arrays.

bench.py's reference arm (`--impl reference`) reads this file so that the
reference process never loads the product library: the check lists are the
same arrays the product builds (configs.c1_code / c4_code, seed 1), frozen
here once. Re-run after any change to the host constructions:

    python scripts/make_bench_fixture.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1202_1060_b200 as P  # noqa: E402


def groups_csr(groups):
    off = np.zeros(len(groups) + 1, np.int32)
    off[1:] = np.cumsum([len(x) for x in groups])
    return off, np.array([c for x in groups for c in x], np.int32)


def main():
    out = {}
    for key, g, s, ebn0 in (
        ("c5_n1008", P.configs.c1_code(), None, 2.0),
        ("c5_n64800", P.configs.c4_code(), None, 1.1),
    ):
        s = (P.configs.c1_schedules(g) if key == "c5_n1008" else P.configs.c4_schedules(g))["ndgsbp"]
        row_off, cols = g.csr()
        goff, gcns = groups_csr(s.groups)
        out[f"{key}_n"] = np.int32(g.n_vars)
        out[f"{key}_row_off"] = np.asarray(row_off, np.int32)
        out[f"{key}_cols"] = np.asarray(cols, np.int32)
        out[f"{key}_grp_off"] = goff
        out[f"{key}_grp_cns"] = gcns
        out[f"{key}_ebn0"] = np.float64(ebn0)
        out[f"{key}_edge_updates_per_iter"] = np.int64(s.edge_updates_per_iter)
    path = os.path.join(ROOT, "bench_fixtures", "c5_workloads.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
