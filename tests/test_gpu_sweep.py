"""run_sweep on the device (sim.hpp:96-186): waves, the min-frame-errors
prefix stop, SimResult records, and the CLI's simulate subcommand."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def test_native_sweep_equals_python_waves(P, torch):
    """ldpcb_run_sweep_host and sim.run_sweep_prefix (the multi-GPU path at
    world size 1, different wave sizes) stop at the same frame."""
    from paper_1202_1060_b200 import sim

    g = P.configs.c1_code()
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 2, True)
    nat = P.run_sweep_native(g, s, [1.25, 1.75], 20, 200000, 150, 1)
    py = sim.run_sweep_prefix(g, s, [1.25, 1.75], 20, 200000, 150, 1)
    small = P.run_sweep_native(g, s, [1.25], 20, 200000, 150, 1, wave_frames=1000)
    for a, b in zip(nat, py):
        b = b.to_record()
        for k in ("frames", "bit_errors", "frame_errors", "converged_frames", "iter_limit"):
            assert a[k] == b[k], k
        assert a["frame_errors"] == 150 and a["frames"] < 200000
    assert all(small[0][k] == nat[0][k] for k in ("frames", "bit_errors", "converged_frames"))
    # max_frames reached before the error target
    capped = P.run_sweep_native(g, s, [2.5], 20, 3000, 10**6, 1)[0]
    assert capped["frames"] == 3000 and capped["frame_errors"] < 10**6


def test_native_sweep_matches_reference_run_sweep(P, torch, rorc):
    """Against the unmodified reference harness (fp64, per-frame regrouping):
    identical stop index and counts up to the <0.1% of chaotic frames."""
    g = P.TannerGraph.random_regular(504, 3, 6, 3)
    rg = rorc.graph(504, *g.csr())
    for kind, G, ov in ((2, 12, 0.4), (1, 8, 0.0), (0, 1, 0.0)):
        s = P.GroupSchedule.per_frame(g, kind, G, ov, 2, True)
        ref = rorc.run_sweep(rg, kind, G, ov, 1, [1.5], 20, 0, 100000, 60, 1, 2, os.cpu_count() or 8)[0]
        got = P.run_sweep_native(g, s, [1.5], 20, 100000, 60, 1)[0]
        assert got["frame_errors"] == ref["frame_errors"] == 60
        assert abs(got["frames"] - ref["frames"]) <= 2
        assert abs(got["bit_errors"] - ref["bit_errors"]) <= 0.03 * ref["bit_errors"]
        assert got["mean_iters_all"] == pytest.approx(ref["mean_iters_all"], rel=0.02)


def test_cli_simulate(P, torch, tmp_path):
    out, csv = tmp_path / "r.jsonl", tmp_path / "r.csv"
    dump = tmp_path / "s.json"
    r = subprocess.run([sys.executable, "-m", "paper_1202_1060_b200.cli", "simulate", "--n", "1008", "--dv", "3",
                        "--dc", "6", "--sched", "ndgsbp", "--groups", "8", "--overlap", "0.25", "--snr", "1.5", "2.0",
                        "--max-iter", "20", "--budgeted", "--frames", "20000", "--min-errors", "40", "--out", str(out),
                        "--csv", str(csv), "--dump-schedule", str(dump)], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    recs = [json.loads(x) for x in out.read_text().splitlines()]
    assert [x["ebn0_db"] for x in recs] == [1.5, 2.0] and all(x["type"] == "sim" for x in recs)
    g = P.TannerGraph.random_regular(1008, 3, 6, 1)
    budget = P.GroupSchedule.nondisjoint(g, 8, 0.25, 2).iteration_budget(20)
    assert all(x["iter_limit"] == budget for x in recs) and budget < 20
    assert recs[0]["frame_errors"] == 40 or recs[0]["frames"] == 20000
    lines = csv.read_text().splitlines()
    assert lines[0].startswith("ebn0_db,frames,") and len(lines) == 3
    sch = json.loads(dump.read_text())
    assert sch["kind"] == "ndgsbp" and sch["groups"] == P.GroupSchedule.nondisjoint(g, 8, 0.25, 2).groups
