"""The CLI surface (ldpc_cli.cpp:63-193) and the JSON records
(json_io.hpp:15-55, data/schema/sim_result.schema.json). CPU only: the
`schedule` subcommand is host code; `simulate` runs in the GPU suite."""
import json
import os
import subprocess
import sys

import pytest

from paper_1202_1060_b200 import cli, sim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCHEMA = "/root/reference/proj/data/schema/sim_result.schema.json"


def _run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_1202_1060_b200.cli", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_schedule_subcommand_matches_reference(rorc):
    rec = json.loads(_run("schedule", "--n", "504", "--dv", "3", "--dc", "6", "--seed-code", "3", "--sched",
                          "ndgsbp", "--groups", "12", "--overlap", "0.4", "--seed-schedule", "123", "--max-iter",
                          "50"))
    cols = rorc.random_regular(504, 3, 6, 3)
    import numpy as np

    rg = rorc.graph(504, np.arange(0, 6 * 252 + 1, 6, dtype=np.int32), cols)
    groups, gsz = rorc.make_schedule(rg, 2, 12, 0.4, 123)
    assert rec["groups"] == groups and rec["group_size"] == gsz
    assert rec["iteration_budget"] == rorc.iteration_budget(252, 50, 2, 12, gsz, 0.4)
    counts = rorc.measure_cocsg(rg, groups)
    assert rec["cocsg"]["transition_counts"] == list(counts)
    assert rec["cocsg"]["average"] == pytest.approx(sum(counts) / len(counts), rel=1e-15)
    assert rec["type"] == "schedule" and rec["kind"] == "ndgsbp" and rec["regroup_each_iteration"] is True
    assert rec["group_sizes"] == [len(x) for x in groups] and rec["n_checks"] == 252 and rec["i_max"] == 50
    assert rec["consecutive_overlaps"] == [len(set(a) & set(b)) for a, b in zip(groups, groups[1:])]


def test_schedule_subcommand_flooding_and_alist(tmp_path):
    from paper_1202_1060_b200 import TannerGraph

    g = TannerGraph.random_regular(96, 3, 6, 5)
    p = tmp_path / "c.alist"
    p.write_text(g.serialize_alist())
    rec = json.loads(_run("schedule", "--code", str(p), "--sched", "bp", "--max-iter", "7"))
    assert rec["groups"] == [list(range(48))] and rec["n_groups"] == 1 and rec["iteration_budget"] == 7
    assert rec["cocsg"] == {"average": None, "transition_counts": []} and rec["regroup_each_iteration"] is False


def test_missing_code_source_is_an_error():
    r = subprocess.run([sys.executable, "-m", "paper_1202_1060_b200.cli", "schedule", "--n", "96"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "--code" in r.stderr


@pytest.mark.skipif(not os.path.exists(SCHEMA), reason="reference schema not present")
def test_sim_record_validates_against_reference_schema():
    import jsonschema

    schema = json.load(open(SCHEMA))
    for c in ([10, 3, 1, 9, 40, 31], [5, 0, 0, 0, 100, 0]):
        jsonschema.validate(sim.aggregate(c, 120, 2.0, 20, 0.5).to_record(), schema)
        d = sim.aggregate(c, 120, 2.0, 20, 0.5).to_record()
        jsonschema.validate(cli._record(d), schema)
    line = cli._dump(cli._record(sim.aggregate([10, 3, 1, 9, 40, 31], 120, 2.0, 20, 0.5).to_record()))
    assert line.startswith('{"ber":') and " " not in line  # nlohmann dump(): sorted keys, compact
