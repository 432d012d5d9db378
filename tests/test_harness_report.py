"""CPU tests of the report projections of the benchmark harness (paper_2304_08232_b200/harness.py): pure host
logic that mirrors /root/reference/proj/include/slab/report.hpp:128-360 (JSON document, CSV rows) and
test_bench.cpp:160-178; no GPU involved — the reports are built by hand."""
import json
import math

import pytest

from paper_2304_08232_b200 import _capi as slab
from paper_2304_08232_b200 import harness


def sample_report():
    cfg = harness.BenchConfig(dims=(8, 8, 8), levels=2, runs=2, fixed_iterations=4, seed=77)
    rep = harness.Report(config=cfg, generation_seconds=0.0123)
    rep.symmetry = harness.SymmetryReport(False, True, 1.5e-13, True, 3.25e-12, 4.0e-6)
    for run in range(2):
        levels = [harness.LevelTimings(0, 512, 1.25e-4 + run * 1e-7, 2.5e-5, 1.75e-4, 123456),
                  harness.LevelTimings(1, 64, 6.0e-5, 0.0, 6.5e-5, 8000)]
        rep.runs.append(harness.RunRecord(run, 3.0e-4 + run * 1e-6, 4, 1.0 / 3.0, False, [64.0, 8.0, 1.0, 0.125, 1.0 / 3.0],
                                          levels))
    rep.aggregate = harness.aggregate_runs(rep.runs, 2)
    return rep


def test_json_round_trip_is_lossless_and_has_the_reference_keys():
    """test_bench.cpp:160-166, report.hpp:128-262"""
    rep = sample_report()
    text = harness.report_to_json(rep)
    assert harness.report_from_json(text) == rep and harness.report_to_json(harness.report_from_json(text)) == text
    doc = json.loads(text)
    assert sorted(doc) == ["aggregate", "config", "generation_seconds", "runs", "symmetry"]
    assert doc["config"]["nx"] == 8 and doc["config"]["fixed_iterations"] == 4 and doc["runs"][1]["run"] == 1
    assert doc["runs"][0]["residual_history"][-1] == 1.0 / 3.0  # doubles survive exactly


def test_csv_projection_round_trips_losslessly():
    """test_bench.cpp:168-176, report.hpp:270-360: rows (run, level, kernel, value), level empty on per-run rows"""
    rep = sample_report()
    rows = harness.report_to_rows(rep)
    assert len(rows) == 2 * (2 * 4 + 4)
    assert [r.kernel for r in rows[:4]] == ["smoother_seconds", "transfer_seconds", "mg_seconds", "nnz_visited"]
    assert [r.kernel for r in rows[8:12]] == ["solve_seconds", "iterations", "final_residual", "converged"]
    assert rows[8].level is None and rows[0].level == 0 and rows[4].level == 1
    text = harness.rows_to_csv(rows)
    assert text.splitlines()[0] == "run,level,kernel,value" and text.endswith("\n")
    back = harness.csv_to_rows(text)
    assert back == rows and harness.rows_to_csv(back) == text == harness.report_to_csv(rep)
    assert any(r.value == 1.0 / 3.0 for r in back)  # shortest round-trip formatting of doubles


def test_csv_rejects_malformed_input():
    """report.hpp:326-347: wrong header, wrong field count, unparsable numbers"""
    for bad in ("", "bad,header\n", "run,level,kernel,value\n1,2,3\n", "run,level,kernel,value\nx,,k,1\n",
                "run,level,kernel,value\n1,,k,not-a-number\n"):
        with pytest.raises(slab.InvalidArgument):
            harness.csv_to_rows(bad)


def test_aggregate_shares():
    """bench.hpp:133-154: shares are sums over runs divided by the summed solve time"""
    rep = sample_report()
    agg = rep.aggregate
    total = sum(r.solve_seconds for r in rep.runs)
    assert math.isclose(agg.mean_solve_seconds, total / 2)
    assert math.isclose(agg.levels[0].smoother_share, sum(r.levels[0].smoother_seconds for r in rep.runs) / total)
    assert math.isclose(agg.mg_share, sum(l.mg_seconds for r in rep.runs for l in r.levels) / total)
    assert harness.aggregate_runs([], 2) == harness.Aggregate()
