"""The reference CLI (cli.cpp:545-620) on the device build: validate-sgf,
bench-scaling, oracle-compare and extract reports keep the reference's JSON
schema and exit codes."""
import json

import pytest

import paper_2507_09730_b200.frwcap as frwcap
from tests import scenes

pytestmark = pytest.mark.gpu


def test_validate_sgf_passes():
    rc, out, err = frwcap.run_cli(["validate-sgf", "--n", "5", "--grids", "3",
                                   "--samples", "400000", "--seed", "7"])
    rep = json.loads(out)
    assert rc == 0, err
    assert rep["command"] == "validate-sgf" and rep["schema_version"] == 1
    assert rep["results"]["all_pass"]
    assert rep["results"]["uniform_face_symmetry"]["max_abs_err"] <= 1e-9
    for c in rep["results"]["checks"]:
        assert c["sgf_properties_ok"] and abs(c["steps_z"]) <= 4.0
        # n <= 6: the dense-LU cross-check of the device PCG (cli.cpp:271-279)
        assert c["dense_max_abs_diff"] <= 1e-8


def test_bench_scaling_reports_slopes():
    rc, out, err = frwcap.run_cli(["bench-scaling", "--n-list", "8,12,16", "--grids", "2",
                                   "--fdm-max-n", "16"])
    rep = json.loads(out)
    assert rc == 0, err
    rows = rep["results"]["rows"]
    assert [r["n"] for r in rows] == [8, 12, 16]
    # E[steps] grows ~ n^2 (paper: O(N^2) walk length)
    assert 1.6 < rep["results"]["slopes"]["expected_steps"] < 2.4
    for r in rows:
        assert abs(r["measured_mean_steps"] / r["expected_steps"] - 1) < 0.05


def test_oracle_compare_and_extract(tmp_path):
    sc = scenes.load_fixture("plates_uniform")
    f = tmp_path / "s.json"
    f.write_text(sc.to_json())
    rc, out, err = frwcap.run_cli(["oracle-compare", "--structure", str(f), "--mode",
                                   "hybrid-mw", "--tol", "0.02", "--resolution", "96",
                                   "--err-tol", "0.08"])
    rep = json.loads(out)
    assert rep["command"] == "oracle-compare"
    assert rc == (0 if rep["results"]["pass"] else 1)
    assert rep["results"]["err_avg"] < 0.08, err
    rc, out, err = frwcap.run_cli(["extract", "--structure", str(f), "--max-walks", "20000",
                                   "--min-walks", "20000"])
    rep = json.loads(out)
    assert rc == 0 and rep["results"]["walks"] == 20000
    assert "C[" in err


def test_cli_usage_errors():
    assert frwcap.run_cli([])[0] == 2
    assert frwcap.run_cli(["nope"])[0] == 2
    assert frwcap.run_cli(["validate-sgf", "--samples", "10"])[0] == 2
    assert frwcap.run_cli(["bench-scaling", "--n-list", "8"])[0] == 2
