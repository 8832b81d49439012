"""CPU checks of the drop-in Python module (paper_2507_09730_b200.frwcap):
the reference's eight names exist, keyword options and structure files are
validated before any device work (py_module.cpp:20-57, geometry.cpp:173-251),
and without a GPU the calls fail loudly instead of falling back to the CPU."""
import json
import math

import pytest

import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure

TWO_PLATES = json.dumps({
    "units": "nm", "world": {"lo": [0, 0, 0], "hi": [480, 480, 480]}, "background_eps": 1.0,
    "conductors": [{"id": 1, "lo": [90, 90, 150], "hi": [390, 390, 170]},
                   {"id": 2, "lo": [90, 90, 310], "hi": [390, 390, 330]}],
    "master": 1})


def test_reference_names_exported():
    for name in ("analytic_plate_capacitance", "expected_steps_uniform", "extract_file",
                 "extract_json", "reference_capacitance_file", "run_cli", "transit_tv",
                 "__version__"):
        assert hasattr(frwcap, name)
    assert frwcap.__version__ == "1.0.0"


def test_analytic_plate_capacitance():
    """tests/python/test_smoke.py:61-69"""
    c = frwcap.analytic_plate_capacitance([(100.0, 4.0)], 1e-12)
    assert math.isclose(c, 8.8541878128e-12 * 4.0 * 1e-12 / 100e-9, rel_tol=1e-12)
    c2 = frwcap.analytic_plate_capacitance([(50.0, 2.0), (50.0, 8.0)], 1e-12)
    assert math.isclose(c2, 8.8541878128e-12 * 1e-12 / (25e-9 + 6.25e-9), rel_tol=1e-12)


@pytest.mark.gpu
def test_expected_steps_uniform_device_solver():
    """E[tau]/N^2 = 0.3373 +- 5% at n = 24 (test_sgf.cpp:300-304), solved on
    the device (frw_grid_sgf_solve)"""
    s4, s8 = frwcap.expected_steps_uniform(4), frwcap.expected_steps_uniform(8)
    assert 2.5 < s8 / s4 < 6.0
    assert abs(frwcap.expected_steps_uniform(24) / 576 - 0.3373) <= 0.05 * 0.3373


def test_unknown_option_rejected():
    with pytest.raises(ValueError):
        frwcap.extract_json(TWO_PLATES, walks=10)


@pytest.mark.parametrize("kw", [dict(grid_n=1), dict(tol=0.0), dict(batch=0), dict(hop_cap=0),
                                dict(min_walks=10, max_walks=5), dict(gaussian_gap_fraction=1.0),
                                dict(mode="nope"), dict(rng="mt19937")])
def test_bad_config_rejected(kw):
    with pytest.raises(ValueError):
        frwcap.extract_json(TWO_PLATES, **kw)


def test_parse_and_validation_errors():
    with pytest.raises(RuntimeError, match="parse error at line"):
        frwcap.extract_json("{\n  \"units\": \"nm\",\n  oops }", mode="HYBRID-MW")
    bad = json.loads(TWO_PLATES)
    bad["conductors"][1]["id"] = 1
    with pytest.raises(RuntimeError, match="duplicate conductor id"):
        frwcap.extract_json(json.dumps(bad), mode="HYBRID-MW")
    bad = json.loads(TWO_PLATES)
    bad["extra"] = 1
    with pytest.raises(RuntimeError, match="unknown key"):
        frwcap.extract_json(json.dumps(bad), mode="HYBRID-MW")


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        frwcap.extract_json(TWO_PLATES, mode="HYBRID-MW", min_walks=64, max_walks=64)


def test_run_cli_usage_error():
    rc, out, err = frwcap.run_cli(["extract"])
    assert rc == 2 and err
