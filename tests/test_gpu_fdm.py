"""FDM mode on the device (engine.cpp:311-318).

* The FDM transition law equals the solved surface Green's function of the
  transition cube's build_grid (oracle restatement of sgf.cpp:57-299):
  chi-square p > 0.01 over 6n^2 panels.
* Theorem 1 of the paper (MicroWalk is the FDM chain, statistically): FDM
  and HYBRID-MW capacitances agree within 3 combined standard errors.
* Determinism: the same seed gives the same FDM estimate.
"""
import json

import numpy as np
import pytest

import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure
from tests import scenes
from tests.stats import compare_counts

pytestmark = pytest.mark.gpu


def _transit_cube(p, hw, n):
    if n % 2 == 1:
        return np.array(p, float), hw
    delta = hw / (n + 1)
    return np.array(p, float) + delta, (hw - delta) * (1.0 - 1e-12)


def _general_point(oracle, sc, n, rng):
    lo, hi = sc.world[:3], sc.world[3:]
    for _ in range(20000):
        p = lo + (hi - lo) * (0.05 + 0.9 * rng.random(3))
        try:
            hw, _ = oracle.max_free_cube(sc, p)
        except ValueError:
            continue
        if hw < 1e-3:
            continue
        c, h = _transit_cube(p, hw, n)
        ax, _ = oracle.stratified_profile(sc, c, h, n)
        if ax is None:
            return p, c, h
    raise RuntimeError("no general cube found")


def _panel_of(point, c, h, n):
    pitch = 2.0 * h / n
    d = point - c
    axis = int(np.argmax(np.abs(d) / h))
    face = 2 * axis + (1 if d[axis] > 0 else 0)
    b1 = 1 if axis == 0 else 0
    b2 = 1 if axis == 2 else 2
    u = int(round((point[b1] - (c[b1] - h)) / pitch - 0.5))
    v = int(round((point[b2] - (c[b2] - h)) / pitch - 0.5))
    return (face * n + v) * n + u


@pytest.mark.parametrize("name,n", [("highk_cross", 8), ("c3", 12)])
def test_fdm_transition_law(oracle, name, n):
    sc = scenes.load_fixture(name) if name != "c3" else scenes.scene_from_doc(c3_structure())
    text = sc.to_json() if name != "c3" else json.dumps(c3_structure())
    p, c, h = _general_point(oracle, sc, n, np.random.default_rng(5))
    eps, _ = oracle.build_grid(sc, c, h, n)
    exact = oracle.solve_sgf(eps, h, kernels=False)["probs"]
    count = 60000
    states = np.array([oracle.stream_state(9, t) for t in range(count)], np.uint64)
    ev = frwcap.transitions_json(text, np.tile(p, (count, 1)), states, mode="FDM", grid_n=n,
                                 rng="splitmix")
    assert (ev["kind"] == 0).all() and ev["stats"]["fdm"] == count
    panels = np.array([_panel_of(q, c, h, n) for q in ev["point"]])
    hist = np.bincount(panels, minlength=6 * n * n)
    r = compare_counts(exact, hist)
    assert r["p"] > 0.01, r
    # one uniform per FDM transition (sgf.hpp:144-147)
    gamma = 0x9E3779B97F4A7C15
    assert int(ev["state"][0]) == (int(states[0]) + gamma) % (1 << 64)


def test_fdm_matches_microwalk_theorem1():
    doc = json.dumps(c3_structure())
    kw = dict(min_walks=20000, max_walks=20000, seed=3, grid_n=24)
    mw = frwcap.extract_json(doc, mode="HYBRID-MW", **kw)
    fd = frwcap.extract_json(doc, mode="FDM", **kw)
    assert fd["dispatch_stats"]["subsequent"]["fdm"] > 0
    assert fd["dispatch_stats"]["subsequent"]["microwalk"] == 0
    for a, b in zip(mw["terminals"], fd["terminals"]):
        se = np.hypot(a["std_err_farads"], b["std_err_farads"])
        assert abs(a["capacitance_farads"] - b["capacitance_farads"]) <= 3 * se, (a, b)
    fd2 = frwcap.extract_json(doc, mode="FDM", **kw)
    assert [t["capacitance_farads"] for t in fd2["terminals"]] == \
        [t["capacitance_farads"] for t in fd["terminals"]]
