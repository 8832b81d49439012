"""Production-mode lattice jumps (walk.cu `mw_jump`).

Inside one cell of a MicroWalk cube every alpha is 1/2 (microwalk.cpp:97-104
with equal permittivities), so the walk there is the simple symmetric walk
and its first hit of the L-inf sphere of radius m is given by the Green's
function of the (2m-1)^3 interior (frw_lattice_jump_law).  In Philox mode the device replaces
such stretches by one draw from that law.  The transit law must be the
reference's: the exit histogram of a cube agrees with the FDM-solved surface
Green's function of the same cube (sgf.cpp:57-299 via the oracle, chi-square
p > 0.01 -- the north star's MicroWalk criterion), the mean step count with
E[tau] (expected_steps, sgf.cpp:292-299) within 4 standard errors, conductor
exits (MicroWalk-E) have the no-jump law, and full walks give the same
capacitances within 3 combined standard errors.
"""
import json
import os

import numpy as np
import pytest
from scipy import stats as st

import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure
from tests import scenes
from tests.stats import compare_counts
from tests.walk_helpers import upload_scene

pytestmark = pytest.mark.gpu
N = 24


def _transits(ctx, cube, count, seed, jumps, with_conductors=False):
    cubes = np.tile(np.asarray(cube, np.float64), (count, 1))
    return ctx.structure_transits_philox(N, cubes, seed, jumps=jumps,
                                         with_conductors=with_conductors)


@pytest.mark.parametrize("which", ["uniform", "pocket"])
def test_jump_transit_law_matches_solved_sgf(gpu_ctx, oracle, which):
    sc = scenes.plate_pocket_scene()
    # "uniform": a cube in the plate gap away from the pocket; "pocket": the
    # eps=16 pocket fills the cube's low-x part, background elsewhere
    cube = [500.0, 500.0, 100.0, 95.0] if which == "uniform" else [1200.0, 460.0, 100.0, 95.0]
    upload_scene(gpu_ctx, sc)
    eps, _ = oracle.build_grid(sc, cube[:3], cube[3], N)
    if which == "pocket":
        assert len(np.unique(eps)) == 2
    exact = oracle.solve_sgf(eps, cube[3], kernels=False)["probs"]
    et = oracle.expected_steps(eps)
    count = 400_000
    d = _transits(gpu_ctx, cube, count, seed=5, jumps=True)
    assert (d["kind"] == 0).all()
    r = compare_counts(exact, np.bincount(d["panel"], minlength=6 * N * N))
    assert r["p"] > 0.01, r
    s = d["steps"].astype(np.float64)
    se = s.std() / np.sqrt(count)
    assert abs(s.mean() - et) < 4 * se, (s.mean(), et, se)
    # and without jumps the law is the same
    d0 = _transits(gpu_ctx, cube, count, seed=6, jumps=False)
    r0 = compare_counts(exact, np.bincount(d0["panel"], minlength=6 * N * N))
    assert r0["p"] > 0.01, r0


def test_jump_transits_deterministic_and_differ_from_stepping(gpu_ctx):
    sc = scenes.plate_pocket_scene()
    upload_scene(gpu_ctx, sc)
    cube = [500.0, 500.0, 100.0, 95.0]
    a = _transits(gpu_ctx, cube, 20_000, seed=9, jumps=True)
    b = _transits(gpu_ctx, cube, 20_000, seed=9, jumps=True)
    c = _transits(gpu_ctx, cube, 20_000, seed=9, jumps=False)
    for k in ("panel", "steps", "voxel"):
        assert np.array_equal(a[k], b[k])
    assert not np.array_equal(a["panel"], c["panel"])
    # a step walk's exit parity is fixed by its steps; jumps break that link
    # (E[tau] is added instead of the realised count)
    par_c = (c["steps"] + c["voxel"].sum(axis=1)) % 2
    assert len(np.unique(par_c)) == 1
    par_a = (a["steps"] + a["voxel"].sum(axis=1)) % 2
    assert len(np.unique(par_a)) == 2


def test_jump_conductor_exits_keep_the_law(gpu_ctx):
    """MicroWalk-E cube reaching into both plates: (kind, panel/conductor)
    histograms with and without jumps agree (two-sample chi-square)"""
    sc = scenes.plate_pocket_scene()
    upload_scene(gpu_ctx, sc)
    cube = [900.0, 500.0, 100.0, 160.0]
    count = 300_000
    a = _transits(gpu_ctx, cube, count, seed=3, jumps=True, with_conductors=True)
    b = _transits(gpu_ctx, cube, count, seed=4, jumps=False, with_conductors=True)
    assert ((a["kind"] == 0) | (a["kind"] == 1)).all()

    def cat(d):
        return np.where(d["kind"] == 0, d["panel"], 6 * N * N + d["conductor"])

    ca, cb = cat(a), cat(b)
    m = max(ca.max(), cb.max()) + 1
    ha, hb = np.bincount(ca, minlength=m), np.bincount(cb, minlength=m)
    assert ha[6 * N * N:].sum() > 0.2 * count  # most walks end on a plate
    keep = (ha + hb) >= 10
    tab = np.vstack([ha[keep], hb[keep]])
    chi2, p, dof, _ = st.chi2_contingency(tab)
    assert p > 0.01, (chi2, dof, p)


@pytest.mark.parametrize("mode", ["HYBRID-MW", "MW"])
def test_jump_capacitances_match_stepping(mode):
    """C3 (two coated wires over a plane): jumps on vs off, every terminal
    within 3 combined standard errors; fewer device seconds are expected but
    not asserted.  (The walk engine takes jumps in plain MicroWalk modes;
    MicroWalk-E modes run without them, see frw_run_walks.)"""
    doc = json.dumps(c3_structure())
    walks = 300_000
    out = {}
    old = os.environ.get("FRW_MW_JUMP")
    try:
        for j in ("0", "31"):
            os.environ["FRW_MW_JUMP"] = j
            out[j] = frwcap.extract_json(doc, mode=mode, min_walks=walks, max_walks=walks,
                                         seed=17 if j == "0" else 18)
        assert out["0"].get("mw_jumps", 0) == 0 and out["31"]["mw_jumps"] > walks
    finally:
        if old is None:
            os.environ.pop("FRW_MW_JUMP", None)
        else:
            os.environ["FRW_MW_JUMP"] = old
    for ta, tb in zip(out["0"]["terminals"], out["31"]["terminals"]):
        se = np.hypot(ta["std_err_farads"], tb["std_err_farads"])
        assert abs(ta["capacitance_farads"] - tb["capacitance_farads"]) <= 3 * se, (ta, tb)
    # mean MicroWalk steps per walk (E[tau] bookkeeping for jumps) agree to 2%
    sa, sb = out["0"]["mw_steps"] / walks, out["31"]["mw_steps"] / walks
    assert abs(sa - sb) < 0.02 * sa, (sa, sb)
