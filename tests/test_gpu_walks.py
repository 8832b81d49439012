"""GPU parity of the walk engine (configs C3-C5) through the C ABI and the
drop-in Python API.

* Walk-level bit-exactness: with SplitMix64 parity streams and the oracle's
  own SGF tables injected into the device table, every walk's terminal
  slot, abort flag and first-transition weight equal the oracle's
  (frw_oracle.c run_walk, itself pinned to the reference Engine).
* Statistical parity: Philox capacitances agree with the oracle within 3
  combined standard errors (north_star).
* Engine invariants the reference tests: Maxwell signs / row sum
  (test_engine.cpp:447-496), determinism, launch-shape independence,
  hop cap (test_engine.cpp:598-612), convergence rule.
"""
import json
import os

import numpy as np
import pytest

from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure
from tests import scenes
from tests.walk_helpers import oracle_solver, upload_scene, walk_params

pytestmark = pytest.mark.gpu
PARITY, PHILOX = capi.RNG_SPLITMIX_PARITY, capi.RNG_PHILOX


def _scene(doc):
    return scenes.scene_from_doc(doc)


CASES = {
    "plate_pocket": (scenes.plate_pocket_scene, 8),
    "plate_pocket_odd_n": (scenes.plate_pocket_scene, 9),  # odd lattice: cube centred on p
    "highk_cross_n5": (lambda: scenes.load_fixture("highk_cross"), 5),
    "layered_plates": (scenes.layered_plate_scene, 8),
    "two_plates_small": (scenes.two_plates_small, 12),
    "conformal_staircase": (lambda: scenes.load_fixture("conformal_staircase"), 24),
    "highk_cross": (lambda: scenes.load_fixture("highk_cross"), 24),
    "stratified_stack": (lambda: scenes.load_fixture("stratified_stack"), 24),
    "c3": (lambda: _scene(c3_structure()), 24),
    "c4": (lambda: _scene(c4_structure()), 24),
    "c5": (lambda: _scene(c5_structure()), 24),
}


MODES = {"HYBRID-MW": capi.MODE_HYBRID_MW, "HYBRID-MWE": capi.MODE_HYBRID_MWE}


@pytest.mark.parametrize("grid_min", ["default", "0"])  # "0": geometry bins on every scene
@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("case", sorted(CASES))
def test_walks_bit_exact_vs_oracle(gpu_ctx, oracle, monkeypatch, case, mode, grid_min):
    make, n = CASES[case]
    sc = make()
    if grid_min != "default":
        monkeypatch.setenv("FRW_GRID_MIN", grid_min)
    count = 600 if n == 24 else 2000
    if mode == "HYBRID-MWE" and case in ("c3", "c4", "c5"):
        count = 300  # expanded cubes: the oracle classifies far more voxels
    if case == "c5":
        count = 200  # 200 conductors / 254 dielectrics: the oracle scans them all
    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    p = walk_params(sc, grid_n=n, seed=77, rng=PARITY, n_slots=4096, mode=MODES[mode])
    tally, rec = gpu_ctx.run_walks(p, sc.master_slot(), 0, count, oracle_solver(oracle))
    slot, w, ab = oracle.run_walks(sc, 0, count, threads=8, grid_n=n, mode=mode, seed=77)
    assert np.array_equal(rec["slot"], slot), np.nonzero(rec["slot"] != slot)[0][:10]
    assert np.array_equal(rec["aborted"], ab)
    assert np.array_equal(rec["weight"], w)  # bitwise: same arithmetic, no FMA
    assert (rec["done"] == 1).all()
    # the fixed-order device tallies agree with the per-walk records
    k = sc.n_cond + 1
    for s in range(k):
        assert tally["landed"][s] == np.count_nonzero(rec["slot"] == s)
    assert np.isclose(tally["sum"].sum(), rec["weight"].sum(), rtol=1e-12, atol=0)


def test_walk_offsets_and_slots_are_irrelevant(gpu_ctx, oracle):
    sc = scenes.plate_pocket_scene()
    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    solve = oracle_solver(oracle)
    p = walk_params(sc, grid_n=8, seed=5, rng=PHILOX, n_slots=512)
    _, a = gpu_ctx.run_walks(p, 0, 1000, 3000, solve)
    p2 = walk_params(sc, grid_n=8, seed=5, rng=PHILOX, n_slots=100000)
    _, b = gpu_ctx.run_walks(p2, 0, 1000, 3000, solve)
    _, c = gpu_ctx.run_walks(p2, 0, 2000, 1000, solve)
    for f in ("slot", "weight", "aborted", "mw_steps"):
        assert np.array_equal(a[f], b[f])
        assert np.array_equal(a[f][1000:2000], c[f])


@pytest.mark.parametrize("mode", sorted(MODES))
def test_tail_kernels_agree_bitwise(gpu_ctx, oracle, monkeypatch, mode):
    """k_tail (one lane per walk) and k_flow (transition and MicroWalk roles
    with ring handoffs: roles by SM pair -- the default --, by warp, or as two
    kernels on two streams) run the same walks to the same records, whatever
    the order"""
    sc = _scene(c3_structure())
    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    solve = oracle_solver(oracle)
    p = walk_params(sc, grid_n=24, seed=9, rng=PHILOX, mode=MODES[mode])
    monkeypatch.setenv("FRW_TAIL_WALKS", str(1 << 30))  # everything after round 0
    out = {}
    for k in ("tail", "flow", "flowwarp", "flow2"):
        monkeypatch.setenv("FRW_TAIL_KERNEL", k)
        out[k] = gpu_ctx.run_walks(p, sc.master_slot(), 0, 50_000, solve)
    ta, a = out["tail"]
    for k in ("flow", "flowwarp", "flow2"):
        tb, b = out[k]
        for f in ("slot", "weight", "aborted", "mw_steps", "cached", "microwalk"):
            assert np.array_equal(a[f], b[f]), (k, f)
        assert np.array_equal(ta["sum"], tb["sum"]) and np.array_equal(ta["landed"], tb["landed"]), k


def test_hop_cap_aborts_into_ground(gpu_ctx, oracle):
    """test_engine.cpp:598-612"""
    sc = scenes.plate_scene()
    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    p = walk_params(sc, grid_n=8, seed=3, rng=PARITY, hop_cap=1)
    tally, rec = gpu_ctx.run_walks(p, 0, 0, 512, oracle_solver(oracle))
    slot, w, ab = oracle.run_walks(sc, 0, 512, grid_n=8, mode="HYBRID-MW", seed=3, hop_cap=1)
    assert tally["aborted"] > 0 and tally["aborted"] == int(ab.sum())
    assert np.array_equal(rec["slot"], slot) and np.array_equal(rec["aborted"], ab)
    assert tally["landed"][sc.n_cond] >= tally["aborted"]


def _combined_z(a, sa, b, sb):
    return abs(a - b) / np.sqrt(sa ** 2 + sb ** 2)


@pytest.mark.parametrize("case,walks_gpu,walks_cpu,mode", [
    ("c3", 200_000, 20_000, "HYBRID-MW"), ("highk_cross", 200_000, 20_000, "HYBRID-MW"),
    ("c3", 200_000, 10_000, "HYBRID-MWE"), ("conformal_staircase", 200_000, 20_000, "HYBRID-MWE")])
def test_capacitance_within_3_se_of_oracle(oracle, case, walks_gpu, walks_cpu, mode):
    import paper_2507_09730_b200.frwcap as frwcap
    make, n = CASES[case]
    sc = make()
    g = frwcap.extract_json(sc.to_json(), mode=mode, grid_n=n, min_walks=walks_gpu,
                            max_walks=walks_gpu, seed=11)
    o = oracle.extract(sc, threads=os.cpu_count() or 8, grid_n=n, mode=mode,
                       min_walks=walks_cpu, max_walks=walks_cpu, seed=12)
    assert g["walks"] == walks_gpu
    for tg, to in zip(g["terminals"], o["terminals"]):
        assert tg["conductor_id"] == to["conductor_id"]
        if to["walks_landed"] < 50:
            continue
        z = _combined_z(tg["capacitance_farads"], tg["std_err_farads"],
                        to["capacitance_farads"], to["std_err_farads"])
        assert z < 3.0, (tg, to, z)


def test_extract_api_contract_and_maxwell():
    """tests/python/test_smoke.py:29-44 and test_engine.cpp:447-496"""
    import paper_2507_09730_b200.frwcap as frwcap
    doc = scenes.two_plates_small().to_json()
    res = frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=8192, max_walks=8192, seed=7)
    ids = [t["conductor_id"] for t in res["terminals"]]
    assert ids == [1, 2, -1]
    assert res["walks"] == 8192
    self_row, coup = res["terminals"][0], res["terminals"][1]
    assert self_row["capacitance_farads"] > 5 * self_row["std_err_farads"]
    assert coup["capacitance_farads"] < 0
    sub = res["dispatch_stats"]["subsequent"]
    assert sub["microwalk"] == 0 and sub["fdm"] == 0 and sub["cached"] > 0  # uniform vacuum
    first = res["dispatch_stats"]["first"]
    assert sum(first.values()) == res["walks"]
    row = sum(t["capacitance_farads"] for t in res["terminals"])
    var = sum(t["std_err_farads"] ** 2 for t in res["terminals"])
    assert abs(row) <= 4 * np.sqrt(var)
    assert sum(t["walks_landed"] for t in res["terminals"]) == res["walks"]


def test_extract_deterministic_and_batch_invariant():
    import paper_2507_09730_b200.frwcap as frwcap
    doc = json.dumps(c3_structure())
    kw = dict(mode="HYBRID-MW", min_walks=20000, max_walks=20000, seed=3)
    a = frwcap.extract_json(doc, **kw)
    b = frwcap.extract_json(doc, device_batch=7000, **kw)
    for ta, tb in zip(a["terminals"], b["terminals"]):
        assert ta["capacitance_farads"] == tb["capacitance_farads"]
        assert ta["std_err_farads"] == tb["std_err_farads"]
    c = frwcap.extract_json(doc, **dict(kw, seed=4))
    assert c["terminals"][0]["capacitance_farads"] != a["terminals"][0]["capacitance_farads"]


def test_convergence_rule_stops_on_a_batch_boundary():
    """test_engine.cpp:498-511"""
    import paper_2507_09730_b200.frwcap as frwcap
    doc = scenes.plate_scene().to_json()
    res = frwcap.extract_json(doc, mode="HYBRID-MW", grid_n=8, seed=17, min_walks=1024,
                              max_walks=1 << 20, tol=0.3)
    assert res["converged"]
    assert 1024 <= res["walks"] < (1 << 20)
    assert res["walks"] % 1024 == 0


def test_convergence_independent_of_device_chunks():
    """the stopping rule fires on the same reference batch whether the walks
    come in one device call or in many (folded on a host thread while the
    device runs the next chunk, a speculative chunk discarded)"""
    import paper_2507_09730_b200.frwcap as frwcap
    doc = scenes.plate_scene().to_json()
    kw = dict(mode="HYBRID-MW", grid_n=8, seed=21, min_walks=1024, max_walks=1 << 20, tol=0.05)
    one = frwcap.extract_json(doc, device_batch=1 << 20, **kw)
    many = frwcap.extract_json(doc, device_batch=3072, **kw)
    assert one["converged"] and many["converged"]
    assert one["walks"] == many["walks"] and one["walks"] > 3 * 3072
    for ta, tb in zip(one["terminals"], many["terminals"]):
        assert ta["capacitance_farads"] == tb["capacitance_farads"]
        assert ta["std_err_farads"] == tb["std_err_farads"]
        assert ta["walks_landed"] == tb["walks_landed"]


def test_all_couplings_rule_c4():
    """configs[3]: walk until every coupling has rel. SE < tol (here 5% to
    keep the test short; the bench uses 1%)."""
    import paper_2507_09730_b200.frwcap as frwcap
    res = frwcap.extract_json(json.dumps(c4_structure()), mode="HYBRID-MW", tol=0.05,
                              all_couplings=True, min_walks=4096, max_walks=4_000_000,
                              seed=5, device_batch=1 << 18)
    assert res["converged"]
    for t in res["terminals"][:-1]:
        if t["conductor_id"] == res["master_id"]:
            continue
        assert t["std_err_farads"] <= 0.05 * abs(t["capacitance_farads"])


def test_c5_runs_and_lands_everywhere():
    import paper_2507_09730_b200.frwcap as frwcap
    res = frwcap.extract_json(json.dumps(c5_structure()), mode="HYBRID-MW", min_walks=50000,
                              max_walks=50000, seed=9)
    assert res["walks"] == 50000 and res["aborted"] == 0
    assert res["terminals"][0]["capacitance_farads"] > 0
    assert sum(t["walks_landed"] > 0 for t in res["terminals"]) > 5


def test_default_mode_is_hybrid_mwe_and_dispatch_counts():
    """Reference default mode HYBRID-MWE (engine.hpp:31): every lattice hop
    counts as microwalk_e (engine.cpp:328), none as microwalk."""
    import paper_2507_09730_b200.frwcap as frwcap
    res = frwcap.extract_json(json.dumps(c3_structure()), min_walks=20000, max_walks=20000, seed=2)
    sub = res["dispatch_stats"]["subsequent"]
    assert sub["microwalk"] == 0 and sub["microwalk_e"] > 0 and sub["fdm"] == 0
    assert sum(res["dispatch_stats"]["first"].values()) == res["walks"]


def test_chunk_tally_fold_equals_record_fold():
    """extract folds per-1024-walk device tallies (frw_walk_chunk_tallies) when
    reference batches are whole chunks, and per-walk records otherwise: the
    same walks land in the same slots, the sums agree to rounding, and the
    stopping rule stops on the same batch boundary class"""
    import paper_2507_09730_b200.frwcap as frwcap
    doc = json.dumps(c3_structure())
    kw = dict(mode="HYBRID-MW", min_walks=200_000, max_walks=200_000, seed=9)
    a = frwcap.extract_json(doc, batch=1024, **kw)   # chunk tallies
    b = frwcap.extract_json(doc, batch=1000, **kw)   # per-walk records
    assert a["walks"] == b["walks"] == 200_000
    assert a["dispatch_stats"] == b["dispatch_stats"] and a["mw_steps"] == b["mw_steps"]
    for ta, tb in zip(a["terminals"], b["terminals"]):
        assert ta["walks_landed"] == tb["walks_landed"]
        assert ta["capacitance_farads"] == pytest.approx(tb["capacitance_farads"], rel=1e-12,
                                                         abs=1e-30)
