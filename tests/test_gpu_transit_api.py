"""GPU parity of the reference's single-transit MicroWalk API
(microwalk.hpp:70-100) as restated in csrc/host/microwalk.cpp:

* microwalk_transit over a materialised grid continues the caller's
  SplitMix64 (FRW_RNG_SPLITMIX_STATES): panel / steps equal the reference's
  own microwalk_transit (oracle/_ref) on SplitMix64(seed, t), the exit
  point is surface_panel_center, the state comes back advanced by steps;
* microwalk_transit_lazy and microwalk_e_transit over structure cubes
  (frw_structure_transits): panel, steps, exit point and conductor id equal
  the reference's own functions bit for bit, EngulfedStart included;
* lazy == grid (test_microwalk.cpp:229-250): a lazy transit and a transit on
  build_grid of the same cube give identical exits.
"""
import json

import numpy as np
import pytest

import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c1_grid, c3_structure, random_voxel_grid
from tests import scenes

pytestmark = pytest.mark.gpu
GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def _states(oracle, seed, count, stream0=0):
    return np.array([oracle.stream_state(seed, stream0 + t) for t in range(count)], np.uint64)


def _panel_center(c, h, n, panel):
    """sgf.cpp:38-49 in IEEE doubles (same operation order)"""
    face, rem = divmod(int(panel), n * n)
    u, v = rem % n, rem // n
    axis = face >> 1
    pitch = 2.0 * h / n
    p = [0.0, 0.0, 0.0]
    p[axis] = c[axis] + (1 if face & 1 else -1) * h
    b1 = 1 if axis == 0 else 0
    b2 = 1 if axis == 2 else 2
    p[b1] = c[b1] - h + (u + 0.5) * pitch
    p[b2] = c[b2] - h + (v + 0.5) * pitch
    return p


@pytest.mark.parametrize("which", ["c1", "rv5", "rv8"])
def test_grid_transits_continue_caller_stream(oracle, ref, which):
    eps = {"c1": c1_grid(3)[0], "rv5": random_voxel_grid(5, 9), "rv8": random_voxel_grid(8, 3)}[which]
    n = round(len(eps) ** (1 / 3))
    c, h = np.array([1.5, -2.0, 0.25]), n / 2.0 + 0.125
    count = 4000
    st = _states(oracle, 21, count)
    d = frwcap.transits_grid(eps, list(c), h, st)
    w = ref.microwalk_grid(eps, c, h, seed=21, stream0=0, count=count, threads=8)
    assert np.array_equal(d["panel"], w["panel"]) and np.array_equal(d["steps"], w["steps"])
    assert (d["kind"] == 0).all()
    expect = (st.astype(object) + d["steps"].astype(object) * GAMMA) % (1 << 64)
    assert [int(x) for x in d["state"]] == list(expect)
    for t in range(0, count, 97):
        assert list(d["point"][t]) == _panel_center(c, h, n, d["panel"][t])
        # the exit voxel sits on the panel's face, dir points out of the cube
        vox, dr = d["voxel"][t], d["dir"][t]
        assert vox[dr >> 1] == (n - 1 if dr & 1 else 0)
    # the one-transit-per-call form is the same function
    s = frwcap.transits_grid(eps, list(c), h, st[:40], single=True)
    for k in ("panel", "steps", "state", "voxel", "dir"):
        assert np.array_equal(s[k], d[k][:40])


def test_grid_transits_masked_conductor_exits(oracle):
    from tests.golden.make_golden import staircase_scene
    eps, mask = oracle.build_grid(staircase_scene(), [-10.0, 0, 0], 10.0, 5, mask=True)
    st = _states(oracle, 64, 3000)
    d = frwcap.transits_grid(eps, [-10.0, 0.0, 0.0], 10.0, st, mask=mask)
    w = oracle.microwalk_grid(eps, np.array([-10.0, 0, 0]), 10.0, 64, 0, 3000, mask=mask)
    assert np.array_equal(np.where(d["kind"] == 0, d["panel"], -1), w["panel"])
    assert np.array_equal(d["steps"], w["steps"])
    cx = np.flatnonzero(d["kind"] == 1)
    assert len(cx) > 0
    n = 5
    for t in cx[:50]:
        vox, dr = d["voxel"][t].copy(), int(d["dir"][t])
        nb = vox.copy()
        nb[dr >> 1] += 1 if dr & 1 else -1
        assert d["cond"][t] == mask[(nb[2] * n + nb[1]) * n + nb[0]] >= 0


def _free_points(sc, ref_s, rng, count):
    lo, hi = sc.world[:3], sc.world[3:]
    pts, hws = [], []
    while len(pts) < count:
        p = lo + (hi - lo) * (0.05 + 0.9 * rng.random(3))
        try:
            hw, _ = ref_s.max_free_cube(p)
        except ValueError:
            continue
        if hw > 1e-3:
            pts.append(p)
            hws.append(hw)
    return np.array(pts), np.array(hws)


def _transit_cube(p, hw, n):
    if n % 2 == 1:
        return list(p), hw
    delta = hw / (n + 1)
    return [p[0] + delta, p[1] + delta, p[2] + delta], (hw - delta) * (1.0 - 1e-12)


SCENES = {
    "c3": lambda: scenes.scene_from_doc(c3_structure()),
    "conformal_staircase": lambda: scenes.load_fixture("conformal_staircase"),
    "highk_cross": lambda: scenes.load_fixture("highk_cross"),
}


@pytest.mark.parametrize("name", sorted(SCENES))
@pytest.mark.parametrize("n", [7, 24])
def test_lazy_transits_match_reference(oracle, ref, name, n):
    sc = SCENES[name]()
    rs = ref.structure(sc)
    pts, hws = _free_points(sc, rs, np.random.default_rng(n), 60)
    cubes = np.array([_transit_cube(p, h, n)[0] + [_transit_cube(p, h, n)[1]]
                      for p, h in zip(pts, hws)])
    seed = 1000 + n
    st = _states(oracle, seed, len(cubes))
    d = frwcap.transits_structure(sc.to_json(), cubes, n, False, states=st)
    for t, cb in enumerate(cubes):
        w = rs.microwalk_lazy(cb[:3], cb[3], n, seed, t, 1)
        assert d["kind"][t] == 0
        assert d["panel"][t] == w["panel"][0] and d["steps"][t] == w["steps"][0]
        assert list(d["point"][t]) == list(w["point"][0])
    s = frwcap.transits_structure(sc.to_json(), cubes[:10], n, False, states=st[:10], single=True)
    for k in ("panel", "steps", "point", "state"):
        assert np.array_equal(s[k], d[k][:10])


@pytest.mark.parametrize("name", sorted(SCENES))
def test_expanded_transits_match_reference(oracle, ref, name):
    sc = SCENES[name]()
    rs = ref.structure(sc)
    n, expansion = 24, 5.0
    pts, hws = _free_points(sc, rs, np.random.default_rng(7), 40)
    seed = 99
    st = _states(oracle, seed, len(pts))
    cubes = np.concatenate([pts, hws[:, None]], axis=1)
    d = frwcap.transits_structure(sc.to_json(), cubes, n, True, expansion=expansion, states=st,
                                  single=True)
    conductor_exits = 0
    for t in range(len(pts)):
        try:
            w = rs.microwalk_e(pts[t], hws[t], expansion, n, seed, t, 1)
        except LookupError:  # EngulfedStart in the reference
            assert d["kind"][t] == -1
            continue
        assert d["kind"][t] in (0, 1)
        assert d["steps"][t] == w["steps"][0]
        assert list(d["point"][t]) == list(w["point"][0])
        if d["kind"][t] == 0:
            assert d["panel"][t] == w["panel"][0]
        else:
            conductor_exits += 1
            assert w["panel"][0] == -1 and d["cond"][t] == w["cond"][0]
    assert conductor_exits > 0


def test_lazy_equals_grid(oracle, ref):
    """test_microwalk.cpp:229-250: lazy field and materialised grid agree"""
    doc = c3_structure()
    text = json.dumps(doc)
    sc = scenes.scene_from_doc(doc)
    n = 24
    pts, hws = _free_points(sc, ref.structure(sc), np.random.default_rng(3), 1)
    c, h = [float(x) for x in pts[0]], float(hws[0])
    eps, mask, tag, axis = frwcap.build_grid(text, c, h, n)
    assert mask is None
    st = _states(oracle, 5, 2000)
    g = frwcap.transits_grid(eps, c, h, st)
    lz = frwcap.transits_structure(text, np.array([c + [h]] * 2000), n, False, states=st)
    for k in ("panel", "steps", "point", "voxel", "dir", "state"):
        assert np.array_equal(g[k], lz[k]), k
    # build_grid matches the oracle's voxelisation
    oe, _ = oracle.build_grid(sc, c, h, n)
    assert np.array_equal(eps, oe)


def test_neighbor_weights_known_answers():
    """test_microwalk.cpp:64-98: uniform interior 1/6; interface 3/4 vs 1/4"""
    n = 4
    eps = np.full(n ** 3, 2.0)
    b = frwcap.neighbor_weights(eps, [1, 1, 1])
    assert np.allclose(b, 1 / 6, rtol=0, atol=1e-15)
    eps2 = eps.copy()
    eps2[(1 * n + 1) * n + 2] = 6.0  # +x neighbour of (1,1,1) has eps 6
    b2 = frwcap.neighbor_weights(eps2, [1, 1, 1])
    a = [0.5, 0.75, 0.5, 0.5, 0.5, 0.5]
    assert np.allclose(b2, np.array(a) / sum(a), rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        frwcap.neighbor_weights(eps, [4, 0, 0])


def test_c_abi_states_and_structure_transits(gpu_ctx, oracle, ref):
    """the same through the C ABI (capi): FRW_RNG_SPLITMIX_STATES batches and
    frw_structure_transits"""
    eps = random_voxel_grid(6, 4)
    st = _states(oracle, 8, 3000)
    gpu_ctx.upload_grid(eps, np.zeros(3), 3.0)
    g = gpu_ctx.microwalk_batch(0, states=st, per_transit=True)
    w = ref.microwalk_grid(eps, np.zeros(3), 3.0, seed=8, stream0=0, count=3000, threads=8)
    assert np.array_equal(g["panel"], w["panel"]) and np.array_equal(g["steps"], w["steps"])
    sc = scenes.load_fixture("highk_cross")
    rs = ref.structure(sc)
    from tests.walk_helpers import upload_scene
    upload_scene(gpu_ctx, sc)
    pts, hws = _free_points(sc, rs, np.random.default_rng(11), 30)
    cubes = np.concatenate([pts, hws[:, None]], axis=1)
    st = _states(oracle, 12, 30)
    d = gpu_ctx.structure_transits(24, cubes, st)
    for t in range(30):
        r = rs.microwalk_lazy(cubes[t, :3], cubes[t, 3], 24, 12, t, 1)
        assert d["panel"][t] == r["panel"][0] and d["steps"][t] == r["steps"][0]
        assert list(d["point"][t]) == list(r["point"][0])


@pytest.mark.parametrize("mode", ["HYBRID-MW", "HYBRID-MWE"])
@pytest.mark.parametrize("name", ["c3", "highk_cross"])
def test_engine_transitions_compose_the_walk_engine(name, mode):
    """Engine::first_transition / Engine::transition (engine.hpp:146-159) on
    the device, composed into run_walk (engine.cpp:352-376) on the host,
    reproduce the device walk engine's per-walk outcome bit for bit (same
    SplitMix64 streams, same SGF tables)"""
    text = json.dumps(c3_structure()) if name == "c3" else SCENES[name]().to_json()
    kw = dict(mode=mode, rng="splitmix", seed=31, grid_n=24)
    dev = frwcap.run_walks_json(text, 0, 300, **kw)
    comp = frwcap.walks_by_transitions(text, 0, 300, False, **kw)
    assert np.array_equal(comp["slot"], dev["slot"])
    assert np.array_equal(comp["weight"], dev["weight"])
    assert np.array_equal(comp["aborted"], dev["aborted"])
    st = comp["stats"]
    assert st["first_stratified"] + st["first_shrunk"] + st["first_layered"] + \
        st["first_homogenized"] >= 300
    assert (st["microwalk"] if mode == "HYBRID-MW" else st["microwalk_e"]) > 0
    one = frwcap.walks_by_transitions(text, 0, 12, True, **kw)
    for k in ("slot", "weight", "aborted"):
        assert np.array_equal(one[k], comp[k][:12])
