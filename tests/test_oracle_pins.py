"""Pin the CPU oracle (oracle/frw_oracle.c) before trusting it.

1. against golden vectors produced by the reference's own sources
   (tests/golden/make_golden.py -> oracle/_ref), bit for bit where the
   reference is integer/ordering work, to the solver tolerance for the SGF;
2. against the reference's known-answer tests (test_sgf.cpp,
   test_microwalk.cpp) that survive without Eigen;
3. live against oracle/_ref when it is built (this container).
"""
import os

import numpy as np
import pytest

from paper_2507_09730_b200.workloads import SplitMix64, c1_grid, random_voxel_grid
from tests.golden.make_golden import layered_scene, random_scene, staircase_scene

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


# ---------------------------------------------------------------- rng
def test_splitmix_streams_match(oracle):
    for seed, stream in [(1, 0), (7, 12345), (2 ** 63 + 5, 2 ** 40)]:
        py = SplitMix64(seed, stream)
        st = oracle.stream_state(seed, stream)
        assert st == py.state
        u = oracle.uniforms(seed, stream, 5)
        assert np.array_equal(u, np.array([py.uniform() for _ in range(5)]))


# ---------------------------------------------------------------- MicroWalk
@pytest.mark.parametrize("name", ["c1_s1", "c2_s1", "rv4_s11", "rv6_s12", "rv1_s2", "rv2_s3"])
def test_grid_transits_match_reference_vectors(oracle, gold, name):
    eps = gold[f"mw_{name}_eps"]
    n = round(len(eps) ** (1 / 3))
    want_p, want_s = gold[f"mw_{name}_panel"], gold[f"mw_{name}_steps"]
    got = oracle.microwalk_grid(eps, np.zeros(3), n / 2.0, seed=3, stream0=0,
                                count=len(want_p), threads=4)
    assert np.array_equal(got["panel"], want_p)
    assert np.array_equal(got["steps"], want_s)


def test_masked_staircase_transits_match(oracle, gold):
    eps, mask = gold["mw_stair_eps"], gold["mw_stair_mask"]
    assert (mask >= 0).any()
    got = oracle.microwalk_grid(eps, np.array([-10.0, 0, 0]), 10.0, seed=64, stream0=2,
                                count=len(gold["mw_stair_panel"]), mask=mask)
    assert np.array_equal(got["panel"], gold["mw_stair_panel"])
    assert np.array_equal(got["steps"], gold["mw_stair_steps"])
    # the oracle's voxelisation of the staircase equals the reference's
    e2, m2 = oracle.build_grid(staircase_scene(), [-10.0, 0, 0], 10.0, 5, mask=True)
    assert np.array_equal(e2, eps) and np.array_equal(m2, mask)


@pytest.mark.parametrize("n", [5, 6])
def test_lazy_transits_match(oracle, gold, n):
    c, hw = gold[f"lazy{n}_center"], float(gold[f"lazy{n}_hw"][0])
    got = oracle.microwalk_lazy(layered_scene(), c, hw, n, seed=61, stream0=5, count=300)
    assert np.array_equal(got["panel"], gold[f"lazy{n}_panel"])
    assert np.array_equal(got["steps"], gold[f"lazy{n}_steps"])
    assert np.array_equal(got["point"], gold[f"lazy{n}_point"])  # bit-exact continuation


def test_lazy_equals_materialized(oracle):
    """test_microwalk.cpp:229-250: lazy transits == materialized-grid transits."""
    sc = layered_scene()
    for n in (5, 6):
        hw0 = 6.0
        c = np.zeros(3)
        if n % 2 == 0:
            d = hw0 / (n + 1)
            c, hw = c + d, (hw0 - d) * (1.0 - 1e-12)
        else:
            hw = hw0
        eps, _ = oracle.build_grid(sc, c, hw, n)
        a = oracle.microwalk_lazy(sc, c, hw, n, seed=61, stream0=5, count=300)
        b = oracle.microwalk_grid(eps, c, hw, seed=61, stream0=5, count=300)
        assert np.array_equal(a["panel"], b["panel"]) and np.array_equal(a["steps"], b["steps"])


def test_n1_exits_in_one_step(oracle):
    """test_microwalk.cpp:100-117"""
    r = oracle.microwalk_grid(np.array([3.0]), np.zeros(3), 0.5, seed=1, stream0=0, count=6000)
    assert (r["steps"] == 1).all()
    assert set(np.unique(r["panel"])) == set(range(6))


def test_step_cap_raises(oracle):
    """test_microwalk.cpp:364-370"""
    with pytest.raises(RuntimeError):
        oracle.microwalk_grid(np.ones(8 ** 3), np.zeros(3), 4.0, 66, 0, 10, step_cap=2)


# ---------------------------------------------------------------- SGF
@pytest.mark.parametrize("name", ["rv4_s11", "rv6_s12"])
def test_sgf_matches_reference_vectors(oracle, gold, name):
    eps = gold[f"mw_{name}_eps"]
    s = oracle.solve_sgf(eps)
    assert np.abs(s["probs"] - gold[f"sgf_{name}_probs"]).max() < 1e-10
    assert np.abs(s["kernels"] - gold[f"sgf_{name}_kernels"]).max() < 1e-9
    assert abs(oracle.expected_steps(eps) - gold[f"sgf_{name}_esteps"][0]) < 1e-7


def test_sgf_known_answers(oracle):
    # n=1: six unit couplings, probs 1/6, E[tau]=1 (test_sgf.cpp:111-123)
    s = oracle.solve_sgf(np.array([7.5]))
    assert np.allclose(s["probs"], 1 / 6, rtol=1e-12)
    assert abs(oracle.expected_steps(np.array([7.5])) - 1.0) < 1e-12
    # probabilities normalise, kernels sum to zero (test_sgf.cpp:212-222)
    g = random_voxel_grid(5, 13, 0)
    s = oracle.solve_sgf(g)
    assert abs(s["probs"].sum() - 1) < 1e-9 and (s["probs"] >= 0).all()
    assert np.abs(s["kernels"].sum(axis=1)).max() < 1e-9
    # eps scaling invariance (test_sgf.cpp:270-279)
    s2 = oracle.solve_sgf(g * 37.5)
    assert np.abs(s2["probs"] - s["probs"]).max() < 1e-8


def test_sgf_linear_field_exactness(oracle):
    """test_sgf.cpp:235-259: the SGF reproduces linear potentials."""
    for n in (4, 5):
        s = oracle.solve_sgf(np.full(n ** 3, 2.5))
        d, b = np.array([0.37, -1.21, 0.52]), 0.81
        pcs = np.array([_panel_center(n, p) for p in range(6 * n * n)])
        phi = pcs @ d + b
        c = (n - 1) // 2
        sp = np.array([-n / 2 + (c + 0.5)] * 3)
        assert abs(s["probs"] @ phi - (sp @ d + b)) < 1e-8
        for a in range(3):
            assert abs(s["kernels"][a] @ phi - d[a]) < 1e-6


def _panel_center(n, p):
    face, rem = divmod(p, n * n)
    v, u = divmod(rem, n)
    ax = face // 2
    out = [0.0, 0.0, 0.0]
    out[ax] = (-1 if face % 2 == 0 else 1) * n / 2
    b1 = 1 if ax == 0 else 0
    b2 = 1 if ax == 2 else 2
    out[b1] = -n / 2 + (u + 0.5)
    out[b2] = -n / 2 + (v + 0.5)
    return out


def test_expected_steps_square_law(oracle):
    """E[tau]/N^2 = 0.3373 +- 5% at n=24 (test_sgf.cpp:300-304)."""
    e = oracle.expected_steps(np.ones(24 ** 3))
    assert abs(e / 576 - 0.3373) <= 0.05 * 0.3373


def test_dense_absorption_row_agrees(oracle):
    """Independent dense solve of the absorbing chain (oracle.cpp:15-88 restated
    in numpy) agrees with the PCG solve to 1e-8 (test_sgf.cpp:178-193)."""
    for n, sd in ((3, 1), (4, 2)):
        eps = random_voxel_grid(n, 42, sd)
        row = _dense_row(eps, n)
        assert np.abs(row - oracle.solve_sgf(eps, kernels=False)["probs"]).max() < 1e-8


def _dense_row(eps, n):
    E = eps.reshape(n, n, n)
    m = n ** 3
    A = np.zeros((m, m))
    B = np.zeros((m, 6 * n * n))
    for k in range(n):
        for j in range(n):
            for i in range(n):
                r = (k * n + j) * n + i
                diag = 0.0
                for d, (di, dj, dk) in enumerate(((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0),
                                                  (0, 0, -1), (0, 0, 1))):
                    a, b, c = i + di, j + dj, k + dk
                    if not (0 <= a < n and 0 <= b < n and 0 <= c < n):
                        ax = d // 2
                        u = j if ax == 0 else i
                        v = j if ax == 2 else k
                        B[r, (d * n + v) * n + u] += 1
                        diag += 1
                        continue
                    al = E[c, b, a] / (E[c, b, a] + E[k, j, i])
                    A[r, (c * n + b) * n + a] -= al
                    diag += al
                A[r, r] = diag
    c = (n - 1) // 2
    e = np.zeros(m)
    e[(c * n + c) * n + c] = 1
    return B.T @ np.linalg.solve(A.T, e)


# ---------------------------------------------------------------- geometry
@pytest.mark.parametrize("sd", [1, 2, 3])
def test_geometry_queries_match_reference_vectors(oracle, gold, sd):
    sc = random_scene(sd)
    assert np.array_equal(gold[f"geo{sd}_scene"],
                          np.concatenate([sc.cond_box.ravel(), sc.diel_box.ravel(), sc.diel_eps]))
    pts = gold[f"geo{sd}_pts"]
    for p, e, c, f in zip(pts, gold[f"geo{sd}_eps"], gold[f"geo{sd}_cond"], gold[f"geo{sd}_free"]):
        assert oracle.permittivity_at(sc, p) == e
        ci = oracle.conductor_at(sc, p, 0.5)
        assert (-1 if ci < 0 else int(sc.cond_id[ci])) == c
        try:
            h = oracle.max_free_cube(sc, p)[0]
        except ValueError:
            h = -1.0
        assert h == f
    for p, ax, layers in zip(pts[:100], gold[f"geo{sd}_prof_axis"], gold[f"geo{sd}_prof_layers"]):
        try:
            a, lay = oracle.stratified_profile(sc, p, 3.0, 6)
        except ValueError:
            a, lay = -2, None
        assert (-1 if a is None else a) == ax
        if a is not None and a >= 0:
            assert np.array_equal(lay, layers)


def test_round_sig(oracle):
    for x in (3.9, 7.000000001, 1234567.89, 2.5e-7, 25.0):
        r = oracle.round_sig(x)
        assert abs(r - float(f"{x:.6g}")) <= 1e-15 * abs(x)


# ---------------------------------------------------------------- live reference
def test_live_reference_grid(oracle, ref):
    eps, c, h, _ = c1_grid(5)
    a = oracle.microwalk_grid(eps, c, h, seed=9, stream0=100, count=3000, threads=4)
    b = ref.microwalk_grid(eps, c, h, seed=9, stream0=100, count=3000, threads=4)
    assert np.array_equal(a["panel"], b["panel"]) and np.array_equal(a["steps"], b["steps"])
    assert np.array_equal(a["hist"], b["hist"])


def test_live_reference_engine_walks(oracle, ref):
    """Walk-level bit parity of the restated engine against the reference's
    Engine (first_transition/transition) on a small stratified + general scene."""
    from tests.scenes import plate_pocket_scene
    sc = plate_pocket_scene()
    kw = dict(grid_n=8, mode="HYBRID-MW", seed=77)
    s1, w1, a1 = oracle.run_walks(sc, 0, 200, **kw)
    s2, w2, a2 = ref.structure(sc).run_walks(0, 200, **kw)
    assert np.array_equal(s1, s2) and np.array_equal(a1, a2)
    assert np.allclose(w1, w2, rtol=1e-9, atol=0)
