"""The device solver of materialised grids (frw_grid_sgf_solve, restating
assemble_system / solve_sgf / expected_steps, sgf.cpp:57-299) against the
oracle and the reference's test_sgf.cpp properties, plus the transit
invariants of test_microwalk.cpp that need no RNG alignment."""
import numpy as np
import pytest

import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import random_voxel_grid
from tests import scenes

pytestmark = pytest.mark.gpu


def _panel_centers(n, c, h):
    P = 6 * n * n
    out = np.empty((P, 3))
    pitch = 2.0 * h / n
    for q in range(P):
        face, rem = divmod(q, n * n)
        u, v = rem % n, rem // n
        ax = face >> 1
        p = [0.0, 0.0, 0.0]
        p[ax] = c[ax] + (1 if face & 1 else -1) * h
        b1 = 1 if ax == 0 else 0
        b2 = 1 if ax == 2 else 2
        p[b1] = c[b1] - h + (u + 0.5) * pitch
        p[b2] = c[b2] - h + (v + 0.5) * pitch
        out[q] = p
    return out


@pytest.mark.parametrize("n,seed", [(3, 1), (5, 2), (8, 3), (12, 4)])
def test_random_grids_match_oracle(gpu_ctx, oracle, n, seed):
    """test_sgf.cpp:178-193 / :281-298 (dense-oracle matches) against the
    oracle's restated solve"""
    eps = random_voxel_grid(n, seed)
    probs, ker, steps = gpu_ctx.grid_sgf_solve(eps)
    o = oracle.solve_sgf(eps, n / 2.0, kernels=True)
    assert np.allclose(probs[0], o["probs"], rtol=0, atol=1e-9)
    assert np.allclose(ker[0], o["kernels"], rtol=0, atol=1e-8)
    assert abs(steps[0] - oracle.expected_steps(eps)) <= 1e-8 * steps[0]


def test_normalisation_kernels_and_scale_invariance(gpu_ctx):
    """test_sgf.cpp:195-222, :270-279"""
    eps = np.stack([random_voxel_grid(7, s) for s in range(6)])
    probs, ker, _ = gpu_ctx.grid_sgf_solve(eps)
    assert np.allclose(probs.sum(axis=1), 1.0, atol=1e-9) and (probs >= 0).all()
    assert np.abs(ker.sum(axis=2)).max() <= 1e-9
    p2, k2, _ = gpu_ctx.grid_sgf_solve(eps * 7.25)
    assert np.allclose(p2, probs, rtol=0, atol=1e-12)


def test_linear_fields_and_octahedral_symmetry(gpu_ctx):
    """test_sgf.cpp:224-268: constant and linear boundary data are
    reproduced at the start node on a uniform lattice; odd n gives the full
    octahedral symmetry (every face carries 1/6)"""
    n, h = 9, 4.5
    probs, ker, _ = gpu_ctx.grid_sgf_solve(np.full(n ** 3, 3.9), h)
    p = probs[0]
    pc = _panel_centers(n, np.zeros(3), h)
    # tolerances of test_sgf.cpp:235-268 (linear 1e-8 / 1e-6, symmetry 1e-8)
    assert abs(p.sum() - 1) < 1e-9
    for a in range(3):
        assert abs(p @ pc[:, a]) < 1e-8  # linear field through the centre
        g = ker[0][a] @ pc[:, a]          # gradient of f = x_a is 1
        assert abs(g - 1.0) < 1e-6
    faces = p.reshape(6, n * n).sum(axis=1)
    assert np.allclose(faces, 1 / 6, atol=1e-8)


def test_transits_are_bit_transparent_to_power_of_two_scaling(oracle):
    """test_microwalk.cpp:209-227"""
    eps = random_voxel_grid(6, 9)
    st = np.array([oracle.stream_state(4, t) for t in range(5000)], np.uint64)
    a = frwcap.transits_grid(eps, [0, 0, 0], 3.0, st)
    b = frwcap.transits_grid(eps * 32.0, [0, 0, 0], 3.0, st)
    for k in ("panel", "steps", "state"):
        assert np.array_equal(a[k], b[k])


def test_expansion_one_is_the_plain_transit(oracle, ref):
    """test_microwalk.cpp:252-276: microwalk_e_transit with expansion 1 on a
    conductor-free cube equals microwalk_transit_lazy on transit_cube"""
    sc = scenes.load_fixture("highk_cross")
    rs = ref.structure(sc)
    rng = np.random.default_rng(2)
    lo, hi = sc.world[:3], sc.world[3:]
    pts, hws = [], []
    while len(pts) < 20:
        p = lo + (hi - lo) * (0.05 + 0.9 * rng.random(3))
        try:
            hw, _ = rs.max_free_cube(p)
        except ValueError:
            continue
        pts.append(p)
        hws.append(hw)
    n = 12
    st = np.array([oracle.stream_state(6, t) for t in range(20)], np.uint64)
    e = frwcap.transits_structure(sc.to_json(), np.c_[pts, hws], n, True, expansion=1.0,
                                  states=st, single=True)
    cubes = []
    for p, hw in zip(pts, hws):
        delta = hw / (n + 1)
        cubes.append(list(np.array(p) + delta) + [(hw - delta) * (1.0 - 1e-12)])
    lz = frwcap.transits_structure(sc.to_json(), np.array(cubes), n, False, states=st)
    for k in ("panel", "steps", "point", "state"):
        assert np.array_equal(e[k], lz[k]), k


def test_n1_transit_is_uniform_over_six_panels(oracle):
    """test_microwalk.cpp:100-117"""
    st = np.array([oracle.stream_state(8, t) for t in range(60000)], np.uint64)
    d = frwcap.transits_grid(np.array([2.5]), [0, 0, 0], 0.5, st)
    assert (d["steps"] == 1).all()
    counts = np.bincount(d["panel"], minlength=6)
    assert np.allclose(counts / counts.sum(), 1 / 6, atol=0.01)
