"""Host direct solves of the transition-cube system (csrc/host/direct.cpp):

* direct_sgf -- band L D L^T of s_ii, the counterpart of the reference's
  SimplicialLDLT fallback (sgf.cpp:162-211) and the solver of masked
  (conductor-voxel) grids: probabilities, gradient kernels and E[steps]
  against the oracle's Jacobi-PCG restatement (unmasked) and the reference
  build's solve_sgf (masked: surface then conductor panels in (node,
  direction) order, sgf.cpp:94-118);
* exact_absorption_row -- the dense LU row (oracle.hpp:14-19), validate-sgf's
  n <= 6 cross-check (cli.cpp:271-279).

CPU only: nothing here touches the device."""
import numpy as np
import pytest

import paper_2507_09730_b200.frwcap as frwcap
from oracle.oracle import Oracle


def _grid(n, seed, masked=False):
    rng = np.random.default_rng(seed)
    eps = rng.exponential(10.0, n ** 3) + 1e-9
    if not masked:
        return eps, None
    mask = np.full(n ** 3, -1, np.int32)
    idx = rng.choice(n ** 3, n ** 3 // 6, replace=False)
    c = (n - 1) // 2
    idx = idx[idx != (c * n + c) * n + c]
    mask[idx] = rng.integers(0, 3, len(idx))
    return eps, mask


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11])
def test_direct_equals_oracle_solve(n):
    eps, _ = _grid(n, 10 + n)
    d = frwcap.direct_sgf(eps)
    o = Oracle().solve_sgf(eps, half_width=n / 2.0, kernels=True)
    assert abs(d["probs"].sum() - 1.0) < 1e-12
    assert np.abs(d["probs"] - o["probs"]).max() < 1e-9   # the oracle's PCG stops at 1e-10
    assert np.abs(d["kernels"] - o["kernels"]).max() < 1e-9
    assert d["expected_steps"] == pytest.approx(Oracle().expected_steps(eps), rel=1e-9)


@pytest.mark.parametrize("n", [3, 4, 6])
def test_dense_row_equals_direct(n):
    eps, _ = _grid(n, 30 + n)
    row = frwcap.exact_absorption_row(eps)
    assert np.abs(row - frwcap.direct_sgf(eps)["probs"]).max() < 1e-13


@pytest.mark.parametrize("n", [4, 7, 10])
def test_masked_grid_vs_reference(ref, n):
    eps, mask = _grid(n, 50 + n, masked=True)
    d = frwcap.direct_sgf(eps, mask=mask)
    r = ref.solve_sgf(eps, mask=mask, kernels=True)
    assert len(d["probs"]) == len(r["probs"]) > 6 * n * n  # conductor panels appended
    assert np.abs(d["probs"] - r["probs"]).max() < 1e-9
    assert np.abs(d["kernels"] - r["kernels"]).max() < 1e-9
    row = frwcap.exact_absorption_row(eps, mask=mask)
    assert np.abs(row - d["probs"]).max() < 1e-13


def test_uniform_known_answers():
    # n = 1: six faces, 1/6 each, one step (sgf.cpp known answers)
    d = frwcap.direct_sgf(np.ones(1))
    assert np.allclose(d["probs"], 1 / 6, atol=1e-15) and d["expected_steps"] == pytest.approx(1.0)
    # odd uniform lattice: each face absorbs 1/6 (cli.cpp:303-320)
    n = 7
    p = frwcap.direct_sgf(np.full(n ** 3, 3.9))["probs"]
    assert np.abs(p.reshape(6, -1).sum(axis=1) - 1 / 6).max() < 1e-12
    with pytest.raises(ValueError):
        frwcap.exact_absorption_row(np.ones(13 ** 3))  # past the cost cap


def test_masked_grid_solves_directly():
    """conductor-voxel grids (build_grid with allow_conductors) solve through
    the host direct factorisation: surface then conductor panels, summing to 1"""
    from tests import scenes
    sc = scenes.load_fixture("plates_uniform")
    eps, mask, _, _ = frwcap.build_grid(sc.to_json(), [480.0, 480.0, 400.0], 200.0, 9, True)
    assert mask is not None and (np.asarray(mask) >= 0).any()
    d = frwcap.direct_sgf(eps, 200.0, mask)
    assert len(d["probs"]) > 6 * 81 and abs(d["probs"].sum() - 1) < 1e-12
