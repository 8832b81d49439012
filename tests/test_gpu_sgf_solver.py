"""Device stratified-SGF miss solver (sgf_solve.cu) against the oracle's
restated solve (frw_oracle.c, pinned to the reference shim), and the walk
engine's NULL-callback path that solves its own table misses."""
import numpy as np
import pytest

from paper_2507_09730_b200 import capi
from tests import scenes
from tests.walk_helpers import oracle_solver, upload_scene, walk_params

pytestmark = pytest.mark.gpu

KEYS = [
    (24, 0, [3.9] * 24),
    (24, 2, [2.5] * 7 + [3.9] * 10 + [4.2] * 7),
    (24, 1, [7.0] * 3 + [1.0] * 21),
    (21, 0, [2.5, 25.0] * 10 + [3.9]),
    (8, 2, [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0]),
    (2, 0, [3.0, 5.0]),
    (1, 0, [7.5]),
]


@pytest.mark.parametrize("n,axis,layers", KEYS)
def test_device_solver_matches_oracle(gpu_ctx, oracle, n, axis, layers):
    probs, ker = gpu_ctx.sgf_solve(n, [axis], [layers])
    pitch, want_p, _, want_k = oracle_solver(oracle)(n, axis, np.array(layers))
    assert pitch == 1.0
    assert np.abs(probs[0] - want_p).max() < 1e-10
    assert abs(probs[0].sum() - 1) < 1e-9
    assert np.abs(ker[0] - want_k).max() < 1e-8
    assert np.abs(ker[0].sum(axis=1)).max() < 1e-9  # kernel zero-sum (test_sgf.cpp:212-222)


def test_device_solver_batch_of_many_keys(gpu_ctx, oracle):
    rng = np.random.default_rng(3)
    n = 24
    layers = np.round(rng.choice([2.5, 3.9, 4.2, 7.0], size=(300, n)), 6)
    axes = rng.integers(0, 3, size=300)
    probs, ker = gpu_ctx.sgf_solve(n, axes, layers)
    for q in (0, 137, 299):
        _, want_p, _, want_k = oracle_solver(oracle)(n, int(axes[q]), layers[q])
        assert np.abs(probs[q] - want_p).max() < 1e-10
        assert np.abs(ker[q] - want_k).max() < 1e-8


def test_walks_with_device_solved_table_match_oracle_statistically(gpu_ctx, oracle):
    """NULL miss callback: the engine fills its own table on the device."""
    sc = scenes.layered_plate_scene()
    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    p = walk_params(sc, grid_n=8, seed=21, rng=capi.RNG_PHILOX)
    t, rec = gpu_ctx.run_walks(p, sc.master_slot(), 0, 200_000, None)
    assert t["misses"] > 0 and (rec["done"] == 1).all()
    o = oracle.extract(sc, threads=8, grid_n=8, mode="HYBRID-MW", min_walks=40_000,
                       max_walks=40_000, seed=22)
    w = len(rec)
    for k, to in enumerate(o["terminals"]):
        sel = rec["slot"] == k
        mean = rec["weight"][sel].sum() / w
        var = ((rec["weight"] * sel) ** 2).sum() / w - mean ** 2
        se = np.sqrt(var / (w - 1))
        z = abs(mean - to["capacitance_farads"]) / np.hypot(se, to["std_err_farads"])
        assert z < 3.0, (k, mean, to)
