"""GPU parity of the single-cube MicroWalk kernel (configs C1/C2), through
the C ABI (include/frw_gpu.h via paper_2507_09730_b200.capi).

* bit-exact integer first-hit panel and step count against the oracle when
  both consume the same injected SplitMix64(seed, stream) streams;
* chi-square p > 0.01 of the boundary-hit histogram against the FDM-solved
  surface Green's function (north_star), TV within the reference's bounds;
* mean steps within 3 SE of the exact expected_steps solve;
* edge cases the reference tests: n=1, even n, masked (conductor) lattices,
  step cap, engulfed start, empty batch.
"""
import numpy as np
import pytest

from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c1_grid, c2_grid, random_voxel_grid
from tests.stats import compare_counts, expected_tv

pytestmark = pytest.mark.gpu
PARITY, PHILOX = capi.RNG_SPLITMIX_PARITY, capi.RNG_PHILOX


def _bitexact(ctx, oracle, eps, center, hw, count, seed, stream0=0, mask=None, blocks=0):
    ctx.upload_grid(eps, center, hw, mask=mask)
    g = ctx.microwalk_batch(count, seed=seed, stream_begin=stream0, rng=PARITY,
                            per_transit=True, blocks=blocks)
    w = oracle.microwalk_grid(eps, center, hw, seed=seed, stream0=stream0, count=count,
                              mask=mask, threads=8)
    assert np.array_equal(g["panel"], w["panel"])
    assert np.array_equal(g["steps"], w["steps"])
    assert np.array_equal(g["hist"], w["hist"])
    assert g["step_sum"] == int(w["steps"].sum())
    assert g["step_sumsq"] == int((w["steps"].astype(np.int64) ** 2).sum())
    return g


def test_c1_parity_bit_exact(gpu_ctx, oracle):
    eps, c, h, _ = c1_grid(1)
    _bitexact(gpu_ctx, oracle, eps, c, h, 200_000, seed=11)


@pytest.mark.parametrize("seed", [2, 3, 17])
def test_c1_other_inclusions_bit_exact(gpu_ctx, oracle, seed):
    eps, c, h, _ = c1_grid(seed)
    _bitexact(gpu_ctx, oracle, eps, c, h, 50_000, seed=seed, stream0=10 ** 9)


def test_c2_parity_bit_exact(gpu_ctx, oracle):
    eps, c, h, _ = c2_grid(1)
    _bitexact(gpu_ctx, oracle, eps, c, h, 40_000, seed=5)


def test_kernel_variants_bit_exact(gpu_ctx, oracle):
    """every table placement runs the same walk: mw_grid_fast (records
    addressable by 16-bit shared addresses: C2), the shared-memory kernel
    with record ids (n=24 random grid: 13.8k records, 110 KB), and the
    global-memory kernel (n=61 block cube: 0.5 MB map, beyond shared memory)"""
    for eps, resident in ((c2_grid(1)[0], True), (random_voxel_grid(24, 64), True),
                          (c2_grid(3, n=61)[0], False)):
        n = round(len(eps) ** (1 / 3))
        gpu_ctx.upload_grid(eps, np.zeros(3), n / 2.0)
        assert gpu_ctx.grid_info()["smem_resident"] == resident
        _bitexact(gpu_ctx, oracle, eps, np.zeros(3), n / 2.0, 3000 if n > 41 else 20_000,
                  seed=n, stream0=7)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 12, 24])
def test_random_voxel_grids_bit_exact(gpu_ctx, oracle, n):
    eps = random_voxel_grid(n, 40 + n)
    _bitexact(gpu_ctx, oracle, eps, np.zeros(3), n / 2.0, 20_000, seed=n)


def test_launch_shape_does_not_change_parity(gpu_ctx, oracle):
    eps, c, h, _ = c1_grid(4)
    _bitexact(gpu_ctx, oracle, eps, c, h, 30_000, seed=8, blocks=3)


def test_masked_staircase_bit_exact(gpu_ctx, oracle):
    from tests.golden.make_golden import staircase_scene
    c = np.array([-10.0, 0, 0])
    eps, mask = oracle.build_grid(staircase_scene(), c, 10.0, 5, mask=True)
    g = _bitexact(gpu_ctx, oracle, eps, c, 10.0, 50_000, seed=64, mask=mask)
    assert g["cond_exits"] > 0
    assert set(np.unique(g["cond"][g["panel"] < 0])) == {7}


def test_philox_launch_independent_and_seeded(gpu_ctx):
    eps, c, h, _ = c1_grid(1)
    gpu_ctx.upload_grid(eps, c, h)
    a = gpu_ctx.microwalk_batch(300_000, seed=3, rng=PHILOX, per_transit=True)
    b = gpu_ctx.microwalk_batch(300_000, seed=3, rng=PHILOX, per_transit=True, blocks=7)
    assert np.array_equal(a["panel"], b["panel"]) and np.array_equal(a["steps"], b["steps"])
    d = gpu_ctx.microwalk_batch(300_000, seed=4, rng=PHILOX)
    assert not np.array_equal(a["hist"], d["hist"])
    # stream offsets index the same counter space
    e = gpu_ctx.microwalk_batch(1000, seed=3, stream_begin=1000, rng=PHILOX, per_transit=True)
    assert np.array_equal(e["panel"], a["panel"][1000:2000])


@pytest.mark.parametrize("rng", [PHILOX, PARITY])
def test_c1_histogram_matches_fdm_sgf(gpu_ctx, oracle, rng):
    """configs[0]: 1e6 transitions vs the FDM-solved SGF, chi-square p > 0.01."""
    eps, c, h, _ = c1_grid(1)
    exact = oracle.solve_sgf(eps, kernels=False)["probs"]
    gpu_ctx.upload_grid(eps, c, h)
    g = gpu_ctx.microwalk_batch(1_000_000, seed=2024, rng=rng)
    rep = compare_counts(exact, g["hist"])
    assert rep["p"] > 0.01, rep
    assert rep["tv"] <= 2.5 * expected_tv(exact, 1_000_000)
    # mean steps within 3 SE of the exact fundamental-matrix count
    n = 1_000_000
    mean = g["step_sum"] / n
    var = (g["step_sumsq"] - g["step_sum"] ** 2 / n) / (n - 1)
    assert abs(mean - oracle.expected_steps(eps)) <= 3 * np.sqrt(var / n)


@pytest.mark.parametrize("n,seed", [(4, 11), (6, 12)])
def test_random_grid_exit_law(gpu_ctx, oracle, n, seed):
    """test_microwalk.cpp:119-140 at 1e6 samples: TV <= 0.01 and chi-square pass."""
    from paper_2507_09730_b200.workloads import SplitMix64  # noqa: F401
    eps = random_voxel_grid(n, seed)
    exact = oracle.solve_sgf(eps, kernels=False)["probs"]
    gpu_ctx.upload_grid(eps)
    g = gpu_ctx.microwalk_batch(1_000_000, seed=seed, rng=PHILOX)
    rep = compare_counts(exact, g["hist"])
    assert rep["tv"] <= 0.01 and rep["p"] > 0.01, rep


def test_acceptance_transit_law_20_grids(gpu_ctx, oracle):
    """acceptance_main.cpp:65-90: 20 random n=4 grids, 1e6 transits each,
    TV <= 0.01 (the reference budget is 120 s on CPU)."""
    worst = 0.0
    for gi in range(20):
        eps = random_voxel_grid(4, 1, 1000 + gi)
        exact = oracle.solve_sgf(eps, kernels=False)["probs"]
        gpu_ctx.upload_grid(eps)
        g = gpu_ctx.microwalk_batch(1_000_000, seed=1, stream_begin=2000 * 10 ** 6 + gi * 10 ** 6,
                                    rng=PHILOX)
        rep = compare_counts(exact, g["hist"])
        worst = max(worst, rep["tv"])
        assert rep["chi2"] <= rep["crit_1e3"], (gi, rep)
    assert worst <= 0.01


def test_acceptance_step_law(gpu_ctx, oracle):
    """acceptance_main.cpp:95-132: mean steps within 3 SE on n=4/8 random grids."""
    for n in (4, 8):
        for gi in range(5):
            eps = random_voxel_grid(n, 2, 100 * n + gi)
            gpu_ctx.upload_grid(eps)
            S = 100_000
            g = gpu_ctx.microwalk_batch(S, seed=2, stream_begin=200 * n + gi, rng=PHILOX)
            mean = g["step_sum"] / S
            sd = np.sqrt((g["step_sumsq"] - g["step_sum"] ** 2 / S) / (S - 1))
            z = (mean - oracle.expected_steps(eps)) / (sd / np.sqrt(S))
            assert abs(z) <= 3.0, (n, gi, z)


@pytest.mark.slow
def test_c2_histogram_and_steps(gpu_ctx, oracle):
    """configs[1]: 1e7 transitions on the 41^3 block cube."""
    eps, c, h, _ = c2_grid(1)
    exact = oracle.solve_sgf(eps, kernels=False)["probs"]
    gpu_ctx.upload_grid(eps, c, h)
    n = 10_000_000
    g = gpu_ctx.microwalk_batch(n, seed=99, rng=PHILOX)
    rep = compare_counts(exact, g["hist"])
    assert rep["p"] > 0.01, rep
    mean = g["step_sum"] / n
    var = (g["step_sumsq"] - g["step_sum"] ** 2 / n) / (n - 1)
    assert abs(mean - oracle.expected_steps(eps)) <= 3 * np.sqrt(var / n)


def test_step_cap_raises(gpu_ctx):
    gpu_ctx.upload_grid(np.ones(8 ** 3))
    with pytest.raises(capi.StepCapExceeded):
        gpu_ctx.microwalk_batch(10, seed=66, rng=PARITY, step_cap=2)
    # the context stays usable afterwards
    g = gpu_ctx.microwalk_batch(10, seed=66, rng=PARITY)
    assert int(g["hist"].sum()) == 10


def test_engulfed_start_raises(gpu_ctx):
    mask = np.full(27, -1, np.int32)
    mask[13] = 4
    gpu_ctx.upload_grid(np.ones(27), mask=mask)
    with pytest.raises(capi.EngulfedStart):
        gpu_ctx.microwalk_batch(10, rng=PARITY)


def test_empty_batch(gpu_ctx):
    gpu_ctx.upload_grid(np.ones(27))
    g = gpu_ctx.microwalk_batch(0, rng=PHILOX)
    assert int(g["hist"].sum()) == 0 and g["step_sum"] == 0


def test_n1_one_step(gpu_ctx):
    gpu_ctx.upload_grid(np.array([3.0]))
    g = gpu_ctx.microwalk_batch(60_000, rng=PHILOX, per_transit=True)
    assert (g["steps"] == 1).all()
    rep = compare_counts(np.full(6, 1 / 6), g["hist"])
    assert rep["tv"] <= 0.01 and rep["p"] > 0.01

