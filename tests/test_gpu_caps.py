"""Structures past the device's fast-path capacities run, and match the
reference (geometry.cpp:47-62, microwalk.cpp:44-71 have no such caps):

* more than 63 distinct permittivities: the MicroWalk cells use job-local
  classes and divide the pair alphas out of the palette when it exceeds the
  shared-memory pair table;
* more than 64 boxes reaching into one MicroWalk cube: the hop runs on a
  dense voxel grid (k_mw_dense), and a first-transition ladder-branch-2 cube
  classifies its voxel centres one by one.

Walk records are compared bitwise with the reference Engine (parity streams,
its own SGF tables injected), and production-mode capacitances with the
reference's Engine::extract within 3 combined standard errors."""
import math
import os

import numpy as np
import pytest

from paper_2507_09730_b200 import capi
from tests.scenes import block_array_scene
from tests.test_gpu_ref_parity import _sgf1_solver
from tests.walk_helpers import upload_scene, walk_params

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8
MODES = {"HYBRID-MW": capi.MODE_HYBRID_MW, "HYBRID-MWE": capi.MODE_HYBRID_MWE}


@pytest.mark.parametrize("distinct", [True, False])
@pytest.mark.parametrize("mode", sorted(MODES))
def test_dense_cubes_bit_exact_vs_reference_engine(gpu_ctx, ref, tmp_path, mode, distinct):
    sc = block_array_scene(distinct=distinct)
    assert sc.n_diel == 1000 and (len(set(sc.diel_eps)) > 63) == distinct
    count = 96
    path = tmp_path / "ref.sgf"
    slot, w, ab = ref.structure(sc).run_walks(0, count, threads=THREADS, cache_out=str(path),
                                              grid_n=24, mode=mode, seed=31)
    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    p = walk_params(sc, grid_n=24, seed=31, rng=capi.RNG_SPLITMIX_PARITY, n_slots=4096,
                    mode=MODES[mode])
    tally, rec = gpu_ctx.run_walks(p, sc.master_slot(), 0, count, _sgf1_solver(path))
    assert tally["mw_dense_hops"] > 0  # the dense path ran
    assert np.array_equal(rec["slot"], slot), np.nonzero(rec["slot"] != slot)[0][:10]
    assert np.array_equal(rec["aborted"], ab)
    assert np.array_equal(rec["weight"], w)


@pytest.mark.parametrize("mode", sorted(MODES))
def test_dense_cubes_production_vs_reference_extract(ref, tmp_path, mode):
    import paper_2507_09730_b200.frwcap as frwcap
    sc = block_array_scene()
    text = sc.to_json()
    frwcap.sgf_cache_clear()
    g = frwcap.extract_json(text, mode=mode, grid_n=24, min_walks=100_000, max_walks=100_000,
                            seed=5)
    assert g["mw_dense_hops"] > 0
    path = str(tmp_path / "dev.sgf")
    frwcap.sgf_cache_save(path)
    r = ref.structure(sc).extract(threads=THREADS, cache_in=path, grid_n=24, mode=mode,
                                  min_walks=4096, max_walks=4096, seed=6)
    for k, tg in enumerate(g["terminals"]):
        if r["landed"][k] < 50:
            continue
        se = math.hypot(tg["std_err_farads"], r["std_err"][k])
        z = abs(tg["capacitance_farads"] - r["value"][k]) / se
        assert z < 3.0, (k, tg, r["value"][k], z)


@pytest.mark.parametrize("n,count", [(80, 160), (128, 48)])
@pytest.mark.parametrize("mode", sorted(MODES))
def test_large_lattice_bit_exact_vs_reference_engine(gpu_ctx, ref, tmp_path, mode, n, count):
    """grid_n past 64 (the reference takes any lattice size,
    engine.cpp:69-82): stratification probes classify slice centres one by
    one, the stratified-SGF direct solve stages its DST basis in dynamic
    shared memory, and the walks equal the reference Engine's bit for bit
    on the device-solved tables (the same SGF1 file on both sides)."""
    import paper_2507_09730_b200.frwcap as frwcap
    from paper_2507_09730_b200.workloads import c3_structure
    from tests.scenes import scene_from_doc
    sc = scene_from_doc(c3_structure())
    cache = frwcap.SgfCache()

    def solve(nn, axis, layers):
        probs = np.asarray(cache.get(nn, axis, list(layers)))
        kern = np.asarray(cache.kernels(nn, axis, list(layers)))
        return 1.0, probs, np.cumsum(probs), kern

    upload_scene(gpu_ctx, sc)
    gpu_ctx.sgf_clear()
    p = walk_params(sc, grid_n=n, seed=41, rng=capi.RNG_SPLITMIX_PARITY, n_slots=4096,
                    mode=MODES[mode])
    tally, rec = gpu_ctx.run_walks(p, sc.master_slot(), 0, count, solve)
    assert tally["misses"] > 0 and (rec["done"] == 1).all()
    path = tmp_path / "dev.sgf"
    cache.save(str(path))
    slot, w, ab = ref.structure(sc).run_walks(0, count, threads=THREADS, cache_in=str(path),
                                              grid_n=n, mode=mode, seed=41)
    assert np.array_equal(rec["slot"], slot), np.nonzero(rec["slot"] != slot)[0][:10]
    assert np.array_equal(rec["aborted"], ab)
    assert np.array_equal(rec["weight"], w)
    # production mode (Philox, lattice jumps up to radius 31) runs at this size
    p = walk_params(sc, grid_n=n, seed=42, rng=capi.RNG_PHILOX, mode=MODES[mode])
    tally, rec = gpu_ctx.run_walks(p, sc.master_slot(), 0, 4096, None)
    assert (rec["done"] == 1).all() and tally["landed"].sum() == 4096
