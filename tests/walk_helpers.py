"""Helpers for the walk-engine parity tests: host-exact engine parameters
(restating gaussian_surface, engine.cpp:84-124, and the snap distance,
engine.cpp:186-187) and an SGF solver callback backed by the oracle."""
import json

import numpy as np

from paper_2507_09730_b200 import capi


def gaussian_params(sc, gap_fraction=0.5, snap_tol=1e-4):
    m = sc.master_slot()
    mb = sc.cond_box[m]
    gap = float("inf")
    for a in range(3):
        gap = min(gap, mb[a] - sc.world[a])
        gap = min(gap, sc.world[3 + a] - mb[3 + a])
    for c in range(sc.n_cond):
        if c == m:
            continue
        cb = sc.cond_box[c]
        g = 0.0
        for a in range(3):
            g = max(g, max(mb[a] - cb[3 + a], cb[a] - mb[3 + a]))
        gap = min(gap, max(g, 0.0))
    inflate = gap_fraction * gap
    box = [mb[a] - inflate for a in range(3)] + [mb[3 + a] + inflate for a in range(3)]
    ex, ey, ez = box[3] - box[0], box[4] - box[1], box[5] - box[2]
    f = [ey * ez, ey * ez, ex * ez, ex * ez, ex * ey, ex * ey]
    total = 0.0
    for v in f:
        total += v
    cdf, acc = [], 0.0
    for v in f:
        acc += v / total
        cdf.append(acc)
    cdf[5] = 1.0
    area = total * 1e-9 * 1e-9
    he = max((box[3 + a] - box[a]) / 2 for a in range(3))
    return box, cdf, area, snap_tol * he


def walk_params(sc, grid_n=24, seed=1, rng=capi.RNG_PHILOX, hop_cap=10000, n_slots=0,
                mode=capi.MODE_HYBRID_MW, gap_fraction=0.5, snap_tol=1e-4):
    box, cdf, area, snap = gaussian_params(sc, gap_fraction, snap_tol)
    d6 = capi.C.c_double * 6
    return capi.WalkParams(grid_n, mode, 5.0, snap, hop_cap, seed, rng, n_slots, d6(*box),
                           d6(*cdf), area)


def oracle_solver(oracle):
    """(n, axis, rounded layers) -> canonical unit-pitch SGF via the oracle
    (the oracle's own cache does exactly this, frw_oracle.c cache_get)."""
    def solve(n, axis, layers):
        idx = np.indices((n, n, n))  # [k, j, i]
        coord = {0: idx[2], 1: idx[1], 2: idx[0]}[axis]
        eps = np.asarray(layers)[coord].reshape(-1)
        s = oracle.solve_sgf(eps, half_width=n / 2.0, kernels=True)
        cdf = np.cumsum(s["probs"])  # sequential running sum, like the C cache
        return s["pitch"], s["probs"], cdf, s["kernels"]
    return solve


def upload_scene(ctx, sc):
    ctx.upload_structure(sc.cond_id, sc.cond_box, sc.diel_box, sc.diel_eps,
                         sc.background_eps, sc.world)


def scene_json(sc):
    return sc.to_json()


def load_json_scene(doc):
    from tests.scenes import scene_from_doc
    return scene_from_doc(json.loads(doc) if isinstance(doc, str) else doc)
