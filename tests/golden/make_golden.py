"""Generate the golden fixtures from the REFERENCE's own code.

Runs oracle/_ref/libfrwref.so -- the reference's microwalk.cpp, geometry.cpp,
engine.cpp and sgf_cache.cpp compiled unmodified from /root/reference (plus
the restated Eigen-free sgf.cpp shim) -- and stores small input/output
vectors under tests/golden/.  The CPU tests pin the C restatement
(oracle/frw_oracle.c) against these files, so the pin holds on machines
where /root/reference is absent.  Re-run with
    python tests/golden/make_golden.py
after `make -C oracle ref`.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, Scene  # noqa: E402
from paper_2507_09730_b200.workloads import (SplitMix64, c1_grid, c2_grid,  # noqa: E402
                                             random_voxel_grid)


def staircase_scene():
    """test_microwalk.cpp:278-329: conductor 7 swallows the +x part."""
    return Scene(np.array([7], np.int32), np.array([[-9.9, -11, -11, 2, 11, 11]], float),
                 np.zeros((0, 6)), np.zeros(0), 2.0, np.array([-40, -40, -40, 40, 40, 40.0]), 7)


def layered_scene():
    """test_microwalk.cpp:30-38 layered_structure (plus a far conductor so
    the scene validates)."""
    return Scene(np.array([1], np.int32), np.array([[30, 30, 30, 35, 35, 35]], float),
                 np.array([[-40, -40, -40, 40, 40, -2], [-40, -40, -2, 40, 40, 3],
                           [1, -5, -40, 12, 9, 40]], float),
                 np.array([3.9, 7.5, 22.0]), 1.0, np.array([-40, -40, -40, 40, 40, 40.0]), 1)


def random_scene(seed, n_cond=12, n_diel=10):
    """Random boxes in a 100^3 world, seeded (test_geometry.cpp:184-231 style)."""
    r = SplitMix64(seed, 0)
    cb, ids = [], []
    for i in range(n_cond):
        lo = [r.uniform() * 90 - 50 for _ in range(3)]
        ext = [1 + r.uniform() * 10 for _ in range(3)]
        cb.append(lo + [lo[a] + ext[a] for a in range(3)])
        ids.append(100 + i)
    db, de = [], []
    for i in range(n_diel):
        lo = [r.uniform() * 90 - 50 for _ in range(3)]
        ext = [1 + r.uniform() * 40 for _ in range(3)]
        db.append(lo + [min(lo[a] + ext[a], 50.0) for a in range(3)])
        de.append(1.0 + 20 * r.uniform())
    return Scene(np.array(ids, np.int32), np.array(cb), np.array(db), np.array(de), 2.5,
                 np.array([-60, -60, -60, 60, 60, 60.0]), ids[0])


def main():
    ref = Ref()
    out = {}
    # -- single-cube transits (microwalk_transit) --------------------------------
    grids = {
        "c1_s1": c1_grid(1)[0],
        "c2_s1": c2_grid(1)[0],
        "rv4_s11": random_voxel_grid(4, 11),
        "rv6_s12": random_voxel_grid(6, 12),
        "rv1_s2": random_voxel_grid(1, 2),
        "rv2_s3": random_voxel_grid(2, 3),
    }
    for name, eps in grids.items():
        n = round(len(eps) ** (1 / 3))
        cnt = 400 if n > 30 else 2000
        r = ref.microwalk_grid(eps, np.zeros(3), n / 2.0, seed=3, stream0=0, count=cnt)
        out[f"mw_{name}_eps"] = eps
        out[f"mw_{name}_panel"] = r["panel"]
        out[f"mw_{name}_steps"] = r["steps"]
    # masked staircase grid (MicroWalk-E lattice, test_microwalk.cpp:278-329)
    h = ref.structure(staircase_scene())
    c, hw = np.array([-10.0, 0, 0]), 10.0
    eps, mask, _, _ = h.build_grid(c, hw, 5, allow_conductors=True)
    r = ref.microwalk_grid(eps, c, hw, seed=64, stream0=2, count=2000, mask=mask)
    out.update(mw_stair_eps=eps, mw_stair_mask=mask, mw_stair_panel=r["panel"],
               mw_stair_steps=r["steps"])
    # -- SGF solves (restated sgf.cpp) and expected steps ---------------------------
    for name in ("rv4_s11", "rv6_s12"):
        s = ref.solve_sgf(grids[name])
        out[f"sgf_{name}_probs"] = s["probs"]
        out[f"sgf_{name}_kernels"] = s["kernels"]
        out[f"sgf_{name}_esteps"] = np.array([ref.expected_steps(grids[name])])
    # -- geometry queries on random scenes --------------------------------------------
    for sd in (1, 2, 3):
        sc = random_scene(sd)
        hh = ref.structure(sc)
        rr = SplitMix64(sd, 99)
        pts, eps_at, cond_at, free_h = [], [], [], []
        for _ in range(400):
            p = [rr.uniform() * 118 - 59 for _ in range(3)]
            pts.append(p)
            eps_at.append(hh.permittivity_at(p))
            cid = hh.conductor_at(p, 0.5)
            cond_at.append(-1 if cid is None else cid)
            try:
                free_h.append(hh.max_free_cube(p)[0])
            except ValueError:
                free_h.append(-1.0)
        out[f"geo{sd}_scene"] = np.concatenate([sc.cond_box.ravel(), sc.diel_box.ravel(),
                                                sc.diel_eps])
        out[f"geo{sd}_pts"] = np.array(pts)
        out[f"geo{sd}_eps"] = np.array(eps_at)
        out[f"geo{sd}_cond"] = np.array(cond_at, np.int32)
        out[f"geo{sd}_free"] = np.array(free_h)
        # stratification probe on cubes around sample points
        prof_axis, prof_layers = [], []
        for p in pts[:100]:
            try:
                ax, layers = hh.stratified_profile(p, 3.0, 6)
            except ValueError:  # slice centre outside the world: reference throws
                ax, layers = -2, None
            prof_axis.append(-1 if ax is None else ax)
            prof_layers.append(np.zeros(6) if layers is None else layers)
        out[f"geo{sd}_prof_axis"] = np.array(prof_axis, np.int32)
        out[f"geo{sd}_prof_layers"] = np.array(prof_layers)
    # lazy transits on the layered scene (microwalk_transit_lazy)
    hl = ref.structure(layered_scene())
    for n in (5, 6):
        p, hw0 = np.zeros(3), 6.0
        if n % 2 == 0:
            d = hw0 / (n + 1)
            cc, hw = p + d, (hw0 - d) * (1.0 - 1e-12)
        else:
            cc, hw = p, hw0
        r = hl.microwalk_lazy(cc, hw, n, seed=61, stream0=5, count=300)
        out[f"lazy{n}_center"] = cc
        out[f"lazy{n}_hw"] = np.array([hw])
        out[f"lazy{n}_panel"] = r["panel"]
        out[f"lazy{n}_steps"] = r["steps"]
        out[f"lazy{n}_point"] = r["point"]
    # -- the reference's fixture structures, parsed by its own parse_structure
    fx_dir = "/root/reference/proj/tests/fixtures"
    for fn in sorted(os.listdir(fx_dir)):
        with open(os.path.join(fx_dir, fn)) as f:
            sc = ref.parse(f.read())
        key = "fx_" + fn.replace(".json", "")
        out[key + "_cond_id"] = sc.cond_id
        out[key + "_cond_box"] = sc.cond_box
        out[key + "_diel_box"] = sc.diel_box
        out[key + "_diel_eps"] = sc.diel_eps
        out[key + "_misc"] = np.array([sc.background_eps, sc.master_id, *sc.world])
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    meta = {"generator": "tests/golden/make_golden.py",
            "source": "oracle/_ref/libfrwref.so (reference sources from /root/reference/proj)",
            "keys": sorted(out)}
    with open(os.path.join(HERE, "reference_vectors.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
