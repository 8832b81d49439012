"""Scenes restated from the reference's unit tests and fixtures."""
import json
import os

import numpy as np

from oracle.oracle import Scene

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")


def plate_scene():
    """test_engine.cpp:16-23: two 1000x1000 plates 200 nm apart, master 1."""
    return Scene(np.array([1, 2], np.int32),
                 np.array([[0, 0, -50, 1000, 1000, 0], [0, 0, 200, 1000, 1000, 250]], float),
                 np.zeros((0, 6)), np.zeros(0), 1.0,
                 np.array([-2000, -2000, -2000, 3000, 3000, 3000.0]), 1)


def layered_plate_scene():
    """test_engine.cpp:27-32: plates with two dielectric films in the gap."""
    s = plate_scene()
    return Scene(s.cond_id, s.cond_box,
                 np.array([[-2000, -2000, 0, 3000, 3000, 80], [-2000, -2000, 80, 3000, 3000, 200]],
                          float), np.array([3.9, 7.5]), 1.0, s.world, 1)


def plate_pocket_scene():
    """test_engine.cpp:513-520: plates plus a general eps=16 pocket."""
    s = plate_scene()
    return Scene(s.cond_id, s.cond_box, np.array([[1100, 400, 30, 1180, 520, 170]], float),
                 np.array([16.0]), 1.0, s.world, 1)


def two_plates_small():
    """tests/python/test_smoke.py:13-22 TWO_PLATES."""
    return Scene(np.array([1, 2], np.int32),
                 np.array([[90, 90, 150, 390, 390, 170], [90, 90, 310, 390, 390, 330]], float),
                 np.zeros((0, 6)), np.zeros(0), 1.0, np.array([0, 0, 0, 480, 480, 480.0]), 1)


FIXTURE_NAMES = ("conformal_staircase", "highk_cross", "plates_uniform", "stratified_stack")


def load_fixture(name):
    """The reference's tests/fixtures/<name>.json as parsed by the reference's
    own parse_structure (stored by tests/golden/make_golden.py)."""
    g = np.load(GOLD)
    k = "fx_" + name
    misc = g[k + "_misc"]
    return Scene(g[k + "_cond_id"], g[k + "_cond_box"], g[k + "_diel_box"].reshape(-1, 6),
                 g[k + "_diel_eps"], float(misc[0]), misc[2:8].copy(), int(misc[1]))


def scene_from_doc(doc):
    cb = np.array([c["lo"] + c["hi"] for c in doc["conductors"]], float)
    ids = np.array([c["id"] for c in doc["conductors"]], np.int32)
    d = doc.get("dielectrics", [])
    db = np.array([x["lo"] + x["hi"] for x in d], float).reshape(-1, 6)
    de = np.array([x["eps"] for x in d], float)
    w = doc["world"]
    return Scene(ids, cb, db, de, float(doc.get("background_eps", 1.0)),
                 np.array(w["lo"] + w["hi"], float), int(doc["master"]))


def block_array_scene(nx=10, edge=30.0, pitch=70.0, seed=9, distinct=True):
    """Two plates 800 nm apart with an nx^3 array of small dielectric blocks
    between them (edge 30 nm, pitch 70 nm), each block its own permittivity
    (distinct=True: nx^3 distinct values, far more than 63): a transition
    cube in the gap holds far more than 64 boxes, so its MicroWalk hop runs
    on the dense grid and the palette exceeds the shared-memory pair table."""
    from paper_2507_09730_b200.workloads import SplitMix64
    r = SplitMix64(seed, 0)
    span = (nx - 1) * pitch + edge
    lo0 = -span / 2
    boxes, eps = [], []
    for k in range(nx):
        for j in range(nx):
            for i in range(nx):
                lo = [lo0 + i * pitch, lo0 + j * pitch, lo0 + k * pitch]
                boxes.append(lo + [v + edge for v in lo])
                eps.append(2.0 + 20.0 * r.uniform() if distinct else 7.0)
    cond = np.array([[-600, -600, -600, -400, 600, 600], [400, -600, -600, 600, 600, 600]],
                    float)
    return Scene(np.array([1, 2], np.int32), cond, np.array(boxes), np.array(eps), 1.0,
                 np.array([-3000, -3000, -3000, 3000, 3000, 3000.0]), 1)
