"""Seeded synthetic workloads for the BASELINE.json configs (C1-C5).

The paper's industrial structures (RT1-RT8, Cases 1-2) are proprietary and
absent; these generators stand in for them with the shapes, sizes and value
distributions BASELINE.json names.  Every random draw comes
from the reference's SplitMix64 (rng.hpp:12-40), restated here in integer
Python so inputs are bit-identical on every host.
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    """SplitMix64::mix (rng.hpp:30-35)."""
    z = (z + _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class SplitMix64:
    """rng.hpp:12-40: per-(seed, stream) independent sequences."""

    def __init__(self, seed: int, stream: int | None = None):
        if stream is None:
            self.state = mix64(seed & _M64)
        else:
            self.state = mix64((mix64(seed & _M64) + ((stream + 1) * _GAMMA)) & _M64)

    def next(self) -> int:
        self.state = (self.state + _GAMMA) & _M64
        return mix64(self.state)

    def uniform(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        return self.next() % n


# ---------------------------------------------------------------------------
# single-cube MicroWalk workloads (configs[0], configs[1])

def c1_grid(seed: int = 1, n: int = 21):
    """C1: n^3 unit-pitch cube, eps 3.9 with one eps 7.0 inclusion box whose
    corner indices are uniform on the grid (random_block_grid's recipe,
    oracle.cpp:322-339, with a fixed eps).  Returns (eps, center, half_width,
    meta)."""
    rng = SplitMix64(seed, 0)
    eps = np.full((n, n, n), 3.9)  # [k, j, i] -> x fastest when flattened
    lo, hi = [], []
    for _ in range(3):
        x = int(rng.uniform() * n)
        y = int(rng.uniform() * n)
        lo.append(min(min(x, y), n - 1))
        hi.append(min(max(x, y), n - 1))
    eps[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1] = 7.0
    return eps.reshape(-1).copy(), np.zeros(3), n / 2.0, dict(box_lo=lo, box_hi=hi)


C2_PALETTE = (2.5, 3.9, 7.5, 25.0)


def c2_grid(seed: int = 1, n: int = 41, block: int = 4):
    """C2: n^3 cube, eps piecewise constant on block^3-node blocks, each block
    uniform on {2.5, 3.9, 7.5, 25.0} (blocks drawn x-fastest from
    SplitMix64(seed, 0)); the last block along each axis is 1 node thick."""
    rng = SplitMix64(seed, 0)
    nb = (n + block - 1) // block
    pal = np.array(C2_PALETTE)
    blocks = np.empty((nb, nb, nb))
    for bk in range(nb):
        for bj in range(nb):
            for bi in range(nb):
                blocks[bk, bj, bi] = pal[rng.below(len(pal))]
    idx = np.arange(n) // block
    eps = blocks[idx[:, None, None], idx[None, :, None], idx[None, None, :]]
    return eps.reshape(-1).copy(), np.zeros(3), n / 2.0, dict(blocks=nb)


def random_voxel_grid(n: int, seed: int, stream: int | None = None):
    """oracle.cpp:315-320: eps ~ Exp(rate 0.1) per voxel, unit-pitch cube."""
    rng = SplitMix64(seed, stream)
    out = np.empty(n ** 3)
    for i in range(n ** 3):
        out[i] = max(-10.0 * np.log1p(-rng.uniform()), 1e-9)
    return out


# ---------------------------------------------------------------------------
# full-walk structures (configs[2..4]); coordinates in nm.  A structure is a
# dict in the reference's JSON schema (geometry.cpp:124-259) so it feeds
# both the drop-in API (extract_json) and the oracle.

def _box(lo, hi):
    return {"lo": [float(v) for v in lo], "hi": [float(v) for v in hi]}


def _inflate(lo, hi, d):
    return [v - d for v in lo], [v + d for v in hi]


def c3_structure():
    """C3: two 100x100x5000 wires (100 nm apart) 200 nm above a 2x2 um
    ground plane (thickness pinned to 100 nm); three full-width z layers of
    200 nm (eps 2.5/3.9/4.2) declared first, then a 20 nm eps=7.0 coating
    around each wire.  Wire 1 (id 1) is the master."""
    w1 = ([-150, -2500, 200], [-50, 2500, 300])
    w2 = ([50, -2500, 200], [150, 2500, 300])
    plane = ([-1000, -1000, -100], [1000, 1000, 0])
    world = ([-5000, -5000, -1000], [5000, 5000, 2000])
    diel = [
        dict(eps=2.5, **_box([-5000, -5000, 0], [5000, 5000, 200])),
        dict(eps=3.9, **_box([-5000, -5000, 200], [5000, 5000, 400])),
        dict(eps=4.2, **_box([-5000, -5000, 400], [5000, 5000, 600])),
        dict(eps=7.0, **_box(*_inflate(*w1, 20))),
        dict(eps=7.0, **_box(*_inflate(*w2, 20))),
    ]
    return {"units": "nm", "world": _box(*world), "background_eps": 1.0,
            "conductors": [dict(id=1, **_box(*w1)), dict(id=2, **_box(*w2)),
                           dict(id=3, **_box(*plane))],
            "dielectrics": diel, "master": 1}


def c4_structure(seed: int = 4):
    """C4: 3-layer crossing bus, 5 wires per layer along x / y / x (width 50,
    pitch 100, length 600; wire thickness pinned to 50 nm, vertical layer
    gap 100 nm), ILD slabs eps 2.7/3.0/3.9, 10 nm eps=7.5 liners, 10 seeded
    LDE blocks (edges U(20,100) nm, eps U(4,25)).  Master: the middle wire of
    the middle layer."""
    rng = SplitMix64(seed, 0)
    cond, liners = [], []
    z0 = [0, 150, 300]
    cid = 1
    master = None
    for layer in range(3):
        for w in range(5):
            c = -200 + 100 * w
            if layer == 1:   # along y
                lo, hi = [c - 25, -300, z0[layer]], [c + 25, 300, z0[layer] + 50]
            else:            # along x
                lo, hi = [-300, c - 25, z0[layer]], [300, c + 25, z0[layer] + 50]
            cond.append(dict(id=cid, **_box(lo, hi)))
            liners.append(dict(eps=7.5, **_box(*_inflate(lo, hi, 10))))
            if layer == 1 and w == 2:
                master = cid
            cid += 1
    world = ([-1500, -1500, -800], [1500, 1500, 1150])
    diel = [
        dict(eps=2.7, **_box([-1500, -1500, -800], [1500, 1500, 100])),
        dict(eps=3.0, **_box([-1500, -1500, 100], [1500, 1500, 250])),
        dict(eps=3.9, **_box([-1500, -1500, 250], [1500, 1500, 1150])),
    ] + liners
    for _ in range(10):
        e = [20 + 80 * rng.uniform() for _ in range(3)]
        lo = [-350 + (700 - e[0]) * rng.uniform(), -350 + (700 - e[1]) * rng.uniform(),
              -50 + (450 - e[2]) * rng.uniform()]
        eps = 4 + 21 * rng.uniform()
        diel.append(dict(eps=eps, **_box(lo, [lo[a] + e[a] for a in range(3)])))
    return {"units": "nm", "world": _box(*world), "background_eps": 1.0,
            "conductors": cond, "dielectrics": diel, "master": master}


def c5_structure(seed: int = 5, n_cond: int = 200, n_blocks: int = 50):
    """C5: n_cond non-overlapping box conductors (edges U(50,500) nm,
    rejection-sampled with >= 60 nm clearance so coatings never touch another
    conductor) in a 10x10x2 um domain; 4 z layers of 500 nm (eps pinned to
    2.5/3.0/3.9/4.2), 20 nm eps=7.0 coatings, n_blocks eps=25 blocks (edges
    pinned to U(50,300) nm).  Masters: the first 10 conductors."""
    rng = SplitMix64(seed, 0)
    dom = [10000.0, 10000.0, 2000.0]
    boxes = []
    tries = 0
    while len(boxes) < n_cond:
        tries += 1
        if tries > 200000:
            raise RuntimeError("c5_structure: rejection sampling failed")
        e = [50 + 450 * rng.uniform() for _ in range(3)]
        lo = [100 + (dom[a] - 200 - e[a]) * rng.uniform() for a in range(3)]
        hi = [lo[a] + e[a] for a in range(3)]
        ok = True
        for blo, bhi in boxes:
            gap = max(max(blo[a] - hi[a], lo[a] - bhi[a]) for a in range(3))
            if gap < 60:
                ok = False
                break
        if ok:
            boxes.append((lo, hi))
    diel = [dict(eps=e, **_box([0, 0, 500 * q], [dom[0], dom[1], 500 * (q + 1)]))
            for q, e in enumerate((2.5, 3.0, 3.9, 4.2))]
    diel += [dict(eps=7.0, **_box(*_inflate(lo, hi, 20))) for lo, hi in boxes]
    for _ in range(n_blocks):
        e = [50 + 250 * rng.uniform() for _ in range(3)]
        lo = [(dom[a] - e[a]) * rng.uniform() for a in range(3)]
        diel.append(dict(eps=25.0, **_box(lo, [lo[a] + e[a] for a in range(3)])))
    cond = [dict(id=i + 1, **_box(lo, hi)) for i, (lo, hi) in enumerate(boxes)]
    return {"units": "nm", "world": _box([0, 0, 0], dom), "background_eps": 1.0,
            "conductors": cond, "dielectrics": diel, "master": 1}
