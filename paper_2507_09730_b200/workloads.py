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
