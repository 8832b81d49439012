"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and the stencil-table compilation reproduces the
reference's f64 direction scan bit for bit (emulated on the host)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c1_grid, c2_grid, random_voxel_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(frw_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    names = _declared("frw_gpu.h")
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_device():
    # on a CPU-only host the context must fail loudly, never emulate
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(capi.FrwError):
        capi.Context(0)


M64 = (1 << 64) - 1


def _emulate(oracle, eps, seed, count, mask=None):
    """Host replay of the kernel's table-driven step (mw_grid.cu): padded
    map with an absorbing halo, five 11-bit SWAR lanes, exact fallback."""
    n = round(len(eps) ** (1 / 3))
    mp, rec, full = capi.grid_compile(eps, mask)
    npad = n + 2
    exit_rec = len(rec) - 1
    strides = [-1, 1, -npad, npad, -npad * npad, npad * npad]
    ones = sum(1 << (12 * d) for d in range(5))
    guard = ones << 11
    c = (n - 1) // 2
    out = []
    for t in range(count):
        st = oracle.stream_state(seed, t)
        idx = ((c + 1) * npad + (c + 1)) * npad + (c + 1)
        node = [c, c, c]
        steps = 0
        while True:
            steps += 1
            st = (st + 0x9E3779B97F4A7C15) & M64
            z = int(oracle.lib.frwo_mix(st))
            r = int(mp[idx])
            rc = int(rec[r])
            d1 = ((z >> 53) * ones + rc) & M64               # SWAR lanes
            d = bin(d1 & (guard | 1 << 63)).count("1")        # x11 > T_d
            # 11-bit tie: lane d reads 2047 (mw_grid_fast); the same test as
            # "some lane's low 11 bits are all ones" (mw_grid_kernel)
            tie = ((d1 >> (12 * d)) & 0x7FF) == 0x7FF
            assert tie == ((((d1 + ones) ^ d1) & guard) != 0)
            if tie:
                d = sum((z >> 11) >= int(full[r, q]) for q in range(5))
            prev = list(node)
            node[d >> 1] += 1 if d & 1 else -1
            idx += strides[d]
            if int(mp[idx]) == exit_rec:                      # absorbing node
                ax = d >> 1
                if not 0 <= node[ax] < n:
                    i, j, k = prev
                    u = j if ax == 0 else i
                    v = j if ax == 2 else k
                    out.append(((d * n + v) * n + u, steps))
                else:
                    out.append((-1, steps))
                break
    return np.array(out)


@pytest.mark.parametrize("which", ["c1", "c2", "rv3", "rv6"])
def test_threshold_tables_replay_reference_bit_exact(oracle, which):
    eps = {"c1": c1_grid(1)[0], "c2": c2_grid(1)[0], "rv3": random_voxel_grid(3, 5),
           "rv6": random_voxel_grid(6, 12)}[which]
    n = round(len(eps) ** (1 / 3))
    cnt = 40 if n > 30 else 300
    e = _emulate(oracle, eps, 3, cnt)
    w = oracle.microwalk_grid(eps, np.zeros(3), n / 2.0, 3, 0, cnt)
    assert np.array_equal(e[:, 0], w["panel"]) and np.array_equal(e[:, 1], w["steps"])


def test_threshold_tables_masked(oracle):
    from tests.golden.make_golden import staircase_scene
    eps, mask = oracle.build_grid(staircase_scene(), [-10.0, 0, 0], 10.0, 5, mask=True)
    # the emulator assumes a unit cube; panels/steps do not depend on geometry
    e = _emulate(oracle, eps, 64, 300, mask)
    w = oracle.microwalk_grid(eps, np.array([-10.0, 0, 0]), 10.0, 64, 0, 300, mask=mask)
    assert np.array_equal(e[:, 0], w["panel"]) and np.array_equal(e[:, 1], w["steps"])


def test_record_counts_fit_shared_memory():
    for eps in (c1_grid(1)[0], c2_grid(1)[0]):
        n = round(len(eps) ** (1 / 3))
        _, rec, _ = capi.grid_compile(eps)
        smem = (2 * (n + 2) ** 3 + 15) // 16 * 16 + (8 * rec.shape[0] + 15) // 16 * 16
        assert smem <= 227 * 1024


def test_packed_thresholds_are_monotone_prefixes():
    """lane d holds 2047 minus the top 11 bits of X_d; X_d is non-decreasing;
    the halo and only the halo maps to the exit record"""
    eps = c2_grid(1)[0]
    mp, rec_all, full = capi.grid_compile(eps)
    rec, full = rec_all[:-1], full[:-1]  # the last record is the exit record
    assert (np.diff(full.astype(np.float64), axis=1) >= 0).all()
    assert int(rec_all[-1]) == sum(1 << (12 * d + 11) for d in range(5)) | 1 << 63  # exit: dir 6
    lanes = np.stack([(rec >> np.uint64(12 * d)) & np.uint64(4095) for d in range(5)], axis=1)
    assert np.array_equal(lanes, 2047 - np.minimum(full >> np.uint64(42), np.uint64(2047)))
    n = 41
    m3 = mp.reshape(n + 2, n + 2, n + 2)
    ex = len(rec)
    assert (m3[0] == ex).all() and (m3[-1] == ex).all() and (m3[:, 0] == ex).all()
    assert (m3[:, :, -1] == ex).all() and (m3[1:-1, 1:-1, 1:-1] < ex).all()


def test_invalid_grid_rejected():
    with pytest.raises(capi.FrwError):
        capi.grid_compile(np.array([1.0, -2.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0]))


def _bisect_threshold(acc, s):
    """the definition: smallest x in [0, 2^53] with fl(x*s) >= acc*2^53"""
    import math
    target = math.ldexp(acc, 53)
    lo, hi = 0, 1 << 53
    while lo < hi:
        mid = (lo + hi) // 2
        if float(mid) * s >= target:
            hi = mid
        else:
            lo = mid + 1
    return lo


@pytest.mark.parametrize("which", ["c2", "rv6"])
def test_exact_thresholds_match_bisection(which):
    """frw_grid_compile's X_d (quotient estimate + exact walk) equal the
    bisection definition for every record, recomputing the alphas from the
    grid as microwalk.cpp:91-109 does"""
    eps = c2_grid(1)[0] if which == "c2" else random_voxel_grid(6, 12)
    n = round(len(eps) ** (1 / 3))
    mp, rec, full = capi.grid_compile(eps)
    e3 = eps.reshape(n, n, n)  # [k][j][i]
    seen = set()
    npad = n + 2
    for v in range(n ** 3):
        k, j, i = v // (n * n), (v // n) % n, v % n
        r = int(mp[((k + 1) * npad + (j + 1)) * npad + (i + 1)])
        if r in seen:
            continue
        seen.add(r)
        ev = float(e3[k, j, i])
        acc, s = [], 0.0
        for d in range(6):
            nb = [i, j, k]
            nb[d >> 1] += 1 if d & 1 else -1
            if not 0 <= nb[d >> 1] < n:
                a = 1.0
            else:
                en = float(e3[nb[2], nb[1], nb[0]])
                a = en / (en + ev)
            s += a
            acc.append(s)
        for d in range(5):
            assert int(full[r, d]) == _bisect_threshold(acc[d], s), (r, d)
