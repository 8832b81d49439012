"""StratifiedSgfCache of the B200 build (sgf_cache.hpp / sgf_cache.cpp):
SGF1 files interchange with the reference's own cache code in both
directions (CPU), and on the device: cached solves equal the reference's,
LRU eviction at capacity, hit/miss accounting, scale-factor keys
(test_cache.cpp:50-260)."""
import numpy as np
import pytest

import paper_2507_09730_b200.frwcap as frwcap

N = 6
KEYS = [(0, [2.0] * N), (2, [2.5, 2.5, 3.9, 3.9, 7.0, 7.0]), (1, [1.0, 4.0, 4.0, 4.0, 9.5, 9.5])]


def _ref_file(ref, tmp_path):
    path = str(tmp_path / "ref.sgf")
    ref.cache_save(N, [k[0] for k in KEYS], np.array([k[1] for k in KEYS]), path)
    return path


def test_reference_sgf1_file_loads_unchanged(ref, tmp_path):
    path = _ref_file(ref, tmp_path)
    c = frwcap.SgfCache()
    assert c.load(path) == len(KEYS)
    assert c.stats()["size"] == len(KEYS)
    for axis, layers in KEYS:
        mine = c.find(N, axis, layers)
        theirs, _ = ref.cache_load_probs(path, N, axis, layers)
        assert np.array_equal(mine, theirs)
        assert c.kernels(N, axis, layers).shape == (3, 6 * N * N)


def test_b200_sgf1_file_loads_in_the_reference(ref, tmp_path):
    src = _ref_file(ref, tmp_path)
    c = frwcap.SgfCache()
    c.load(src)
    out = str(tmp_path / "b200.sgf")
    c.save(out)
    for axis, layers in KEYS:
        theirs, loaded = ref.cache_load_probs(out, N, axis, layers)
        assert loaded == len(KEYS)
        assert np.array_equal(theirs, c.find(N, axis, layers))


def test_corrupt_files_are_rejected(ref, tmp_path):
    src = _ref_file(ref, tmp_path)
    raw = open(src, "rb").read()
    bad = tmp_path / "bad.sgf"
    for blob in (b"SGF2" + raw[4:], raw[:-3], raw + b"\x00"):
        bad.write_bytes(blob)
        with pytest.raises(RuntimeError):
            frwcap.SgfCache().load(str(bad))


@pytest.mark.gpu
def test_device_solves_equal_the_reference_cache(ref, tmp_path):
    path = _ref_file(ref, tmp_path)
    c = frwcap.SgfCache()
    for axis, layers in KEYS:
        mine = c.get(N, axis, layers)
        theirs, _ = ref.cache_load_probs(path, N, axis, layers)
        assert np.allclose(mine, theirs, rtol=0, atol=1e-9)
        assert abs(mine.sum() - 1) < 1e-9
    st = c.stats()
    assert st["misses"] == len(KEYS) and st["hits"] == 0
    c.get(N, *KEYS[1])
    assert c.stats()["hits"] == 1


@pytest.mark.gpu
def test_lru_eviction_and_scale_keys():
    c = frwcap.SgfCache(2)
    k1, k2, k3 = KEYS
    c.get(N, *k1)
    c.get(N, *k2)
    c.get(N, *k1)  # k1 is now the most recent
    c.get(N, *k3)  # evicts k2 (test_cache.cpp:151-166)
    assert c.find(N, *k2) is None
    assert c.find(N, *k1) is not None and c.find(N, *k3) is not None
    # a global scale factor is a distinct key with the same law (test_cache.cpp:124-135)
    d = frwcap.SgfCache()
    a = d.get(N, k2[0], k2[1])
    b = d.get(N, k2[0], [2 * x for x in k2[1]])
    assert d.stats()["size"] == 2
    assert np.allclose(a, b, rtol=0, atol=1e-12)
