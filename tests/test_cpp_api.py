"""The C++ API mirror as a C++ caller sees it: libfrwcap.so (csrc/host
without the Python bindings) and examples/frwcap_main, built by
__graft_entry__.build().  On a CPU-only host the binary fails loudly; on the
device its microwalk_transit agrees bit for bit with the oracle and its
extract with the Python module."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2507_09730_b200.workloads import random_voxel_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2507_09730_b200", "lib", "frwcap_main")


def _run(*args):
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_cpp_library_and_example_are_built():
    assert os.path.exists(os.path.join(ROOT, "paper_2507_09730_b200", "lib", "libfrwcap.so"))
    assert os.path.exists(EXE)


def test_no_cpu_fallback_in_cpp():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    r = _run("transit", 4, 1, 3)
    assert r.returncode == 2 and "no CPU fallback" in r.stderr


@pytest.mark.gpu
def test_cpp_microwalk_transit_matches_oracle(oracle):
    """microwalk_transit(grid, SplitMix64(7, t)) through libfrwcap"""
    n, count = 6, 2000
    r = _run("transit", n, 1, count)
    assert r.returncode == 0, r.stderr
    got = np.array([[int(x) for x in line.split()] for line in r.stdout.split("\n") if line])
    eps = random_voxel_grid(n, 1, 0)  # random_voxel_grid(n, SplitMix64(1, 0)) as in C++
    w = oracle.microwalk_grid(eps, np.zeros(3), n / 2.0, 7, 0, count)
    assert np.array_equal(got[:, 0], w["panel"]) and np.array_equal(got[:, 1], w["steps"])


@pytest.mark.gpu
def test_cpp_extract_matches_python(tmp_path):
    from tests import scenes
    import paper_2507_09730_b200.frwcap as frwcap
    sc = scenes.load_fixture("highk_cross")
    f = tmp_path / "s.json"
    f.write_text(sc.to_json())
    r = _run("extract", f, 50000)
    assert r.returncode == 0, r.stderr
    rows = [line.split() for line in r.stdout.split("\n") if line.startswith("C ")]
    py = frwcap.extract_json(sc.to_json(), mode="HYBRID-MW", rng="splitmix", min_walks=50000,
                             max_walks=50000)
    for row, t in zip(rows, py["terminals"]):
        assert int(row[1]) == t["conductor_id"]
        assert float(row[2]) == t["capacitance_farads"]
