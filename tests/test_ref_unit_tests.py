"""The reference's own C++ unit tests, compiled unchanged against the B200
C++ frwcap mirror (the source-level drop-in).

`paper_2507_09730_b200/build.py::build_ref_unit_tests` compiles
/root/reference/proj/tests/{doctest_main,test_geometry,test_cache,
test_engine}.cpp in place -- the sources are not copied into this repo --
with the forwarding headers csrc/host/frwcap/*.hpp (so `#include
"frwcap/engine.hpp"` resolves to the mirror) and a doctest stand-in
(tests/cpp/doctest_shim, doctest itself is absent from the image).  The
binaries (tests/cpp/_bin, git-ignored) travel to the GPU box.
test_geometry is host-only; test_cache and test_engine drive the device
(SGF solves, Engine::first_transition/transition/extract)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(__file__), "cpp", "_bin")


def _run(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1800)
    summary = r.stderr.strip().splitlines()[-1] if r.stderr.strip() else ""
    assert r.returncode == 0, r.stderr[-4000:]
    assert " 0 failed;" in summary, summary
    return summary


def test_reference_geometry_suite():
    _run("test_geometry")


@pytest.mark.gpu
def test_reference_cache_suite():
    _run("test_cache")


@pytest.mark.gpu
def test_reference_engine_suite():
    _run("test_engine")
