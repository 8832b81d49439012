"""In-tree build of the native libraries (nvcc/g++, no JIT cache).

* lib/libfrwgpu.so  -- CUDA kernels for sm_100a + the C ABI (include/frw_gpu.h)
* _core*.so         -- pybind11 module: the C++ `frwcap` API mirror over the
                       C ABI (bindings/py_module.cpp of the reference)
The oracle (test infrastructure) is built by oracle/Makefile.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_INC = "/usr/local/cuda/include"
CUDA_LIB = "/usr/local/cuda/lib64"


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_gpu_lib(force=False):
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "libfrwgpu.so")
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = cu + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) \
        + [os.path.join(ROOT, "include", "frw_gpu.h")]
    # -fmad=false: geometry/voxel-centre arithmetic must round like the
    # reference (x86-64 baseline, no FMA contraction)
    # FRW_NVCC_EXTRA: extra flags for A/B builds of kernel knobs (-D...)
    extra = os.environ.get("FRW_NVCC_EXTRA", "").split()
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-fmad=false", "-Xptxas", "-v",
           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), *extra,
           "-o", out, *cu, "-ldl"]
    # the flags of the last build sit next to the library: a variant build
    # (FRW_NVCC_EXTRA) is rebuilt by the next default build() even when no
    # source changed
    stamp = out + ".flags"
    flags = " ".join(cmd)
    old = open(stamp).read() if os.path.exists(stamp) else None
    if force or old != flags or _stale(out, deps):
        _run(cmd)
        with open(stamp, "w") as f:
            f.write(flags)
    return out


def build_core(force=False):
    """pybind11 `_core` (host C++ engine) linked against libfrwgpu.so."""
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    if not host:
        return None
    import pybind11
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    out = os.path.join(PKG, "_core" + suffix)
    deps = host + glob.glob(os.path.join(CSRC, "host", "*.hpp")) + \
        glob.glob(os.path.join(CSRC, "host", "frwcap", "*.hpp")) + \
        [os.path.join(ROOT, "include", "frw_gpu.h"), os.path.join(LIB, "libfrwgpu.so")]
    if force or _stale(out, deps):
        json_inc = os.path.join(sysconfig.get_paths()["purelib"],
                                "include/cudnn_frontend/thirdparty/nlohmann")
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CSRC, "host"),
              "-I", pybind11.get_include(), "-I", sysconfig.get_paths()["include"],
              "-I", json_inc, "-I", CUDA_INC, "-o", out, *host,
              "-L", LIB, "-lfrwgpu", "-Wl,-rpath,$ORIGIN/lib", "-lpthread"])
    return out


def build_cpp_lib(force=False):
    """libfrwcap.so: the C++ API mirror (csrc/host, without the Python
    bindings) for C++ callers of the reference's frwcap API, plus the example
    caller examples/frwcap_main."""
    host = sorted(p for p in glob.glob(os.path.join(CSRC, "host", "*.cpp"))
                  if not p.endswith("py_module.cpp"))
    out = os.path.join(LIB, "libfrwcap.so")
    exe = os.path.join(LIB, "frwcap_main")
    deps = host + glob.glob(os.path.join(CSRC, "host", "*.hpp")) + \
        [os.path.join(ROOT, "include", "frw_gpu.h"), os.path.join(LIB, "libfrwgpu.so")]
    json_inc = os.path.join(sysconfig.get_paths()["purelib"],
                            "include/cudnn_frontend/thirdparty/nlohmann")
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(CSRC, "host"), "-I", json_inc]
    if force or _stale(out, deps):
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-ffp-contract=off", *inc,
              "-o", out, *host, "-L", LIB, "-lfrwgpu", "-Wl,-rpath,$ORIGIN", "-lpthread"])
    src = os.path.join(ROOT, "examples", "frwcap_main.cpp")
    if os.path.exists(src) and (force or _stale(exe, [src, out])):
        _run(["g++", "-O2", "-std=c++20", *inc, "-o", exe, src, "-L", LIB, "-lfrwcap",
              "-lfrwgpu", "-Wl,-rpath,$ORIGIN", "-lpthread"])
    return out


REF_TESTS = ("test_geometry", "test_cache", "test_engine")


def build_ref_unit_tests(force=False):
    """The reference's own doctest suites (proj/tests/test_{geometry,cache,
    engine}.cpp, compiled in place and unchanged) against the C++ frwcap
    mirror (csrc/host, forwarding headers csrc/host/frwcap/*.hpp), with the
    doctest stand-in tests/cpp/doctest_shim: the C++ source-level drop-in
    check.  Binaries go to tests/cpp/_bin (git-ignored; they travel to the
    GPU box).  Needs /root/reference (present in the build container only)."""
    ref = "/root/reference/proj/tests"
    if not os.path.isdir(ref):
        return []
    out_dir = os.path.join(ROOT, "tests", "cpp", "_bin")
    os.makedirs(out_dir, exist_ok=True)
    json_inc = os.path.join(sysconfig.get_paths()["purelib"],
                            "include/cudnn_frontend/thirdparty/nlohmann")
    shim = os.path.join(ROOT, "tests", "cpp", "doctest_shim")
    lib = os.path.join(LIB, "libfrwcap.so")
    inc = ["-I", shim, "-I", os.path.join(CSRC, "host"), "-I", os.path.join(ROOT, "include"),
           "-I", json_inc]
    built = []
    for t in REF_TESTS:
        exe = os.path.join(out_dir, t)
        srcs = [os.path.join(ref, "doctest_main.cpp"), os.path.join(ref, t + ".cpp")]
        deps = srcs + [lib, os.path.join(shim, "doctest.h")] + \
            glob.glob(os.path.join(CSRC, "host", "*.hpp"))
        if force or _stale(exe, deps):
            _run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", *inc, "-o", exe, *srcs,
                  "-L", LIB, "-lfrwcap", "-lfrwgpu", "-Wl,-rpath," + LIB, "-lpthread"])
        built.append(exe)
    return built


def build_oracle(with_ref=None):
    tgts = ["all"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj")
    if with_ref:
        tgts.append("ref")
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), *tgts])


def build_all(force=False):
    build_gpu_lib(force)
    build_core(force)
    build_cpp_lib(force)
    build_oracle()
    build_ref_unit_tests(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
