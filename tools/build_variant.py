"""Build an experiment variant of libfrwgpu.so here (nvcc cross-compiles) into
paper_2507_09730_b200/lib/variants/<name>/libfrwgpu.so; on the GPU box
tools/use_variant.sh <name> copies it over the default library.
usage: build_variant.py <name> "<extra nvcc flags>" """
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_09730_b200 import build as b
import glob
name, flags = sys.argv[1], sys.argv[2].split()
# optional third argument: a git revision whose csrc/*.cu{,h} and frw_internal.h to build
rev = sys.argv[3] if len(sys.argv) > 3 else None
out_dir = os.path.join(b.LIB, "variants", name)
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, "libfrwgpu.so")
cu = sorted(glob.glob(os.path.join(b.CSRC, "*.cu")))
if rev:
    src = os.path.join("/tmp", "variant_src_" + name)
    os.makedirs(src, exist_ok=True)
    for f in glob.glob(os.path.join(b.CSRC, "*.cu*")) + glob.glob(os.path.join(b.CSRC, "*.h")):
        rel = os.path.relpath(f, b.ROOT)
        data = subprocess.run(["git", "-C", b.ROOT, "show", f"{rev}:{rel}"], capture_output=True).stdout
        open(os.path.join(src, os.path.basename(f)), "wb").write(data)
    cu = sorted(glob.glob(os.path.join(src, "*.cu")))
cmd = [b.NVCC, "-O3", "-std=c++17", *b.ARCH, "-lineinfo", "-fmad=false", "-Xptxas", "-v",
       "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(b.ROOT, "include"), *flags,
       "-o", out, *cu, "-ldl"]
r = subprocess.run(cmd, capture_output=True, text=True)
open(os.path.join(out_dir, "build.log"), "w").write(r.stdout + r.stderr)
print(name, "rc", r.returncode, out)
sys.exit(r.returncode)
