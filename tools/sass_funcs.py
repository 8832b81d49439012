"""SASS bytes of one kernel per source function (nvdisasm -g line info): which
inlined routines make a kernel's code large (instruction-fetch stalls).
usage: sass_funcs.py <kernel-substring> [lib] [top]"""
import collections, os, re, subprocess, sys, tempfile
kern = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2507_09730_b200/lib/libfrwgpu.so"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.startswith("walk") and f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
src = open(os.path.join(root, "paper_2507_09730_b200/csrc/walk.cu")).read().split("\n")
pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:__global__|__device__|__host__ __device__|static|inline)[^(]*?\b(\w+)\s*\(")
starts = []
for i, l in enumerate(src, 1):
    m = pat.match(l)
    if m:
        starts.append((i, m.group(1)))
    elif re.match(r"^\s+(k_\w+)\(", l) and "__global__" in src[i - 2]:
        starts.append((i, re.match(r"^\s+(k_\w+)\(", l).group(1)))
def fn(ln):
    f = "?"
    for s, n in starts:
        if s <= ln: f = n
        else: break
    return f
inside, cur, cnt = False, None, collections.Counter()
for l in sass.split("\n"):
    if l.lstrip().startswith(".section"):
        inside = ".text." in l and kern in l
        continue
    if not inside: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        f = m.group(1).split("/")[-1]; ln = int(m.group(2))
        cur = f + ":" + (fn(ln) if f == "walk.cu" else str(ln)); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l): cnt[cur] += 16
tot = sum(cnt.values())
print(kern, "SASS bytes", tot)
for k, v in cnt.most_common(top): print(f"  {v:8d} {100 * v / tot:5.1f}% {k}")
