"""Per-function issue share of one kernel in an .ncu-rep: source lines of
walk.cu (and frw_rng.cuh) grouped by the enclosing function definition.
Usage: ncu_funcs.py rep [kernel-regex] [source-file]"""
import collections, csv, re, subprocess, sys, os

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
srcs = {"walk.cu": os.path.join(root, "paper_2507_09730_b200/csrc/walk.cu"),
        "frw_rng.cuh": os.path.join(root, "paper_2507_09730_b200/csrc/frw_rng.cuh"),
        "mw_grid.cu": os.path.join(root, "paper_2507_09730_b200/csrc/mw_grid.cu")}
starts = {}
pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:__global__|__device__|__host__ __device__|static|inline)[^(]*?\b(\w+)\s*\(")
for k, p in srcs.items():
    st = []
    lines = open(p).read().split("\n")
    for i, l in enumerate(lines, 1):
        m = pat.match(l)
        if m:
            st.append((i, m.group(1)))
        elif re.match(r"^\s+(k_\w+)\(", l) and i > 1 and "__global__" in lines[i - 2]:
            st.append((i, re.match(r"^\s+(k_\w+)\(", l).group(1)))
    starts[k] = st
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
def f(x):
    try: return float(x.replace(",", ""))
    except ValueError: return 0.0
fname, cur, hdr = None, None, None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 9: continue
    if r[0] != "":
        ln = int(r[0]); fn = "?"
        for s, name in starts.get(fname, []):
            if s <= ln: fn = name
            else: break
        cur = f"{fname}:{fn}"; continue
    agg[cur][0] += f(r[7]); agg[cur][1] += f(r[8]); agg[cur][2] += f(r[4])
tot = sum(v[0] for v in agg.values()) or 1; stot = sum(v[2] for v in agg.values()) or 1
print(f"total warp instructions {tot:.3e}")
for k, (ie, te, smp) in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
    if ie: print(f"  {k:40s} inst {100*ie/tot:5.1f}%  stall {100*smp/stot:5.1f}%  lanes {te/ie:4.1f}  inst {ie:.3e}")
