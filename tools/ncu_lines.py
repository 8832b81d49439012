"""Per-source-line issue share and active lanes of one kernel in an .ncu-rep
(ncu --page source --print-source cuda,sass).  Usage: ncu_lines.py rep [regex] [top]"""
import collections, csv, subprocess, sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


cur, fname, tot = None, None, 0.0
agg = collections.defaultdict(lambda: [0.0, 0.0, "", 0.0])
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9:
        continue
    if r[0] != "":
        cur = (fname, r[0])
        agg[cur][2] = r[1].strip()[:72]
        continue
    ie, te, smp = f(r[7]), f(r[8]), f(r[4])
    agg[cur][0] += ie
    agg[cur][1] += te
    agg[cur][3] += smp
    tot += ie
stot = sum(v[3] for v in agg.values()) or 1
print(f"total warp instructions {tot:.3e}; lanes {sum(v[1] for v in agg.values()) / max(tot, 1):.2f}")
for k, (ie, te, src, smp) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    if ie:
        print(f"{k[0][:12]:12s} {k[1]:>5s} inst {100 * ie / tot:5.1f}% stall {100 * smp / stot:5.1f}% "
              f"lanes {te / ie:4.1f}  {src}")
