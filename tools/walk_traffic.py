"""Per-kernel time, DRAM bytes and active lanes of one warm walk-engine call
from an ncu CSV (tools/ncu_walks.sh), and the engine's DRAM bytes per walk.
usage: walk_traffic.py <csv> <walks> <label> > out.json"""
import collections, csv, json, sys

fn, walks, label = sys.argv[1], float(sys.argv[2]), sys.argv[3]
rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
h = rows[0]
ki, vi, ui, mi, idi = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit",
                                             "Metric Name", "ID"))
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "": 1}
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[(r[idi], r[ki].split("(")[0].split("::")[-1])][r[mi]] = \
        float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
agg = collections.defaultdict(lambda: dict(launches=0, ms=0.0, dram_read=0.0, dram_write=0.0,
                                           lane_ms=0.0))
for (_, k), m in per.items():
    a = agg[k]
    a["launches"] += 1
    t = m.get("gpu__time_duration.sum", 0.0)
    a["ms"] += t
    a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
    a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
    a["lane_ms"] += m.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0.0) * t
tot_ms = sum(a["ms"] for a in agg.values())
tot_b = sum(a["dram_read"] + a["dram_write"] for a in agg.values())
kern = {}
for k, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
    kern[k] = dict(launches=a["launches"], ms=round(a["ms"], 3),
                   share=round(a["ms"] / tot_ms, 3) if tot_ms else 0,
                   dram_bytes=a["dram_read"] + a["dram_write"],
                   dram_bytes_per_walk=(a["dram_read"] + a["dram_write"]) / walks,
                   active_lanes=round(a["lane_ms"] / a["ms"], 2) if a["ms"] else None)
top = next(iter(kern))
print(json.dumps(dict(label=label, walks=walks, source=fn,
                      note="ncu launch times are serialised and cold-cache: compare shares",
                      kernels=kern, total_ms=round(tot_ms, 3),
                      dram_bytes_per_walk=tot_b / walks, dominant_kernel=top,
                      dominant_dram_bytes_per_walk=kern[top]["dram_bytes_per_walk"]), indent=1))
