"""FDM mode vs HYBRID-MW on C3 / fixtures (Theorem 1 check, scratch tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure

walks = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 24
doc = json.dumps(c3_structure())
for mode in ("HYBRID-MW", "FDM", "FDM"):
    t = time.time()
    r = frwcap.extract_json(doc, mode=mode, min_walks=walks, max_walks=walks, seed=3, grid_n=n)
    dt = time.time() - t
    print(mode, f"wall={dt:.2f}s dev={r['t_device_seconds']:.3f}s", r["dispatch_stats"]["subsequent"],
          [(round(x["capacitance_farads"] * 1e18, 2), round(x["std_err_farads"] * 1e18, 2))
           for x in r["terminals"]], flush=True)
