"""Quick walk-engine timing on C3-C5 (scratch tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure

which = sys.argv[1:] or ["c3"]
for name in which:
    doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    for walks in (100_000, 1_000_000, 1_000_000):
        t = time.time()
        r = frwcap.extract_json(doc, mode=os.environ.get("FRW_MODE", "HYBRID-MW"), min_walks=walks, max_walks=walks, seed=7)
        dt = time.time() - t
        print(f"{name} walks={walks} wall={dt:.2f}s dev={r['t_device_seconds']:.3f}s mw={r['t_mw_seconds']:.3f}s "
              f"walks/s(dev)={walks / r['t_device_seconds']:.3e} misses={r['cache']['misses']} "
              f"stats={r['dispatch_stats']} steps/walk={r['mw_steps'] / walks:.1f} "
              f"C={[round(t_['capacitance_farads'] * 1e18, 2) for t_ in r['terminals'][:4]]}", flush=True)
