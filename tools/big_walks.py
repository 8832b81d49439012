"""Device walks/s of large calls (the bench's C4/C5 regime): C5 one master x
1e7 walks, C4 and C3 at 8e6 fixed walks, warm tables."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure
for name, W in (("c5", 10_000_000), ("c4", 8_000_000), ("c3", 8_000_000)):
    doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=1 << 18, max_walks=1 << 18, seed=1)
    for rep in range(2):
        t = time.time()
        r = frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=W, max_walks=W, seed=7 + rep)
        print(f"{name} walks={W} dev={r['t_device_seconds']:.3f}s walks/s(dev)={W / r['t_device_seconds']:.3e} "
              f"wall={time.time() - t:.2f}s", flush=True)
