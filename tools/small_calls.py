"""Device time of small warm calls (the regime of a resumed batch of parked walks): k_flow
against k_tail.  usage: small_calls.py [c3 c5]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure
for name in sys.argv[1:] or ["c5"]:
    doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=1 << 20, max_walks=1 << 20, seed=1)
    for W in (128, 2048, 16384, 131072):
        for k in ("flow", "tail"):
            os.environ["FRW_TAIL_KERNEL"] = k
            ts = []
            for rep in range(4):
                r = frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=W, max_walks=W, seed=7 + rep)
                if r["cache"]["misses"] == 0:
                    ts.append(r["t_device_seconds"])
            print(f"{name} walks={W} {k}: device ms {[round(t * 1e3, 2) for t in ts]}", flush=True)
