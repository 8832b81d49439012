"""Trace one cold extract (FRW_TRACE_ROUNDS=1 set by the caller)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
mode = sys.argv[2] if len(sys.argv) > 2 else "HYBRID-MW"
walks = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
t = time.time()
r = frwcap.extract_json(doc, mode=mode, min_walks=walks, max_walks=walks, seed=7)
print("wall", time.time() - t, "dev", r["t_device_seconds"], "misses", r["cache"]["misses"], file=sys.stderr)
