"""Warm the SGF table, then run 1e6 walks of a config (for ncu launch lists)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
walks = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
kw = dict(mode=os.environ.get("FRW_MODE", "HYBRID-MW"), seed=7)
frwcap.extract_json(doc, min_walks=walks, max_walks=walks, **kw)   # warm table
# the warm run is bracketed by cuProfilerStart/Stop: `ncu --profile-from-start off`
# captures only its launches
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
cu.cuProfilerStart()
r = frwcap.extract_json(doc, min_walks=walks, max_walks=walks, **kw)
cu.cuProfilerStop()
print(name, "device s", r["t_device_seconds"], "mw s", r["t_mw_seconds"], "misses", r["cache"]["misses"])
