"""Steps taken / jumps per walk and device walks/s of warm 1e6-walk calls."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure
tag = os.environ.get("TAG", "")
for name in sys.argv[1:] or ["c3"]:
    doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    mode = os.environ.get("FRW_MODE", "HYBRID-MW")
    frwcap.extract_json(doc, mode=mode, min_walks=1_000_000, max_walks=1_000_000, seed=8)
    best = None
    for rep in range(2):
        r = frwcap.extract_json(doc, mode=mode, min_walks=1_000_000, max_walks=1_000_000, seed=8)
        if best is None or r["t_device_seconds"] < best["t_device_seconds"]:
            best = r
    r, w = best, 1e6
    print(f"{tag} {name} {mode} walks/s(dev)={w / r['t_device_seconds']:.3e} taken/walk="
          f"{(r['mw_steps'] - r['mw_jump_steps']) / w:.1f} jumps/walk={r['mw_jumps'] / w:.1f} "
          f"Etau/walk={r['mw_steps'] / w:.1f} C={[round(t['capacitance_farads'] * 1e18, 2) for t in r['terminals'][:3]]} "
          f"se={[round(t['std_err_farads'] * 1e18, 2) for t in r['terminals'][:3]]}", flush=True)
