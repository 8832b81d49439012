"""A/B of MicroWalk lattice jumps (FRW_MW_JUMP) on C3-C5: device walks/s,
mean MicroWalk steps per walk and the capacitance row with and without jumps
(z-scores of the differences).  Scratch tool."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure

which = sys.argv[1:] or ["c3"]
walks = int(os.environ.get("WALKS", 1_000_000))
modes = os.environ.get("MODES", "HYBRID-MW,HYBRID-MWE").split(",")
for name in which:
    doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    for mode in modes:
        rows = {}
        for jump in ("0", "31"):
            os.environ["FRW_MW_JUMP"] = jump.split("/")[0]
            os.environ["FRW_MW_JUMP_TWICE"] = jump.split("/")[1] if "/" in jump else "0"
            frwcap.extract_json(doc, mode=mode, min_walks=walks, max_walks=walks, seed=7)  # warm
            best = None
            for rep in range(3):
                r = frwcap.extract_json(doc, mode=mode, min_walks=walks, max_walks=walks,
                                        seed=11 + rep)
                if best is None or r["t_device_seconds"] < best["t_device_seconds"]:
                    best = r
            rows[jump] = best
            print(f"{name} {mode} jump={jump} walks/s(dev)={walks / best['t_device_seconds']:.3e} "
                  f"mw_s={best['t_mw_seconds']:.3f} steps/walk={best['mw_steps'] / walks:.1f} "
                  f"jumps/walk={best.get('mw_jumps', 0) / walks:.1f}",
                  flush=True)
        a, b = rows["0"]["terminals"], rows["31"]["terminals"]
        zs = []
        for ta, tb in zip(a, b):
            se = (ta["std_err_farads"] ** 2 + tb["std_err_farads"] ** 2) ** 0.5
            zs.append((ta["capacitance_farads"] - tb["capacitance_farads"]) / se if se > 0 else 0.0)
        print(f"  C(no jump)[:4] aF={[round(t['capacitance_farads'] * 1e18, 2) for t in a[:4]]}")
        print(f"  C(jump)[:4]    aF={[round(t['capacitance_farads'] * 1e18, 2) for t in b[:4]]}")
        print(f"  max|z|={max(abs(z) for z in zs):.2f} over {len(zs)} terminals", flush=True)
