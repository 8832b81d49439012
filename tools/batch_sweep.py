"""Walk-engine throughput vs device_batch (walks per frw_run_walks call):
each call drains its pool through the run-to-completion tail once, so larger
calls amortise it.  Scratch tool."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c5_structure

walks = int(os.environ.get("WALKS", 8 * 2 ** 20))
for name in sys.argv[1:] or ["c3", "c5"]:
    doc = json.dumps({"c3": c3_structure, "c5": c5_structure}[name]())
    # warm: SGF table and the largest page-locked record buffers
    frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=walks, max_walks=walks, seed=3,
                        device_batch=2 ** 23)
    for db in (2 ** 20, 2 ** 21, 2 ** 22, 2 ** 23):
        r = min((frwcap.extract_json(doc, mode="HYBRID-MW", min_walks=walks, max_walks=walks,
                                     seed=5 + k, device_batch=db) for k in range(2)),
                key=lambda x: x["t_total_seconds"])
        print(f"{name} walks={walks} device_batch={db} walks/s(dev)={walks / r['t_device_seconds']:.3e} "
              f"wall={walks / r['t_total_seconds']:.3e}", flush=True)
