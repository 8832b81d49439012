"""MicroWalk step-class statistics of a config through the C ABI (scratch)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle
from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure
from tests.scenes import scene_from_doc
from tests.walk_helpers import oracle_solver, upload_scene, walk_params
O = Oracle()
ctx = capi.Context(0)
for name in sys.argv[1:] or ["c3"]:
    sc = scene_from_doc({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    upload_scene(ctx, sc); ctx.sgf_clear()
    p = walk_params(sc, grid_n=24, seed=3, rng=capi.RNG_PHILOX)
    ctx.run_walks(p, sc.master_slot(), 0, 100000, oracle_solver(O), records=False)
    t, _ = ctx.run_walks(p, sc.master_slot(), 0, 1000000, oracle_solver(O), records=False)
    print(name, "mw_steps", t["mw_steps"], "general frac %.3f" % (t["mw_general_steps"] / t["mw_steps"]),
          "cell changes per 100 steps %.2f" % (100 * t["mw_cell_changes"] / t["mw_steps"]),
          "mw_ms", round(t["mw_ms"], 1), "total_ms", round(t["total_ms"], 1), flush=True)
