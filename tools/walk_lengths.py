"""Per-walk length distribution (cached hops, MicroWalk hops, MicroWalk
steps) of a config through the C ABI: what bounds the run-to-completion tail."""
import os, sys
import numpy as np
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
    t, rec = ctx.run_walks(p, sc.master_slot(), 0, 1000000, oracle_solver(O), records=True)
    for f in ("cached", "microwalk", "mw_steps"):
        x = rec[f].astype(np.float64)
        q = np.percentile(x, [50, 90, 99, 99.9, 99.99])
        print(name, f, "mean %.1f" % x.mean(), "pcts(50,90,99,99.9,99.99)", np.round(q, 1),
              "max", int(x.max()), "share of top 1%% %.3f" % (np.sort(x)[-len(x) // 100:].sum() / x.sum()),
              flush=True)
    print(name, "total_ms", round(t["total_ms"], 1), "mw_ms", round(t["mw_ms"], 1), flush=True)
