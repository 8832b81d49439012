"""Several contexts on one GPU (Config::devices = [0, 0, ...], one host thread and one
stream each): the latency-bound late rounds and tails of one context overlap the other's
work.  Wall time of warm 1e6-walk calls (scratch tool).
usage: dual_ctx.py [c3 c4 c5]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure, c4_structure, c5_structure

W = int(os.environ.get("WALKS", 1_000_000))
for name in sys.argv[1:] or ["c3"]:
    doc = json.dumps({"c3": c3_structure, "c4": c4_structure, "c5": c5_structure}[name]())
    for G in (1, 2, 3, 4):
        for tail_div in (1, G) if G > 1 else (1,):
            os.environ["FRW_TAIL_WALKS"] = str(148 * 1024 // tail_div)
            kw = dict(mode="HYBRID-MW", min_walks=W, max_walks=W, devices=[0] * G)
            if G > 1:
                kw["device_batch"] = -(-W // G // 1024) * 1024
            best = 1e9
            for rep in range(4):
                t = time.perf_counter()
                r = frwcap.extract_json(doc, seed=7 + rep, **kw)
                dt = time.perf_counter() - t
                if rep:
                    best = min(best, dt)
            print(f"{name} contexts={G} tail_walks={os.environ['FRW_TAIL_WALKS']} wall(best of 3)={best*1e3:.1f} ms "
                  f"walks/s={W / best:.3e} dev={r['t_device_seconds']*1e3:.1f} ms "
                  f"C={[round(t_['capacitance_farads'] * 1e18, 2) for t_ in r['terminals'][:3]]}", flush=True)
