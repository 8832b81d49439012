"""Single-walker step latency of the single-cube kernel: tiny counts (one
transit per warp / per SM), kernel time over the longest transit's steps.
usage: step_latency.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c1_grid, c2_grid

ctx = capi.Context(0)
clk = ctx.sm_clock_khz * 1e3
for name, (eps, c, h, _) in (("C1", c1_grid(1)), ("C2", c2_grid(1))):
    ctx.upload_grid(eps, c, h)
    n = ctx.n
    for count in (1, 8, 64):
        out_steps = ctx.alloc(4 * count)
        hist = ctx.alloc(6 * n * n * 8); mom = ctx.alloc(32)
        res = []
        for seed in range(1, 9):
            ctx.event_record(0)
            p = capi.MwParams(capi.RNG_PHILOX, seed, 0, count, 0, 1, None)
            o = capi.MwOut(None, out_steps, None, hist, mom, mom + 8, mom + 16, None)
            ctx._check(ctx.L.frw_microwalk_batch_dev(ctx.h, capi.C.byref(p), capi.C.byref(o)))
            ctx.event_record(1)
            ms = ctx.elapsed_ms()
            st = np.zeros(count, np.int32); ctx.d2h(st, out_steps)
            res.append((ms, int(st.max())))
        ctx.check()
        ms = np.array([r[0] for r in res]); mx = np.array([r[1] for r in res])
        A = np.vstack([mx, np.ones_like(mx)]).T
        slope, icpt = np.linalg.lstsq(A, ms, rcond=None)[0]
        print(f"{name} count {count:3d} one CTA: max steps {mx.tolist()} ms {np.round(ms,3).tolist()} "
              f"-> {slope*1e-3*clk:.0f} cycles/step, fixed {icpt*1e3:.1f} us")
        ctx.free(out_steps); ctx.free(hist); ctx.free(mom)
