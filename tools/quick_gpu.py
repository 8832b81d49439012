"""Quick GPU sanity: smoke parity + C1/C2 device timings (scratch tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__ as g
from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c1_grid, c2_grid

g.smoke()
ctx = capi.Context(0)
print("device", ctx.name, ctx.sm_count, ctx.sm_clock_khz)
print("smem probe GB/s", ctx.smem_bandwidth() / 1e9)
for name, (eps, c, h, _), count in (("C1", c1_grid(1), 1_000_000), ("C2", c2_grid(1), 10_000_000)):
    ctx.upload_grid(eps, c, h)
    print(name, ctx.grid_info())
    n = ctx.n
    hist = ctx.alloc(6 * n * n * 8); mom = ctx.alloc(32)
    for rng in (capi.RNG_PHILOX, capi.RNG_SPLITMIX_PARITY):
        for it in range(4):
            ctx.memset(hist, 6 * n * n * 8); ctx.memset(mom, 32)
            ctx.event_record(0)
            ctx.microwalk_batch_dev(count, hist, mom, seed=it + 1, rng=rng)
            ctx.event_record(1)
            ms = ctx.elapsed_ms()
        ctx.check()
        m = np.zeros(4, np.uint64); ctx.d2h(m, mom)
        h = np.zeros(6 * n * n, np.uint64); ctx.d2h(h, hist)
        steps = int(m[0])
        print(f"{name} rng={rng} {ms:.3f} ms  {count/ms*1e3:.3e} transits/s  {steps/ms*1e3:.3e} steps/s "
              f"mean steps {steps/count:.2f} hist sum {int(h.sum())}")
    ctx.free(hist); ctx.free(mom)
