"""Single-cube kernel time vs transit count (C1, C2): separates the
steady-state step rate from the per-launch ramp and the longest-transit tail.
usage: c1_sweep.py [counts...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c1_grid, c2_grid

counts = [int(float(x)) for x in sys.argv[1:]] or [250_000, 500_000, 1_000_000, 2_000_000, 4_000_000, 8_000_000]
ctx = capi.Context(0)
for name, (eps, c, h, _) in (("C1", c1_grid(1)), ("C2", c2_grid(1))):
    ctx.upload_grid(eps, c, h)
    n = ctx.n
    hist = ctx.alloc(6 * n * n * 8); mom = ctx.alloc(32)
    for count in counts:
        if name == "C2" and count > 4_000_000:
            continue
        ts = []
        for it in range(5):
            ctx.memset(hist, 6 * n * n * 8); ctx.memset(mom, 32)
            ctx.event_record(0)
            ctx.microwalk_batch_dev(count, hist, mom, seed=it + 1, rng=capi.RNG_PHILOX)
            ctx.event_record(1)
            ts.append(ctx.elapsed_ms())
        ctx.check()
        m = np.zeros(4, np.uint64); ctx.d2h(m, mom)
        ms = float(np.median(ts))
        print(f"{name} count {count:>9d} {ms:8.3f} ms  {count/ms*1e3:.3e} transits/s  {int(m[0])/ms*1e3:.3e} steps/s")
    ctx.free(hist); ctx.free(mom)
