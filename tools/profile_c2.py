"""Two C2 launches (1e7 Philox transits each) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_09730_b200 import capi
from paper_2507_09730_b200.workloads import c2_grid, c1_grid

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
rng = capi.RNG_PHILOX if (len(sys.argv) < 3 or sys.argv[2] == "philox") else capi.RNG_SPLITMIX_PARITY
eps, c, h, _ = (c2_grid if which == "c2" else c1_grid)(1)
count = 10_000_000 if which == "c2" else 1_000_000
ctx = capi.Context(0)
ctx.upload_grid(eps, c, h)
n = ctx.n
hist = ctx.alloc(6 * n * n * 8); mom = ctx.alloc(32)
for i in range(2):
    ctx.memset(hist, 6 * n * n * 8); ctx.memset(mom, 32)
    ctx.microwalk_batch_dev(count, hist, mom, seed=1 + i, rng=rng)
ctx.check()
m = np.zeros(4, np.uint64); ctx.d2h(m, mom)
print("steps per launch", int(m[0]))
