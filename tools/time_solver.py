"""Time the stratified-key device solver (frw_sgf_solve) on random keys."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_09730_b200 import capi

ctx = capi.Context(0)
rng = np.random.default_rng(1)
for n, cnt in ((24, 1), (24, 16), (24, 128), (24, 512)):
    axes = rng.integers(0, 3, cnt).astype(np.int32)
    layers = np.round(rng.choice([2.5, 3.9, 4.2, 7.0], size=(cnt, n)), 6)
    ctx.sgf_solve(n, axes, layers)  # warm
    t = time.perf_counter()
    ctx.sgf_solve(n, axes, layers)
    dt = time.perf_counter() - t
    print(f"n={n} keys={cnt}: {dt*1e3:.2f} ms  ({dt/cnt*1e6:.1f} us/key)", flush=True)
