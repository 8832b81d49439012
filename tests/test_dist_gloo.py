"""World-size-2 gloo test of the multi-rank tally path (CPU).

Each rank runs its contiguous walk range through the oracle (the walk
records are a pure function of the walk id), folds its tallies, and the
ranks all-reduce them.  The combined estimates must equal a single-process
fold over all walks: landed counts exactly, sums to rounding.
"""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_09730_b200.dist import combine_tallies, estimates, rank_range

WALKS = 600


def _scene():
    from tests.scenes import plate_pocket_scene
    return plate_pocket_scene()


def _fold(slot, w, k):
    s1 = np.zeros(k)
    s2 = np.zeros(k)
    n = np.zeros(k, np.int64)
    for sl, x in zip(slot, w):
        s1[sl] += x
        s2[sl] += x * x
        n[sl] += 1
    return s1, s2, n


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    sc = _scene()
    b, e = rank_range(WALKS, rank, world)
    slot, w, _ = Oracle().run_walks(sc, b, e - b, grid_n=8, mode="HYBRID-MW", seed=5)
    s1, s2, n = _fold(slot, w, sc.n_cond + 1)
    t1, t2, tn = combine_tallies(s1, s2, n)
    out[rank] = (t1.tolist(), t2.tolist(), tn.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_rank_ranges_partition():
    for total in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [rank_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (b0, e0), (b1, _) in zip(spans, spans[1:]):
                assert e0 == b1 and e0 >= b0


def test_two_rank_gloo_allreduce_equals_single_fold(oracle):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    sc = _scene()
    slot, w, _ = oracle.run_walks(sc, 0, WALKS, grid_n=8, mode="HYBRID-MW", seed=5)
    s1, s2, n = _fold(slot, w, sc.n_cond + 1)
    for r in range(2):
        t1, t2, tn = (np.array(x) for x in out[r])
        assert np.array_equal(tn, n)
        assert np.allclose(t1, s1, rtol=1e-12, atol=1e-30)
        assert np.allclose(t2, s2, rtol=1e-12, atol=1e-50)
    a = estimates(t1, t2, WALKS)
    b = estimates(s1, s2, WALKS)
    for (m1, e1), (m2, e2) in zip(a, b):
        assert m1 == pytest.approx(m2, rel=1e-12, abs=1e-30)
        assert e1 == pytest.approx(e2, rel=1e-9, abs=1e-30)
