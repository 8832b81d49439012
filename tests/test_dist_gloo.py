"""World-size-2 gloo test of the product's multi-rank path (CPU).

Each rank runs ``paper_2507_09730_b200.dist.extract_sharded`` -- the
product's partition (contiguous ranges of one walk sequence), tally packing,
all-reduce and estimates.  Only the tally source differs from a GPU run: on
CPU the per-walk outcomes come from the oracle (a pure function of the walk
id, like the device's), folded into the same tally layout the device
returns.  The combined result must equal the single-rank run: landed counts
exactly, sums to rounding.
"""
import json
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_09730_b200.dist import extract_sharded, rank_range

WALKS = 600


def _scene():
    from tests.scenes import plate_pocket_scene
    return plate_pocket_scene()


def _text():
    return _scene().to_json()


def oracle_runner(text, begin, count, allreduce, **kw):
    """tally of walks [begin, begin+count) in the layout of _core.run_walks_tally"""
    from oracle.oracle import Oracle
    from tests.scenes import scene_from_doc
    assert not allreduce  # gloo groups reduce through torch.distributed
    sc = scene_from_doc(json.loads(text))
    slot, w, ab = Oracle().run_walks(sc, begin, count, grid_n=8, mode="HYBRID-MW", seed=5)
    k = sc.n_cond + 1
    s1, s2, n = np.zeros(k), np.zeros(k), np.zeros(k, np.uint64)
    for sl, x in zip(slot, w):
        s1[sl] += x
        s2[sl] += x * x
        n[sl] += 1
    return dict(sum=s1, sumsq=s2, landed=n, walks=count, aborted=int(ab.sum()), resampled=0,
                first=[0] * 4, sub=[0] * 4, mw_steps=0)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = extract_sharded(_text(), WALKS, runner=oracle_runner)
    out[rank] = json.dumps(r)
    dist.barrier()
    dist.destroy_process_group()


def test_rank_ranges_partition():
    for total in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [rank_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (b0, e0), (b1, _) in zip(spans, spans[1:]):
                assert e0 == b1 and e0 >= b0


def test_two_rank_gloo_equals_single_rank():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    one = extract_sharded(_text(), WALKS, runner=oracle_runner)  # no process group: one rank
    assert one["walks"] == WALKS and one["walks_this_rank"] == WALKS
    for r in range(2):
        two = json.loads(out[r])
        assert two["walks"] == WALKS and two["walks_this_rank"] == WALKS // 2
        assert two["aborted"] == one["aborted"]
        for a, b in zip(two["terminals"], one["terminals"]):
            assert a["conductor_id"] == b["conductor_id"]
            assert a["walks_landed"] == b["walks_landed"]  # exact
            assert a["capacitance_farads"] == pytest.approx(b["capacitance_farads"], rel=1e-12,
                                                            abs=1e-30)
            assert a["std_err_farads"] == pytest.approx(b["std_err_farads"], rel=1e-9, abs=1e-30)
    # and the single-rank product fold equals a plain fold of the oracle's walks
    from oracle.oracle import Oracle
    sc = _scene()
    slot, w, _ = Oracle().run_walks(sc, 0, WALKS, grid_n=8, mode="HYBRID-MW", seed=5)
    for k, t in enumerate(one["terminals"]):
        assert t["walks_landed"] == int(np.count_nonzero(slot == k))
