"""Multi-GPU product path on one B200.

* Multi-device Engine (Config::devices, one host thread and context per
  entry; a device listed twice gets two contexts): device chunks of one walk
  sequence go round-robin to the lanes and are folded in walk order, so the
  result equals the one-device run bit for bit -- with a fixed walk count
  and under the stopping rule.
* Sharded extract (paper_2507_09730_b200.dist): the ranges of an emulated
  two-rank run, run through the device path and combined with the
  all-reduce's arithmetic, land exactly as the one-rank run.
* frw_tally_allreduce over a one-rank NCCL communicator is the identity.

Two contexts on one GPU run independent kernels (no cross-context waits),
so this is not a stand-in for a collective between GPUs; the N > 1
collective itself runs under torchrun (bench.py) and its host logic in the
gloo test (tests/test_dist_gloo.py).
"""
import json

import numpy as np
import pytest

from paper_2507_09730_b200 import dist
from paper_2507_09730_b200.workloads import c3_structure, c5_structure

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a["walks"] == b["walks"]
    for x, y in zip(a["terminals"], b["terminals"]):
        assert x["conductor_id"] == y["conductor_id"]
        assert x["walks_landed"] == y["walks_landed"]
        assert x["capacitance_farads"] == y["capacitance_farads"]
        assert x["std_err_farads"] == y["std_err_farads"]


@pytest.mark.parametrize("mode", ["HYBRID-MW", "HYBRID-MWE"])
def test_multi_device_engine_equals_one_device(mode):
    import paper_2507_09730_b200.frwcap as frwcap
    doc = json.dumps(c3_structure())
    kw = dict(mode=mode, min_walks=1_000_000, max_walks=1_000_000, seed=21,
              device_batch=1 << 18)
    one = frwcap.extract_json(doc, **kw)
    two = frwcap.extract_json(doc, devices=[0, 0], **kw)
    three = frwcap.extract_json(doc, devices=[0, 0, 0], **kw)
    _same(one, two)
    _same(one, three)
    assert one["mw_steps"] == two["mw_steps"] == three["mw_steps"]
    # and the default chunking gives the same walks
    _same(one, frwcap.extract_json(doc, mode=mode, min_walks=1_000_000, max_walks=1_000_000,
                                   seed=21))


def test_multi_device_stopping_rule_equals_one_device():
    import paper_2507_09730_b200.frwcap as frwcap
    doc = json.dumps(c3_structure())
    kw = dict(mode="HYBRID-MW", tol=0.003, min_walks=4096, max_walks=20_000_000, seed=5,
              device_batch=1 << 18)
    one = frwcap.extract_json(doc, **kw)
    two = frwcap.extract_json(doc, devices=[0, 0], **kw)
    assert one["converged"] and two["converged"]
    _same(one, two)


def test_sharded_two_rank_emulation_lands_exactly():
    c5 = c5_structure()
    text = json.dumps(c5)
    W = 400_000
    kw = dict(mode="HYBRID-MW", seed=3)
    one = dist.extract_sharded(text, W, **kw)
    parts = []
    for r in range(2):
        b, e = dist.rank_range(W, r, 2)
        t = dist.device_runner(text, b, e - b, False, **kw)
        t["walks"] = e - b
        parts.append(t)
    t = dist.combine_local(parts)
    assert t["walks"] == W
    two = dist.result_from_tally(t, [c["id"] for c in c5["conductors"]], c5["master"])
    assert two["aborted"] == one["aborted"]
    assert two["dispatch_stats"] == one["dispatch_stats"]
    assert two["mw_steps"] == one["mw_steps"]
    for a, b in zip(two["terminals"], one["terminals"]):
        assert a["walks_landed"] == b["walks_landed"]
        assert a["capacitance_farads"] == pytest.approx(b["capacitance_farads"], rel=1e-12,
                                                        abs=1e-30)
    # the sharded tally equals the walk-order fold of extract_json
    import paper_2507_09730_b200.frwcap as frwcap
    ref = frwcap.extract_json(text, min_walks=W, max_walks=W, **kw)
    for a, b in zip(one["terminals"], ref["terminals"]):
        assert a["walks_landed"] == b["walks_landed"]
        assert a["capacitance_farads"] == pytest.approx(b["capacitance_farads"], rel=1e-12,
                                                        abs=1e-30)


def test_nccl_tally_allreduce_single_rank_is_identity():
    from paper_2507_09730_b200 import _core
    dist.init_nccl(0)
    text = json.dumps(c3_structure())
    a = _core.run_walks_tally(text, 0, 200_000, False, mode="HYBRID-MW", seed=8)
    b = _core.run_walks_tally(text, 0, 200_000, True, mode="HYBRID-MW", seed=8)
    assert np.array_equal(a["landed"], b["landed"])
    assert np.array_equal(a["sum"], b["sum"]) and np.array_equal(a["sumsq"], b["sumsq"])
    for k in ("aborted", "resampled", "first", "sub", "mw_steps"):
        assert a[k] == b[k], k
