"""Multi-GPU walk engine: one process per GPU.

Walks are independent and their random streams are a pure function of
(seed, walk id), so the path shards with no data-path collective: rank g of
G runs a contiguous range of the ONE walk sequence of the run (the
reference's per-thread chunking, engine.cpp:437-458), geometry and SGF
tables are replicated, and the only exchange is one all-reduce (sum) of the
per-slot tallies (sum, sum of squares, landed count, dispatch counters).

* On GPUs the all-reduce is the C ABI's ``frw_tally_allreduce``: one
  ``ncclAllReduce`` of the device-resident tally over NVLink / NVSwitch, on
  a communicator the ranks set up with ``frw_nccl_init`` (``init_nccl``).
* In the CPU tests (gloo) the same packed vector goes through
  ``torch.distributed.all_reduce``.

Because a rank's range is a slice of the single-process run, the combined
landed counts equal the one-GPU run's exactly and the sums equal it up to
the association of the final f64 additions.
"""
from __future__ import annotations

import json
import math

import numpy as np

_NCCL_READY: dict = {}


def rank_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of this rank's walks: contiguous chunks, the first
    total % world ranks one longer (engine.cpp:440-455)."""
    chunk, extra = divmod(total, world)
    begin = rank * chunk + min(rank, extra)
    return begin, begin + chunk + (1 if rank < extra else 0)


def _dist():
    try:
        import torch.distributed as d
        if d.is_available() and d.is_initialized():
            return d
    except Exception:
        pass
    return None


def init_nccl(device: int, group=None) -> None:
    """The ranks' NCCL communicator for frw_tally_allreduce: rank 0 draws the
    unique id (ncclGetUniqueId), the process group broadcasts it, and every
    rank calls frw_nccl_init on its device context.  Once per (group, device)."""
    from . import _core
    d = _dist()
    key = (id(group), device)
    if key in _NCCL_READY:
        return
    rank = d.get_rank(group) if d else 0
    world = d.get_world_size(group) if d else 1
    box = [_core.nccl_unique_id() if rank == 0 else None]
    if d is not None and world > 1:
        d.broadcast_object_list(box, src=0, group=group)
    _core.nccl_init(device, box[0], world, rank)
    _NCCL_READY[key] = True


def pack(t: dict) -> np.ndarray:
    """a tally as one f64 vector, the layout frw_tally_allreduce reduces"""
    return np.concatenate([np.asarray(t["sum"], np.float64), np.asarray(t["sumsq"], np.float64),
                           np.asarray(t["landed"], np.float64),
                           np.array([t["aborted"], t["resampled"], *t["first"], *t["sub"],
                                     t["mw_steps"], t["walks"], t.get("mw_jumps", 0),
                                     t.get("mw_jump_steps", 0)], np.float64)])


def unpack(v: np.ndarray, like: dict) -> dict:
    k = len(like["sum"])
    st = v[3 * k:]
    out = dict(like)
    out.update(sum=v[:k].copy(), sumsq=v[k:2 * k].copy(),
               landed=np.rint(v[2 * k:3 * k]).astype(np.uint64),
               aborted=int(st[0]), resampled=int(st[1]),
               first=[int(x) for x in st[2:6]], sub=[int(x) for x in st[6:10]],
               mw_steps=int(st[10]), walks=int(st[11]), mw_jumps=int(st[12]),
               mw_jump_steps=int(st[13]))
    return out


def allreduce_tally(t: dict, group=None) -> dict:
    """sum a tally over the ranks of `group` with torch.distributed (the gloo
    path; on GPUs run_tally(..., allreduce=True) uses frw_tally_allreduce)"""
    d = _dist()
    if d is None or d.get_world_size(group) == 1:
        return t
    import torch
    v = torch.from_numpy(pack(t))
    d.all_reduce(v, group=group)
    return unpack(v.numpy(), t)


def combine_local(tallies: list[dict]) -> dict:
    """the rank tallies of an emulated run combined in rank order (the
    arithmetic of the all-reduce, for single-process checks)"""
    acc = pack(tallies[0])
    for t in tallies[1:]:
        acc = acc + pack(t)
    return unpack(acc, tallies[0])


def device_runner(text: str, begin: int, count: int, allreduce: bool = False, **kw) -> dict:
    """the product's device path: frw_run_walks over the range (drop-in
    Engine, shared SGF cache), optionally frw_tally_allreduce"""
    from . import _core
    return _core.run_walks_tally(text, begin, count, allreduce, **kw)


def estimates(sum_, sumsq, walks):
    """Mean and standard error per slot (engine.cpp:388-400)."""
    w = float(walks)
    out = []
    for s1, s2 in zip(sum_, sumsq):
        mean = s1 / w
        se = 0.0
        if walks > 1:
            se = math.sqrt(max(0.0, (s2 - s1 * s1 / w) / (w - 1)) / w)
        out.append((mean, se))
    return out


def result_from_tally(t: dict, ids: list[int], master: int) -> dict:
    """extract_json's result schema (py_module.cpp:59-98) from a combined tally"""
    terms = []
    est = estimates(t["sum"], t["sumsq"], t["walks"])
    for k, (m, se) in enumerate(est):
        terms.append(dict(conductor_id=ids[k] if k < len(ids) else -1, capacitance_farads=m,
                          std_err_farads=se, walks_landed=int(t["landed"][k])))
    f, s = t["first"], t["sub"]
    return dict(master_id=master, terminals=terms, walks=int(t["walks"]), converged=False,
                aborted=int(t["aborted"]), resampled=int(t["resampled"]),
                dispatch_stats=dict(
                    first=dict(stratified=f[0], shrunk=f[1], layered=f[2], homogenized=f[3]),
                    subsequent=dict(cached=s[0], microwalk=s[1], microwalk_e=s[2], fdm=s[3])),
                mw_steps=int(t["mw_steps"]), mw_jumps=int(t.get("mw_jumps", 0)),
                mw_jump_steps=int(t.get("mw_jump_steps", 0)))


def extract_sharded(text: str, walks: int, group=None, runner=None, device: int | None = None,
                    **kw) -> dict:
    """extract_json for a fixed walk count, sharded over the ranks of `group`
    (default: the default process group, or one rank).  Rank g runs walks
    rank_range(walks, g, G) of the seed's one walk sequence; the tallies are
    combined by one all-reduce: frw_tally_allreduce over NCCL when the group
    uses the nccl backend, torch.distributed otherwise.  `runner(text, begin,
    count, allreduce, **kw)` is the tally source (device_runner by default).
    Every rank returns the combined result; `t_device_seconds` and
    `t_mw_seconds` are this rank's."""
    d = _dist()
    rank = d.get_rank(group) if d else 0
    world = d.get_world_size(group) if d else 1
    b, e = rank_range(walks, rank, world)
    nccl = runner is None and d is not None and world > 1 and d.get_backend(group) == "nccl"
    if runner is None:
        runner = device_runner
    reducer = "frw_tally_allreduce" if nccl else ("torch.distributed" if world > 1 else "none")
    if nccl:
        init_nccl(device if device is not None else kw.get("device", 0), group)
    if device is not None:
        kw["device"] = device
    t = runner(text, b, e - b, nccl, **kw)
    t["walks"] = e - b
    if nccl:
        t["walks"] = walks  # frw_tally_allreduce combined the counters already
    else:
        t = allreduce_tally(t, group)
    doc = json.loads(text)
    ids = [c["id"] for c in doc["conductors"]]
    res = result_from_tally(t, ids, doc["master"])
    res["t_device_seconds"] = t.get("t_device_seconds", 0.0)
    res["t_mw_seconds"] = t.get("t_mw_seconds", 0.0)
    res["walks_this_rank"] = e - b
    res["allreduce"] = reducer
    return res


def combine_tallies(sum_, sumsq, landed, device=None):
    """All-reduce bare per-terminal tallies over the default process group."""
    k = len(sum_)
    t = dict(sum=sum_, sumsq=sumsq, landed=landed, aborted=0, resampled=0, first=[0] * 4,
             sub=[0] * 4, mw_steps=0, walks=0)
    r = allreduce_tally(t)
    return r["sum"][:k], r["sumsq"][:k], r["landed"][:k]
