"""ctypes front-end for the CPU oracle.  TEST INFRASTRUCTURE ONLY.

Two checkers live here:

* ``Oracle`` -- the C restatement ``oracle/liboracle.so`` (frw_oracle.c),
  which every parity test uses as the reference answer.
* ``Ref`` -- ``oracle/_ref/libfrwref.so``: the reference's own, unmodified
  ``microwalk.cpp``/``geometry.cpp``/``engine.cpp``/``sgf_cache.cpp`` compiled
  from /root/reference (plus the restated Eigen-free ``sgf.cpp`` shim).  It
  pins the restatement and is the ``--impl reference`` CPU arm of bench.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libfrwref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint64)
_bp = C.POINTER(C.c_uint8)
_lp = C.POINTER(C.c_int64)

MODES = {"FDM": 0, "MW": 1, "MWE": 2, "HYBRID-MW": 3, "HYBRID-MWE": 4}


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# scene description shared by both checkers (geometry.hpp:94-121)

@dataclass
class Scene:
    cond_id: np.ndarray            # int32 [C]
    cond_box: np.ndarray           # f64 [C,6] lo.xyz hi.xyz
    diel_box: np.ndarray           # f64 [D,6]
    diel_eps: np.ndarray           # f64 [D]
    background_eps: float
    world: np.ndarray              # f64 [6]
    master_id: int
    meta: dict = field(default_factory=dict)

    @property
    def n_cond(self):
        return int(self.cond_id.shape[0])

    @property
    def n_diel(self):
        return int(self.diel_eps.shape[0])

    def master_slot(self):
        return int(np.nonzero(self.cond_id == self.master_id)[0][0])

    def to_json(self) -> str:
        def b(r):
            return {"lo": [float(x) for x in r[:3]], "hi": [float(x) for x in r[3:]]}
        doc = {
            "units": "nm",
            "world": b(self.world),
            "background_eps": float(self.background_eps),
            "conductors": [dict(id=int(i), **b(r)) for i, r in zip(self.cond_id, self.cond_box)],
            "dielectrics": [dict(eps=float(e), **b(r)) for e, r in zip(self.diel_eps, self.diel_box)],
            "master": int(self.master_id),
        }
        return json.dumps(doc)

    def with_master(self, master_id: int) -> "Scene":
        return Scene(self.cond_id, self.cond_box, self.diel_box, self.diel_eps,
                     self.background_eps, self.world, int(master_id), dict(self.meta))


class _Structure(C.Structure):
    _fields_ = [("n_cond", C.c_int), ("cond_id", _ip), ("cond_box", _dp),
                ("n_diel", C.c_int), ("diel_box", _dp), ("diel_eps", _dp),
                ("background_eps", C.c_double), ("world", C.c_double * 6),
                ("master_id", C.c_int32)]


class _Exit(C.Structure):
    _fields_ = [("kind", C.c_int), ("panel", C.c_int), ("conductor_id", C.c_int),
                ("point", C.c_double * 3), ("voxel", C.c_int * 3), ("dir", C.c_int),
                ("steps", C.c_int)]


class _Config(C.Structure):
    _fields_ = [("grid_n", C.c_int), ("expansion", C.c_double), ("mode", C.c_int),
                ("rel_std_tol", C.c_double), ("min_walks", C.c_int64),
                ("max_walks", C.c_int64), ("batch", C.c_int), ("seed", C.c_uint64),
                ("snap_tol", C.c_double), ("hop_cap", C.c_int64),
                ("gaussian_gap_fraction", C.c_double), ("world_margin", C.c_double),
                ("all_couplings_rule", C.c_int)]


class _Result(C.Structure):
    _fields_ = [("value", _dp), ("std_err", _dp), ("landed", _up), ("sum", _dp),
                ("sumsq", _dp), ("walks", C.c_uint64), ("converged", C.c_int),
                ("aborted", C.c_uint64), ("resampled", C.c_uint64),
                ("first", C.c_uint64 * 4), ("sub", C.c_uint64 * 4),
                ("cache_hits", C.c_uint64), ("cache_misses", C.c_uint64),
                ("mw_steps", C.c_uint64), ("t_total_seconds", C.c_double)]


CONFIG_DEFAULTS = dict(grid_n=24, expansion=5.0, mode="HYBRID-MWE", tol=0.01,
                       min_walks=4096, max_walks=4000000, batch=1024, seed=1,
                       snap_tol=1e-4, hop_cap=10000, gaussian_gap_fraction=0.5,
                       world_margin=5.0, all_couplings=False)


def _config(**kw):
    c = dict(CONFIG_DEFAULTS)
    for k, v in kw.items():
        if k not in c:
            raise ValueError(f"unknown option: {k}")
        c[k] = v
    return c


class Oracle:
    """The C restatement (frw_oracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.frwo_last_error.restype = C.c_char_p
        L.frwo_stream_state.restype = C.c_uint64
        L.frwo_stream_state.argtypes = [C.c_uint64, C.c_uint64]
        L.frwo_next.restype = C.c_uint64
        L.frwo_next.argtypes = [_up]
        L.frwo_uniform.restype = C.c_double
        L.frwo_uniform.argtypes = [_up]
        L.frwo_mix.restype = C.c_uint64
        L.frwo_mix.argtypes = [C.c_uint64]
        L.frwo_round_sig.restype = C.c_double
        L.frwo_round_sig.argtypes = [C.c_double, C.c_int]
        L.frwo_expected_steps.restype = C.c_double
        L.frwo_expected_steps.argtypes = [C.c_int, _dp]
        L.frwo_sample_panel.argtypes = [_dp, C.c_int, C.c_double]
        L.frwo_microwalk_grid_batch.argtypes = [
            C.c_int, _dp, _ip, _dp, C.c_double, C.c_uint64, C.c_uint64, C.c_int64,
            C.c_int, C.c_int, _ip, _ip, _up, _dp, _dp]
        L.frwo_solve_sgf.argtypes = [C.c_int, _dp, C.c_double, _dp, _dp, _dp]
        L.frwo_scratch_new.restype = C.c_void_p
        L.frwo_scratch_free.argtypes = [C.c_void_p]
        L.frwo_microwalk_lazy.argtypes = [C.POINTER(_Structure), _dp, C.c_double, C.c_int,
                                          _up, C.c_void_p, C.c_int, C.POINTER(_Exit)]
        L.frwo_microwalk_e.argtypes = [C.POINTER(_Structure), _dp, C.c_double, C.c_double,
                                       C.c_int, _up, C.c_void_p, C.c_int, C.POINTER(_Exit)]
        L.frwo_permittivity_at.argtypes = [C.POINTER(_Structure), _dp, _dp]
        L.frwo_conductor_at.argtypes = [C.POINTER(_Structure), _dp, C.c_double]
        L.frwo_max_free_cube.argtypes = [C.POINTER(_Structure), _dp, _dp, _ip]
        L.frwo_stratified_profile.argtypes = [C.POINTER(_Structure), _dp, C.c_double,
                                              C.c_int, _dp]
        L.frwo_build_grid.argtypes = [C.POINTER(_Structure), _dp, C.c_double, C.c_int,
                                      _dp, _ip]
        L.frwo_extract.argtypes = [C.POINTER(_Structure), C.POINTER(_Config), C.c_int,
                                   C.POINTER(_Result)]
        L.frwo_run_walks.argtypes = [C.POINTER(_Structure), C.POINTER(_Config), C.c_uint64,
                                     C.c_int64, C.c_int, _ip, _dp, _bp]

    def err(self):
        return self.lib.frwo_last_error().decode()

    # -- rng ------------------------------------------------------------
    def stream_state(self, seed, stream):
        return int(self.lib.frwo_stream_state(seed, stream))

    def uniforms(self, seed, stream, count):
        st = C.c_uint64(self.stream_state(seed, stream))
        return np.array([self.lib.frwo_uniform(C.byref(st)) for _ in range(count)])

    def round_sig(self, x, digits=6):
        return self.lib.frwo_round_sig(float(x), digits)

    # -- single-cube MicroWalk -----------------------------------------
    def microwalk_grid(self, eps, center, half_width, seed, stream0, count, mask=None,
                       step_cap=0, threads=1, per_transit=True, hist=True):
        n = int(round(len(eps) ** (1 / 3)))
        eps = np.ascontiguousarray(eps, np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.int32)
        c = np.ascontiguousarray(center, np.float64)
        panel = np.empty(count, np.int32) if per_transit else None
        steps = np.empty(count, np.int32) if per_transit else None
        h = np.zeros(6 * n * n, np.uint64) if hist else None
        s1, s2 = C.c_double(), C.c_double()
        rc = self.lib.frwo_microwalk_grid_batch(
            n, _ptr(eps, _dp), _ptr(m, _ip), _ptr(c, _dp), float(half_width), seed,
            stream0, count, step_cap, threads, _ptr(panel, _ip), _ptr(steps, _ip),
            _ptr(h, _up), C.byref(s1), C.byref(s2))
        if rc:
            raise RuntimeError(self.err())
        return dict(panel=panel, steps=steps, hist=h, step_sum=s1.value, step_sumsq=s2.value)

    def solve_sgf(self, eps, half_width=None, kernels=True):
        n = int(round(len(eps) ** (1 / 3)))
        eps = np.ascontiguousarray(eps, np.float64)
        hw = n / 2.0 if half_width is None else half_width
        probs = np.empty(6 * n * n)
        ker = np.empty((3, 6 * n * n)) if kernels else None
        pitch = C.c_double()
        rc = self.lib.frwo_solve_sgf(n, _ptr(eps, _dp), hw, _ptr(probs, _dp),
                                     _ptr(ker, _dp), C.byref(pitch))
        if rc:
            raise RuntimeError(self.err())
        return dict(probs=probs, cdf=np.cumsum(probs), kernels=ker, pitch=pitch.value)

    def expected_steps(self, eps):
        n = int(round(len(eps) ** (1 / 3)))
        eps = np.ascontiguousarray(eps, np.float64)
        return self.lib.frwo_expected_steps(n, _ptr(eps, _dp))

    def sample_panel(self, cdf, u):
        cdf = np.ascontiguousarray(cdf, np.float64)
        return self.lib.frwo_sample_panel(_ptr(cdf, _dp), len(cdf), float(u))

    # -- structure queries ---------------------------------------------
    def _s(self, sc: Scene):
        keep = (np.ascontiguousarray(sc.cond_id, np.int32),
                np.ascontiguousarray(sc.cond_box, np.float64),
                np.ascontiguousarray(sc.diel_box, np.float64).reshape(-1, 6),
                np.ascontiguousarray(sc.diel_eps, np.float64))
        s = _Structure(sc.n_cond, _ptr(keep[0], _ip), _ptr(keep[1], _dp), sc.n_diel,
                       _ptr(keep[2], _dp), _ptr(keep[3], _dp), float(sc.background_eps),
                       (C.c_double * 6)(*[float(x) for x in sc.world]), int(sc.master_id))
        s._keep = keep
        return s

    def permittivity_at(self, sc, p):
        s, out = self._s(sc), C.c_double()
        pp = np.ascontiguousarray(p, np.float64)
        if self.lib.frwo_permittivity_at(C.byref(s), _ptr(pp, _dp), C.byref(out)):
            raise ValueError(self.err())
        return out.value

    def conductor_at(self, sc, p, tol):
        """declaration index of the first conductor within tol, or -1"""
        pp = np.ascontiguousarray(p, np.float64)
        return self.lib.frwo_conductor_at(C.byref(self._s(sc)), _ptr(pp, _dp), float(tol))

    def max_free_cube(self, sc, p):
        hw, near = C.c_double(), C.c_int32()
        pp = np.ascontiguousarray(p, np.float64)
        if self.lib.frwo_max_free_cube(C.byref(self._s(sc)), _ptr(pp, _dp), C.byref(hw),
                                       C.byref(near)):
            raise ValueError(self.err())
        return hw.value, near.value

    def stratified_profile(self, sc, center, hw, n):
        layers = np.empty(n)
        c = np.ascontiguousarray(center, np.float64)
        ax = self.lib.frwo_stratified_profile(C.byref(self._s(sc)), _ptr(c, _dp), float(hw),
                                              n, _ptr(layers, _dp))
        if ax == -2:
            raise ValueError(self.err())
        return (None, None) if ax < 0 else (ax, layers)

    def build_grid(self, sc, center, hw, n, mask=False):
        eps = np.empty(n ** 3)
        m = np.empty(n ** 3, np.int32) if mask else None
        c = np.ascontiguousarray(center, np.float64)
        if self.lib.frwo_build_grid(C.byref(self._s(sc)), _ptr(c, _dp), float(hw), n,
                                    _ptr(eps, _dp), _ptr(m, _ip)):
            raise ValueError(self.err())
        return eps, m

    def microwalk_lazy(self, sc, center, hw, n, seed, stream0, count, expanded=False,
                       expansion=5.0):
        s = self._s(sc)
        scr = self.lib.frwo_scratch_new()
        c = np.ascontiguousarray(center, np.float64)
        out = dict(panel=np.empty(count, np.int32), steps=np.empty(count, np.int32),
                   point=np.empty((count, 3)), cond=np.empty(count, np.int32))
        try:
            for t in range(count):
                st = C.c_uint64(self.stream_state(seed, stream0 + t))
                e = _Exit()
                if expanded:
                    rc = self.lib.frwo_microwalk_e(C.byref(s), _ptr(c, _dp), float(hw),
                                                   float(expansion), n, C.byref(st), scr, 0,
                                                   C.byref(e))
                else:
                    rc = self.lib.frwo_microwalk_lazy(C.byref(s), _ptr(c, _dp), float(hw), n,
                                                      C.byref(st), scr, 0, C.byref(e))
                if rc:
                    raise RuntimeError(self.err())
                out["panel"][t] = e.panel if e.kind == 0 else -1
                out["steps"][t] = e.steps
                out["point"][t] = list(e.point)
                out["cond"][t] = e.conductor_id
        finally:
            self.lib.frwo_scratch_free(scr)
        return out

    # -- engine ----------------------------------------------------------
    def _cfg(self, **kw):
        c = _config(**kw)
        return _Config(int(c["grid_n"]), float(c["expansion"]), MODES[c["mode"].upper()],
                       float(c["tol"]), int(c["min_walks"]), int(c["max_walks"]),
                       int(c["batch"]), int(c["seed"]), float(c["snap_tol"]),
                       int(c["hop_cap"]), float(c["gaussian_gap_fraction"]),
                       float(c["world_margin"]), int(bool(c["all_couplings"])))

    def extract(self, sc: Scene, threads=1, **kw):
        s, cfg = self._s(sc), self._cfg(**kw)
        k = sc.n_cond + 1
        arr = {nm: np.zeros(k) for nm in ("value", "std_err", "sum", "sumsq")}
        landed = np.zeros(k, np.uint64)
        r = _Result(_ptr(arr["value"], _dp), _ptr(arr["std_err"], _dp), _ptr(landed, _up),
                    _ptr(arr["sum"], _dp), _ptr(arr["sumsq"], _dp))
        if self.lib.frwo_extract(C.byref(s), C.byref(cfg), threads, C.byref(r)):
            raise RuntimeError(self.err())
        ids = list(sc.cond_id) + [-1]
        return dict(
            master_id=sc.master_id, walks=r.walks, converged=bool(r.converged),
            aborted=r.aborted, resampled=r.resampled,
            terminals=[dict(conductor_id=int(ids[i]), capacitance_farads=arr["value"][i],
                            std_err_farads=arr["std_err"][i], walks_landed=int(landed[i]))
                       for i in range(k)],
            sum=arr["sum"], sumsq=arr["sumsq"],
            dispatch_stats=dict(first=dict(zip(("stratified", "shrunk", "layered", "homogenized"),
                                               map(int, r.first))),
                                subsequent=dict(zip(("cached", "microwalk", "microwalk_e", "fdm"),
                                                    map(int, r.sub)))),
            cache=dict(hits=r.cache_hits, misses=r.cache_misses), mw_steps=r.mw_steps,
            t_total_seconds=r.t_total_seconds)

    def run_walks(self, sc: Scene, w0, count, threads=1, **kw):
        s, cfg = self._s(sc), self._cfg(**kw)
        slot = np.empty(count, np.int32)
        w = np.empty(count)
        ab = np.empty(count, np.uint8)
        if self.lib.frwo_run_walks(C.byref(s), C.byref(cfg), w0, count, threads,
                                   _ptr(slot, _ip), _ptr(w, _dp), _ptr(ab, _bp)):
            raise RuntimeError(self.err())
        return slot, w, ab


class Ref:
    """The reference's own sources (oracle/_ref/libfrwref.so)."""

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_microwalk_grid_batch.argtypes = [
            C.c_int, _dp, _ip, _dp, C.c_double, C.c_uint64, C.c_uint64, C.c_int64,
            C.c_int, C.c_int, _ip, _ip, _up, _dp, _dp]
        L.ref_structure_new.restype = C.c_void_p
        L.ref_structure_new.argtypes = [C.c_int, _ip, _dp, C.c_int, _dp, _dp, C.c_double,
                                        _dp, C.c_int32]
        L.ref_structure_parse.restype = C.c_void_p
        L.ref_structure_parse.argtypes = [C.c_char_p, C.c_double]
        L.ref_structure_free.argtypes = [C.c_void_p]
        L.ref_structure_counts.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_structure_dump.argtypes = [C.c_void_p, _ip, _dp, _dp, _dp, _dp, _dp, _ip]
        L.ref_permittivity_at.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_conductor_at.argtypes = [C.c_void_p, _dp, C.c_double, _ip]
        L.ref_max_free_cube.argtypes = [C.c_void_p, _dp, _dp, _ip]
        L.ref_stratified_profile.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, _dp]
        L.ref_build_grid.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, _dp, _ip,
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_microwalk_lazy_batch.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, C.c_uint64,
                                               C.c_uint64, C.c_int64, _ip, _ip, _dp]
        L.ref_microwalk_e_batch.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_int,
                                            C.c_uint64, C.c_uint64, C.c_int64, _ip, _ip, _dp,
                                            _ip]
        L.ref_solve_sgf.argtypes = [C.c_int, _dp, _ip, _dp, C.c_double, _dp, _dp, _dp]
        L.ref_expected_steps.restype = C.c_double
        L.ref_expected_steps.argtypes = [C.c_int, _dp]
        L.ref_round_sig.restype = C.c_double
        L.ref_round_sig.argtypes = [C.c_double, C.c_int]
        L.ref_extract.argtypes = [C.c_void_p, _dp, _lp, C.c_int, _dp, _dp, _up, _up, _dp]
        L.ref_run_walks.argtypes = [C.c_void_p, _dp, _lp, C.c_uint64, C.c_int64, _ip, _dp, _bp]
        L.ref_extract_warm.argtypes = [C.c_void_p, _dp, _lp, C.c_int, _dp, _dp, _up, _up, _dp]
        L.ref_extract_cache.argtypes = [C.c_void_p, _dp, _lp, C.c_int, C.c_char_p, C.c_char_p,
                                        _dp, _dp, _up, _up, _dp]
        L.ref_run_walks_cache.argtypes = [C.c_void_p, _dp, _lp, C.c_uint64, C.c_int64, C.c_int,
                                          C.c_char_p, C.c_char_p, _ip, _dp, _bp]
        L.ref_cache_save.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_char_p]
        L.ref_warm_cache_load.restype = C.c_int64
        L.ref_warm_cache_load.argtypes = [C.c_char_p]
        L.ref_cache_load_probs.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, _dp, _lp]

    def err(self):
        return self.lib.ref_last_error().decode()

    def warm_cache_load(self, path):
        """SGF1 file into the process-wide cache of extract(warm_cache=True)"""
        n = self.lib.ref_warm_cache_load(path.encode())
        if n < 0:
            raise RuntimeError(self.err())
        return n

    def cache_save(self, n, axes, layers, path):
        """SGF1 file written by the reference's StratifiedSgfCache"""
        ax = np.ascontiguousarray(axes, np.int32)
        lay = np.ascontiguousarray(layers, np.float64).reshape(len(ax), n)
        if self.lib.ref_cache_save(n, len(ax), _ptr(ax, _ip), _ptr(lay, _dp), path.encode()):
            raise RuntimeError(self.err())

    def cache_load_probs(self, path, n, axis, layers):
        """the reference's StratifiedSgfCache::load of `path`, then find(key)"""
        lay = np.ascontiguousarray(layers, np.float64)
        probs = np.empty(6 * n * n)
        loaded = C.c_int64()
        rc = self.lib.ref_cache_load_probs(path.encode(), n, axis, _ptr(lay, _dp),
                                           _ptr(probs, _dp), C.byref(loaded))
        if rc == -2:
            return None, loaded.value
        if rc:
            raise RuntimeError(self.err())
        return probs, loaded.value

    def microwalk_grid(self, eps, center, half_width, seed, stream0, count, mask=None,
                       step_cap=0, threads=1, per_transit=True, hist=True):
        n = int(round(len(eps) ** (1 / 3)))
        eps = np.ascontiguousarray(eps, np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.int32)
        c = np.ascontiguousarray(center, np.float64)
        panel = np.empty(count, np.int32) if per_transit else None
        steps = np.empty(count, np.int32) if per_transit else None
        h = np.zeros(6 * n * n, np.uint64) if hist else None
        s1, s2 = C.c_double(), C.c_double()
        rc = self.lib.ref_microwalk_grid_batch(
            n, _ptr(eps, _dp), _ptr(m, _ip), _ptr(c, _dp), float(half_width), seed, stream0,
            count, step_cap, threads, _ptr(panel, _ip), _ptr(steps, _ip), _ptr(h, _up),
            C.byref(s1), C.byref(s2))
        if rc:
            raise RuntimeError(self.err())
        return dict(panel=panel, steps=steps, hist=h, step_sum=s1.value, step_sumsq=s2.value)

    # structure handle -------------------------------------------------------
    def structure(self, sc: Scene):
        ids = np.ascontiguousarray(sc.cond_id, np.int32)
        cb = np.ascontiguousarray(sc.cond_box, np.float64)
        db = np.ascontiguousarray(sc.diel_box, np.float64).reshape(-1, 6)
        de = np.ascontiguousarray(sc.diel_eps, np.float64)
        w = np.ascontiguousarray(sc.world, np.float64)
        h = self.lib.ref_structure_new(sc.n_cond, _ptr(ids, _ip), _ptr(cb, _dp), sc.n_diel,
                                       _ptr(db, _dp), _ptr(de, _dp), float(sc.background_eps),
                                       _ptr(w, _dp), int(sc.master_id))
        return _RefHandle(self, h)

    def parse(self, text: str, world_margin: float = 5.0) -> Scene:
        h = self.lib.ref_structure_parse(text.encode(), world_margin)
        if not h:
            raise ValueError(self.err())
        try:
            nc, nd = C.c_int(), C.c_int()
            self.lib.ref_structure_counts(h, C.byref(nc), C.byref(nd))
            ids = np.empty(nc.value, np.int32)
            cb = np.empty((nc.value, 6))
            db = np.empty((nd.value, 6))
            de = np.empty(nd.value)
            bg = C.c_double()
            w = np.empty(6)
            m = C.c_int32()
            self.lib.ref_structure_dump(h, _ptr(ids, _ip), _ptr(cb, _dp), _ptr(db, _dp),
                                        _ptr(de, _dp), C.byref(bg), _ptr(w, _dp), C.byref(m))
            return Scene(ids, cb, db, de, bg.value, w, m.value)
        finally:
            self.lib.ref_structure_free(h)

    def solve_sgf(self, eps, half_width=None, kernels=True, mask=None, center=(0, 0, 0)):
        n = int(round(len(eps) ** (1 / 3)))
        eps = np.ascontiguousarray(eps, np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.int32)
        c = np.ascontiguousarray(center, np.float64)
        hw = n / 2.0 if half_width is None else half_width
        cap = 6 * n * n + 6 * n ** 3
        probs = np.empty(cap)
        ker = np.empty((3, cap)) if kernels else None
        pitch = C.c_double()
        k = self.lib.ref_solve_sgf(n, _ptr(eps, _dp), _ptr(m, _ip), _ptr(c, _dp), hw,
                                   _ptr(probs, _dp), _ptr(ker, _dp), C.byref(pitch))
        if k < 0:
            raise RuntimeError(self.err())
        out = dict(probs=probs[:k].copy(), pitch=pitch.value)
        if kernels:
            out["kernels"] = np.ascontiguousarray(ker.reshape(-1)[: 3 * k].reshape(3, k))
        return out

    def expected_steps(self, eps):
        n = int(round(len(eps) ** (1 / 3)))
        eps = np.ascontiguousarray(eps, np.float64)
        return self.lib.ref_expected_steps(n, _ptr(eps, _dp))

    def round_sig(self, x, digits=6):
        return self.lib.ref_round_sig(float(x), digits)

    @staticmethod
    def cfg_arrays(**kw):
        c = _config(**kw)
        d = np.array([c["expansion"], c["tol"], c["snap_tol"], c["gaussian_gap_fraction"],
                      c["world_margin"]], np.float64)
        i = np.array([c["grid_n"], MODES[c["mode"].upper()], c["min_walks"], c["max_walks"],
                      c["batch"], c["seed"], c["hop_cap"]], np.int64)
        return d, i


class _RefHandle:
    def __init__(self, ref: Ref, h):
        self.ref, self.h, self.lib = ref, h, ref.lib

    def __del__(self):
        try:
            self.lib.ref_structure_free(self.h)
        except Exception:
            pass

    def permittivity_at(self, p):
        out = C.c_double()
        pp = np.ascontiguousarray(p, np.float64)
        if self.lib.ref_permittivity_at(self.h, _ptr(pp, _dp), C.byref(out)):
            raise ValueError(self.ref.err())
        return out.value

    def conductor_at(self, p, tol):
        """conductor id within tol, or None"""
        cid = C.c_int32()
        pp = np.ascontiguousarray(p, np.float64)
        return cid.value if self.lib.ref_conductor_at(self.h, _ptr(pp, _dp), float(tol),
                                                      C.byref(cid)) else None

    def max_free_cube(self, p):
        hw, near = C.c_double(), C.c_int32()
        pp = np.ascontiguousarray(p, np.float64)
        if self.lib.ref_max_free_cube(self.h, _ptr(pp, _dp), C.byref(hw), C.byref(near)):
            raise ValueError(self.ref.err())
        return hw.value, near.value

    def stratified_profile(self, center, hw, n):
        layers = np.empty(n)
        c = np.ascontiguousarray(center, np.float64)
        ax = self.lib.ref_stratified_profile(self.h, _ptr(c, _dp), float(hw), n,
                                             _ptr(layers, _dp))
        if ax == -2:
            raise ValueError(self.ref.err())
        return (None, None) if ax < 0 else (ax, layers)

    def build_grid(self, center, hw, n, allow_conductors=False):
        eps = np.empty(n ** 3)
        mask = np.full(n ** 3, -1, np.int32)
        tag, ax = C.c_int(), C.c_int()
        c = np.ascontiguousarray(center, np.float64)
        if self.lib.ref_build_grid(self.h, _ptr(c, _dp), float(hw), n, int(allow_conductors),
                                   _ptr(eps, _dp), _ptr(mask, _ip), C.byref(tag), C.byref(ax)):
            raise ValueError(self.ref.err())
        return eps, (mask if allow_conductors else None), tag.value, ax.value

    def microwalk_lazy(self, center, hw, n, seed, stream0, count):
        c = np.ascontiguousarray(center, np.float64)
        out = dict(panel=np.empty(count, np.int32), steps=np.empty(count, np.int32),
                   point=np.empty((count, 3)))
        if self.lib.ref_microwalk_lazy_batch(self.h, _ptr(c, _dp), float(hw), n, seed, stream0,
                                             count, _ptr(out["panel"], _ip),
                                             _ptr(out["steps"], _ip), _ptr(out["point"], _dp)):
            raise RuntimeError(self.ref.err())
        return out

    def microwalk_e(self, p, base_hw, expansion, n, seed, stream0, count):
        pp = np.ascontiguousarray(p, np.float64)
        out = dict(panel=np.empty(count, np.int32), steps=np.empty(count, np.int32),
                   point=np.empty((count, 3)), cond=np.empty(count, np.int32))
        rc = self.lib.ref_microwalk_e_batch(self.h, _ptr(pp, _dp), float(base_hw),
                                            float(expansion), n, seed, stream0, count,
                                            _ptr(out["panel"], _ip), _ptr(out["steps"], _ip),
                                            _ptr(out["point"], _dp), _ptr(out["cond"], _ip))
        if rc == -3:
            raise LookupError("EngulfedStart")
        if rc:
            raise RuntimeError(self.ref.err())
        return out

    def extract(self, threads=1, warm_cache=False, cache_in=None, cache_out=None, **kw):
        """Engine::extract.  warm_cache: a process-wide cache shared by calls;
        cache_in / cache_out: SGF1 files loaded before / saved after the
        call (the CLI's --cache, cli.cpp:186-193)"""
        d, i = Ref.cfg_arrays(**kw)
        nc, nd = C.c_int(), C.c_int()
        self.lib.ref_structure_counts(self.h, C.byref(nc), C.byref(nd))
        k = nc.value + 1
        val, se = np.zeros(k), np.zeros(k)
        landed = np.zeros(k, np.uint64)
        st = np.zeros(14, np.uint64)
        tm = np.zeros(2)
        if cache_in is not None or cache_out is not None:
            rc = self.lib.ref_extract_cache(
                self.h, _ptr(d, _dp), _ptr(i, _lp), threads,
                None if cache_in is None else cache_in.encode(),
                None if cache_out is None else cache_out.encode(), _ptr(val, _dp),
                _ptr(se, _dp), _ptr(landed, _up), _ptr(st, _up), _ptr(tm, _dp))
        else:
            fn = self.lib.ref_extract_warm if warm_cache else self.lib.ref_extract
            rc = fn(self.h, _ptr(d, _dp), _ptr(i, _lp), threads, _ptr(val, _dp),
                    _ptr(se, _dp), _ptr(landed, _up), _ptr(st, _up), _ptr(tm, _dp))
        if rc:
            raise RuntimeError(self.ref.err())
        return dict(value=val, std_err=se, landed=landed, walks=int(st[0]),
                    converged=bool(st[1]), aborted=int(st[2]), resampled=int(st[3]),
                    first=st[4:8].astype(int).tolist(), sub=st[8:12].astype(int).tolist(),
                    cache_hits=int(st[12]), cache_misses=int(st[13]),
                    t_mw_seconds=tm[0], t_total_seconds=tm[1])

    def run_walks(self, w0, count, threads=1, cache_in=None, cache_out=None, **kw):
        """per-walk (slot, weight, aborted) of the reference Engine; its
        stratified-SGF cache starts from cache_in and is saved to cache_out
        (SGF1 files, the reference's own solves)"""
        d, i = Ref.cfg_arrays(**kw)
        slot = np.empty(count, np.int32)
        w = np.empty(count)
        ab = np.empty(count, np.uint8)
        if threads == 1 and cache_in is None and cache_out is None:
            rc = self.lib.ref_run_walks(self.h, _ptr(d, _dp), _ptr(i, _lp), w0, count,
                                        _ptr(slot, _ip), _ptr(w, _dp), _ptr(ab, _bp))
        else:
            rc = self.lib.ref_run_walks_cache(
                self.h, _ptr(d, _dp), _ptr(i, _lp), w0, count, threads,
                None if cache_in is None else cache_in.encode(),
                None if cache_out is None else cache_out.encode(),
                _ptr(slot, _ip), _ptr(w, _dp), _ptr(ab, _bp))
        if rc:
            raise RuntimeError(self.ref.err())
        return slot, w, ab
