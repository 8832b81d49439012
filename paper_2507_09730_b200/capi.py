"""ctypes binding of the C ABI in include/frw_gpu.h (libfrwgpu.so).

This is the reference-facing plugin boundary for the single-cube MicroWalk
path (configs C1/C2) as a Python caller sees it; the walk engine is reached
through the C++ `frwcap` mirror (`paper_2507_09730_b200.frwcap`).  There is
no CPU fallback: if the CUDA library is missing or no device is present the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libfrwgpu.so")

FRW_OK, FRW_EINVAL, FRW_ECUDA, FRW_ESTEPCAP, FRW_EENGULFED, FRW_ESOLVE = 0, -1, -2, -3, -4, -5
FRW_ENOMEM, FRW_EMISS = -6, -7
RNG_SPLITMIX_PARITY, RNG_PHILOX, RNG_SPLITMIX_STATES = 0, 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint64)


class FrwError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class StepCapExceeded(FrwError):
    pass


class EngulfedStart(FrwError):
    pass


class MwParams(C.Structure):
    _fields_ = [("rng_mode", C.c_int), ("seed", C.c_uint64), ("stream_begin", C.c_uint64),
                ("count", C.c_int64), ("step_cap", C.c_int32), ("blocks", C.c_int32),
                ("states", C.c_void_p)]


class MwOut(C.Structure):
    _fields_ = [("panels", C.c_void_p), ("steps", C.c_void_p), ("cond", C.c_void_p),
                ("hist", C.c_void_p), ("step_sum", C.c_void_p), ("step_sumsq", C.c_void_p),
                ("cond_exits", C.c_void_p), ("exit_nd", C.c_void_p)]


class Exit(C.Structure):
    _fields_ = [("kind", C.c_int32), ("panel", C.c_int32), ("conductor", C.c_int32),
                ("dir", C.c_int32), ("voxel", C.c_int32 * 3), ("steps", C.c_int32),
                ("point", C.c_double * 3)]


class StructureDesc(C.Structure):
    _fields_ = [("n_cond", C.c_int32), ("cond_id", C.POINTER(C.c_int32)),
                ("cond_box", C.POINTER(C.c_double)), ("n_diel", C.c_int32),
                ("diel_box", C.POINTER(C.c_double)), ("diel_eps", C.POINTER(C.c_double)),
                ("background_eps", C.c_double), ("world", C.c_double * 6)]


class WalkParams(C.Structure):
    _fields_ = [("grid_n", C.c_int32), ("mode", C.c_int32), ("expansion", C.c_double),
                ("snap", C.c_double), ("hop_cap", C.c_int64), ("seed", C.c_uint64),
                ("rng_mode", C.c_int32), ("n_slots", C.c_int32), ("gauss_box", C.c_double * 6),
                ("face_cdf", C.c_double * 6), ("area_m2", C.c_double)]


class Tally(C.Structure):
    _fields_ = [("sum", C.POINTER(C.c_double)), ("sumsq", C.POINTER(C.c_double)),
                ("landed", C.POINTER(C.c_uint64)), ("aborted", C.c_uint64),
                ("resampled", C.c_uint64), ("first", C.c_uint64 * 4), ("sub", C.c_uint64 * 4),
                ("cache_hits", C.c_uint64), ("cache_misses", C.c_uint64),
                ("mw_steps", C.c_uint64), ("restarts", C.c_uint64),
                ("mw_general_steps", C.c_uint64), ("mw_cell_changes", C.c_uint64),
                ("mw_ms", C.c_double),
                ("total_ms", C.c_double), ("mw_jumps", C.c_uint64),
                ("mw_jump_steps", C.c_uint64), ("mw_dense_hops", C.c_uint64)]


WALK_RECORD = np.dtype([("weight", "<f8"), ("mw_steps", "<u8"), ("slot", "<i4"),
                        ("cached", "<u4"), ("microwalk", "<u4"), ("aborted", "u1"),
                        ("branch", "u1"), ("resampled", "u1"), ("done", "u1")])
MISS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int),
                      C.POINTER(C.c_double))
MODE_MW, MODE_MWE, MODE_HYBRID_MW, MODE_HYBRID_MWE = 1, 2, 3, 4

_lib = None


def lib():
    """Load libfrwgpu.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.frw_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.frw_ctx_destroy.argtypes = [C.c_void_p]
        L.frw_last_error.restype = C.c_char_p
        L.frw_last_error.argtypes = [C.c_void_p]
        L.frw_device_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.c_char_p, C.c_int]
        L.frw_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.frw_synchronize.argtypes = [C.c_void_p]
        L.frw_upload_grid.argtypes = [C.c_void_p, C.c_int, _dp, _ip, C.c_double, C.c_double,
                                      C.c_double, C.c_double]
        L.frw_grid_compile.argtypes = [C.c_int, _dp, _ip, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_int)]
        L.frw_grid_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int)]
        L.frw_grid_h2d_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.frw_microwalk_batch.argtypes = [C.c_void_p, C.POINTER(MwParams), C.POINTER(MwOut)]
        L.frw_microwalk_batch_dev.argtypes = [C.c_void_p, C.POINTER(MwParams), C.POINTER(MwOut)]
        L.frw_microwalk_check.argtypes = [C.c_void_p]
        L.frw_event_record.argtypes = [C.c_void_p, C.c_int]
        L.frw_event_elapsed_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
        L.frw_dev_alloc.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.frw_dev_free.argtypes = [C.c_void_p, C.c_void_p]
        L.frw_dev_memset.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_size_t]
        L.frw_memcpy_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
        L.frw_memcpy_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
        L.frw_smem_bandwidth_probe.argtypes = [C.c_void_p, C.c_int, _dp]
        L.frw_upload_structure.argtypes = [C.c_void_p, C.POINTER(StructureDesc)]
        L.frw_sgf_put.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_double, _dp, _dp, _dp]
        L.frw_sgf_count.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.frw_sgf_clear.argtypes = [C.c_void_p]
        L.frw_sgf_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int), _dp, _dp,
                                    _dp]
        L.frw_grid_sgf_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_double, _dp, _dp,
                                         _dp]
        L.frw_reference_capacitance.argtypes = [C.c_void_p, C.POINTER(StructureDesc), C.c_int,
                                                _dp, _dp]
        L.frw_structure_transits.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _up,
                                             C.c_int32, C.POINTER(Exit)]
        L.frw_lattice_jump_law.argtypes = [C.c_int, _dp, _dp]
        L.frw_structure_transits_philox.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int,
                                                    C.c_uint64, C.c_int, C.c_int32,
                                                    C.POINTER(Exit)]
        _v = C.c_void_p
        L.frw_geometry_queries.argtypes = [_v, C.c_int, _v, C.c_double, _v, _v, _v, _v, _v]
        L.frw_stratified_keys.argtypes = [_v, C.c_int, C.c_int, _v, _v, _v]
        L.frw_nccl_unique_id.argtypes = [_v]
        L.frw_nccl_init.argtypes = [_v, _v, C.c_int, C.c_int]
        L.frw_nccl_destroy.argtypes = [_v]
        L.frw_tally_allreduce.argtypes = [_v, _v, C.POINTER(Tally)]
        L.frw_run_walks.argtypes = [C.c_void_p, C.POINTER(WalkParams), C.c_int32, C.c_uint64,
                                    C.c_int64, MISS_FN, C.c_void_p, C.POINTER(Tally),
                                    C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def grid_compile(eps, mask=None):
    """Host-only stencil-table compilation (no GPU needed)."""
    L = lib()
    eps = np.ascontiguousarray(eps, np.float64)
    n = int(round(len(eps) ** (1 / 3)))
    m = None if mask is None else np.ascontiguousarray(mask, np.int32)
    R = C.c_int()
    rc = L.frw_grid_compile(n, eps.ctypes.data_as(_dp), None if m is None else m.ctypes.data_as(_ip),
                            None, None, None, C.byref(R))
    if rc:
        raise FrwError(rc, "grid_compile failed")
    mp = np.empty((n + 2) ** 3, np.uint16)  # lattice with a one-node halo
    rec = np.empty(R.value, np.uint64)
    full = np.empty((R.value, 5), np.uint64)
    L.frw_grid_compile(n, eps.ctypes.data_as(_dp), None if m is None else m.ctypes.data_as(_ip),
                       _p(mp), _p(rec), _p(full), C.byref(R))
    return mp, rec, full


def lattice_jump_law(m):
    """Host-only: the face law ((2m-1)^2, v-major) and E[tau] of a radius-m
    lattice jump (frw_lattice_jump_law)."""
    side = 2 * m - 1
    face = np.empty(side * side, np.float64)
    et = C.c_double()
    rc = lib().frw_lattice_jump_law(int(m), face.ctypes.data_as(_dp), C.byref(et))
    if rc:
        raise FrwError(rc, "lattice_jump_law failed")
    return face.reshape(side, side), et.value


class Context:
    """One device context (frw_ctx)."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = C.c_void_p()
        rc = self.L.frw_ctx_create(device, C.byref(h))
        if rc:
            raise FrwError(rc, f"frw_ctx_create({device}) failed (is a CUDA device present?)")
        self.h = h
        self.n = None
        sm, clk = C.c_int(), C.c_int()
        name = C.create_string_buffer(256)
        self.L.frw_device_info(self.h, C.byref(sm), C.byref(clk), name, 256)
        self.sm_count, self.sm_clock_khz, self.name = sm.value, clk.value, name.value.decode()

    def close(self):
        if getattr(self, "h", None):
            self.L.frw_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc == 0:
            return
        msg = self.L.frw_last_error(self.h).decode()
        if rc == FRW_ESTEPCAP:
            raise StepCapExceeded(rc, msg)
        if rc == FRW_EENGULFED:
            raise EngulfedStart(rc, msg)
        if rc == FRW_EINVAL:
            raise ValueError(msg)
        raise FrwError(rc, msg)

    # -- single cube ------------------------------------------------------
    def upload_grid(self, eps, center=(0.0, 0.0, 0.0), half_width=None, mask=None):
        eps = np.ascontiguousarray(eps, np.float64)
        n = int(round(len(eps) ** (1 / 3)))
        if n ** 3 != len(eps):
            raise ValueError("eps must hold n^3 values")
        m = None if mask is None else np.ascontiguousarray(mask, np.int32)
        hw = n / 2.0 if half_width is None else float(half_width)
        self._check(self.L.frw_upload_grid(self.h, n, eps.ctypes.data_as(_dp),
                                           None if m is None else m.ctypes.data_as(_ip),
                                           float(center[0]), float(center[1]),
                                           float(center[2]), hw))
        self.n = n

    def grid_info(self):
        r, b, s = C.c_int(), C.c_int(), C.c_int()
        self._check(self.L.frw_grid_info(self.h, C.byref(r), C.byref(b), C.byref(s)))
        h2d = C.c_uint64()
        self._check(self.L.frw_grid_h2d_bytes(self.h, C.byref(h2d)))
        return dict(records=r.value, smem_bytes=b.value, smem_resident=bool(s.value),
                    h2d_bytes=h2d.value)

    def microwalk_batch(self, count, seed=1, stream_begin=0, rng=RNG_PHILOX, step_cap=0,
                        per_transit=False, blocks=0, states=None):
        """Host-buffer batch (frw_microwalk_batch).  `states` (raw SplitMix64
        states, one per transit) selects RNG_SPLITMIX_STATES."""
        n = self.n
        hist = np.zeros(6 * n * n, np.uint64)
        s1, s2, cx = C.c_uint64(), C.c_uint64(), C.c_uint64()
        panel = steps = cond = nd = None
        if states is not None:
            states = np.ascontiguousarray(states, np.uint64)
            count, rng = len(states), RNG_SPLITMIX_STATES
        if per_transit:
            panel = np.empty(count, np.int32)
            steps = np.empty(count, np.int32)
            cond = np.empty(count, np.int32)
            nd = np.empty(count, np.int64)
        p = MwParams(rng, seed, stream_begin, count, step_cap, blocks, _p(states))
        o = MwOut(_p(panel), _p(steps), _p(cond), _p(hist), C.cast(C.byref(s1), C.c_void_p),
                  C.cast(C.byref(s2), C.c_void_p), C.cast(C.byref(cx), C.c_void_p), _p(nd))
        self._check(self.L.frw_microwalk_batch(self.h, C.byref(p), C.byref(o)))
        return dict(hist=hist, step_sum=s1.value, step_sumsq=s2.value, cond_exits=cx.value,
                    panel=panel, steps=steps, cond=cond,
                    voxel=None if nd is None else nd >> 3, dir=None if nd is None else nd & 7)

    # device-resident interface (bench value path) -------------------------
    def alloc(self, nbytes):
        ptr = C.c_void_p()
        self._check(self.L.frw_dev_alloc(self.h, nbytes, C.byref(ptr)))
        return ptr.value

    def free(self, ptr):
        self._check(self.L.frw_dev_free(self.h, C.c_void_p(ptr)))

    def memset(self, ptr, nbytes):
        self._check(self.L.frw_dev_memset(self.h, C.c_void_p(ptr), 0, nbytes))

    def d2h(self, dst: np.ndarray, src_ptr):
        self._check(self.L.frw_memcpy_d2h(self.h, _p(dst), C.c_void_p(src_ptr), dst.nbytes))

    def microwalk_batch_dev(self, count, hist_ptr, mom_ptr, seed=1, stream_begin=0,
                            rng=RNG_PHILOX, step_cap=0, blocks=0):
        p = MwParams(rng, seed, stream_begin, count, step_cap, blocks, None)
        o = MwOut(None, None, None, hist_ptr, mom_ptr, mom_ptr + 8, mom_ptr + 16, None)
        self._check(self.L.frw_microwalk_batch_dev(self.h, C.byref(p), C.byref(o)))

    def check(self):
        self._check(self.L.frw_microwalk_check(self.h))

    def synchronize(self):
        self._check(self.L.frw_synchronize(self.h))

    def event_record(self, which):
        self._check(self.L.frw_event_record(self.h, which))

    def elapsed_ms(self):
        ms = C.c_float()
        self._check(self.L.frw_event_elapsed_ms(self.h, C.byref(ms)))
        return ms.value

    # -- walk engine -------------------------------------------------------
    def upload_structure(self, cond_id, cond_box, diel_box, diel_eps, background_eps, world):
        keep = (np.ascontiguousarray(cond_id, np.int32),
                np.ascontiguousarray(cond_box, np.float64).reshape(-1, 6),
                np.ascontiguousarray(diel_box, np.float64).reshape(-1, 6),
                np.ascontiguousarray(diel_eps, np.float64))
        d = StructureDesc(len(keep[0]), keep[0].ctypes.data_as(_ip),
                          keep[1].ctypes.data_as(_dp), len(keep[3]),
                          keep[2].ctypes.data_as(_dp), keep[3].ctypes.data_as(_dp),
                          float(background_eps), (C.c_double * 6)(*[float(x) for x in world]))
        self._check(self.L.frw_upload_structure(self.h, C.byref(d)))
        self.n_slots_out = len(keep[0]) + 1

    def structure_transits(self, n, cubes, states, with_conductors=False, step_cap=0):
        """frw_structure_transits: one lazy (or expanded) transit per cube
        ([count][4] centre, half width) continuing raw SplitMix64 states."""
        cubes = np.ascontiguousarray(cubes, np.float64).reshape(-1, 4)
        states = np.ascontiguousarray(states, np.uint64)
        out = (Exit * len(states))()
        self._check(self.L.frw_structure_transits(self.h, n, len(states), cubes.ctypes.data_as(_dp),
                                                  int(with_conductors),
                                                  states.ctypes.data_as(_up), step_cap, out))
        a = np.frombuffer(out, dtype=np.dtype([("kind", "<i4"), ("panel", "<i4"),
                                               ("conductor", "<i4"), ("dir", "<i4"),
                                               ("voxel", "<i4", 3), ("steps", "<i4"),
                                               ("point", "<f8", 3)]), count=len(states))
        return {k: a[k].copy() for k in a.dtype.names}

    def structure_transits_philox(self, n, cubes, seed, jumps=True, with_conductors=False,
                                  step_cap=0):
        """frw_structure_transits_philox: production-mode transits of the
        cubes (transit t keyed by Philox (seed, t)), lattice jumps on/off."""
        cubes = np.ascontiguousarray(cubes, np.float64).reshape(-1, 4)
        count = len(cubes)
        out = (Exit * count)()
        self._check(self.L.frw_structure_transits_philox(
            self.h, n, count, cubes.ctypes.data_as(_dp), int(with_conductors), int(seed),
            int(bool(jumps)), step_cap, out))
        a = np.frombuffer(out, dtype=np.dtype([("kind", "<i4"), ("panel", "<i4"),
                                               ("conductor", "<i4"), ("dir", "<i4"),
                                               ("voxel", "<i4", 3), ("steps", "<i4"),
                                               ("point", "<f8", 3)]), count=count)
        return {k: a[k].copy() for k in a.dtype.names}

    def geometry_queries(self, points, tol):
        """frw_geometry_queries: Structure::conductor_at / max_free_cube /
        permittivity_at and the engine's hop prologue, per point"""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        k = len(pts)
        out = dict(conductor_at=np.empty(k, np.int32), free_half_width=np.empty(k),
                   eps=np.empty(k), hop_code=np.empty(k, np.int32), hop_half_width=np.empty(k))
        self._check(self.L.frw_geometry_queries(
            self.h, k, _p(pts), float(tol), _p(out["conductor_at"]), _p(out["free_half_width"]),
            _p(out["eps"]), _p(out["hop_code"]), _p(out["hop_half_width"])))
        return out

    def stratified_keys(self, n, cubes):
        """frw_stratified_keys: (key axis or -1, rounded layers) per cube"""
        cb = np.ascontiguousarray(cubes, np.float64).reshape(-1, 4)
        axis = np.empty(len(cb), np.int32)
        layers = np.empty((len(cb), n))
        self._check(self.L.frw_stratified_keys(self.h, n, len(cb), _p(cb), _p(axis), _p(layers)))
        return axis, layers

    def sgf_put(self, n, axis, layers, pitch, probs, cdf, kernels=None):
        layers = np.ascontiguousarray(layers, np.float64)
        probs = np.ascontiguousarray(probs, np.float64)
        cdf = np.ascontiguousarray(cdf, np.float64)
        k = None if kernels is None else np.ascontiguousarray(kernels, np.float64)
        self._check(self.L.frw_sgf_put(self.h, n, axis, layers.ctypes.data_as(_dp), float(pitch),
                                       probs.ctypes.data_as(_dp), cdf.ctypes.data_as(_dp),
                                       None if k is None else k.ctypes.data_as(_dp)))

    def sgf_solve(self, n, axes, layers, kernels=True):
        """Device miss solver: canonical SGFs of `len(axes)` keys."""
        axes = np.ascontiguousarray(axes, np.int32)
        layers = np.ascontiguousarray(layers, np.float64).reshape(len(axes), n)
        P = 6 * n * n
        probs = np.empty((len(axes), P))
        ker = np.empty((len(axes), 3, P)) if kernels else None
        self._check(self.L.frw_sgf_solve(self.h, n, len(axes), axes.ctypes.data_as(C.POINTER(C.c_int)),
                                         layers.ctypes.data_as(_dp), probs.ctypes.data_as(_dp),
                                         None if ker is None else ker.ctypes.data_as(_dp)))
        return probs, ker

    def grid_sgf_solve(self, eps, half_width=None, kernels=True):
        """frw_grid_sgf_solve of one or more unmasked grids ([count][n^3]):
        probs [count][6n^2], kernels [count][3][6n^2], E[tau] [count]."""
        eps = np.ascontiguousarray(eps, np.float64)
        eps2 = eps.reshape(-1, eps.shape[-1]) if eps.ndim > 1 else eps[None, :]
        n = int(round(eps2.shape[1] ** (1 / 3)))
        cnt = eps2.shape[0]
        hw = n / 2.0 if half_width is None else float(half_width)
        P = 6 * n * n
        probs = np.empty((cnt, P))
        ker = np.empty((cnt, 3, P)) if kernels else None
        steps = np.empty(cnt)
        self._check(self.L.frw_grid_sgf_solve(self.h, n, cnt, eps2.ctypes.data_as(_dp), hw,
                                              probs.ctypes.data_as(_dp),
                                              None if ker is None else ker.ctypes.data_as(_dp),
                                              steps.ctypes.data_as(_dp)))
        return probs, ker, steps

    def sgf_count(self):
        c = C.c_int()
        self._check(self.L.frw_sgf_count(self.h, C.byref(c)))
        return c.value

    def sgf_clear(self):
        self._check(self.L.frw_sgf_clear(self.h))

    def run_walks(self, params: WalkParams, master, walk_begin, count, solver, records=True):
        """frw_run_walks; `solver(n, axis, layers) -> (pitch, probs, cdf, kernels)` fills
        table misses.  Returns (tally dict, records array or None)."""
        nsl = self.n_slots_out
        s1, s2 = np.zeros(nsl), np.zeros(nsl)
        land = np.zeros(nsl, np.uint64)
        t = Tally(s1.ctypes.data_as(_dp), s2.ctypes.data_as(_dp), land.ctypes.data_as(_up))
        rec = np.zeros(count, WALK_RECORD) if records else None
        errors = []

        def cb(user, n, cnt, axes, layers):
            try:
                for q in range(cnt):
                    lay = np.ctypeslib.as_array(layers, shape=(cnt * n,))[q * n:(q + 1) * n].copy()
                    pitch, probs, cdf, ker = solver(n, int(axes[q]), lay)
                    self.sgf_put(n, int(axes[q]), lay, pitch, probs, cdf, ker)
                return 0
            except Exception as e:  # pragma: no cover - surfaced below
                errors.append(e)
                return 1

        fn = MISS_FN(cb) if solver is not None else MISS_FN()  # NULL: device solves
        rc = self.L.frw_run_walks(self.h, C.byref(params), master, walk_begin, count, fn, None,
                                  C.byref(t), None if rec is None else rec.ctypes.data_as(C.c_void_p))
        if errors:
            raise errors[0]
        self._check(rc)
        tally = dict(sum=s1, sumsq=s2, landed=land, aborted=t.aborted, resampled=t.resampled,
                     first=list(t.first), sub=list(t.sub), misses=t.cache_misses,
                     mw_steps=t.mw_steps, restarts=t.restarts, mw_ms=t.mw_ms,
                     mw_general_steps=t.mw_general_steps, mw_cell_changes=t.mw_cell_changes,
                     total_ms=t.total_ms, mw_jumps=t.mw_jumps,
                     mw_jump_steps=t.mw_jump_steps, mw_dense_hops=t.mw_dense_hops)
        return tally, rec

    def smem_bandwidth(self, iters=4096):
        out = C.c_double()
        self._check(self.L.frw_smem_bandwidth_probe(self.h, iters, C.byref(out)))
        return out.value
