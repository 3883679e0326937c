"""ctypes binding of libcosched_b200.so for the reference package ``cosched``.

Drop this file into ``pkg/src/cosched/`` as ``_b200.py`` (it uses relative
imports of the reference's own modules and needs only numpy + ctypes, the
reference's sole dependency, ``pyproject.toml:9-12``), point
``COSCHED_B200_LIB`` at the built ``libcosched_b200.so``, and route
``scheduler.build_graph`` through ``build_graph_b200`` for trained networks
(INTEGRATION.md shows the three-line patch).  One C call,
``cs_build_graph_host`` (include/cosched_b200.h), replaces the per-pair
Python loop of ``scheduler.build_graph`` (scheduler.py:52-78) over
``hwopt.decide_pair`` (hwopt.py:77-87).

Names used from the reference: ``core.enumerate_corun_configs``
(core.py:380-397), ``core.enumerate_solo_splits`` (core.py:400-407),
``core.solo_config`` (core.py:179-181), ``core.TOTAL_CORES/TOTAL_GPCS/
CPU_CAP_MAX/GPU_CAP_MAX`` (core.py:27-35), ``fnn.NetworkWeights``
(fnn.py:42-68), ``estimator.FnnSlowdownModel`` / ``clamp_stats``
(estimator.py:36-67), ``hwopt.PairDecision`` (hwopt.py:24-41) and
``matcher.PairGraph`` (matcher.py:28-63).  tests/test_integration_gpu.py
loads this very file into the drop-in package (which exports the same names)
and checks it against the oracle.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import core, estimator, fnn, hwopt, matcher

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_up = ctypes.POINTER(ctypes.c_uint32)
_u8 = ctypes.POINTER(ctypes.c_uint8)
_MAXB = 8


class _Net(ctypes.Structure):
    _fields_ = [(k, _dp) for k in ("w1", "b1", "w2", "b2", "w_out", "b_out", "feature_bounds")]


class _Grid(ctypes.Structure):
    _fields_ = [("n_grid", ctypes.c_int32), ("knob1", _dp), ("knob2", _dp), ("mask", _up),
                ("n_budgets", ctypes.c_int32), ("n_configs", ctypes.c_int32 * _MAXB),
                ("solo_offsets", ctypes.c_int32 * (_MAXB + 1)), ("solo_knob", _dp)]


class _PairOut(ctypes.Structure):
    _fields_ = [("corun_grid_index", _ip), ("corun_time", _dp), ("corun_chosen", _u8),
                ("weight", _dp)]


class _SoloOut(ctypes.Structure):
    _fields_ = [("solo_time", _dp), ("solo_split", _ip), ("solo_clamps", _ip)]


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.environ.get("COSCHED_B200_LIB", "libcosched_b200.so")
        lib = ctypes.CDLL(path)
        lib.cs_build_graph_workspace_bytes.restype = ctypes.c_size_t
        lib.cs_build_graph_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.POINTER(_Grid)]
        lib.cs_device_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
        lib.cs_device_free.argtypes = [ctypes.c_void_p]
        lib.cs_error_string.restype = ctypes.c_char_p
        lib.cs_build_graph_host.argtypes = [
            ctypes.POINTER(_Net), ctypes.POINTER(_Grid), _dp, _dp, ctypes.c_int32,
            ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t, _dp, _PairOut, _SoloOut,
            ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_void_p]
        _LIB = lib
    return _LIB


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def _knob(cp, gp, cc, gc):
    # the 4 knob slots of normalize_input (core.py:368-371), primary's view
    return (cp[0] / core.TOTAL_CORES, gp[0] / core.TOTAL_GPCS,
            cc / core.CPU_CAP_MAX, gc / core.GPU_CAP_MAX)


def build_graph_b200(inp, rel_eps: float = 1e-5):
    """scheduler.build_graph for a trained network, in one C call."""
    model = inp.model
    w = model.weights if isinstance(model, estimator.FnnSlowdownModel) else model
    if not isinstance(w, fnn.NetworkWeights):
        raise TypeError("build_graph_b200 serves trained FNN models only")
    space, jobs = inp.space, inp.queue
    n = len(jobs)
    configs = core.enumerate_corun_configs(space)
    splits = core.enumerate_solo_splits(space)
    if not configs:
        raise core.ValidationError(f"no co-run configs exist for p_total {space.p_total}")
    if not splits:
        raise core.ValidationError(f"p_total {space.p_total} is unreachable on the cap grids")
    keep = {k: np.ascontiguousarray(getattr(w, k), dtype=np.float64)
            for k in ("w1", "b1", "w2", "b2", "w_out", "b_out", "feature_bounds")}
    net = _Net(*(_p(keep[k]) for k in ("w1", "b1", "w2", "b2", "w_out", "b_out",
                                       "feature_bounds")))
    k1 = np.array([_knob(h.cpu_partition, h.gpu_partition, h.cpu_cap, h.gpu_cap)
                   for h in configs], dtype=np.float64)
    k2 = np.array([_knob(h.cpu_partition[::-1], h.gpu_partition[::-1], h.cpu_cap, h.gpu_cap)
                   for h in configs], dtype=np.float64)          # reversed_partitions view
    mask = np.ones(len(configs), dtype=np.uint32)
    solo = np.array([(1.0, 1.0, c / core.CPU_CAP_MAX, g / core.GPU_CAP_MAX) for c, g in splits],
                    dtype=np.float64)
    grid = _Grid()
    grid.n_grid, grid.knob1, grid.knob2, grid.mask = len(configs), _p(k1), _p(k2), _p(mask, _up)
    grid.n_budgets = 1
    grid.n_configs[0] = len(configs)
    grid.solo_offsets[0], grid.solo_offsets[1] = 0, len(splits)
    grid.solo_knob = _p(solo)

    F = np.ascontiguousarray([j.features for j in jobs], dtype=np.float64)
    T = np.ascontiguousarray([j.base_time for j in jobs], dtype=np.float64)
    P = n * (n - 1) // 2
    W = np.zeros((n, n))
    idx = np.empty(P, np.int32)
    ct = np.empty(P)
    ch = np.empty(P, np.uint8)
    wt = np.empty(P)
    st = np.empty(n)
    ss = np.empty(n, np.int32)
    clamps = (ctypes.c_ulonglong * 1)()
    lib = _lib()
    nbytes = lib.cs_build_graph_workspace_bytes(n, ctypes.byref(grid))
    ws = ctypes.c_void_p()
    if not nbytes or lib.cs_device_alloc(nbytes, ctypes.byref(ws)):
        raise RuntimeError("cosched_b200: workspace allocation failed")
    try:
        rc = lib.cs_build_graph_host(
            ctypes.byref(net), ctypes.byref(grid), _p(F), _p(T), n, rel_eps, ws, nbytes, _p(W),
            _PairOut(_p(idx, _ip), _p(ct), _p(ch, _u8), _p(wt)),
            _SoloOut(_p(st), _p(ss, _ip), None), clamps, None)
    finally:
        lib.cs_device_free(ws)
    if rc:
        msg = lib.cs_error_string(rc).decode()
        raise (core.ValidationError if rc in (-1, -2, -3) else RuntimeError)(msg)
    estimator.clamp_stats.count += int(clamps[0])

    decisions = {}
    p = 0
    for i in range(n):
        for j in range(i + 1, n):
            decisions[(i, j)] = hwopt.PairDecision(
                corun_config=configs[idx[p]], corun_time_s=float(ct[p]),
                solo_configs=(core.solo_config(*splits[ss[i]]), core.solo_config(*splits[ss[j]])),
                solo_time_s=float((0.0 + st[i]) + st[j]), corun_chosen=bool(ch[p]))
            p += 1
    return matcher.PairGraph(W, decisions)
