"""ctypes wrapper of the CPU oracle (cosched_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
Inputs are plain numpy arrays; the knob grid is given as the arrays of a
``KnobGrid`` (or any object with the same attributes).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
HD, IN, NF = 18, 40, 18

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_up = ctypes.POINTER(ctypes.c_uint32)
_u8 = ctypes.POINTER(ctypes.c_uint8)
_lp = ctypes.POINTER(ctypes.c_int64)


class OrcNet(ctypes.Structure):
    _fields_ = [("w1", ctypes.c_double * (HD * IN)), ("b1", ctypes.c_double * HD),
                ("w2", ctypes.c_double * (HD * HD)), ("b2", ctypes.c_double * HD),
                ("wo", ctypes.c_double * HD), ("bo", ctypes.c_double),
                ("bounds", ctypes.c_double * (2 * NF))]


class OrcDecision(ctypes.Structure):
    _fields_ = [("corun_index", ctypes.c_int32), ("corun_time", ctypes.c_double),
                ("solo_split", ctypes.c_int32 * 2), ("solo_time", ctypes.c_double),
                ("corun_chosen", ctypes.c_int32), ("weight", ctypes.c_double),
                ("margin", ctypes.c_double)]


def _has_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    return " fma " in line + " "
    except OSError:
        pass
    return False


_LIB = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        name = "libcosched_oracle_fma.so" if _has_fma() else "libcosched_oracle.so"
        path = os.path.join(HERE, name)
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.orc_predict.restype = ctypes.c_double
        L.orc_predict.argtypes = [ctypes.POINTER(OrcNet), _dp, _dp, _dp]
        L.orc_decide_pair.restype = ctypes.c_int
        L.orc_decide_pair.argtypes = [ctypes.POINTER(OrcNet), _dp, ctypes.c_double, _dp,
                                      ctypes.c_double, _dp, _dp, ctypes.c_int, _dp, ctypes.c_int,
                                      ctypes.POINTER(OrcDecision), _lp]
        L.orc_app_tables.restype = None
        L.orc_solo.restype = ctypes.c_int64
        L.orc_solo.argtypes = [ctypes.POINTER(OrcNet), _dp, _dp, ctypes.c_int, _dp, _ip,
                               ctypes.c_int, _dp, _ip]
        L.orc_app_tables.argtypes = [ctypes.POINTER(OrcNet), _dp, ctypes.c_int, _dp, _dp]
        L.orc_sweep.restype = ctypes.c_int
        L.orc_sweep.argtypes = [ctypes.POINTER(OrcNet), _dp, _dp, ctypes.c_int, _dp, _dp, _up,
                                ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int, _ip, _dp, _u8, _dp, _dp, _lp]
        _LIB = L
    return _LIB


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def net_of(weights) -> OrcNet:
    """OrcNet from anything with w1/b1/w2/b2/w_out/b_out/feature_bounds arrays."""
    n = OrcNet()
    n.w1[:] = np.asarray(weights.w1, dtype=float).ravel().tolist()
    n.b1[:] = np.asarray(weights.b1, dtype=float).ravel().tolist()
    n.w2[:] = np.asarray(weights.w2, dtype=float).ravel().tolist()
    n.b2[:] = np.asarray(weights.b2, dtype=float).ravel().tolist()
    n.wo[:] = np.asarray(weights.w_out, dtype=float).ravel().tolist()
    n.bo = float(np.asarray(weights.b_out, dtype=float).ravel()[0])
    n.bounds[:] = np.asarray(weights.feature_bounds, dtype=float).ravel().tolist()
    return n


def predict(weights, f1, co, knob) -> float:
    """FnnSlowdownModel.predict_slowdown, unfloored, direct (unfactored) form."""
    net = net_of(weights)
    f1 = np.ascontiguousarray(f1, dtype=float)
    knob = np.ascontiguousarray(knob, dtype=float)
    cop = None if co is None else _p(np.ascontiguousarray(co, dtype=float))
    return lib().orc_predict(ctypes.byref(net), _p(f1), cop, _p(knob))


def decide_pair(weights, fi, ti, fj, tj, knob1, knob2, solo_knob) -> dict:
    """Direct-form hwopt.decide_pair for one budget; knob arrays (C, 4) / (S, 4)."""
    net = net_of(weights)
    k1 = np.ascontiguousarray(knob1, dtype=float)
    k2 = np.ascontiguousarray(knob2, dtype=float)
    sk = np.ascontiguousarray(solo_knob, dtype=float)
    fi = np.ascontiguousarray(fi, dtype=float)
    fj = np.ascontiguousarray(fj, dtype=float)
    out = OrcDecision()
    clamps = ctypes.c_int64(0)
    rc = lib().orc_decide_pair(ctypes.byref(net), _p(fi), float(ti), _p(fj), float(tj), _p(k1),
                               _p(k2), len(k1), _p(sk), len(sk), ctypes.byref(out),
                               ctypes.byref(clamps))
    if rc:
        raise ValueError(f"orc_decide_pair failed ({rc})")
    return {"corun_index": out.corun_index, "corun_time": out.corun_time,
            "solo_split": (out.solo_split[0], out.solo_split[1]), "solo_time": out.solo_time,
            "corun_chosen": bool(out.corun_chosen), "weight": out.weight, "margin": out.margin,
            "clamps": clamps.value}


def sweep(weights, features, base_time, grid, pair_begin=0, pair_end=None, threads=None) -> dict:
    """Factored fp64 sweep (all budgets of `grid`) over pairs [pair_begin, pair_end)."""
    net = net_of(weights)
    F = np.ascontiguousarray(features, dtype=float)
    T = np.ascontiguousarray(base_time, dtype=float)
    n = F.shape[0]
    P_all = n * (n - 1) // 2
    pair_end = P_all if pair_end is None else pair_end
    P = pair_end - pair_begin
    L = grid.n_budgets
    A = np.empty((n, HD)); B = np.empty((n, HD))
    lib().orc_app_tables(ctypes.byref(net), _p(F), n, _p(A), _p(B))
    solo_off = np.ascontiguousarray(grid.solo_offsets, dtype=np.int32)
    sk = np.ascontiguousarray(grid.solo_knob if len(grid.solo_knob) else np.zeros((1, 4)))
    solo_time = np.empty((L, n)); solo_split = np.empty((L, n), dtype=np.int32)
    solo_clamps_one = lib().orc_solo(ctypes.byref(net), _p(A), _p(T), n, _p(sk),
                                     _p(solo_off, _ip), L, _p(solo_time), _p(solo_split, _ip))
    idx = np.empty((L, max(P, 1)), dtype=np.int32)
    ct = np.empty((L, max(P, 1))); w = np.empty((L, max(P, 1))); mg = np.empty((L, max(P, 1)))
    ch = np.empty((L, max(P, 1)), dtype=np.uint8)
    clamps = np.zeros(L, dtype=np.int64)
    k1 = np.ascontiguousarray(grid.knob1 if grid.n_grid else np.zeros((1, 4)))
    k2 = np.ascontiguousarray(grid.knob2 if grid.n_grid else np.zeros((1, 4)))
    mask = np.ascontiguousarray(grid.mask if grid.n_grid else np.zeros(1, dtype=np.uint32))
    threads = threads or os.cpu_count() or 1
    rc = lib().orc_sweep(ctypes.byref(net), _p(F), _p(T), n, _p(k1), _p(k2), _p(mask, _up),
                         grid.n_grid, L, _p(solo_time), pair_begin, pair_end, threads,
                         _p(idx, _ip), _p(ct), _p(ch, _u8), _p(w), _p(mg), _p(clamps, _lp))
    if rc:
        raise ValueError(f"orc_sweep failed ({rc})")
    return {"corun_grid_index": idx[:, :P], "corun_time": ct[:, :P],
            "corun_chosen": ch[:, :P].astype(bool), "weight": w[:, :P], "margin": mg[:, :P],
            "solo_time": solo_time, "solo_split": solo_split, "corun_clamps": clamps,
            "solo_clamps_one_pass": solo_clamps_one, "A": A, "B": B}
