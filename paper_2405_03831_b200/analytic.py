"""The analytic slowdown oracle as a model the GPU sweep serves.

The reference's ``simenv`` oracle (``pkg/src/cosched/simenv.py:62-233``) is
the model behind every exact-estimate optimality test of the reference
(``test_acceptance.py:185-250``).  Through the plugin protocol it is called
one scalar ``predict_slowdown`` at a time, like any duck-typed model; here it
is recognized (this module's ``OracleSlowdownModel`` or the reference's own,
by class name and ``params`` fields) and ``scheduler.build_graph`` runs it as
one GPU sweep (``cs_analytic_sweep``).

The oracle factors exactly:

    slowdown(self | other, hc) = (resource(self, hc) * power(self, hc)) * contention(self, other)

(``simenv.py:182-218``, left to right as Python evaluates it), so the host
builds, per app and config, the product ``resource * power`` for the member-1
view and for the reversed-partition member-2 view (numpy, no FMA: the same
IEEE operations as the reference), and the kernel multiplies by the pair's
contention, floors at 0.5, scales by the base time and reduces -- in fp64
without contraction, bit-identical to the reference.

The scalar functions below restate simenv.py line by line (file:line cited)
for callers that query single slowdowns; they are not used by the sweep.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields
from typing import Optional, Sequence

import numpy as np

from .core import (CPU_CAP_MAX, GPU_CAP_MAX, TOTAL_CORES, TOTAL_GPCS, ConfigSpace, JobProfile,
                   ValidationError)

_IPC_SCALE = 4.0      # simenv.py:58
_PCT_SCALE = 100.0    # simenv.py:59


@dataclass(frozen=True)
class OracleParams:
    """Coefficients of the analytic oracle (simenv.py:62-131, same defaults)."""

    cpu_scaling: float = 0.35
    gpu_scaling: float = 0.40
    cpu_mem_scaling: float = 0.55
    gpu_mem_scaling: float = 1.05
    cpu_threshold_floor: float = 100.0
    cpu_threshold_span: float = 150.0
    gpu_threshold_floor: float = 150.0
    gpu_threshold_span: float = 100.0
    cpu_power_penalty: float = 0.45
    gpu_power_penalty: float = 0.45
    compute_compute: float = 0.15
    memory_memory: float = 0.30
    compute_memory: float = 0.05
    noise_sigma: float = 0.03
    seed: int = 0

    def __post_init__(self) -> None:
        if min(self.cpu_scaling, self.gpu_scaling, self.cpu_mem_scaling, self.gpu_mem_scaling) < 0:
            raise ValidationError("scaling exponents must be >= 0")
        if self.noise_sigma < 0:
            raise ValidationError("noise_sigma must be >= 0")
        if not (0 < self.cpu_threshold_floor
                and self.cpu_threshold_floor + self.cpu_threshold_span <= CPU_CAP_MAX):
            raise ValidationError("CPU sensitivity thresholds must stay within the cap grid")
        if not (0 < self.gpu_threshold_floor
                and self.gpu_threshold_floor + self.gpu_threshold_span <= GPU_CAP_MAX):
            raise ValidationError("GPU sensitivity thresholds must stay within the cap grid")

    def to_json(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_json(cls, data: dict) -> "OracleParams":
        return cls(**data)


_PARAM_NAMES = tuple(f.name for f in fields(OracleParams))


def _intensity_arrays(features: np.ndarray) -> dict:
    """job_intensities (simenv.py:154-168) for a (N, 18) feature matrix."""
    f = np.asarray(features, dtype=np.float64)

    def frac(col, scale):
        return np.clip(f[:, col] / scale, 0.0, 1.0)

    cpu_dep = frac(0, _PCT_SCALE)
    gpu_dep = frac(14, _PCT_SCALE)
    cpu_mem = (frac(4, _PCT_SCALE) + frac(6, _PCT_SCALE)) / 2.0
    gpu_mem = (frac(11, _PCT_SCALE) + frac(13, _PCT_SCALE)) / 2.0
    compute = (frac(3, _IPC_SCALE) + frac(14, _PCT_SCALE)) / 2.0
    memory = (cpu_mem + gpu_mem) / 2.0                       # JobIntensities.memory
    return dict(cpu_dep=cpu_dep, gpu_dep=gpu_dep, cpu_mem=cpu_mem, gpu_mem=gpu_mem,
                compute=compute, memory=memory)


def _resource_power(p, I: dict, cores, gpcs, ccap, gcap) -> np.ndarray:
    """resource * power of simenv.oracle_slowdown (simenv.py:202-216), broadcast
    over apps (axis 0) and configs (axis 1), in the reference's operation order."""
    cpu_dep, gpu_dep = I["cpu_dep"][:, None], I["gpu_dep"][:, None]
    cpu_slope = p.cpu_scaling * cpu_dep + p.cpu_mem_scaling * I["cpu_mem"][:, None]
    gpu_slope = p.gpu_scaling * gpu_dep + p.gpu_mem_scaling * I["gpu_mem"][:, None]
    resource = ((1.0 + cpu_slope * (1.0 - cores / TOTAL_CORES))
                * (1.0 + gpu_slope * (1.0 - gpcs / TOTAL_GPCS)))
    cpu_thr = p.cpu_threshold_floor + p.cpu_threshold_span * cpu_dep
    gpu_thr = p.gpu_threshold_floor + p.gpu_threshold_span * gpu_dep
    power = ((1.0 + p.cpu_power_penalty * np.maximum(0.0, cpu_thr - ccap) / p.cpu_threshold_span)
             * (1.0 + p.gpu_power_penalty * np.maximum(0.0, gpu_thr - gcap) / p.gpu_threshold_span))
    return resource * power


def oracle_slowdown(params, j1: JobProfile, j2: Optional[JobProfile], hc) -> float:
    """Scalar restatement of simenv.oracle_slowdown (simenv.py:182-218)."""
    if j2 is None and not hc.is_solo:
        raise ValidationError("solo oracle query requires solo partitions")
    if j2 is not None and not hc.is_corun:
        raise ValidationError("co-run oracle query requires co-run partitions")
    I = _intensity_arrays(np.asarray(j1.features)[None, :])
    rp = _resource_power(params, I, np.array([[hc.cpu_partition[0]]]),
                         np.array([[hc.gpu_partition[0]]]), np.array([[float(hc.cpu_cap)]]),
                         np.array([[float(hc.gpu_cap)]]))[0, 0]
    contention = 1.0 if j2 is None else float(_contention(params, I, _intensity_arrays(
        np.asarray(j2.features)[None, :]))[0])
    return float(rp) * contention


def _contention(p, A: dict, B: dict) -> np.ndarray:
    """interference_factor (simenv.py:171-179) for aligned rows of A (self), B (other)."""
    return 1.0 + (p.compute_compute * A["compute"] * B["compute"]
                  + p.memory_memory * A["memory"] * B["memory"]
                  + p.compute_memory * (A["compute"] * B["memory"] + A["memory"] * B["compute"]))


class OracleSlowdownModel:
    """The analytic oracle behind the plugin protocol (simenv.py:221-233)."""

    def __init__(self, params: OracleParams):
        self.params = params

    def predict_slowdown(self, primary, co_job, hc, space) -> float:
        return oracle_slowdown(self.params, primary, co_job, hc)


def oracle_params_of(model):
    """The params when `model` is the analytic oracle (this module's or the
    reference's ``simenv.OracleSlowdownModel``), else None."""
    if type(model).__name__ != "OracleSlowdownModel":
        return None
    p = getattr(model, "params", None)
    if p is None or not all(hasattr(p, k) for k in _PARAM_NAMES if k not in ("noise_sigma", "seed")):
        return None
    return p


# --------------------------------------------------------------------------
def host_tables(params, features: np.ndarray, grid) -> dict:
    """Config-major products resource*power for both member views, the
    per-app intensities the kernel needs for the contention, and the solo
    results (host, exact)."""
    I = _intensity_arrays(features)
    cfg = grid.configs
    cores1 = np.array([c[0][0] for c in cfg], dtype=np.float64)[None, :]
    cores2 = np.array([c[0][1] for c in cfg], dtype=np.float64)[None, :]
    gpcs1 = np.array([c[1][0] for c in cfg], dtype=np.float64)[None, :]
    gpcs2 = np.array([c[1][1] for c in cfg], dtype=np.float64)[None, :]
    ccap = np.array([float(c[2]) for c in cfg], dtype=np.float64)[None, :]
    gcap = np.array([float(c[3]) for c in cfg], dtype=np.float64)[None, :]
    # integer partitions in the reference: cores / TOTAL_CORES is int / int
    rp1 = _resource_power(params, I, cores1.astype(np.int64), gpcs1.astype(np.int64), ccap, gcap)
    rp2 = _resource_power(params, I, cores2.astype(np.int64), gpcs2.astype(np.int64), ccap, gcap)
    return {"rp1": np.ascontiguousarray(rp1.T), "rp2": np.ascontiguousarray(rp2.T),
            "compute": np.ascontiguousarray(I["compute"]),
            "memory": np.ascontiguousarray(I["memory"])}


def solo_results(params, features: np.ndarray, base_time: np.ndarray, grid):
    """Per (budget, app) best exclusive split (estimator.py:139-180 with the oracle):
    (solo_time (L, N), solo_split (L, N), solo_clamps (L, N))."""
    I = _intensity_arrays(features)
    L, N = grid.n_budgets, len(base_time)
    st = np.full((L, N), np.nan)
    ss = np.full((L, N), -1, dtype=np.int32)
    sc = np.zeros((L, N), dtype=np.int32)
    for l, splits in enumerate(grid.solo_splits):
        if not splits:
            continue
        cc = np.array([[float(c) for c, _ in splits]])
        gc = np.array([[float(g) for _, g in splits]])
        full_c = np.full_like(cc, TOTAL_CORES, dtype=np.int64)
        full_g = np.full_like(gc, TOTAL_GPCS, dtype=np.int64)
        s = _resource_power(params, I, full_c, full_g, cc, gc) * 1.0   # contention 1.0
        clamp = s < 0.5
        t = np.where(clamp, 0.5, s) * base_time[:, None]
        k = np.argmin(t, axis=1)                   # first minimum (estimator.py:175)
        st[l] = t[np.arange(N), k]
        ss[l] = k
        sc[l] = clamp.sum(axis=1)
    return st, ss, sc


def analytic_sweep(params, jobs: Sequence[JobProfile], spaces, with_matrix: bool = True):
    """build_graph's arrays for the analytic oracle, on the GPU (cs_analytic_sweep)."""
    import torch
    from . import _native as nat
    from .device import require_cuda
    from .grid import KnobGrid
    from .sweep import SweepResult
    if isinstance(spaces, ConfigSpace):
        spaces = (spaces,)
    grid = KnobGrid(tuple(spaces))
    grid.check_nonempty()
    feats = np.stack([np.asarray(j.features, dtype=np.float64) for j in jobs])
    bt = np.array([float(j.base_time) for j in jobs], dtype=np.float64)
    n, L, G = len(jobs), grid.n_budgets, grid.n_grid
    P = n * (n - 1) // 2
    tab = host_tables(params, feats, grid)
    st, ss, sc = solo_results(params, feats, bt, grid)
    dev = require_cuda()
    d = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
    d_rp1, d_rp2 = d(tab["rp1"]), d(tab["rp2"])
    d_cmp, d_mem, d_bt, d_st = d(tab["compute"]), d(tab["memory"]), d(bt), d(st)
    d_mask = torch.as_tensor(grid.mask.view(np.int32)).to(dev)
    idx = torch.empty((L, max(P, 1)), dtype=torch.int32, device=dev)
    ct = torch.empty((L, max(P, 1)), dtype=torch.float64, device=dev)
    ch = torch.empty((L, max(P, 1)), dtype=torch.uint8, device=dev)
    wt = torch.empty((L, max(P, 1)), dtype=torch.float64, device=dev)
    W = torch.zeros((L, n, n), dtype=torch.float64, device=dev) if with_matrix else None
    clamps = torch.zeros(L, dtype=torch.int64, device=dev)
    coef = (ctypes.c_double * 3)(params.compute_compute, params.memory_memory,
                                 params.compute_memory)
    out = nat.CsPairOut(ctypes.cast(idx.data_ptr(), nat.c_int32_p),
                        ctypes.cast(ct.data_ptr(), nat.c_double_p),
                        ctypes.cast(ch.data_ptr(), nat.c_uint8_p),
                        ctypes.cast(wt.data_ptr(), nat.c_double_p))
    lib = nat.sweep_lib()
    nat.check(lib.cs_analytic_sweep(
        d_rp1.data_ptr(), d_rp2.data_ptr(), d_cmp.data_ptr(), d_mem.data_ptr(), coef,
        d_bt.data_ptr(), d_st.data_ptr(), d_mask.data_ptr(), n, G, L, out,
        W.data_ptr() if W is not None else None, clamps.data_ptr(),
        torch.cuda.current_stream(dev).cuda_stream), "cs_analytic_sweep")
    torch.cuda.synchronize(dev)
    res = SweepResult(
        n=n, grid=grid, pair_begin=0, pair_end=P,
        corun_grid_index=idx[:, :P].cpu().numpy(), corun_time=ct[:, :P].cpu().numpy(),
        corun_chosen=ch[:, :P].cpu().numpy().astype(bool), weight=wt[:, :P].cpu().numpy(),
        solo_time=st, solo_split=ss, solo_clamps=sc,
        clamps=clamps.cpu().numpy().astype(np.int64) + (n - 1) * sc.sum(axis=1),
        queue_len=0, screen_error=0.0,
        matrix=W.cpu().numpy() if W is not None else None)
    return res
