"""Batched pair x knob sweep: the entry point behind hwopt/scheduler for FNN models.

``sweep_pairs(weights, jobs, spaces)`` runs the fused GPU pipeline once over
every unordered pair of ``jobs`` (row-major i < j, scheduler.py:61) for up to 8
budgets and returns a ``SweepResult`` of host arrays.  ``hwopt.decide_pair``
is the 2-job special case; ``scheduler.build_graph`` wraps the result in a
``PairGraph`` with a lazy ``decisions`` mapping.
"""

from __future__ import annotations

import os

import threading
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from .core import ConfigSpace, JobProfile, ValidationError
from .device import DEFAULT_REL_EPS, SweepPlan, require_cuda, to_device_inputs
from .grid import KnobGrid

_PLAN_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_PLAN_CACHE_SIZE = 8
_GRID_CACHE: "OrderedDict[tuple, KnobGrid]" = OrderedDict()
_CACHE_LOCK = threading.RLock()     # the two caches are shared by caller threads


def knob_grid(spaces: Sequence[ConfigSpace]) -> KnobGrid:
    key = tuple(spaces)
    with _CACHE_LOCK:
        g = _GRID_CACHE.get(key)
        if g is None:
            g = KnobGrid(key)
            _GRID_CACHE[key] = g
            while len(_GRID_CACHE) > 32:
                _GRID_CACHE.popitem(last=False)
        return g


def plan_for(weights, spaces: Sequence[ConfigSpace], n: int, pair_begin: int = 0,
             pair_end: Optional[int] = None, with_matrix: bool = True,
             rel_eps: float = DEFAULT_REL_EPS, kernel: str = "tcgen05") -> SweepPlan:
    """A cached SweepPlan (buffers are reused across calls of the same shape)."""
    dev = require_cuda()
    key = (id(weights), tuple(spaces), n, pair_begin, pair_end, with_matrix, rel_eps, kernel,
           str(dev), os.environ.get("COSCHED_TC_KIND"))
    with _CACHE_LOCK:
        hit = _PLAN_CACHE.get(key)
        if hit is not None and hit[0] is weights:
            _PLAN_CACHE.move_to_end(key)
            return hit[1]
        plan = SweepPlan(weights, knob_grid(spaces), n, pair_begin, pair_end, dev,
                         with_matrix=with_matrix, rel_eps=rel_eps, kernel=kernel)
        _PLAN_CACHE[key] = (weights, plan)      # holds `weights` so its id stays unique
        while len(_PLAN_CACHE) > _PLAN_CACHE_SIZE:
            _PLAN_CACHE.popitem(last=False)
    return plan


@dataclass
class SweepResult:
    """Host copies of one sweep.  Budget-major arrays: [l, p] / [l, app]."""

    n: int
    grid: KnobGrid
    pair_begin: int
    pair_end: int
    corun_grid_index: np.ndarray     # (L, P) int32, union-grid index of the best config
    corun_time: np.ndarray           # (L, P) float64
    corun_chosen: np.ndarray         # (L, P) bool
    weight: np.ndarray               # (L, P) float64 = winning_time
    solo_time: np.ndarray            # (L, N) float64, best exclusive time per app
    solo_split: np.ndarray           # (L, N) int32, index into grid.solo_splits[l]
    solo_clamps: np.ndarray          # (L, N) int32, floored solo predictions per app
    clamps: np.ndarray               # (L,) floor clamps as the reference would count them
    queue_len: int                   # (pair, budget)s re-scanned exactly in fp64
    screen_error: float              # largest fp32-screen vs fp64 relative gap seen
    exact_rows: int = 0              # rows whose floor clamps were re-counted in fp64
    matrix: Optional[np.ndarray] = field(default=None)   # (L, N, N) symmetric weights

    def corun_local_index(self, l: int) -> np.ndarray:
        """Best config as an index into budget l's own enumerate_corun_configs list."""
        return self.grid.local_index[l][self.corun_grid_index[l]]

    def solo_pair_time(self, l: int, i, j):
        """(0.0 + t_i) + t_j exactly as estimator.solorun_time sums (estimator.py:168-178)."""
        st = self.solo_time[l]
        return (0.0 + st[i]) + st[j]


class _PairWeights:
    """(L, P) winning times read from the symmetric matrix on first use: with
    the matrix on the host, copying the per-pair array as well would move the
    same 8 bytes per pair over PCIe twice."""

    def __init__(self, matrix: np.ndarray, n: int, pair_begin: int, pair_end: int):
        self._m, self._n, self._b, self._e = matrix, n, pair_begin, pair_end
        self._a = None

    def _array(self) -> np.ndarray:
        if self._a is None:
            iu, ju = np.triu_indices(self._n, 1)
            iu, ju = iu[self._b:self._e], ju[self._b:self._e]
            self._a = np.stack([self._m[l][iu, ju] for l in range(self._m.shape[0])])
        return self._a

    def __getitem__(self, k):
        return self._array()[k]

    def __array__(self, dtype=None, copy=None):
        a = self._array()
        return a if dtype is None else a.astype(dtype)

    def __len__(self):
        return self._m.shape[0]

    @property
    def shape(self):
        return (self._m.shape[0], self._e - self._b)


def _d2h(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> a fresh numpy array.  numpy advises huge pages for
    large allocations, so the destination is not faulted in 4 KB at a time
    (torch's .cpu() buffers are: ~2 GB/s for the 134 MB matrix at 4,096 apps)."""
    out = np.empty(tuple(t.shape), dtype=torch.empty((), dtype=t.dtype).numpy().dtype)
    torch.from_numpy(out).copy_(t)
    return out


def _inputs(jobs: Sequence[JobProfile]):
    feats = np.stack([np.asarray(j.features, dtype=np.float64) for j in jobs])
    bt = np.array([float(j.base_time) for j in jobs], dtype=np.float64)
    return feats, bt


def run_plan(plan: SweepPlan, features: np.ndarray, base_time: np.ndarray,
             with_matrix: bool = True) -> SweepResult:
    """One sweep through `plan` and the host copies of its results.  Holds the
    plan's lock from launch to read-back, so threads sharing a cached plan
    (concurrent decide_pair / build_graph calls) never see each other's
    buffers."""
    with plan.lock:
        d_f, d_b = to_device_inputs(features, base_time, plan.device)
        eps = plan.rel_eps
        with torch.cuda.device(plan.device):
            plan.launch(d_f, d_b, rel_eps=eps)
            c = plan.read_counters()            # synchronizes the stream
            # a network far outside the trained range: the fp32 screen's observed
            # error is not well inside rel_eps -- widen the ambiguity band (more
            # pairs go to the exact fp64 resolve; results identical) and redo
            while (c.screen_error > 0.25 * eps or c.verify_fail) and 16.0 * eps < 0.1:
                eps = min(max(16.0 * eps, 16.0 * c.screen_error), 0.099)
                plan.launch(d_f, d_b, rel_eps=eps)
                c = plan.read_counters()
            P = plan.P
            matrix = _d2h(plan.matrix) if (with_matrix and plan.matrix is not None) else None
            res = SweepResult(
                n=plan.n, grid=plan.grid, pair_begin=plan.pair_begin, pair_end=plan.pair_end,
                corun_grid_index=_d2h(plan.corun_grid_index[:, :P]),
                corun_time=_d2h(plan.corun_time[:, :P]),
                corun_chosen=_d2h(plan.corun_chosen[:, :P]).view(bool),
                weight=(_PairWeights(matrix, plan.n, plan.pair_begin, plan.pair_end)
                        if matrix is not None else _d2h(plan.weight[:, :P])),
                solo_time=_d2h(plan.solo_time),
                solo_split=_d2h(plan.solo_split),
                solo_clamps=_d2h(plan.solo_clamps),
                clamps=c.clamps, queue_len=c.queue_len, screen_error=c.screen_error,
                exact_rows=c.exact_rows, matrix=matrix)
    if res.screen_error > 0.25 * eps or c.verify_fail:
        raise RuntimeError(f"fp32 screen error {res.screen_error:.3g} is too close to rel_eps "
                           f"{eps:.3g}; argmin parity is no longer guaranteed")
    return res


def sweep_pairs(weights, jobs: Sequence[JobProfile], spaces, pair_begin: int = 0,
                pair_end: Optional[int] = None, with_matrix: bool = True,
                need_corun: bool = True, need_solo: bool = True,
                kernel: str = "tcgen05") -> SweepResult:
    """Evaluate every (pair, config) of `jobs` for each budget in `spaces` on the GPU.

    Raises the reference's ValidationErrors for an empty co-run space
    (hwopt.py:62-64) / unreachable budget (estimator.py:165-167) when the
    corresponding part of the result is needed."""
    if isinstance(spaces, ConfigSpace):
        spaces = (spaces,)
    jobs = list(jobs)
    if len(jobs) < 2:
        raise ValidationError("a sweep needs at least two jobs")
    knob_grid(tuple(spaces)).check_nonempty(corun=need_corun, solo=need_solo)
    feats, bt = _inputs(jobs)
    plan = plan_for(weights, tuple(spaces), len(jobs), pair_begin, pair_end, with_matrix,
                    kernel=kernel)
    return run_plan(plan, feats, bt, with_matrix)
