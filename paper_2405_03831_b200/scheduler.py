"""End-to-end scheduling of a job queue (mirrors ``cosched.scheduler``).

``build_graph`` (scheduler.py:52-78) is the hot path's driver.  For a trained
network it is ONE fused GPU sweep over all N(N-1)/2 pairs (``sweep_pairs``):
the symmetric weight matrix is scattered on the device and the per-edge
``PairDecision``s are built lazily from the result arrays on access
(``PairDecisions``), so the 8.4M-pair case never materializes Python objects
it does not need.  ``schedule`` (81-107) matches on the host (native blossom)
and emits job sets exactly as the reference does.
"""

from __future__ import annotations

import json
from collections.abc import Mapping
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import analytic, estimator
from .core import (ConfigSpace, HardwareConfig, JobSet, Schedule, SchedulingParams, ValidationError,
                   normalize_input, solo_config)
from .fnn import forward_batch
from .hwopt import PairDecision, decide_pair
from .matcher import PairGraph, min_weight_perfect_matching


@dataclass(frozen=True)
class SchedulerInput:
    """Queued jobs, knob space, window parameters and the model (scheduler.py:32-49)."""

    queue: tuple
    space: ConfigSpace
    params: SchedulingParams
    model: object

    def __post_init__(self) -> None:
        queue = tuple(self.queue)
        if not queue:
            raise ValidationError("queue must not be empty")
        if len(queue) != self.params.window:
            raise ValidationError(
                f"queue length {len(queue)} must equal the window {self.params.window}")
        object.__setattr__(self, "queue", queue)


def pair_index(n: int, i: int, j: int) -> int:
    """Row-major linear index of the unordered pair i < j (scheduler.py:61)."""
    return i * (2 * n - i - 1) // 2 + (j - i - 1)


class PairDecisions(Mapping):
    """Lazy ``{(i, j): PairDecision}`` view over one budget of a SweepResult."""

    def __init__(self, result, budget: int = 0):
        self._r = result
        self._l = budget
        self._n = result.n
        self._splits = result.grid.solo_splits[budget]
        self._cfg_cache: dict = {}

    def __len__(self) -> int:
        return self._n * (self._n - 1) // 2

    def corun_flags(self) -> np.ndarray:
        """corun_chosen of every pair, row-major i < j (no PairDecision objects)."""
        return np.asarray(self._r.corun_chosen[self._l], dtype=bool)

    def potentials(self) -> np.ndarray:
        """Per-app best solo times: every pair weight is min(co-run, solo_i +
        solo_j) <= pot_i + pot_j, which the native matcher uses to solve the
        benefit form of the matching (cm_min_weight_perfect_matching_pot)."""
        return np.ascontiguousarray(self._r.solo_time[self._l], dtype=np.float64)

    def __iter__(self):
        n = self._n
        for i in range(n):
            for j in range(i + 1, n):
                yield (i, j)

    def __contains__(self, key) -> bool:
        try:
            i, j = key
        except (TypeError, ValueError):
            return False
        return isinstance(i, (int, np.integer)) and isinstance(j, (int, np.integer)) \
            and 0 <= i < j < self._n

    def _config(self, g: int) -> HardwareConfig:
        hc = self._cfg_cache.get(g)
        if hc is None:
            hc = HardwareConfig(*self._r.grid.configs[g])
            self._cfg_cache[g] = hc
        return hc

    def __getitem__(self, key) -> PairDecision:
        if key not in self:
            raise KeyError(key)
        i, j = int(key[0]), int(key[1])
        r, l = self._r, self._l
        p = pair_index(self._n, i, j) - r.pair_begin
        g = int(r.corun_grid_index[l, p])
        st = r.solo_time[l]
        si, sj = int(r.solo_split[l, i]), int(r.solo_split[l, j])
        return PairDecision(
            corun_config=self._config(g),
            corun_time_s=float(r.corun_time[l, p]),
            solo_configs=(solo_config(*self._splits[si]), solo_config(*self._splits[sj])),
            solo_time_s=float((0.0 + st[i]) + st[j]),
            corun_chosen=bool(r.corun_chosen[l, p]))


def build_graph_gpu(jobs: Sequence, space: ConfigSpace, weights) -> PairGraph:
    """The fused GPU sweep as a PairGraph (lazy decisions); updates clamp_stats."""
    from .sweep import sweep_pairs
    res = sweep_pairs(weights, jobs, space, with_matrix=True)
    estimator.clamp_stats.count += int(res.clamps[0])
    return PairGraph.trusted(res.matrix[0], PairDecisions(res, 0))


def build_graph(inp: SchedulerInput, jobs: int = 1) -> PairGraph:
    """Optimize every unordered pair and assemble the weighted pair graph.

    ``jobs`` keeps the reference's meaning (worker threads) for plugin models;
    a trained network and the analytic oracle (``simenv.OracleSlowdownModel``)
    are one GPU sweep regardless.
    """
    weights = estimator.fnn_weights_of(inp.model)
    if weights is not None:
        return build_graph_gpu(inp.queue, inp.space, weights)
    oracle_params = analytic.oracle_params_of(inp.model)
    if oracle_params is not None:
        # the analytic oracle (simenv.OracleSlowdownModel): one exact GPU sweep
        res = analytic.analytic_sweep(oracle_params, inp.queue, inp.space)
        estimator.clamp_stats.count += int(res.clamps[0])
        return PairGraph.trusted(res.matrix[0], PairDecisions(res, 0))
    n = len(inp.queue)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]

    def edge(pair):
        return decide_pair(inp.model, inp.queue[pair[0]], inp.queue[pair[1]], inp.space)

    if jobs > 1:
        with ThreadPoolExecutor(max_workers=jobs) as pool:
            decisions = list(pool.map(edge, pairs))
    else:
        decisions = [edge(p) for p in pairs]
    w = np.zeros((n, n))
    payload = {}
    for (i, j), d in zip(pairs, decisions):
        w[i, j] = w[j, i] = d.winning_time
        payload[(i, j)] = d
    return PairGraph(w, payload)


def emit_schedule(inp: SchedulerInput, graph: PairGraph, matched) -> Schedule:
    """Job sets from matched pairs; solo-flagged pairs split in edge order (scheduler.py:90-107)."""
    sets, configs, flags = [], [], []
    for i, j in matched:
        d = graph.decisions[(i, j)]
        if d.corun_chosen:
            sets.append(JobSet((inp.queue[i], inp.queue[j])))
            configs.append((d.corun_config,))
            flags.append(True)
        else:
            for k, hc in zip((i, j), d.solo_configs):
                sets.append(JobSet((inp.queue[k],)))
                configs.append((hc,))
                flags.append(False)
    out = Schedule(tuple(sets), tuple(configs), tuple(flags))
    out.validate_against(inp.queue, inp.space)
    return out


def schedule(inp: SchedulerInput, jobs: int = 1) -> Schedule:
    """Dispatch plan for the queue: sweep, match, emit."""
    graph = build_graph(inp, jobs=jobs)
    return emit_schedule(inp, graph, min_weight_perfect_matching(graph))


def set_time(model, js: JobSet, configs: Sequence, corun: bool, space: ConfigSpace) -> float:
    """Predicted dispatch time of one emitted set (scheduler.py:110-116)."""
    if corun:
        return estimator.corun_time(model, js, configs[0], space)
    hc = configs[0]
    return estimator.solo_app_time(model, js.jobs[0], hc.cpu_cap, hc.gpu_cap, space)


def _set_times(sched: Schedule, model, space: ConfigSpace, passes: int = 1) -> list:
    """set_time of every emitted set.  For a trained network all the set's
    slowdown queries (two per co-run set, member 2 on reversed partitions; one
    per solo set) go to the GPU as ONE forward_batch instead of a device round
    trip per query; floors, clamp counting (``passes`` times, as often as the
    reference evaluates each query) and the max / sum are applied on the host
    in the reference's order, so the values equal the scalar path's."""
    weights = estimator.fnn_weights_of(model)
    if weights is None:
        out = [set_time(model, js, cs, fl, space)
               for js, cs, fl in zip(sched.job_sets, sched.configs, sched.corun_flags)]
        for _ in range(passes - 1):
            for js, cs, fl in zip(sched.job_sets, sched.configs, sched.corun_flags):
                set_time(model, js, cs, fl, space)
        return out
    rows, owners = [], []
    for k, (js, cs, fl) in enumerate(zip(sched.job_sets, sched.configs, sched.corun_flags)):
        hc = cs[0]
        if fl:
            if len(js) == 1:
                rows.append(normalize_input(js.jobs[0], None, hc, space, weights.feature_bounds))
                owners.append((k, 0))
            else:
                for m in range(len(js)):
                    view = hc if m == 0 else hc.reversed_partitions()
                    rows.append(normalize_input(js.jobs[m], js.jobs[1 - m], view, space,
                                                weights.feature_bounds))
                    owners.append((k, m))
        else:
            rows.append(normalize_input(js.jobs[0], None, solo_config(hc.cpu_cap, hc.gpu_cap),
                                        space, weights.feature_bounds))
            owners.append((k, 0))
    preds = forward_batch(weights, np.stack(rows)) if rows else np.zeros(0)
    floor = estimator.SLOWDOWN_FLOOR
    estimator.clamp_stats.count += passes * int(np.count_nonzero(preds < floor))
    member_times: dict = {}
    for (k, m), y in zip(owners, preds):
        y = float(y)
        member_times.setdefault(k, []).append((floor if y < floor else y) * sched.job_sets[k].jobs[m].base_time)
    return [max(member_times[k]) for k in range(len(sched.job_sets))]


def predicted_makespan(sched: Schedule, model, space: ConfigSpace) -> float:
    return sum(_set_times(sched, model, space))


def schedule_to_json(sched: Schedule, model, space: ConfigSpace) -> dict:
    times = _set_times(sched, model, space, passes=2)   # set loop + predicted_makespan
    sets = [{"jobs": [job.job_id for job in js.jobs], "corun": bool(fl),
             "configs": [hc.to_json() for hc in cs], "predicted_s": t}
            for js, cs, fl, t in zip(sched.job_sets, sched.configs, sched.corun_flags, times)]
    return {"p_total_w": space.p_total, "sets": sets, "total_predicted_s": sum(times)}


def write_schedule_json(sched: Schedule, model, space: ConfigSpace, path) -> None:
    with open(path, "w") as fh:
        json.dump(schedule_to_json(sched, model, space), fh, indent=2, sort_keys=True)
        fh.write("\n")
