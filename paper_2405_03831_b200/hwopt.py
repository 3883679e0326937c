"""Per-pair hardware-setup optimization (mirrors ``cosched.hwopt``, hwopt.py:1-87).

For a trained network the three entry points run the fused GPU sweep on the
single pair (a 2-job ``sweep_pairs``); results carry the reference's exact
semantics: first-minimum argmin in enumeration order, co-run wins ties,
``ValidationError`` on an empty co-run space or an unreachable budget, and
``clamp_stats`` advanced by the number of floored predictions the reference
would have made.  Any other ``predict_slowdown`` plugin is scanned by calling
it, as the reference does.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import estimator
from .core import (ConfigSpace, HardwareConfig, JobProfile, JobSet, ValidationError,
                   enumerate_corun_configs, solo_config)


@dataclass(frozen=True)
class PairDecision:
    """Best co-run setup, best solo splits, and which dispatch mode wins."""

    corun_config: HardwareConfig
    corun_time_s: float
    solo_configs: tuple
    solo_time_s: float
    corun_chosen: bool

    def __post_init__(self) -> None:
        if self.corun_chosen != (self.corun_time_s <= self.solo_time_s):
            raise ValidationError("corun_chosen must reflect corun_time <= solo_time")

    @property
    def winning_time(self) -> float:
        return self.corun_time_s if self.corun_chosen else self.solo_time_s


def _gpu_pair(weights, j1: JobProfile, j2: JobProfile, space: ConfigSpace,
              corun: bool = True, solo: bool = True):
    from .sweep import sweep_pairs
    return sweep_pairs(weights, (j1, j2), space, with_matrix=False, need_corun=corun,
                       need_solo=solo)


def _corun_from(res, space: ConfigSpace):
    cp, gp, cc, gc = res.grid.configs[int(res.corun_grid_index[0, 0])]
    return HardwareConfig(cp, gp, cc, gc), float(res.corun_time[0, 0])


def _solo_from(res):
    splits = res.grid.solo_splits[0]
    s1, s2 = (splits[int(k)] for k in res.solo_split[0, :2])
    return solo_config(*s1), solo_config(*s2), float(res.solo_pair_time(0, 0, 1))


def optimize_corun(model, j1: JobProfile, j2: JobProfile, space: ConfigSpace):
    """Fastest co-run config for the pair and its CoRunTime (hwopt.py:44-65)."""
    weights = estimator.fnn_weights_of(model)
    if weights is not None:
        res = _gpu_pair(weights, j1, j2, space, solo=False)
        _account(res, corun=True, solo=False)
        return _corun_from(res, space)
    js = JobSet((j1, j2))
    best = None
    for hc in enumerate_corun_configs(space):
        t = estimator.corun_time(model, js, hc, space)
        if best is None or t < best[1]:
            best = (hc, t)
    if best is None:
        raise ValidationError(f"no co-run configs exist for p_total {space.p_total}")
    return best


def optimize_solo_pair(model, j1: JobProfile, j2: JobProfile, space: ConfigSpace):
    """Each job's best exclusive split and the time-sharing total (hwopt.py:68-74)."""
    weights = estimator.fnn_weights_of(model)
    if weights is not None:
        res = _gpu_pair(weights, j1, j2, space, corun=False)
        _account(res, corun=False, solo=True)
        return _solo_from(res)
    total, splits = estimator.solorun_time(model, JobSet((j1, j2)), space)
    return solo_config(*splits[0]), solo_config(*splits[1]), total


def decide_pair(model, j1: JobProfile, j2: JobProfile, space: ConfigSpace) -> PairDecision:
    """Both optimizations, co-run chosen on <= (hwopt.py:77-87)."""
    weights = estimator.fnn_weights_of(model)
    if weights is not None:
        res = _gpu_pair(weights, j1, j2, space)
        _account(res, corun=True, solo=True)
        hc, t = _corun_from(res, space)
        s1, s2, st = _solo_from(res)
        return PairDecision(hc, t, (s1, s2), st, bool(res.corun_chosen[0, 0]))
    hc, t = optimize_corun(model, j1, j2, space)
    s1, s2, st = optimize_solo_pair(model, j1, j2, space)
    return PairDecision(hc, t, (s1, s2), st, t <= st)


def _account(res, corun: bool, solo: bool) -> None:
    """Advance clamp_stats as the reference's scalar calls would have."""
    solo_part = int(res.solo_clamps[0, 0] + res.solo_clamps[0, 1])
    total = int(res.clamps[0])
    if corun and solo:
        estimator.clamp_stats.count += total
    elif solo:
        estimator.clamp_stats.count += solo_part
    else:
        estimator.clamp_stats.count += total - solo_part
