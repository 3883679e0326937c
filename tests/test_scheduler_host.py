"""Scheduler/optimizer semantics on the plugin path (duck-typed models, host only).

A ``predict_slowdown`` object that is not the trained network is a caller
plugin; the package calls it exactly as the reference does (the FNN sweep is
the GPU path, tested in test_*_gpu.py).  These restate the reference's KATs
(test_hwopt.py:62-138, test_scheduler.py:49-70) against this package.
"""

import numpy as np
import pytest

import paper_2405_03831_b200 as cs
from paper_2405_03831_b200 import core, estimator
from paper_2405_03831_b200.scheduler import PairDecisions, pair_index


class Flat:
    def predict_slowdown(self, primary, co_job, hc, space):
        return 1.0


class Analytic:
    """Deterministic toy: slowdown grows with the co-runner's counters, falls with share."""

    def predict_slowdown(self, primary, co_job, hc, space):
        share = hc.cpu_partition[0] / 32 + hc.gpu_partition[0] / 8
        inter = 0.0 if co_job is None else 0.002 * float(np.sum(co_job.features[:4]))
        cap = (250 - hc.cpu_cap) / 500 + (250 - hc.gpu_cap) / 500
        return 1.0 + inter + cap + (2.0 - share) * 0.3 * primary.features[0] / 100


def _jobs(n):
    return [s.job for s in cs.generate_workload(0, cs.mixed_archetypes(n))]


def test_ties_take_first_config_and_corun():
    j = _jobs(2)
    hc, t = cs.optimize_corun(Flat(), j[0], j[1], core.default_space())
    assert hc == core.enumerate_corun_configs(core.default_space())[0]
    d = cs.decide_pair(Flat(), j[0], j[1], core.default_space())
    assert d.corun_chosen == (d.corun_time_s <= d.solo_time_s)


def test_graph_threaded_equals_serial_and_decisions():
    jobs = _jobs(6)
    inp = cs.SchedulerInput(tuple(jobs), core.default_space(), core.SchedulingParams(6), Analytic())
    g1 = cs.build_graph(inp, jobs=1)
    g4 = cs.build_graph(inp, jobs=4)
    assert np.array_equal(g1.weights, g4.weights)
    assert len(g1.decisions) == 15 and list(g1.decisions) == list(g4.decisions)
    for (i, j), d in g1.decisions.items():
        assert g1.weights[i, j] == d.winning_time == cs.decide_pair(
            Analytic(), jobs[i], jobs[j], core.default_space()).winning_time
    s = cs.schedule(inp)
    s.validate_against(jobs, core.default_space())


def test_unknown_model_rejected():
    with pytest.raises(core.ValidationError, match="not a slowdown model"):
        estimator.as_model(object())


def test_floor_counts_clamps():
    class Zero:
        def predict_slowdown(self, *a):
            return 0.1
    estimator.clamp_stats.reset()
    j = _jobs(1)[0]
    t = estimator.solo_app_time(Zero(), j, 200, 200, core.default_space())
    assert t == 0.5 * j.base_time and estimator.clamp_stats.count == 1


def test_lazy_decisions_view(weights):
    """PairDecisions over a SweepResult-shaped object (filled by the oracle here)."""
    import oracle
    from paper_2405_03831_b200.grid import KnobGrid
    from paper_2405_03831_b200.sweep import SweepResult
    n = 10
    F, T = cs.synth.workload_arrays(0, cs.mixed_archetypes(n))
    grid = KnobGrid([core.default_space(400.0)])
    r = oracle.sweep(weights, F, T, grid)
    res = SweepResult(n=n, grid=grid, pair_begin=0, pair_end=45,
                      corun_grid_index=r["corun_grid_index"], corun_time=r["corun_time"],
                      corun_chosen=r["corun_chosen"], weight=r["weight"],
                      solo_time=r["solo_time"], solo_split=r["solo_split"],
                      solo_clamps=np.zeros((1, n), np.int32), clamps=np.zeros(1, np.int64),
                      queue_len=0, screen_error=0.0)
    dec = PairDecisions(res)
    assert len(dec) == 45 and (3, 7) in dec and (7, 3) not in dec and (2, 2) not in dec
    keys = list(dec.keys())
    assert keys[0] == (0, 1) and keys[-1] == (8, 9)
    d = dec[(3, 7)]
    p = pair_index(n, 3, 7)
    assert d.winning_time == r["weight"][0, p]
    assert d.corun_config == core.HardwareConfig(*grid.configs[r["corun_grid_index"][0, p]])
    with pytest.raises(KeyError):
        dec[(7, 3)]
