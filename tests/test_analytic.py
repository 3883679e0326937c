"""The analytic oracle model (analytic.py) against the
reference's simenv oracle (tests/golden/analytic.json, make_golden.py stage
`analytic`).  CPU: the scalar restatement through the plugin path
(hwopt.decide_pair calls predict_slowdown like the reference).  GPU: the batched
sweep behind scheduler.build_graph, bit-identical."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, pair_index
import paper_2405_03831_b200 as cs
from paper_2405_03831_b200 import analytic, core, estimator, synth

with open(os.path.join(GOLDEN, "analytic.json")) as fh:
    DOC = json.load(fh)


def _model(doc_entry):
    return analytic.OracleSlowdownModel(analytic.OracleParams.from_json(doc_entry["params_json"]))


def _jobs(n, seed):
    return synth.generate_jobs(seed, synth.mixed_archetypes(n))


def test_scalar_restatement_matches_reference_decisions():
    g = DOC["graphs"][0]
    model = _model(g)
    jobs = _jobs(g["n"], g["seed"])
    space = core.default_space(g["budget"])
    configs = core.enumerate_corun_configs(space)
    for row in g["pairs"][::7]:
        d = cs.decide_pair(model, jobs[row["i"]], jobs[row["j"]], space)
        assert d.corun_config == configs[row["corun_index"]]
        assert d.corun_time_s == row["corun_time_s"]          # bit-exact
        assert d.solo_time_s == row["solo_time_s"]
        assert d.corun_chosen == row["corun_chosen"]


def test_params_validation_and_recognition():
    with pytest.raises(cs.ValidationError):
        analytic.OracleParams(cpu_scaling=-1.0)
    assert analytic.oracle_params_of(analytic.OracleSlowdownModel(analytic.OracleParams())) is not None

    class OracleSlowdownModel:           # the reference's class, by name and fields
        def __init__(self):
            self.params = analytic.OracleParams()
    assert analytic.oracle_params_of(OracleSlowdownModel()) is not None
    assert analytic.oracle_params_of(object()) is None


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(4))
def test_gpu_build_graph_equals_reference(k):
    g = DOC["graphs"][k]
    n = g["n"]
    model = _model(g)
    jobs = _jobs(n, g["seed"])
    space = core.default_space(g["budget"])
    inp = cs.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=n), model)
    graph = cs.build_graph(inp)
    configs = core.enumerate_corun_configs(space)
    for row in g["pairs"]:
        d = graph.decisions[(row["i"], row["j"])]
        assert d.corun_config == configs[row["corun_index"]]
        assert d.corun_time_s == row["corun_time_s"]
        assert d.solo_time_s == row["solo_time_s"]
        assert d.corun_chosen == row["corun_chosen"]
        assert graph.weights[row["i"], row["j"]] == row["winning_time"]
    sched = cs.schedule(inp)
    assert [[j.job_id for j in js.jobs] for js in sched.job_sets] == g["schedule_sets"]
    assert [bool(f) for f in sched.corun_flags] == g["schedule_flags"]


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(2))
def test_gpu_five_budget_samples(k):
    entry = DOC["samples"][k]
    n = entry["n"]
    jobs = _jobs(n, entry["seed"])
    spaces = [core.ConfigSpace(p_total=p, cap_sum_levels=tuple(entry["cap_sum_levels"]))
              for p in (entry["p_total"], 400.0)]
    res = analytic.analytic_sweep(analytic.OracleParams(), jobs, spaces, with_matrix=False)
    local = res.corun_local_index(0)
    for row in entry["pairs"]:
        p = pair_index(n, row["i"], row["j"])
        assert local[p] == row["corun_index"]
        assert res.corun_time[0, p] == row["corun_time_s"]
        assert res.corun_chosen[0, p] == row["corun_chosen"]
        assert res.weight[0, p] == row["winning_time"]
