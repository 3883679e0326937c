"""The drop-in API (hwopt / scheduler / estimator) against the reference fixtures, on GPU."""

import numpy as np
import pytest

from conftest import pair_index, space_for, workload
import paper_2405_03831_b200 as cs
from paper_2405_03831_b200 import core, estimator, synth

pytestmark = pytest.mark.gpu
REL = 1e-12


def _hc(t):
    return core.HardwareConfig(tuple(t[0]), tuple(t[1]), t[2], t[3])


def test_decide_pair_matches_reference_samples(weights, samples):
    entry = samples["n4096_400"]
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(4096))
    space = space_for(entry)
    configs = core.enumerate_corun_configs(space)
    splits = core.enumerate_solo_splits(space)
    for row in entry["pairs"][:25]:
        d = cs.decide_pair(weights, jobs[row["i"]], jobs[row["j"]], space)
        assert d.corun_config == configs[row["corun_index"]]
        assert d.corun_chosen == row["corun_chosen"]
        assert abs(d.corun_time_s - row["corun_time_s"]) <= REL * row["corun_time_s"]
        assert abs(d.solo_time_s - row["solo_time_s"]) <= REL * row["solo_time_s"]
        assert [(hc.cpu_cap, hc.gpu_cap) for hc in d.solo_configs] == \
            [splits[k] for k in row["solo_split_index"]]
        hc, t = cs.optimize_corun(weights, jobs[row["i"]], jobs[row["j"]], space)
        assert hc == d.corun_config and t == d.corun_time_s
        s1, s2, st = cs.optimize_solo_pair(weights, jobs[row["i"]], jobs[row["j"]], space)
        assert (s1, s2) == d.solo_configs and st == d.solo_time_s


@pytest.mark.parametrize("budget", ["400", "350"])
def test_build_graph_and_schedule_match_reference(weights, paper20, budget):
    sp = paper20["spaces"][budget]
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(20))
    space = core.default_space(float(budget))
    inp = cs.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=20), weights)
    estimator.clamp_stats.reset()
    graph = cs.build_graph(inp, jobs=4)
    assert estimator.clamp_stats.count == sp["clamp_count_build_graph"]
    assert len(graph.decisions) == 190
    assert list(graph.decisions.keys()) == [(p["i"], p["j"]) for p in sp["pairs"]]
    for p in sp["pairs"]:
        d = graph.decisions[(p["i"], p["j"])]
        assert d.corun_config == _hc(p["corun_config"])
        assert d.corun_chosen == p["corun_chosen"]
        assert abs(d.winning_time - p["winning_time"]) <= REL * p["winning_time"]
        assert graph.weights[p["i"], p["j"]] == d.winning_time
    matched = cs.min_weight_perfect_matching(graph)
    _assert_matching_parity(graph, matched, [tuple(m) for m in sp["matching"]], sp["matching_weight"])
    sched = cs.schedule(inp)
    ref = sp["schedule"]
    mk = cs.predicted_makespan(sched, weights, space)
    assert abs(mk - ref["predicted_makespan"]) <= 1e-12 * ref["predicted_makespan"]
    if [list(m) for m in matched] == sp["matching"]:
        assert [[j.job_id for j in js.jobs] for js in sched.job_sets] == ref["job_sets"]
        assert list(sched.corun_flags) == ref["corun_flags"]
        assert [[_hc(t) for t in cfgs] for cfgs in ref["configs"]] == [list(c) for c in sched.configs]


def _assert_matching_parity(graph, ours, ref_pairs, ref_weight):
    """Optimal total equal to the reference's; the pair set may differ only on a
    tie (time-shared pairs weigh solo_i + solo_j, so swapping partners among
    them leaves the total unchanged up to fp64 rounding)."""
    w_ours = cs.matching_weight(graph, ours)
    assert abs(w_ours - ref_weight) <= 1e-12 * ref_weight
    if list(ours) != list(ref_pairs):
        w_ref_on_ours = cs.matching_weight(graph, ref_pairs)
        assert abs(w_ref_on_ours - w_ours) <= 1e-12 * w_ours, "not a tie: pair sets differ"


def test_full_256_schedule_matches_reference_matching(weights, n256):
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(256))
    inp = cs.SchedulerInput(tuple(jobs), core.default_space(400.0),
                            core.SchedulingParams(window=256), weights)
    graph = cs.build_graph(inp)
    matched = cs.min_weight_perfect_matching(graph)
    _assert_matching_parity(graph, matched, [tuple(int(v) for v in m) for m in n256["matching"]],
                            float(n256["matching_weight"]))


def test_empty_search_spaces_raise_like_the_reference(weights):
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(2))
    with pytest.raises(core.ValidationError, match="no co-run configs"):
        cs.optimize_corun(weights, jobs[0], jobs[1], core.default_space(300.0))
    # 300 W has solo splits but no co-run level: the solo optimizer still works
    s1, s2, t = cs.optimize_solo_pair(weights, jobs[0], jobs[1], core.default_space(300.0))
    assert s1.cap_sum == 300.0 and t > 0
    with pytest.raises(core.ValidationError, match="unreachable"):
        cs.decide_pair(weights, jobs[0], jobs[1], core.default_space(360.0))
    hc, t = cs.optimize_corun(weights, jobs[0], jobs[1], core.default_space(360.0))
    assert hc.cap_sum == 350.0


def test_scalar_predictions_match_sweep(weights):
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(6))
    space = core.default_space(400.0)
    d = cs.decide_pair(weights, jobs[2], jobs[5], space)
    t = cs.corun_time(weights, core.JobSet((jobs[2], jobs[5])), d.corun_config, space)
    assert abs(t - d.corun_time_s) <= REL * t
    total, splits = cs.solorun_time(weights, core.JobSet((jobs[2], jobs[5])), space)
    assert abs(total - d.solo_time_s) <= REL * total


def test_graph_csv_fast_path_matches_generic(tmp_path, weights):
    """graph_to_csv on a sweep graph (flag arrays, no PairDecision objects) writes
    exactly what the generic per-edge path writes (matcher.py:132-142)."""
    jobs = synth.generate_jobs(2, synth.mixed_archetypes(40))
    inp = cs.SchedulerInput(tuple(jobs), core.default_space(400.0),
                            core.SchedulingParams(window=40), weights)
    g = cs.build_graph(inp)
    fast, slow = tmp_path / "fast.csv", tmp_path / "slow.csv"
    cs.matcher.graph_to_csv(g, fast)
    plain = cs.PairGraph(g.weights, {k: g.decisions[k] for k in g.decisions})
    cs.matcher.graph_to_csv(plain, slow)
    assert fast.read_text() == slow.read_text()


def test_batched_set_times_equal_the_scalar_path(weights):
    """predicted_makespan / schedule_to_json send every set's slowdown queries
    to the GPU as one forward_batch; the times, their sum and the clamp counter
    must equal the reference-shaped scalar path (one query per call)."""
    from paper_2405_03831_b200 import scheduler
    n = 96
    jobs = synth.generate_jobs(3, synth.mixed_archetypes(n))
    space = core.default_space(350.0)
    inp = cs.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=n), weights)
    sched = cs.schedule(inp)
    assert any(sched.corun_flags) and not all(sched.corun_flags)
    estimator.clamp_stats.reset()
    scalar = [scheduler.set_time(weights, js, c, f, space)
              for js, c, f in zip(sched.job_sets, sched.configs, sched.corun_flags)]
    c_scalar = estimator.clamp_stats.count
    estimator.clamp_stats.reset()
    assert scheduler._set_times(sched, weights, space) == scalar
    assert estimator.clamp_stats.count == c_scalar
    assert cs.predicted_makespan(sched, weights, space) == sum(scalar)
    doc = cs.schedule_to_json(sched, estimator.FnnSlowdownModel(weights), space)
    assert [s["predicted_s"] for s in doc["sets"]] == scalar
    assert doc["total_predicted_s"] == sum(scalar)
