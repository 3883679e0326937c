"""The tcgen05 screen (k_sweep_tc3) and the SIMT screen agree with the oracle bit-for-bit."""

import numpy as np
import pytest

import oracle
from conftest import workload
from paper_2405_03831_b200 import core, synth
from paper_2405_03831_b200.grid import KnobGrid
from paper_2405_03831_b200.sweep import sweep_pairs

pytestmark = pytest.mark.gpu


def _check(res, ref, L):
    for l in range(L):
        assert np.array_equal(res.corun_grid_index[l], ref["corun_grid_index"][l])
        assert np.array_equal(res.corun_chosen[l], ref["corun_chosen"][l])
        assert np.array_equal(res.corun_time[l], ref["corun_time"][l])
        assert np.array_equal(res.weight[l], ref["weight"][l])


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
@pytest.mark.parametrize("n,seed,budgets", [
    (20, 0, (400.0,)), (2, 1, (400.0,)), (67, 2, (350.0,)), (131, 3, (400.0, 350.0)),
    (256, 0, (400.0,))])
def test_screen_kernels_match_oracle(weights, kernel, n, seed, budgets):
    spaces = [core.default_space(p) for p in budgets]
    jobs = synth.generate_jobs(seed, synth.mixed_archetypes(n))
    res = sweep_pairs(weights, jobs, spaces, with_matrix=False, kernel=kernel)
    F, T = workload(n, seed)
    ref = oracle.sweep(weights, F, T, KnobGrid(spaces))
    _check(res, ref, len(spaces))
    assert res.screen_error < 2.5e-6, res.screen_error


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
def test_five_budgets_and_fine_grid_shards(weights, kernel):
    levels = (300, 325, 350, 375, 400)
    spaces = [core.ConfigSpace(p_total=p, cap_sum_levels=levels) for p in (300.0, 325.0, 350.0, 375.0, 400.0)]
    n = 1024
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(n))
    F, T = workload(n)
    b, e = 123_456, 123_456 + 5000
    res = sweep_pairs(weights, jobs, spaces, b, e, with_matrix=False, kernel=kernel)
    _check(res, oracle.sweep(weights, F, T, KnobGrid(spaces), b, e), 5)
    fine = [core.ConfigSpace(cpu_caps=tuple(100.0 + 6.25 * k for k in range(25)),
                             gpu_caps=tuple(150.0 + 6.25 * k for k in range(17)), p_total=400.0)]
    res = sweep_pairs(weights, jobs, fine, b, e, with_matrix=False, kernel=kernel)
    _check(res, oracle.sweep(weights, F, T, KnobGrid(fine), b, e), 1)


def test_out_of_fp16_range_network_falls_back_and_stays_exact(weights):
    """A network whose layer-1 activations exceed the fp16 range cannot use the
    tensor-core screen; the default plan must switch to the fp32 SIMT screen and
    still match the oracle exactly."""
    from paper_2405_03831_b200 import fnn
    from paper_2405_03831_b200.device import fp16_screen_safe
    big = fnn.NetworkWeights(weights.w1 * 5000.0, weights.b1 * 5000.0, weights.w2, weights.b2,
                             weights.w_out, weights.b_out, weights.feature_bounds)
    assert fp16_screen_safe(weights) and not fp16_screen_safe(big)
    n = 48
    jobs = synth.generate_jobs(5, synth.mixed_archetypes(n))
    spaces = [core.default_space(400.0)]
    res = sweep_pairs(big, jobs, spaces, with_matrix=False)
    F, T = workload(n, 5)
    _check(res, oracle.sweep(big, F, T, KnobGrid(spaces)), 1)


@pytest.mark.parametrize("kind", ["a03342", "3342"])
@pytest.mark.parametrize("n,seed,budgets", [
    (20, 0, (400.0,)), (131, 3, (400.0, 350.0)), (300, 4, (375.0,))])
def test_alternative_screen_instances_match_oracle(weights, monkeypatch, kind, n, seed, budgets):
    """The measured alternatives of k_sweep_tc3 stay parity-exact: the stream-K
    schedule (0xA03342: items cut between group slots, merged by their last
    piece -- at n=20 every item is split into several pieces) and the instance
    without register rebalancing (0x3342)."""
    monkeypatch.setenv("COSCHED_TC_KIND", kind)
    spaces = [core.default_space(p) for p in budgets]
    jobs = synth.generate_jobs(seed, synth.mixed_archetypes(n))
    res = sweep_pairs(weights, jobs, spaces, with_matrix=False, kernel="tcgen05")
    F, T = workload(n, seed)
    ref = oracle.sweep(weights, F, T, KnobGrid(spaces))
    _check(res, ref, len(spaces))


@pytest.mark.parametrize("n,seed", [(3, 5), (40, 6)])
def test_eight_budgets_small_n_stream_k(weights, n, seed):
    """The most budgets a sweep takes (8, so the stream-K partials carry
    3 x 8 + 1 fields per thread) on small N, where the screen splits the
    configs of every work item across group slots."""
    levels = (300, 325, 350, 375, 400, 425, 450, 475)
    spaces = [core.ConfigSpace(p_total=float(p), cap_sum_levels=levels) for p in levels]
    jobs = synth.generate_jobs(seed, synth.mixed_archetypes(n))
    res = sweep_pairs(weights, jobs, spaces, with_matrix=True, kernel="tcgen05")
    F, T = workload(n, seed)
    ref = oracle.sweep(weights, F, T, KnobGrid(spaces))
    _check(res, ref, len(spaces))
