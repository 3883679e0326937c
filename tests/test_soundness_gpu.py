"""Parity where the fp32 screen is weakest: near-tie configs and predictions at the floor.

The screen only nominates; exactness comes from (a) the fp64 re-evaluation of
every winner, (b) an fp64 re-evaluation of the runner-up when it lies within
64 rel_eps (the pair falls back to the exact re-scan should the two be
ordered wrongly), (c) the exact fp64 re-scan of every pair whose runner-up is
within rel_eps, and (d) an fp64 re-count of the floor clamps of every (pair, member) row with a
screened prediction within tau = rel_eps / 2 of the 0.5 floor
(estimator.py:98-109).  These networks are built to hit each case; the
argmin, the times and clamp_stats must equal the fp64 oracle exactly.
"""

import numpy as np
import pytest

import oracle
from conftest import workload
from paper_2405_03831_b200 import core, fnn, synth
from paper_2405_03831_b200.grid import KnobGrid
from paper_2405_03831_b200.sweep import sweep_pairs

pytestmark = pytest.mark.gpu


def _net(w, w1=None, b1=None, wo=None, bo=None):
    return fnn.NetworkWeights(w.w1 if w1 is None else w1, w.b1 if b1 is None else b1, w.w2, w.b2,
                              w.w_out if wo is None else wo, w.b_out if bo is None else bo,
                              w.feature_bounds)


def _check_exact(net, n, seed, spaces, kernel="tcgen05"):
    jobs = synth.generate_jobs(seed, synth.mixed_archetypes(n))
    res = sweep_pairs(net, jobs, spaces, with_matrix=False, kernel=kernel)
    F, T = workload(n, seed)
    grid = KnobGrid(spaces)
    ref = oracle.sweep(net, F, T, grid)
    for l in range(len(spaces)):
        assert np.array_equal(res.corun_grid_index[l], ref["corun_grid_index"][l])
        assert np.array_equal(res.corun_time[l], ref["corun_time"][l])
        assert np.array_equal(res.corun_chosen[l], ref["corun_chosen"][l])
        assert np.array_equal(res.weight[l], ref["weight"][l])
        # clamp_stats over build_graph: every co-run prediction + both members'
        # solo splits once per pair (estimator.py:139-180 inside decide_pair)
        solo_part = (n - 1) * int(res.solo_clamps[l].sum())
        assert int(res.clamps[l]) == int(ref["corun_clamps"][l]) + solo_part, l
    return res


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
@pytest.mark.parametrize("scale", [1e-9, 3e-6, 2e-5, 3e-4])
def test_near_tie_configs(weights, kernel, scale):
    """Knob columns of W1 scaled down: every config of a pair lies within
    ~scale of the others -- exact ties in fp32 (1e-9), inside the re-scan
    band (3e-6), inside the runner-up check band (2e-5, 3e-4)."""
    w1 = np.array(weights.w1)
    w1[:, 0:4] *= scale
    net = _net(weights, w1=w1)
    res = _check_exact(net, 40, 2, [core.default_space(400.0), core.default_space(350.0)], kernel)
    if scale < 1e-5:
        assert res.queue_len > 0          # the exact re-scan did the work


@pytest.mark.parametrize("kernel", ["tcgen05", "simt"])
@pytest.mark.parametrize("spread", [1e-6, 1e-4, 3e-3])
def test_predictions_straddling_the_floor(weights, kernel, spread):
    """Output layer squeezed around 0.5: y = 0.5 + spread * (...).  With
    spread 1e-6 nearly every row has a prediction within tau of the floor
    (fp64 re-count of nearly everything); 1e-4 and 3e-3 mix screened and
    re-counted rows."""
    wo = np.array(weights.w_out) * spread
    # centre the squeezed output on 0.5 for this workload
    F, T = workload(32, 4)
    grid = KnobGrid([core.default_space(400.0)])
    ref0 = oracle.sweep(_net(weights, wo=wo, bo=np.zeros(1)), F, T, grid)
    A = ref0["A"]
    # typical hidden output: median of wo.h2 over a few rows (host numpy, fp64)
    W1, b1, W2, b2 = (np.asarray(x) for x in (weights.w1, weights.b1, weights.w2, weights.b2))
    x = np.maximum(A[:8] + W1[:, 0:4] @ np.array([0.5, 0.5, 0.8, 0.8]) + b1, 0)
    med = float(np.median(np.maximum(x @ W2.T + b2, 0) @ wo.ravel()))
    net = _net(weights, wo=wo, bo=np.array([0.5 - med]))
    res = _check_exact(net, 32, 4, [core.default_space(400.0)], kernel)
    assert int(res.clamps[0]) > 0


def test_floor_crowded_multi_budget(weights):
    wo = np.array(weights.w_out) * 1e-7
    net = _net(weights, wo=wo, bo=np.array([0.5]))
    levels = (300, 325, 350, 375, 400)
    spaces = [core.ConfigSpace(p_total=p, cap_sum_levels=levels) for p in (325.0, 350.0, 400.0)]
    _check_exact(net, 24, 1, spaces)


def test_host_abi_counts_floor_clamps_exactly(weights):
    from paper_2405_03831_b200 import host_abi
    wo = np.array(weights.w_out) * 1e-4
    net = _net(weights, wo=wo, bo=np.array([0.5]))
    n = 40
    F, T = workload(n, 9)
    grid = KnobGrid([core.default_space(400.0)])
    out = host_abi.build_graph_host(net, grid, F, T)
    ref = oracle.sweep(net, F, T, grid)
    iu, ju = np.triu_indices(n, 1)
    assert np.array_equal(out["weights"][0][iu, ju], ref["weight"][0])
    solo_part = (n - 1) * int(out["solo_clamps"][0].sum()) if "solo_clamps" in out else None
    if solo_part is not None:
        assert int(out["clamps"][0]) == int(ref["corun_clamps"][0]) + solo_part
