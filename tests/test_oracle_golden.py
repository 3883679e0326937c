"""Pin the CPU oracle (oracle/cosched_oracle.c) to the UNMODIFIED reference.

Every fixture under tests/golden/ was produced by the reference package itself
(tests/golden/make_golden.py).  The oracle must reproduce the reference's
chosen config index, co-run flag and solo splits exactly, and its times to
<= 1e-12 relative (the only difference is fp64 summation order: the reference
goes through numpy BLAS, fnn.py:163-165).  CPU only.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, pair_index, space_for, workload
from paper_2405_03831_b200 import core, synth
from paper_2405_03831_b200.grid import KnobGrid

REL = 1e-12


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.max(np.abs(a - b) / np.abs(b)) if a.size else 0.0


def test_workload_generator_is_bit_identical():
    with open(os.path.join(GOLDEN, "workloads.json")) as fh:
        pins = json.load(fh)
    for key, pin in pins.items():
        seed, n = (int(v) for v in key.split(":"))
        f, b = synth.workload_arrays(seed, synth.mixed_archetypes(n))
        assert hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest() == pin["features_sha256"]
        assert hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest() == pin["base_time_sha256"]
        ids = synth.job_ids(synth.mixed_archetypes(n))
        assert ids[0] == pin["first_job_id"] and ids[-1] == pin["last_job_id"]


@pytest.mark.parametrize("budget", ["400", "350"])
def test_factored_sweep_matches_reference_paper20(weights, paper20, budget):
    sp = paper20["spaces"][budget]
    F, T = np.array(paper20["features"]), np.array(paper20["base_time"])
    grid = KnobGrid([core.default_space(float(budget))])
    assert grid.n_configs[0] == sp["n_corun_configs"]
    r = oracle.sweep(weights, F, T, grid)
    rows = sp["pairs"]
    assert [(p["i"], p["j"]) for p in rows] == [(i, j) for i in range(20) for j in range(i + 1, 20)]
    local = grid.local_index[0][r["corun_grid_index"][0]]
    assert local.tolist() == [p["corun_index"] for p in rows]
    assert r["corun_chosen"][0].tolist() == [p["corun_chosen"] for p in rows]
    assert _rel(r["corun_time"][0], [p["corun_time_s"] for p in rows]) <= REL
    assert _rel(r["weight"][0], [p["winning_time"] for p in rows]) <= REL
    for p in rows:
        assert [r["solo_split"][0, p["i"]], r["solo_split"][0, p["j"]]] == p["solo_split_index"]
    # clamp_stats over build_graph: co-run clamps + (n-1) solo passes per app
    total = int(r["corun_clamps"][0]) + 19 * int(r["solo_clamps_one_pass"])
    assert total == sp["clamp_count_build_graph"]


def test_factored_sweep_matches_full_reference_graph_256(weights, n256):
    F, T = workload(256)
    grid = KnobGrid([core.default_space(400.0)])
    r = oracle.sweep(weights, F, T, grid)
    local = grid.local_index[0][r["corun_grid_index"][0]]
    assert np.array_equal(local, n256["corun_index"])
    assert np.array_equal(r["corun_chosen"][0], n256["corun_chosen"].astype(bool))
    assert _rel(r["corun_time"][0], n256["corun_time"]) <= REL
    assert _rel(r["weight"][0], n256["winning_time"]) <= REL
    assert np.array_equal(r["solo_split"][0], n256["solo_split"])


@pytest.mark.parametrize("key", ["n4096_400", "n4096_350", "n1024_b300", "n1024_b325",
                                 "n1024_b350", "n1024_b375", "n1024_b400", "n4096_fine400",
                                 "n256s1_400"])
def test_oracle_matches_reference_samples(weights, samples, key):
    entry = samples[key]
    n, seed = entry["n"], entry["seed"]
    F, T = workload(n, seed)
    space = space_for(entry)
    grid = KnobGrid([space])
    if "n_corun_configs" in entry:
        assert grid.n_configs[0] == entry["n_corun_configs"]
        assert len(grid.solo_splits[0]) == entry["n_solo_splits"]
    k1 = grid.knob1[grid.budget_configs[0]]
    k2 = grid.knob2[grid.budget_configs[0]]
    for row in entry["pairs"][:60]:
        i, j = row["i"], row["j"]
        # direct form (normalize_input + unfactored forward)
        d = oracle.decide_pair(weights, F[i], T[i], F[j], T[j], k1, k2, grid.solo_knob)
        assert d["corun_index"] == row["corun_index"]
        assert d["corun_chosen"] == row["corun_chosen"]
        assert list(d["solo_split"]) == row["solo_split_index"]
        assert abs(d["corun_time"] - row["corun_time_s"]) <= REL * row["corun_time_s"]
        assert abs(d["solo_time"] - row["solo_time_s"]) <= REL * row["solo_time_s"]
        # factored form on the one-pair shard
        p = pair_index(n, i, j)
        r = oracle.sweep(weights, F, T, grid, p, p + 1, threads=1)
        assert grid.local_index[0][r["corun_grid_index"][0, 0]] == row["corun_index"]
        assert abs(r["weight"][0, 0] - row["winning_time"]) <= REL * row["winning_time"]


def test_direct_and_factored_agree_on_budget_sweep(weights):
    n = 48
    F, T = workload(n, 3)
    spaces = [core.ConfigSpace(p_total=p, cap_sum_levels=(300, 325, 350, 375, 400))
              for p in (300.0, 325.0, 350.0, 375.0, 400.0)]
    grid = KnobGrid(spaces)
    assert grid.n_configs == [30, 70, 120, 170, 220]
    r = oracle.sweep(weights, F, T, grid)
    for l in range(5):
        cfg = grid.budget_configs[l]
        lo, hi = grid.solo_offsets[l], grid.solo_offsets[l + 1]
        for (i, j) in [(0, 1), (3, 17), (10, 47), (46, 47)]:
            p = pair_index(n, i, j)
            d = oracle.decide_pair(weights, F[i], T[i], F[j], T[j], grid.knob1[cfg],
                                   grid.knob2[cfg], grid.solo_knob[lo:hi])
            assert grid.local_index[l][r["corun_grid_index"][l, p]] == d["corun_index"]
            assert r["corun_chosen"][l, p] == d["corun_chosen"]
            assert abs(r["weight"][l, p] - d["weight"]) <= REL * d["weight"]
