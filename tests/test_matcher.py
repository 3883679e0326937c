"""Native matcher (csrc/matching.cpp) vs the reference's matcher fixtures and brute force. CPU."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2405_03831_b200 import matcher
from paper_2405_03831_b200.core import ValidationError


def random_graph(n, seed):
    """Same generator as tests/golden/make_golden.py."""
    rng = np.random.default_rng([seed, n, 7])
    w = np.triu(rng.uniform(10.0, 100.0, size=(n, n)), 1)
    return w + w.T


with open(os.path.join(GOLDEN, "matching.json")) as fh:
    CASES = json.load(fh)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c['n']}s{c['seed']}")
def test_matches_reference_matcher(case):
    W = np.array(case["weights"]) if case.get("integer_ties") else random_graph(case["n"], case["seed"])
    g = matcher.PairGraph(W)
    pairs = matcher.min_weight_perfect_matching(g)
    total = matcher.matching_weight(g, pairs)
    assert abs(total - case["weight"]) <= 1e-12 * case["weight"]
    if not case.get("integer_ties"):       # continuous weights: unique optimum
        assert [list(p) for p in pairs] == case["pairs"]
    if "brute_force_weight" in case:
        assert abs(total - case["brute_force_weight"]) <= 1e-12 * case["brute_force_weight"]


@pytest.mark.parametrize("n", [2, 4, 6, 8, 10])
def test_against_brute_force_many_seeds(n):
    for seed in range(25):
        rng = np.random.default_rng([seed, n, 11])
        w = np.triu(rng.integers(0, 6, size=(n, n)).astype(float), 1)   # heavy ties
        g = matcher.PairGraph(w + w.T)
        pairs = matcher.min_weight_perfect_matching(g)
        assert sorted(v for p in pairs for v in p) == list(range(n))
        _, best = matcher.brute_force_matching(g)
        assert matcher.matching_weight(g, pairs) == best


def test_dual_certificate_random_256():
    """Optimality without an oracle: a perfect matching M is minimum iff no
    alternating cycle improves it; spot-check with 2-opt swaps on every matched
    pair couple (a necessary condition, exhaustive over O(n^2) swaps)."""
    W = random_graph(256, 42)
    g = matcher.PairGraph(W)
    pairs = matcher.min_weight_perfect_matching(g)
    P = np.array(pairs)
    a, b = P[:, 0], P[:, 1]
    base = W[a, b]
    for k in range(len(P)):
        cur = base[k] + base
        alt1 = W[a[k], a] + W[b[k], b]
        alt2 = W[a[k], b] + W[b[k], a]
        alt1[k] = alt2[k] = np.inf
        assert np.all(alt1 >= cur - 1e-9) and np.all(alt2 >= cur - 1e-9)


def test_max_weight_matching_general():
    w = np.array([[0, 5, 1, 0], [5, 0, 9, 0], [1, 9, 0, 2], [0, 0, 2, 0]], dtype=float)
    mate = matcher.max_weight_matching(w)
    # best: (0,1)+(2,3) = 7 vs (1,2) = 9 -> (1,2) alone or (1,2)+(0,3=0)
    assert mate[1] == 2 and mate[2] == 1


def test_pairgraph_validation():
    with pytest.raises(ValidationError, match="square"):
        matcher.PairGraph(np.zeros((2, 3)))
    with pytest.raises(ValidationError, match="even"):
        matcher.PairGraph(np.zeros((3, 3)))
    with pytest.raises(ValidationError, match="symmetric"):
        matcher.PairGraph(np.array([[0, 1.0], [2.0, 0]]))
    with pytest.raises(ValidationError, match=">= 0"):
        matcher.PairGraph(np.array([[0, -1.0], [-1.0, 0]]))
    g = matcher.PairGraph(np.array([[7.0, 1.0], [1.0, 9.0]]))
    assert g.weights[0, 0] == 0 and not g.weights.flags.writeable


def test_brute_force_limit():
    with pytest.raises(ValidationError):
        matcher.brute_force_matching(matcher.PairGraph(np.ones((14, 14)) - np.eye(14)))


def test_graph_csv(tmp_path):
    g = matcher.PairGraph(random_graph(4, 0))
    p = tmp_path / "g.csv"
    matcher.graph_to_csv(g, p)
    rows = p.read_text().splitlines()
    assert rows[0] == "i,j,weight,corun_flag" and len(rows) == 7


@pytest.mark.parametrize("n,k", [(40, 1), (64, 2), (128, 4), (200, 24)])
def test_sparse_candidates_plus_certificate_equal_dense(n, k):
    """cm_min_weight_perfect_matching_k: a starved candidate graph (k lightest
    edges per vertex, possibly without any perfect matching) must still end at
    the complete graph's optimum via the dual certificate / edge-addition loop."""
    from paper_2405_03831_b200 import _native as nat
    for seed in range(3):
        W = random_graph(n, 100 + seed)
        g = matcher.PairGraph(W)
        out = {}
        for kk in (k, 0):
            mate = np.empty(n, dtype=np.int32)
            rc = nat.match_lib().cm_min_weight_perfect_matching_k(
                nat.ptr(np.ascontiguousarray(W)), n, kk, nat.ptr(mate, nat.c_int32_p))
            assert rc == 0
            out[kk] = sorted((v, int(mate[v])) for v in range(n) if v < mate[v])
        assert out[k] == out[0]


def test_potential_form_equals_direct_on_sweep_graphs():
    """cm_min_weight_perfect_matching_pot (benefit form, solo-time potentials)
    reaches the same optimum as the direct solve on real pair graphs (oracle
    sweep of the synthetic workload), and rejects potentials that do not bound
    the weights."""
    import oracle
    from conftest import workload
    from paper_2405_03831_b200 import _native as nat, core, fnn
    from paper_2405_03831_b200.grid import KnobGrid
    w = fnn.load_weights(os.path.join(GOLDEN, "weights.json"))
    for n, budget in ((64, 400.0), (150, 350.0)):
        F, T = workload(n, 3)
        r = oracle.sweep(w, F, T, KnobGrid([core.default_space(budget)]))
        W = np.zeros((n, n))
        iu, ju = np.triu_indices(n, 1)
        W[iu, ju] = r["weight"][0]
        W = np.ascontiguousarray(W + W.T)
        pot = np.ascontiguousarray(r["solo_time"][0])
        g = matcher.PairGraph(W)
        out = {}
        for name, call in (("pot", lambda m: nat.match_lib().cm_min_weight_perfect_matching_pot(
                                nat.ptr(W), n, nat.ptr(pot), 8, nat.ptr(m, nat.c_int32_p))),
                           ("direct", lambda m: nat.match_lib().cm_min_weight_perfect_matching_k(
                                nat.ptr(W), n, 0, nat.ptr(m, nat.c_int32_p)))):
            mate = np.empty(n, dtype=np.int32)
            assert call(mate) == 0
            out[name] = matcher.matching_weight(g, [(v, int(mate[v])) for v in range(n) if v < mate[v]])
        assert abs(out["pot"] - out["direct"]) <= 1e-12 * out["direct"]
        bad = np.ascontiguousarray(pot * 0.4)
        mate = np.empty(n, dtype=np.int32)
        assert nat.match_lib().cm_min_weight_perfect_matching_pot(
            nat.ptr(W), n, nat.ptr(bad), 8, nat.ptr(mate, nat.c_int32_p)) == -4


def _mate_weight(W, mate):
    n = len(mate)
    assert sorted(int(x) for x in mate) == list(range(n))
    assert all(mate[int(mate[v])] == v and mate[v] != v for v in range(n))
    return sum(W[v, int(mate[v])] for v in range(n) if v < mate[v])


def test_warm_started_solver_on_a_512_app_sweep_graph():
    """The auction-priced, warm-started certified solver (benefit and reflected
    forms, two candidate degrees) reaches the dense solve's optimum on a real
    512-app pair graph (oracle sweep) -- the size where several certificate
    rounds and blossoms actually occur."""
    import oracle
    from conftest import workload
    from paper_2405_03831_b200 import _native as nat, core, fnn
    from paper_2405_03831_b200.grid import KnobGrid
    w = fnn.load_weights(os.path.join(GOLDEN, "weights.json"))
    n = 512
    F, T = workload(n, 5)
    r = oracle.sweep(w, F, T, KnobGrid([core.default_space(400.0)]))
    W = np.zeros((n, n))
    iu, ju = np.triu_indices(n, 1)
    W[iu, ju] = r["weight"][0]
    W = np.ascontiguousarray(W + W.T)
    pot = np.ascontiguousarray(r["solo_time"][0])
    lib = nat.match_lib()
    out = []
    for call in (lambda m: lib.cm_min_weight_perfect_matching_pot(nat.ptr(W), n, nat.ptr(pot), 48, nat.ptr(m, nat.c_int32_p)),
                 lambda m: lib.cm_min_weight_perfect_matching_pot(nat.ptr(W), n, nat.ptr(pot), 4, nat.ptr(m, nat.c_int32_p)),
                 lambda m: lib.cm_min_weight_perfect_matching_k(nat.ptr(W), n, 8, nat.ptr(m, nat.c_int32_p)),
                 lambda m: lib.cm_min_weight_perfect_matching_k(nat.ptr(W), n, 0, nat.ptr(m, nat.c_int32_p))):
        mate = np.empty(n, dtype=np.int32)
        assert call(mate) == 0
        out.append(_mate_weight(W, mate))
    assert max(out) - min(out) <= 1e-12 * min(out)


def test_all_time_share_graph_is_fully_degenerate_but_solved():
    """Every pair time-shares (w = pot_i + pot_j: zero benefit everywhere), so
    every perfect matching is optimal -- the solver must still return one."""
    from paper_2405_03831_b200 import _native as nat
    n = 64
    pot = np.ascontiguousarray(np.random.default_rng(3).uniform(1.0, 9.0, n))
    W = np.ascontiguousarray(pot[:, None] + pot[None, :])
    np.fill_diagonal(W, 0.0)
    mate = np.empty(n, dtype=np.int32)
    assert nat.match_lib().cm_min_weight_perfect_matching_pot(
        nat.ptr(W), n, nat.ptr(pot), 8, nat.ptr(mate, nat.c_int32_p)) == 0
    assert abs(_mate_weight(W, mate) - pot.sum()) <= 1e-12 * pot.sum()
