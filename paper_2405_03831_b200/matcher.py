"""Pair graph container and minimum-weight perfect matching.

Mirrors ``cosched.matcher`` (``pkg/src/cosched/matcher.py``): ``PairGraph``
(28-63) is the consumer contract of the sweep, ``min_weight_perfect_matching``
(78-88) reflects the weights to ``(max + 1) - w`` and takes a maximum-weight
matching, which is perfect on a complete graph with an even vertex count.  The
matching itself runs in the native exact-integer blossom solver
(``csrc/matching.cpp``, host C++) instead of the
reference's interpreted O(n^3) loop; it stays on the host CPU as north_star
asks.  ``brute_force_matching`` is the reference's (n-1)!! oracle.
"""

from __future__ import annotations

import csv
from collections.abc import Mapping
from dataclasses import dataclass
from typing import Iterator, Optional

import numpy as np

from . import _native as nat
from .core import ValidationError

BRUTE_FORCE_MAX_VERTICES = 12


@dataclass(frozen=True)
class PairGraph:
    """Complete graph over a window: symmetric, finite, non-negative weights.

    ``decisions`` optionally maps (i, j), i < j, to the per-edge optimizer
    payload; the GPU build hands a lazy mapping (scheduler.PairDecisions).
    """

    weights: np.ndarray
    decisions: Optional[Mapping] = None

    def __post_init__(self) -> None:
        w = np.array(self.weights, dtype=float)
        if w.ndim != 2 or w.shape[0] != w.shape[1]:
            raise ValidationError(f"weights must be square, got shape {w.shape}")
        n = w.shape[0]
        if n < 2 or n % 2:
            raise ValidationError(f"vertex count must be even and >= 2, got {n}")
        off = ~np.eye(n, dtype=bool)
        if not np.isfinite(w[off]).all():
            raise ValidationError("edge weights must be finite")
        if (w[off] < 0).any():
            raise ValidationError("edge weights must be >= 0")
        if not np.array_equal(w[off], w.T[off]):
            raise ValidationError("weights must be symmetric")
        np.fill_diagonal(w, 0.0)
        w.flags.writeable = False
        object.__setattr__(self, "weights", w)

    @classmethod
    def trusted(cls, weights: np.ndarray, decisions=None) -> "PairGraph":
        """Wrap a matrix produced by the sweep (symmetric by construction,
        zero diagonal) without the O(n^2) re-validation; checks the shape only."""
        w = np.asarray(weights, dtype=np.float64)
        n = w.shape[0]
        if w.ndim != 2 or w.shape[1] != n or n < 2 or n % 2:
            raise ValidationError(f"vertex count must be even and >= 2, got shape {w.shape}")
        if not w.flags.c_contiguous:
            w = np.ascontiguousarray(w)
        w.flags.writeable = False
        obj = object.__new__(cls)
        object.__setattr__(obj, "weights", w)
        object.__setattr__(obj, "decisions", decisions)
        return obj

    @property
    def n(self) -> int:
        return self.weights.shape[0]


def matching_weight(graph: PairGraph, pairs) -> float:
    """Sum of matched weights in canonical (sorted) edge order (matcher.py:66-69)."""
    canon = sorted((min(p), max(p)) for p in pairs)
    return sum(graph.weights[i, j] for i, j in canon)


def _check_perfect(n: int, pairs) -> None:
    if sorted(v for p in pairs for v in p) != list(range(n)):
        raise ValidationError("matching does not cover every vertex exactly once")


def min_weight_perfect_matching(graph: PairGraph) -> list:
    """Perfect matching of minimum total weight, as sorted (i, j) pairs.

    A graph built by the GPU sweep carries per-app potentials (the solo times,
    ``PairDecisions.potentials``): the native solver then maximizes the
    co-run benefit instead (cm_min_weight_perfect_matching_pot), which avoids
    the degeneracy of the many equal-weight time-share pairings.  Either way
    the result is a certified optimum of the complete graph (LP dual check)."""
    n = graph.n
    lib = nat.match_lib()
    w = np.ascontiguousarray(graph.weights, dtype=np.float64)
    mate = np.empty(n, dtype=np.int32)
    pot_fn = getattr(graph.decisions, "potentials", None)
    rc = None
    if pot_fn is not None:
        pot = pot_fn()
        k = 48
        rc = lib.cm_min_weight_perfect_matching_pot(nat.ptr(w), n, nat.ptr(pot), k,
                                                    nat.ptr(mate, nat.c_int32_p))
    if rc is None or rc == -4:
        rc = lib.cm_min_weight_perfect_matching(nat.ptr(w), n, nat.ptr(mate, nat.c_int32_p))
    if rc == -2:
        raise ValidationError("edge weights span too many orders of magnitude for exact matching")
    if rc != 0:
        raise ValidationError(f"matching failed (code {rc})")
    pairs = [(v, int(mate[v])) for v in range(n) if v < mate[v]]
    _check_perfect(n, pairs)
    return sorted(pairs)


def max_weight_matching(weights) -> np.ndarray:
    """Native maximum-weight (not necessarily perfect) matching; mate array, -1 = single."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    n = w.shape[0]
    mate = np.empty(n, dtype=np.int32)
    rc = nat.match_lib().cm_max_weight_matching(nat.ptr(w), n, nat.ptr(mate, nat.c_int32_p))
    if rc:
        raise ValidationError(f"matching failed (code {rc})")
    return mate


def iter_perfect_matchings(n: int) -> Iterator[list]:
    """Every perfect matching of n vertices, lowest free vertex paired first."""
    if n % 2:
        raise ValidationError(f"vertex count must be even, got {n}")

    def rec(free):
        if not free:
            yield []
            return
        head, rest = free[0], free[1:]
        for k, other in enumerate(rest):
            for tail in rec(rest[:k] + rest[k + 1:]):
                yield [(head, other)] + tail

    yield from rec(list(range(n)))


def brute_force_matching(graph: PairGraph):
    """Exact optimum by enumeration (oracle path; n <= 12)."""
    n = graph.n
    if n > BRUTE_FORCE_MAX_VERTICES:
        raise ValidationError(
            f"brute force supports at most {BRUTE_FORCE_MAX_VERTICES} vertices, got {n}")
    best, best_w = None, np.inf
    for pairs in iter_perfect_matchings(n):
        total = matching_weight(graph, pairs)
        if total < best_w:
            best, best_w = pairs, total
    return sorted(best), best_w


def graph_to_csv(graph: PairGraph, path) -> None:
    """One row per edge: i, j, repr(weight), co-run flag (matcher.py:132-142).

    For a graph from the GPU sweep the flags come straight from the result
    arrays (no per-edge PairDecision objects: 8.4M of them at N=4,096)."""
    n = graph.n
    dec = graph.decisions
    flags_fn = getattr(dec, "corun_flags", None)
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["i", "j", "weight", "corun_flag"])
        if flags_fn is not None and len(dec) == n * (n - 1) // 2:
            flags = flags_fn()
            W = graph.weights
            p = 0
            for i in range(n):
                row = W[i].tolist()
                out.writerows([i, j, repr(row[j]), int(flags[p + (j - i - 1)])]
                              for j in range(i + 1, n))
                p += n - i - 1
            return
        for i in range(n):
            for j in range(i + 1, n):
                flag = ""
                if dec and (i, j) in dec:
                    flag = int(dec[(i, j)].corun_chosen)
                out.writerow([i, j, repr(float(graph.weights[i, j])), flag])
