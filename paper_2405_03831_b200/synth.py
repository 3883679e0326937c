"""Synthetic job profiles -- the input generator of every benchmark config.

Reproduces ``simenv.generate_workload`` / ``mixed_archetypes``
(simenv.py:264-311) bit-for-bit (pinned by tests/golden/workloads.json): one
``numpy.random.default_rng([seed, 100])`` stream, per job 18 uniform counter
draws inside its archetype's ranges, then one base time in U(15, 45) s.
``simenv.generate_workload`` wraps the same draws in ``SyntheticJobSpec``s,
exactly as the reference returns them.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .core import JobProfile

ARCHETYPES = ("cpu-bound", "gpu-bound", "memory-bound", "balanced")

# (low, high) per counter, in JobProfile.features order (simenv.py:264-285).
ARCHETYPE_RANGES = {
    "cpu-bound": [(85, 98), (500, 3000), (100, 1000), (2.6, 3.6), (10, 25), (1, 5), (5, 15),
                  (1, 6), (0.5, 3), (0.2, 2), (4, 12), (5, 15), (5, 15), (5, 15), (3, 10),
                  (1, 6), (5, 20), (2, 10)],
    "gpu-bound": [(8, 20), (200, 1500), (50, 500), (0.8, 1.6), (20, 40), (2, 8), (8, 20),
                  (2, 8), (1, 5), (0.5, 3), (55, 80), (20, 45), (30, 60), (25, 50), (82, 97),
                  (20, 48), (60, 90), (15, 40)],
    "memory-bound": [(40, 60), (2000, 8000), (1000, 5000), (0.5, 1.1), (55, 80), (5, 15),
                     (30, 55), (5, 15), (5, 15), (2, 8), (70, 92), (70, 90), (30, 60),
                     (60, 85), (12, 25), (8, 20), (30, 60), (8, 24)],
    "balanced": [(45, 70), (800, 4000), (200, 2000), (1.4, 2.4), (30, 50), (3, 10), (15, 30),
                 (3, 10), (2, 8), (1, 4), (35, 60), (30, 55), (20, 45), (30, 55), (35, 60),
                 (10, 30), (40, 70), (10, 30)],
}
BASE_TIME_RANGE = (15.0, 45.0)


def mixed_archetypes(n_jobs: int) -> list:
    """Round-robin archetype labels."""
    return [ARCHETYPES[k % len(ARCHETYPES)] for k in range(n_jobs)]


def workload_arrays(seed: int, archetypes: Sequence[str]):
    """(features (N, 18) float64, base_time (N,) float64) without building objects."""
    rng = np.random.default_rng([seed, 100])
    n = len(archetypes)
    feats = np.empty((n, 18))
    bt = np.empty(n)
    for k, arch in enumerate(archetypes):
        for c, (lo, hi) in enumerate(ARCHETYPE_RANGES[arch]):
            feats[k, c] = rng.uniform(lo, hi)
        bt[k] = float(rng.uniform(*BASE_TIME_RANGE))
    return feats, bt


def job_ids(archetypes: Sequence[str]) -> list:
    return [f"job{k:02d}-{a}" for k, a in enumerate(archetypes)]


def generate_jobs(seed: int, archetypes: Sequence[str]) -> list:
    """The JobProfiles of ``simenv.generate_workload`` (``[s.job for s in ...]``),
    in the reference's order and naming (``jobNN-<archetype>``)."""
    feats, bt = workload_arrays(seed, archetypes)
    return [JobProfile(jid, feats[k], bt[k]) for k, jid in enumerate(job_ids(archetypes))]
