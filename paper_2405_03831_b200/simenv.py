"""The parts of ``cosched.simenv`` the hot path's callers and tests use.

Mirrors the reference's public names (``pkg/src/cosched/simenv.py``):

* the synthetic workload generator -- ``SyntheticJobSpec`` (simenv.py:240-256),
  ``generate_job`` / ``generate_workload`` / ``mixed_archetypes``
  (simenv.py:290-311), ``workload_to_json`` / ``load_workload``
  (simenv.py:314-326).  The draws are those of ``synth.workload_arrays``
  (one ``default_rng([seed, 100])`` stream, 18 counters then the base time
  per job), so the specs are bit-identical to the reference's;
* the analytic oracle model -- ``OracleParams``, ``OracleSlowdownModel``,
  ``oracle_slowdown`` (simenv.py:63-237), served by ``analytic.py`` (its
  batched form is the exact GPU sweep ``cs_analytic_sweep``);
* the training dataset -- ``generate_dataset``, ``Dataset``, ``DatasetRow``
  and the CSV form (simenv.py:330-505), in ``dataset.py``.

The policy harness (``run_policy``, reports) and the CLI stay out of scope
(SURVEY.md §2).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .analytic import OracleParams, OracleSlowdownModel, oracle_slowdown  # noqa: F401
from .dataset import (DATASET_INPUT_COLUMNS, Dataset, DatasetRow, dataset_to_csv,  # noqa: F401
                      generate_dataset, load_dataset_csv)
from .core import JobProfile, ValidationError
from .synth import ARCHETYPE_RANGES, ARCHETYPES, BASE_TIME_RANGE, job_ids, mixed_archetypes  # noqa: F401


@dataclass(frozen=True)
class SyntheticJobSpec:
    """A generated job together with the archetype that shaped it."""

    archetype: str
    job: JobProfile

    def __post_init__(self) -> None:
        if self.archetype not in ARCHETYPES:
            raise ValidationError(f"unknown archetype {self.archetype!r}")

    def to_json(self) -> dict:
        return {"archetype": self.archetype, "job": self.job.to_json()}

    @classmethod
    def from_json(cls, data: dict) -> "SyntheticJobSpec":
        return cls(archetype=data["archetype"], job=JobProfile.from_json(data["job"]))


def generate_job(rng: np.random.Generator, archetype: str, job_id: str) -> SyntheticJobSpec:
    """One job: 18 uniform counter draws in its archetype's ranges, then the base time."""
    if archetype not in ARCHETYPE_RANGES:
        raise ValidationError(f"unknown archetype {archetype!r}")
    features = np.array([rng.uniform(lo, hi) for lo, hi in ARCHETYPE_RANGES[archetype]])
    base_time = float(rng.uniform(*BASE_TIME_RANGE))
    return SyntheticJobSpec(archetype, JobProfile(job_id, features, base_time))


def generate_workload(seed: int, archetypes: Sequence[str]) -> list:
    """One job per requested archetype label, deterministically (simenv.py:297-306)."""
    rng = np.random.default_rng([seed, 100])
    return [generate_job(rng, arch, jid) for arch, jid in zip(archetypes, job_ids(archetypes))]


def workload_to_json(specs: Sequence[SyntheticJobSpec]) -> list:
    return [s.to_json() for s in specs]


def load_workload(path) -> list:
    with open(path) as fh:
        data = json.load(fh)
    if not isinstance(data, list):
        raise ValidationError(f"workload file {path} must hold a JSON list")
    return [SyntheticJobSpec.from_json(d) for d in data]
