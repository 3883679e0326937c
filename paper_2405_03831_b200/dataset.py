"""Training-corpus generation: ``cosched.simenv.generate_dataset`` and its CSV form.

Mirrors ``pkg/src/cosched/simenv.py:330-505`` (``DatasetRow``, ``Dataset``,
``_sample_pairs``, ``generate_dataset``, ``DATASET_INPUT_COLUMNS``,
``dataset_to_csv``, ``load_dataset_csv``).  The corpus is bit-identical to the
reference's: the same seeded draws in the same order (workload, pair picks,
one lognormal noise draw per row), and the clean labels are the analytic
oracle evaluated with the same IEEE operations -- taken from the
config-major resource x power tables and pairwise contention that
``analytic.host_tables`` builds for the GPU analytic sweep, so every (pair,
config, ordering) label is one product rp[view][config][primary] x
contention(primary, co) instead of a Python call per row.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .analytic import _contention, _intensity_arrays, host_tables
from .core import ConfigSpace, HardwareConfig, ValidationError, enumerate_corun_configs, normalize_input
from .fnn import LabeledSample
from .grid import KnobGrid


@dataclass(frozen=True)
class DatasetRow:
    """One labeled training point plus its provenance (simenv.py:330-340)."""

    sample: LabeledSample
    clean_target: float
    pair_id: str
    split: str
    primary_id: str
    co_id: str
    hc: HardwareConfig


@dataclass
class Dataset:
    rows: list
    jobs: list
    bounds: np.ndarray

    def samples(self, split: str) -> list:
        return [r.sample for r in self.rows if r.split == split]

    def rows_for(self, split: str) -> list:
        return [r for r in self.rows if r.split == split]


def _sample_pairs(n_jobs: int, n_pairs: int, train_pairs: int, rng: np.random.Generator,
                  archetypes: Sequence[str]):
    """Stratified pair selection (simenv.py:355-390): train picks prefer an
    unseen archetype combination, then the least-covered jobs; test pairs are
    the next random picks."""
    all_pairs = [(i, j) for i in range(n_jobs) for j in range(i + 1, n_jobs)]
    remaining = [all_pairs[k] for k in rng.permutation(len(all_pairs))]
    counts = [0] * n_jobs
    seen: set = set()
    train = []
    combo = lambda p: frozenset((archetypes[p[0]], archetypes[p[1]]))
    for _ in range(train_pairs):
        best = min(range(len(remaining)),
                   key=lambda k: (combo(remaining[k]) in seen,
                                  max(counts[remaining[k][0]], counts[remaining[k][1]]),
                                  counts[remaining[k][0]] + counts[remaining[k][1]], k))
        i, j = remaining.pop(best)
        counts[i] += 1
        counts[j] += 1
        seen.add(combo((i, j)))
        train.append((i, j))
    return train, remaining[:n_pairs - train_pairs]


def generate_dataset(params, space: ConfigSpace, n_jobs: int = 8, n_pairs: int = 16,
                     train_pairs: int = 12, seed: Optional[int] = None) -> Dataset:
    """Label random job pairs under every co-run config, both orderings
    (simenv.py:393-469).  Defaults: 16 pairs x 100 configs x 2 orderings =
    3,200 points, 2,400 of them training; labels carry multiplicative
    lognormal noise of ``params.noise_sigma``; bounds are the per-slot maxima
    of the training rows."""
    from .simenv import generate_workload, mixed_archetypes
    if seed is None:
        seed = params.seed
    if n_pairs < 1:
        raise ValidationError("n_pairs must be >= 1")
    if n_pairs > n_jobs * (n_jobs - 1) // 2:
        raise ValidationError(f"cannot draw {n_pairs} distinct pairs from {n_jobs} jobs")
    if not 1 <= train_pairs < n_pairs:
        raise ValidationError("train_pairs must satisfy 1 <= train_pairs < n_pairs")

    jobs = generate_workload(seed, mixed_archetypes(n_jobs))
    rng = np.random.default_rng([seed, 200])
    train_picks, test_picks = _sample_pairs(n_jobs, n_pairs, train_pairs, rng,
                                            [s.archetype for s in jobs])
    configs = enumerate_corun_configs(space)
    if not configs:
        raise ValidationError(f"no co-run configs for p_total {space.p_total}")

    # clean labels for every (job, config, view) and pairwise contention, with
    # the reference's operation order (resource * power) * contention
    feats = np.stack([np.asarray(s.job.features, dtype=np.float64) for s in jobs])
    grid = KnobGrid((space,))
    tab = host_tables(params, feats, grid)
    rp = (tab["rp1"], tab["rp2"])                      # [view] (G x N), config-major
    # one budget: the grid is that budget's config list in enumerate_corun_configs order
    assert grid.n_grid == len(configs)
    I = _intensity_arrays(feats)
    contention = _contention(params, {k: v[:, None] for k, v in I.items()},
                             {k: v[None, :] for k, v in I.items()})   # [self][other]

    raw = []
    for split, (i, j) in [("train", p) for p in train_picks] + [("test", p) for p in test_picks]:
        pair_id = f"{jobs[i].job.job_id}+{jobs[j].job.job_id}"
        for g, hc in enumerate(configs):
            for primary, co, view, v in ((i, j, hc, 0), (j, i, hc.reversed_partitions(), 1)):
                clean = float(rp[v][g, primary]) * float(contention[primary, co])
                noise = float(np.exp(rng.normal(0.0, params.noise_sigma))) \
                    if params.noise_sigma > 0 else 1.0
                raw.append((pair_id, split, jobs[primary].job, jobs[co].job, view, clean,
                            clean * noise))

    bounds = np.zeros(36)
    for _, split, primary, co, _, _, _ in raw:
        if split == "train":
            bounds[:18] = np.maximum(bounds[:18], primary.features)
            bounds[18:] = np.maximum(bounds[18:], co.features)
    if np.any(bounds <= 0):
        raise ValidationError("training rows left a zero normalization bound")
    rows = [DatasetRow(sample=LabeledSample(normalize_input(primary, co, view, space, bounds), label),
                       clean_target=clean, pair_id=pair_id, split=split, primary_id=primary.job_id,
                       co_id=co.job_id, hc=view)
            for pair_id, split, primary, co, view, clean, label in raw]
    return Dataset(rows=rows, jobs=jobs, bounds=bounds)


DATASET_INPUT_COLUMNS = (["rc_norm", "rg_norm", "pc_norm", "pg_norm"]
                         + [f"j1_f{k}" for k in range(1, 19)]
                         + [f"j2_f{k}" for k in range(1, 19)])


def dataset_to_csv(dataset: Dataset, path) -> None:
    """40 input columns + target + pair id + split tag, one row per point."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(DATASET_INPUT_COLUMNS + ["slowdown", "pair_id", "split"])
        for row in dataset.rows:
            w.writerow([repr(float(v)) for v in row.sample.input]
                       + [repr(float(row.sample.target)), row.pair_id, row.split])


def load_dataset_csv(path):
    """Read a dataset CSV back as (samples, pair_ids, splits)."""
    samples, pair_ids, splits = [], [], []
    expected = DATASET_INPUT_COLUMNS + ["slowdown", "pair_id", "split"]
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        if next(reader, None) != expected:
            raise ValidationError(f"dataset CSV {path} has an unexpected header")
        for line_no, row in enumerate(reader, start=2):
            if len(row) != len(expected):
                raise ValidationError(f"dataset CSV {path} line {line_no}: expected "
                                      f"{len(expected)} fields, got {len(row)}")
            try:
                values = [float(v) for v in row[:41]]
            except ValueError as exc:
                raise ValidationError(f"dataset CSV {path} line {line_no}: {exc}") from exc
            samples.append(LabeledSample(np.array(values[:40]), values[40]))
            pair_ids.append(row[41])
            splits.append(row[42])
    return samples, pair_ids, splits
