"""Shared fixtures.  Markers: `gpu` = needs a B200 (run with -m gpu)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (sm_100a B200)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def weights():
    from paper_2405_03831_b200 import fnn
    return fnn.load_weights(os.path.join(GOLDEN, "weights.json"))


@pytest.fixture(scope="session")
def paper20():
    with open(os.path.join(GOLDEN, "paper20.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def samples():
    with open(os.path.join(GOLDEN, "samples.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def n256():
    return dict(np.load(os.path.join(GOLDEN, "n256_400.npz")))


def workload(n, seed=0):
    from paper_2405_03831_b200 import synth
    return synth.workload_arrays(seed, synth.mixed_archetypes(n))


def space_for(entry):
    """ConfigSpace of a samples.json entry."""
    from paper_2405_03831_b200 import core
    kw = {"p_total": entry["p_total"], "cap_sum_levels": tuple(entry["cap_sum_levels"])}
    if entry.get("grid") == "fine":
        kw["cpu_caps"] = tuple(entry["cpu_caps"])
        kw["gpu_caps"] = tuple(entry["gpu_caps"])
    return core.ConfigSpace(**kw)


def pair_index(n, i, j):
    return i * (2 * n - i - 1) // 2 + (j - i - 1)
