"""The reference-side ctypes binding (integration/cosched_b200_binding.py).

The binding is written against the reference package's module names; the
drop-in package exports the same names, so the file is loaded here as a
submodule of it (``paper_2405_03831_b200._b200``), exactly as it would sit in
``cosched/_b200.py``.
"""

import importlib.util
import os
import sys

import numpy as np
import pytest

import oracle
from conftest import ROOT, workload
import paper_2405_03831_b200 as cs
from paper_2405_03831_b200 import _native, core, estimator, synth
from paper_2405_03831_b200.grid import KnobGrid


def _binding():
    name = "paper_2405_03831_b200._b200"
    if name in sys.modules:
        return sys.modules[name]
    path = os.path.join(ROOT, "integration", "cosched_b200_binding.py")
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    os.environ["COSCHED_B200_LIB"] = _native.SWEEP_LIB
    return mod


def test_binding_loads_and_binds_symbols():
    b = _binding()
    lib = b._lib()
    for name in ("cs_build_graph_host", "cs_build_graph_workspace_bytes", "cs_device_alloc",
                 "cs_device_free", "cs_error_string"):
        assert hasattr(lib, name)


@pytest.mark.gpu
@pytest.mark.parametrize("n,budget", [(20, 400.0), (64, 350.0)])
def test_binding_build_graph_matches_oracle_and_dropin(weights, n, budget):
    b = _binding()
    jobs = synth.generate_jobs(1, synth.mixed_archetypes(n))
    space = core.default_space(budget)
    inp = cs.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=n), weights)
    estimator.clamp_stats.reset()
    g = b.build_graph_b200(inp)
    c_bind = estimator.clamp_stats.count
    estimator.clamp_stats.reset()
    ref = cs.build_graph(inp)
    assert estimator.clamp_stats.count == c_bind
    assert np.array_equal(g.weights, ref.weights)
    assert list(g.decisions.keys()) == list(ref.decisions.keys())
    for k in g.decisions:
        assert g.decisions[k] == ref.decisions[k]
    F, T = workload(n, 1)
    orc = oracle.sweep(weights, F, T, KnobGrid([space]))
    iu, ju = np.triu_indices(n, 1)
    assert np.array_equal(g.weights[iu, ju], orc["weight"][0])
