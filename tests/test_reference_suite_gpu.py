"""The reference's OWN unit tests, run against the drop-in on the GPU.

``pkg/tests/test_{core,hwopt,estimator,scheduler,matcher,fnn}.py`` of the
unmodified reference are executed in a subprocess whose ``cosched`` package is
the alias in ``tests/ref_alias`` (every ``cosched.X`` is the drop-in's module
``paper_2405_03831_b200.X``).  The test files are read from the staged copy
``baseline/_ref/ref_tests`` (``tools/stage_reference.sh``: git-ignored, it
travels to the GPU box with the tree) or, in this container, straight from
``/root/reference/pkg/tests``.  Nothing is copied into the repository.

The FNN paths of these tests (``build_graph`` / ``decide_pair`` with a
trained network, the floor clamp counter) have no CPU fallback, hence -m gpu.
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

CANDIDATES = (os.path.join(ROOT, "baseline", "_ref", "ref_tests"), "/root/reference/pkg/tests")
SUITES = ("test_core", "test_hwopt", "test_estimator", "test_scheduler", "test_matcher", "test_fnn")


def _ref_tests():
    for d in CANDIDATES:
        if os.path.isfile(os.path.join(d, "conftest.py")):
            return d
    return None


def _run(suite, tmp_path):
    d = _ref_tests()
    if d is None:
        pytest.skip("reference tests not staged (tools/stage_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "ref_alias"), ROOT,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", os.path.join(d, f"{suite}.py"), "-q", "-p",
           "no:cacheprovider", "--rootdir", str(tmp_path), "-c", os.devnull]
    res = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                         timeout=900)
    tail = "\n".join((res.stdout + res.stderr).splitlines()[-40:])
    assert res.returncode == 0, tail
    assert " passed" in res.stdout, tail
    # the alias must really have served the drop-in, not an installed reference
    probe = subprocess.run([sys.executable, "-c", "import cosched, cosched.hwopt as h; "
                            "print(h.__name__)"], cwd=str(tmp_path), env=env,
                           capture_output=True, text=True)
    assert probe.stdout.strip() == "paper_2405_03831_b200.hwopt", probe.stdout + probe.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_dropin(suite, tmp_path):
    _run(suite, tmp_path)


@pytest.mark.parametrize("suite", ("test_core", "test_hwopt", "test_matcher"))
def test_reference_suite_cpu_parts(suite, tmp_path):
    """The suites whose paths never reach a kernel (enumeration, validation,
    plugin-model optimization, matching) also pass here without a GPU."""
    _run(suite, tmp_path)
