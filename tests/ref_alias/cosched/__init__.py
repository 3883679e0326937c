"""Alias package: the reference's import paths (``cosched.*``) bound to the drop-in.

TEST INFRASTRUCTURE.  ``tests/test_reference_suite_gpu.py`` runs the
reference's own unit tests (``pkg/tests/test_{core,hwopt,estimator,scheduler,
matcher}.py``) with this directory first on ``sys.path``, so every
``from cosched.X import Y`` in them resolves to the drop-in package
``paper_2405_03831_b200``.  The submodules are the drop-in's module objects
themselves (``sys.modules`` aliases), so a test that resets or patches
``cosched.estimator.clamp_stats`` acts on the state the drop-in uses.
"""

import sys

import paper_2405_03831_b200 as _dropin
from paper_2405_03831_b200 import core, estimator, fnn, hwopt, matcher, scheduler, simenv

for _name, _mod in {"core": core, "estimator": estimator, "fnn": fnn, "hwopt": hwopt,
                    "matcher": matcher, "scheduler": scheduler, "simenv": simenv}.items():
    sys.modules[f"{__name__}.{_name}"] = _mod

from paper_2405_03831_b200 import *  # noqa: E402,F401,F403

__version__ = _dropin.__version__
