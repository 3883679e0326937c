"""cosched_b200 -- B200-native pair x knob sweep behind the ``cosched`` API.

Drop-in for the optimizer/scheduler path of the reference package ``cosched``
(arXiv 2405.03831, ``pkg/src/cosched``): the same public names for the hot
path (``build_graph``, ``decide_pair``, ``optimize_corun``, ...), with the
exhaustive (pair x knob) evaluation of a trained FNN done by hand-written
sm_100a kernels (``csrc/sweep.cu``) through a C ABI (``include/cosched_b200.h``)
and the matching by a native exact blossom solver (``csrc/matching.cpp``).
See DESIGN.md.
"""

__version__ = "0.1.0"

from .core import (ConfigSpace, HardwareConfig, JobProfile, JobSet, Schedule,
                   SchedulingParams, ValidationError, default_space, enumerate_corun_configs,
                   enumerate_solo_splits, normalize_input, solo_config)
from .fnn import (LabeledSample, NetworkWeights, TrainingConfig, TrainingDivergedError, backward,
                  forward, forward_batch, initialize_weights, load_weights, save_weights, train)
from .estimator import (FnnSlowdownModel, SlowdownQuery, as_model, clamp_stats, corun_app_time,
                        corun_time, slowdown, solo_app_time, solorun_time)
from .hwopt import PairDecision, decide_pair, optimize_corun, optimize_solo_pair
from .matcher import PairGraph, brute_force_matching, matching_weight, min_weight_perfect_matching
from .scheduler import (SchedulerInput, build_graph, predicted_makespan, schedule,
                        schedule_to_json, set_time)
from .simenv import (OracleParams, OracleSlowdownModel, SyntheticJobSpec, generate_dataset,
                     generate_workload, mixed_archetypes, oracle_slowdown)
from .grid import KnobGrid

__all__ = [name for name in dir() if not name.startswith("_")]


def __getattr__(name):
    # sweep_pairs / SweepPlan import torch; keep `import paper_2405_03831_b200` light
    if name in ("sweep_pairs", "SweepResult", "plan_for"):
        from . import sweep
        return getattr(sweep, name)
    if name == "train_many":
        from .trainer import train_many
        return train_many
    if name == "SweepPlan":
        from .device import SweepPlan
        return SweepPlan
    raise AttributeError(name)
