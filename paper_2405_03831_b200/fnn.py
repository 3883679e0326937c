"""The 40-18-18-1 slowdown regressor: parameters, persistence and inference.

Mirrors ``cosched.fnn`` (``pkg/src/cosched/fnn.py``) for what the sweep needs:
``NetworkWeights`` (fnn.py:42-68), the versioned JSON document
(``save_weights``/``load_weights``, fnn.py:311-359), seeded Glorot init
(fnn.py:122-143) and inference (``forward``/``forward_batch``,
fnn.py:146-165).  Inference runs on the GPU through the C ABI
(``cs_forward_rows``), in fp64, with no CPU fallback.

Training mirrors fnn.py:23-28, 71-119 and 168-308 (``TrainingConfig``,
``LabeledSample``, ``Gradients``, ``EpochStats``, ``split_dataset``,
``epoch_batch_order``, ``sgd_step``, ``backward``, ``train``,
``write_loss_csv``): the seeded split / permutations / init are the
reference's numpy draws (host), while every gradient step runs on the GPU --
``backward`` as one kernel launch, ``train`` as ONE persistent kernel per run
that walks all epochs and batches with the parameters resident in shared
memory (``csrc/train.cu``, ``include/cosched_train.h``).  ``train_many``
trains several seeds concurrently, one SM each.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .core import INPUT_DIM, NUM_FEATURES, ValidationError

HIDDEN_DIM = 18
WEIGHTS_FORMAT_VERSION = 1


def _param(name: str, value, shape) -> np.ndarray:
    arr = np.array(value, dtype=np.float64, copy=True)
    if arr.shape != shape:
        raise ValidationError(f"{name} must have shape {shape}, got {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValidationError(f"{name} contains non-finite entries")
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class NetworkWeights:
    """Dense layer parameters plus the normalization maxima they were trained with."""

    w1: np.ndarray          # (18, 40)
    b1: np.ndarray          # (18,)
    w2: np.ndarray          # (18, 18)
    b2: np.ndarray          # (18,)
    w_out: np.ndarray       # (1, 18)
    b_out: np.ndarray       # (1,)
    feature_bounds: np.ndarray  # (36,)

    def __post_init__(self) -> None:
        spec = (("w1", "layer_1 weights", (HIDDEN_DIM, INPUT_DIM)),
                ("b1", "layer_1 biases", (HIDDEN_DIM,)),
                ("w2", "layer_2 weights", (HIDDEN_DIM, HIDDEN_DIM)),
                ("b2", "layer_2 biases", (HIDDEN_DIM,)),
                ("w_out", "output weights", (1, HIDDEN_DIM)),
                ("b_out", "output biases", (1,)),
                ("feature_bounds", "feature_bounds", (2 * NUM_FEATURES,)))
        for attr, label, shape in spec:
            object.__setattr__(self, attr, _param(label, getattr(self, attr), shape))
        if (self.feature_bounds <= 0).any():
            raise ValidationError("feature_bounds entries must be > 0")

    # contiguous fp64 views handed to the C ABI (cs_network)
    def abi_arrays(self) -> dict:
        return {k: np.ascontiguousarray(getattr(self, k), dtype=np.float64)
                for k in ("w1", "b1", "w2", "b2", "w_out", "b_out", "feature_bounds")}


def initialize_weights(seed: int, feature_bounds) -> NetworkWeights:
    """Seeded Glorot-uniform init; hidden biases 0, output bias 1 (fnn.py:122-143)."""
    rng = np.random.default_rng(seed)

    def glorot(rows: int, cols: int) -> np.ndarray:
        lim = np.sqrt(6.0 / (rows + cols))
        return rng.uniform(-lim, lim, size=(rows, cols))

    w1 = glorot(HIDDEN_DIM, INPUT_DIM)
    w2 = glorot(HIDDEN_DIM, HIDDEN_DIM)
    wo = glorot(1, HIDDEN_DIM)
    return NetworkWeights(w1, np.zeros(HIDDEN_DIM), w2, np.zeros(HIDDEN_DIM), wo, np.ones(1),
                          feature_bounds)


def save_weights(weights: NetworkWeights, path) -> None:
    """Write the version-1 JSON document (fnn.py:311-324)."""
    doc = {
        "version": WEIGHTS_FORMAT_VERSION,
        "input_dim": INPUT_DIM,
        "hidden_dim": HIDDEN_DIM,
        "layer_1": {"weights": weights.w1.tolist(), "biases": weights.b1.tolist()},
        "layer_2": {"weights": weights.w2.tolist(), "biases": weights.b2.tolist()},
        "output": {"weights": weights.w_out.tolist(), "biases": weights.b_out.tolist()},
        "feature_bounds": weights.feature_bounds.tolist(),
    }
    with open(path, "w") as fh:
        json.dump(doc, fh)
        fh.write("\n")


def load_weights(path) -> NetworkWeights:
    """Read and validate a weight document; lossless inverse of save_weights."""
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except (json.JSONDecodeError, UnicodeDecodeError) as exc:
        raise ValidationError(f"weights file {path} is not valid JSON: {exc}") from exc
    if not isinstance(doc, dict):
        raise ValidationError(f"weights file {path} must hold a JSON object")
    if doc.get("version") != WEIGHTS_FORMAT_VERSION:
        raise ValidationError(f"unsupported weights format version {doc.get('version')!r} "
                              f"(expected {WEIGHTS_FORMAT_VERSION})")
    try:
        fields = (doc["layer_1"]["weights"], doc["layer_1"]["biases"],
                  doc["layer_2"]["weights"], doc["layer_2"]["biases"],
                  doc["output"]["weights"], doc["output"]["biases"], doc["feature_bounds"])
    except KeyError as exc:
        raise ValidationError(f"weights file {path} is missing field {exc}") from exc
    try:
        return NetworkWeights(*(np.asarray(f, dtype=float) for f in fields))
    except ValueError as exc:
        if isinstance(exc, ValidationError):
            raise
        raise ValidationError(f"weights file {path} has a malformed array: {exc}") from exc


def forward_batch(weights: NetworkWeights, X) -> np.ndarray:
    """ReLU(w_out ReLU(W2 ReLU(W1 x + b1) + b2) + b_out) for a (batch, 40) matrix,
    evaluated on the GPU in fp64 (fnn.py:161-165)."""
    from .device import forward_rows
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != INPUT_DIM:
        raise ValidationError(f"input must have shape (batch, {INPUT_DIM}), got {X.shape}")
    return forward_rows(weights, X)


def forward(weights: NetworkWeights, x) -> float:
    """One input vector (fnn.py:146-158): shape and finiteness checked first."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (INPUT_DIM,):
        raise ValidationError(f"input must have {INPUT_DIM} entries, got {x.shape}")
    bad = ~np.isfinite(x)
    if bad.any():
        raise ValidationError(f"input entry {int(np.argmax(bad))} is not finite")
    return float(forward_batch(weights, x[None, :])[0])


# ---------------------------------------------------------------------------
# training (fnn.py:23-28, 71-119, 168-308)
# ---------------------------------------------------------------------------

class TrainingDivergedError(RuntimeError):
    """Raised when the training loss stops being finite (fnn.py:23-28)."""

    def __init__(self, epoch: int):
        super().__init__(f"training loss became non-finite at epoch {epoch}")
        self.epoch = epoch


@dataclass(frozen=True)
class TrainingConfig:
    """SGD hyperparameters; defaults follow the standard recipe (fnn.py:71-89)."""

    learning_rate: float = 0.001
    batch_size: int = 4
    epochs: int = 200
    seed: int = 0
    validation_fraction: float = 0.2

    def __post_init__(self) -> None:
        if self.learning_rate <= 0:
            raise ValidationError("learning_rate must be > 0")
        if self.batch_size < 1:
            raise ValidationError("batch_size must be >= 1")
        if self.epochs < 1:
            raise ValidationError("epochs must be >= 1")
        if not 0.0 < self.validation_fraction < 1.0:
            raise ValidationError("validation_fraction must be in (0, 1)")


@dataclass(frozen=True)
class LabeledSample:
    """One normalized 40-vector input and its slowdown target (fnn.py:92-107)."""

    input: np.ndarray
    target: float

    def __post_init__(self) -> None:
        x = np.asarray(self.input, dtype=float)
        if x.shape != (INPUT_DIM,):
            raise ValidationError(f"sample input must have {INPUT_DIM} entries, got {x.shape}")
        x = x.copy()
        x.setflags(write=False)
        object.__setattr__(self, "input", x)
        if not np.isfinite(self.target):
            raise ValidationError("sample target must be finite")


@dataclass
class Gradients:
    """Parameter gradients, congruent with NetworkWeights (fnn.py:110-119)."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray


@dataclass(frozen=True)
class EpochStats:
    epoch: int
    train_mse: float
    val_mse: float


_PARAM_SHAPES = (("w1", (HIDDEN_DIM, INPUT_DIM)), ("b1", (HIDDEN_DIM,)),
                 ("w2", (HIDDEN_DIM, HIDDEN_DIM)), ("b2", (HIDDEN_DIM,)),
                 ("w_out", (1, HIDDEN_DIM)), ("b_out", (1,)))
N_PARAMS = sum(int(np.prod(s)) for _, s in _PARAM_SHAPES)     # CT_NPARAM = 1099


def flat_params(weights) -> np.ndarray:
    """The flat fp64 parameter vector of include/cosched_train.h."""
    return np.concatenate([np.asarray(getattr(weights, k), dtype=np.float64).ravel()
                           for k, _ in _PARAM_SHAPES])


def _split_params(vec: np.ndarray) -> dict:
    out, i = {}, 0
    for k, shape in _PARAM_SHAPES:
        size = int(np.prod(shape))
        out[k] = np.array(vec[i:i + size]).reshape(shape)
        i += size
    return out


def weights_from_flat(vec: np.ndarray, feature_bounds) -> NetworkWeights:
    return NetworkWeights(feature_bounds=feature_bounds, **_split_params(vec))


def split_dataset(dataset: Sequence[LabeledSample], cfg: TrainingConfig):
    """Seeded shuffle split into (train, validation) lists (fnn.py:219-231)."""
    rng = np.random.default_rng([cfg.seed, 0])
    order = rng.permutation(len(dataset))
    n_val = int(len(dataset) * cfg.validation_fraction)
    return [dataset[i] for i in order[n_val:]], [dataset[i] for i in order[:n_val]]


def epoch_batch_order(cfg: TrainingConfig, n_train: int, epoch: int) -> np.ndarray:
    """The deterministic sample permutation of one epoch (fnn.py:234-237)."""
    rng = np.random.default_rng([cfg.seed, 1 + epoch])
    return rng.permutation(n_train)


def sgd_step(weights: NetworkWeights, grads: Gradients, lr: float) -> NetworkWeights:
    """One plain SGD update; fresh weights, inputs untouched (fnn.py:247-257)."""
    return NetworkWeights(
        w1=weights.w1 - lr * grads.w1, b1=weights.b1 - lr * grads.b1,
        w2=weights.w2 - lr * grads.w2, b2=weights.b2 - lr * grads.b2,
        w_out=weights.w_out - lr * grads.w_out, b_out=weights.b_out - lr * grads.b_out,
        feature_bounds=weights.feature_bounds)


def backward(weights: NetworkWeights, batch: Sequence[LabeledSample]):
    """Gradients of the batch mean squared error plus the loss (fnn.py:174-210),
    computed on the GPU (ct_backward).  The ReLU subgradient at 0 is 0."""
    if len(batch) == 0:
        raise ValidationError("backward needs a nonempty batch")
    from .trainer import device_backward
    g, loss = device_backward(weights, batch)
    return Gradients(**_split_params(g)), loss


def train(dataset: Sequence[LabeledSample], cfg: TrainingConfig, feature_bounds=None):
    """Mini-batch SGD training, bit-reproducible for a fixed seed (fnn.py:260-297).

    Same split, init and per-epoch permutations as the reference (its numpy
    draws); the epochs themselves run as one persistent GPU kernel.  The
    per-epoch train MSE averages the batch losses as seen before each update,
    the validation MSE is taken after the epoch.

    Raises:
        TrainingDivergedError: when a batch loss stops being finite.
    """
    from .trainer import train_many
    return train_many(dataset, [cfg], feature_bounds)[0]


def write_loss_csv(history: Sequence[EpochStats], path) -> None:
    """Training log: one row per epoch (fnn.py:362-369)."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["epoch", "train_mse", "val_mse"])
        for row in history:
            writer.writerow([row.epoch, repr(row.train_mse), repr(row.val_mse)])
