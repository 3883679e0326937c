"""The 40-18-18-1 slowdown regressor: parameters, persistence and inference.

Mirrors ``cosched.fnn`` (``pkg/src/cosched/fnn.py``) for what the sweep needs:
``NetworkWeights`` (fnn.py:42-68), the versioned JSON document
(``save_weights``/``load_weights``, fnn.py:311-359), seeded Glorot init
(fnn.py:122-143) and inference (``forward``/``forward_batch``,
fnn.py:146-165).  Inference runs on the GPU through the C ABI
(``cs_forward_rows``), in fp64, with no CPU fallback.  Training (backprop,
SGD, dataset split; fnn.py:168-308) is out of scope for this build: it is
offline, ~50 s on a CPU and not on the sweep path.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

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
