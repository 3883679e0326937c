"""Device-side training (csrc/train.cu) against the reference's own numbers.

Fixtures come from the unmodified reference (tests/golden/make_golden.py,
stages ``weights`` and ``training``).  The kernel evaluates every dot product
as a sequential fp64 FMA chain while numpy's BLAS picks its own order, so
gradients agree to rounding (REL_GRAD) and a training run agrees to the
accumulated rounding of its steps (REL_TRAIN); everything that does not go
through a dot product -- the replayed per-batch losses, train_many vs train,
the divergence epoch -- must agree exactly.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2405_03831_b200 import analytic, core, fnn, simenv

pytestmark = pytest.mark.gpu

REL_GRAD = 1e-12      # one backward pass: rounding of 40-term dot products
REL_TRAIN = 1e-9      # 20 epochs x 1,140 SGD steps
REL_ACCEPT = 1e-6     # the 400-epoch acceptance recipe (228k steps)
PARAMS = ("w1", "b1", "w2", "b2", "w_out", "b_out")

with open(os.path.join(GOLDEN, "training.json")) as fh:
    TRAINING = json.load(fh)


@pytest.fixture(scope="module")
def corpus():
    return simenv.generate_dataset(analytic.OracleParams(noise_sigma=0.0), core.default_space(400.0), seed=0)


def _rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("case", TRAINING["backward"], ids=lambda c: f"b{c['size']}")
def test_backward_matches_reference_gradients(corpus, case):
    w0 = fnn.initialize_weights(case["init_seed"], corpus.bounds)
    batch = corpus.samples("train")[case["start"]:case["start"] + case["size"]]
    g, loss = fnn.backward(w0, batch)
    assert abs(loss - case["loss"]) <= REL_GRAD * abs(case["loss"])
    for k in PARAMS:
        assert _rel(getattr(g, k), case[k]) <= REL_GRAD, k


def test_train_20_epochs_matches_reference(corpus):
    ref = TRAINING["train"]
    cfg = fnn.TrainingConfig(**ref["cfg"])
    w, hist = fnn.train(corpus.samples("train"), cfg, feature_bounds=corpus.bounds)
    assert [h.epoch for h in hist] == list(range(cfg.epochs))
    got = np.array([[h.train_mse, h.val_mse] for h in hist])
    want = np.array([[h[1], h[2]] for h in ref["history"]])
    assert _rel(got, want) <= REL_TRAIN
    for k in PARAMS:
        assert _rel(getattr(w, k), ref[k]) <= REL_TRAIN, k
    assert np.array_equal(w.feature_bounds, corpus.bounds)


def test_acceptance_recipe_reproduces_the_shipped_weights(corpus):
    """The 400-epoch recipe that produced tests/golden/weights.json with the
    reference (test_acceptance.py:144-157) reproduces it on the device."""
    ref = fnn.load_weights(os.path.join(GOLDEN, "weights.json"))
    cfg = fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=400, seed=2,
                             validation_fraction=0.05)
    w, hist = fnn.train(corpus.samples("train"), cfg, feature_bounds=corpus.bounds)
    for k in PARAMS:
        assert _rel(getattr(w, k), getattr(ref, k)) <= REL_ACCEPT, k
    assert hist[-1].train_mse < hist[0].train_mse


def test_train_many_equals_single_runs_bit_for_bit(corpus):
    from paper_2405_03831_b200.trainer import train_many
    data = corpus.samples("train")[:400]
    cfgs = [fnn.TrainingConfig(learning_rate=0.002, batch_size=3, epochs=4, seed=s) for s in (2, 7, 11)]
    many = train_many(data, cfgs, corpus.bounds)
    for cfg, (w, hist) in zip(cfgs, many):
        w1, h1 = fnn.train(data, cfg, feature_bounds=corpus.bounds)
        assert hist == h1
        for k in PARAMS:
            assert np.array_equal(getattr(w, k), getattr(w1, k)), k


def test_epoch_zero_replay_is_exact(corpus):
    """history[0].train_mse equals an independent replay with backward +
    sgd_step (fnn.py:247-257) -- the kernel's step IS backward + w - lr * g."""
    data = corpus.samples("train")[:60]
    cfg = fnn.TrainingConfig(epochs=1, seed=9, batch_size=5, learning_rate=0.01)
    _, hist = fnn.train(data, cfg)
    tr, _ = fnn.split_dataset(data, cfg)
    w = fnn.initialize_weights(cfg.seed, np.ones(36))
    order = fnn.epoch_batch_order(cfg, len(tr), 0)
    losses = []
    for s in range(0, len(order), cfg.batch_size):
        g, loss = fnn.backward(w, [tr[i] for i in order[s:s + cfg.batch_size]])
        losses.append(loss)
        w = fnn.sgd_step(w, g, cfg.learning_rate)
    assert hist[0].train_mse == float(np.mean(losses))


def test_divergence_reports_the_epoch():
    rng = np.random.default_rng(0)
    data = [fnn.LabeledSample(rng.uniform(0, 1, 40), 1e200) for _ in range(16)]
    with pytest.raises(fnn.TrainingDivergedError, match="epoch 0") as exc:
        fnn.train(data, fnn.TrainingConfig(epochs=50, seed=0))
    assert exc.value.epoch == 0


def test_memorizes_a_single_point_and_large_batches():
    x = np.zeros(40)
    x[0] = 0.5
    _, hist = fnn.train([fnn.LabeledSample(x, 1.5)] * 5, fnn.TrainingConfig(epochs=400, learning_rate=0.01))
    assert hist[-1].train_mse < 1e-4
    # a batch larger than the kernel's shared-memory chunk (32 rows)
    rng = np.random.default_rng(1)
    data = [fnn.LabeledSample(rng.uniform(0, 1, 40), float(rng.uniform(1, 2))) for _ in range(200)]
    cfg = fnn.TrainingConfig(epochs=2, batch_size=77, seed=4, learning_rate=0.01)
    _, hist = fnn.train(data, cfg)
    tr, _ = fnn.split_dataset(data, cfg)
    g, loss = fnn.backward(fnn.initialize_weights(4, np.ones(36)),
                           [tr[i] for i in fnn.epoch_batch_order(cfg, len(tr), 0)[:77]])
    assert np.isfinite(loss) and np.isfinite(hist[-1].train_mse)
