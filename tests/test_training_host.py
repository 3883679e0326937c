"""Training-corpus generation and the host side of training, against the
reference's fixtures (tests/golden/make_golden.py stage ``training``). CPU."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2405_03831_b200 import analytic, core, fnn, simenv
from paper_2405_03831_b200.core import ValidationError

with open(os.path.join(GOLDEN, "training.json")) as fh:
    TRAINING = json.load(fh)


@pytest.mark.parametrize("case", TRAINING["datasets"], ids=lambda c: f"s{c['noise_sigma']}_{c['p_total']}")
def test_dataset_csv_bytes_equal_the_reference(case, tmp_path):
    """generate_dataset + dataset_to_csv reproduce the reference's corpus byte
    for byte (simenv.py:393-469): seeded pair picks, oracle labels, noise draws,
    bounds and normalization."""
    ds = simenv.generate_dataset(analytic.OracleParams(noise_sigma=case["noise_sigma"], seed=case["seed"]),
                                 core.default_space(case["p_total"]))
    assert len(ds.rows) == case["rows"]
    path = tmp_path / "d.csv"
    simenv.dataset_to_csv(ds, path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == case["csv_sha256"]
    samples, pair_ids, splits = simenv.load_dataset_csv(path)
    assert len(samples) == len(ds.rows)
    assert all(np.array_equal(a.input, r.sample.input) and a.target == r.sample.target
               for a, r in zip(samples, ds.rows))
    assert set(splits) == {"train", "test"}
    assert not {p for p, s in zip(pair_ids, splits) if s == "train"} & \
        {p for p, s in zip(pair_ids, splits) if s == "test"}


def test_dataset_argument_checks():
    p = analytic.OracleParams()
    sp = core.default_space(400.0)
    with pytest.raises(ValidationError):
        simenv.generate_dataset(p, sp, n_pairs=0)
    with pytest.raises(ValidationError):
        simenv.generate_dataset(p, sp, n_jobs=4, n_pairs=7)
    with pytest.raises(ValidationError):
        simenv.generate_dataset(p, sp, n_pairs=4, train_pairs=4)


def test_training_config_and_sample_validation():
    for bad in ({"learning_rate": 0.0}, {"batch_size": 0}, {"epochs": 0},
                {"validation_fraction": 1.0}):
        with pytest.raises(ValidationError):
            fnn.TrainingConfig(**bad)
    with pytest.raises(ValidationError):
        fnn.LabeledSample(np.zeros(39), 1.0)
    with pytest.raises(ValidationError):
        fnn.LabeledSample(np.zeros(40), float("nan"))
    s = fnn.LabeledSample(np.zeros(40), 1.0)
    assert not s.input.flags.writeable


def test_split_and_epoch_orders_are_the_reference_draws():
    data = [fnn.LabeledSample(np.full(40, k / 10.0), 1.0) for k in range(10)]
    cfg = fnn.TrainingConfig(seed=3, validation_fraction=0.3)
    tr, va = fnn.split_dataset(data, cfg)
    order = np.random.default_rng([3, 0]).permutation(10)
    assert [id(s) for s in va] == [id(data[i]) for i in order[:3]]
    assert [id(s) for s in tr] == [id(data[i]) for i in order[3:]]
    assert np.array_equal(fnn.epoch_batch_order(cfg, 7, 4), np.random.default_rng([3, 5]).permutation(7))


def test_flat_parameter_layout_roundtrip():
    w = fnn.initialize_weights(4, np.ones(36))
    v = fnn.flat_params(w)
    assert v.shape == (fnn.N_PARAMS,) == (1099,)
    again = fnn.weights_from_flat(v, w.feature_bounds)
    for k in ("w1", "b1", "w2", "b2", "w_out", "b_out"):
        assert np.array_equal(getattr(w, k), getattr(again, k))


def test_sgd_step_and_loss_csv(tmp_path):
    w = fnn.initialize_weights(1, np.ones(36))
    g = fnn.Gradients(**{k: np.ones_like(getattr(w, k)) for k in ("w1", "b1", "w2", "b2", "w_out", "b_out")})
    w2 = fnn.sgd_step(w, g, 0.5)
    assert np.array_equal(w2.w1, w.w1 - 0.5) and np.array_equal(w2.b_out, w.b_out - 0.5)
    path = tmp_path / "loss.csv"
    fnn.write_loss_csv([fnn.EpochStats(0, 1.5, 1.25), fnn.EpochStats(1, 0.5, 0.75)], path)
    assert path.read_text().splitlines()[:2] == ["epoch,train_mse,val_mse", "0,1.5,1.25"]


def test_training_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: the device path is exercised by test_training_gpu.py")
    data = [fnn.LabeledSample(np.zeros(40), 1.0)] * 5
    with pytest.raises(RuntimeError, match="CUDA"):
        fnn.train(data, fnn.TrainingConfig(epochs=1))
    with pytest.raises(RuntimeError, match="CUDA"):
        fnn.backward(fnn.initialize_weights(0, np.ones(36)), data[:2])
