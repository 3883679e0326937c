"""GPU driver of the training API (fnn.backward / fnn.train / train_many).

The reference trains with a numpy loop, one Python dispatch per batch
(``pkg/src/cosched/fnn.py:260-297``).  Here the host only reproduces the
reference's seeded draws -- the train/validation split (fnn.py:219-231), the
Glorot init (fnn.py:122-143) and every epoch's permutation (fnn.py:234-237)
-- uploads them once, and ``ct_train_sgd`` (csrc/train.cu) runs every epoch
and batch of a run inside ONE persistent CTA with the parameters resident in
shared memory.  Several runs (seeds) train concurrently, one CTA each.  The
per-batch losses and per-row validation errors come back to the host, which
averages them with numpy exactly as the reference's ``EpochStats`` does.
There is no CPU fallback: a missing extension or device raises.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from . import _native as nat
from .core import INPUT_DIM, NUM_FEATURES, ValidationError
from .fnn import (N_PARAMS, EpochStats, LabeledSample, TrainingConfig, TrainingDivergedError,
                  epoch_batch_order, flat_params, initialize_weights, split_dataset,
                  weights_from_flat)


def _check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc == -1:
        raise ValidationError(f"{what}: invalid argument")
    raise RuntimeError(f"{what}: CUDA error (code {rc})")


def _stack(samples: Sequence[LabeledSample]):
    X = np.ascontiguousarray(np.stack([s.input for s in samples]), dtype=np.float64)
    t = np.ascontiguousarray([float(s.target) for s in samples], dtype=np.float64)
    return X, t


def device_backward(weights, batch: Sequence[LabeledSample]):
    """(flat gradient, loss) of one batch via ct_backward."""
    import torch
    from .device import require_cuda
    dev = require_cuda()
    X, t = _stack(batch)
    d_p = torch.as_tensor(flat_params(weights)).to(dev)
    d_x, d_t = torch.as_tensor(X).to(dev), torch.as_tensor(t).to(dev)
    d_rows = torch.arange(len(batch), dtype=torch.int32, device=dev)
    d_g = torch.empty(N_PARAMS, dtype=torch.float64, device=dev)
    d_loss = torch.empty(1, dtype=torch.float64, device=dev)
    _check(nat.train_lib().ct_backward(d_p.data_ptr(), d_x.data_ptr(), d_t.data_ptr(),
                                       d_rows.data_ptr(), len(batch), d_g.data_ptr(),
                                       d_loss.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
           "ct_backward")
    return d_g.cpu().numpy(), float(d_loss.cpu().numpy()[0])


def train_many(dataset: Sequence[LabeledSample], cfgs: Sequence[TrainingConfig],
               feature_bounds=None):
    """``fnn.train`` for several configs at once -- one CTA per config.

    The configs must share ``learning_rate``, ``batch_size``, ``epochs`` and
    ``validation_fraction`` (one kernel launch); ``seed`` may differ.  Returns
    one ``(weights, history)`` per config, each equal to what ``fnn.train``
    returns for it; a diverged run raises ``TrainingDivergedError`` (the first
    one in config order)."""
    import torch
    from .device import require_cuda
    if len(dataset) == 0:
        raise ValidationError("training dataset must be nonempty")
    if not cfgs:
        return []
    c0 = cfgs[0]
    for c in cfgs:
        if (c.learning_rate, c.batch_size, c.epochs, c.validation_fraction) != \
                (c0.learning_rate, c0.batch_size, c0.epochs, c0.validation_fraction):
            raise ValidationError("train_many: configs may differ only in seed")
    if feature_bounds is None:
        feature_bounds = np.ones(2 * NUM_FEATURES)
    index = {id(s): k for k, s in enumerate(dataset)}
    runs = []
    for c in cfgs:
        tr, va = split_dataset(dataset, c)
        if not tr:
            raise ValidationError("validation_fraction leaves no training samples")
        runs.append((tr, va))
    n_train, n_val = len(runs[0][0]), len(runs[0][1])
    R, E, B = len(cfgs), c0.epochs, c0.batch_size
    nb = (n_train + B - 1) // B
    X, t = _stack(dataset)
    train_rows = np.empty((R, n_train), dtype=np.int32)
    val_rows = np.empty((R, max(n_val, 1)), dtype=np.int32)
    order = np.empty((R, E, n_train), dtype=np.int32)
    params = np.empty((R, N_PARAMS), dtype=np.float64)
    for r, (c, (tr, va)) in enumerate(zip(cfgs, runs)):
        train_rows[r] = [index[id(s)] for s in tr]
        if n_val:
            val_rows[r] = [index[id(s)] for s in va]
        for e in range(E):
            order[r, e] = epoch_batch_order(c, n_train, e)
        params[r] = flat_params(initialize_weights(c.seed, feature_bounds))
    dev = require_cuda()
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
    d_x, d_t, d_tr, d_va, d_ord, d_par = d(X), d(t), d(train_rows), d(val_rows), d(order), d(params)
    d_bl = torch.empty((R, E, nb), dtype=torch.float64, device=dev)
    d_vs = torch.empty((R, E, max(n_val, 1)), dtype=torch.float64, device=dev)
    d_st = torch.empty(R, dtype=torch.int32, device=dev)
    _check(nat.train_lib().ct_train_sgd(
        d_x.data_ptr(), d_t.data_ptr(), d_tr.data_ptr(), n_train, d_va.data_ptr(), n_val,
        d_ord.data_ptr(), E, B, float(c0.learning_rate), R, d_par.data_ptr(), d_bl.data_ptr(),
        d_vs.data_ptr(), d_st.data_ptr(), torch.cuda.current_stream(dev).cuda_stream), "ct_train_sgd")
    status = d_st.cpu().numpy()
    bl, vs, par = d_bl.cpu().numpy(), d_vs.cpu().numpy(), d_par.cpu().numpy()
    out = []
    for r in range(R):
        if status[r] >= 0:
            raise TrainingDivergedError(int(status[r]))
        hist = [EpochStats(epoch=e, train_mse=float(np.mean(bl[r, e])),
                           val_mse=float(np.mean(vs[r, e, :n_val])) if n_val else float("nan"))
                for e in range(E)]
        out.append((weights_from_flat(par[r], feature_bounds), hist))
    return out
