/*
 * cosched_train.h -- C ABI of the device-side trainer of the slowdown network.
 *
 * Replaces the reference's numpy training loop (cosched.fnn, pkg/src/cosched/
 * fnn.py:174-297: backward, sgd_step, train) with one persistent CUDA kernel
 * per training run: the whole epoch x batch loop (forward, backprop, SGD
 * update) runs on the device in fp64, the parameters live in shared memory
 * and never leave the SM until the run ends.  Independent runs (e.g. seeds)
 * train concurrently, one CTA each.
 *
 * Parameters are a flat fp64 vector of CT_NPARAM entries in the order
 *   w1 (18 x 40, row-major) | b1 (18) | w2 (18 x 18) | b2 (18) | w_out (18) | b_out (1)
 * which is the field order of fnn.NetworkWeights.
 *
 * All pointers are device pointers; every call is asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default stream).  Return codes are those of
 * cosched_b200.h (CS_OK = 0, CS_ERR_ARG = -1, CS_ERR_CUDA = -2).
 */
#ifndef COSCHED_TRAIN_H
#define COSCHED_TRAIN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define CT_INPUT 40
#define CT_HIDDEN 18
#define CT_NPARAM (CT_HIDDEN * CT_INPUT + CT_HIDDEN + CT_HIDDEN * CT_HIDDEN + CT_HIDDEN + CT_HIDDEN + 1)

const char *ct_version(void);

/* Gradients of the batch mean squared error and the loss itself
 * (fnn.backward, fnn.py:174-210): rows d_x[d_rows[b]] (b < n) of the
 * (.. x 40) input matrix with targets d_t[d_rows[b]].  d_grad gets CT_NPARAM
 * entries in the parameter order, d_loss one double.  The ReLU subgradient at
 * exactly 0 is 0.  n >= 1. */
int ct_backward(const double *d_params, const double *d_x, const double *d_t,
                const int32_t *d_rows, int32_t n, double *d_grad, double *d_loss, void *stream);

/* Mini-batch SGD (fnn.train, fnn.py:240-297) for `runs` independent runs, one
 * CTA each.  Run r:
 *   d_params[r * CT_NPARAM ..]           in: initial weights, out: trained weights
 *   d_train_rows[r * n_train + i]        dataset row of training position i
 *   d_val_rows[r * n_val + i]            dataset row of validation position i
 *   d_order[(r * epochs + e) * n_train + s]  training position visited s-th in epoch e
 *   d_batch_loss[(r * epochs + e) * nb + q]  loss of batch q of epoch e (before its
 *                                        update), nb = ceil(n_train / batch)
 *   d_val_sq[(r * epochs + e) * n_val + i]   squared validation error after epoch e
 *   d_status[r]                          -1, or the epoch whose batch loss stopped
 *                                        being finite (the run stops there, as
 *                                        TrainingDivergedError does)
 * Each step applies w <- w - lr * grad per entry (sgd_step, fnn.py:230-238),
 * without FMA contraction.  The host averages the per-batch losses and the
 * per-row squared errors the way numpy does (EpochStats). */
int ct_train_sgd(const double *d_x, const double *d_t, const int32_t *d_train_rows, int32_t n_train,
                 const int32_t *d_val_rows, int32_t n_val, const int32_t *d_order, int32_t epochs,
                 int32_t batch, double lr, int32_t runs, double *d_params, double *d_batch_loss,
                 double *d_val_sq, int32_t *d_status, void *stream);

#ifdef __cplusplus
}
#endif
#endif
