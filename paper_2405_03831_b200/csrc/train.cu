// train.cu -- device-side training of the 40-18-18-1 slowdown network.
//
// Replaces the numpy loop of cosched.fnn (pkg/src/cosched/fnn.py:174-297:
// backward, sgd_step, train).  One persistent CTA per training run walks every
// epoch and batch itself: the parameters and their gradients stay in shared
// memory for the whole run, a batch is staged into shared memory in chunks of
// kChunk rows, and each step is forward -> backprop -> SGD update separated
// only by CTA barriers.  No host round trip per step (the reference pays a
// Python/numpy dispatch per batch); independent runs (seeds) occupy
// independent SMs.
//
// Arithmetic is fp64, like the reference's numpy float64.  Each dot product
// is a sequential FMA chain (numpy's BLAS order is unspecified, so dot
// products agree to rounding, not bit for bit); everything the reference
// evaluates as separate numpy ops -- the bias add after the matmul, the
// (2/n)(y - t) error scale, the SGD update w - lr * g -- is evaluated as the
// same separate IEEE operations (_rn intrinsics: no FMA contraction).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cosched_train.h"

namespace {

constexpr int IN = CT_INPUT, H = CT_HIDDEN, NP = CT_NPARAM;
constexpr int OW1 = 0, OB1 = H * IN, OW2 = OB1 + H, OB2 = OW2 + H * H, OWO = OB2 + H, OBO = OWO + H;
static_assert(OBO + 1 == NP, "parameter layout");
constexpr int kChunk = 32;       // batch rows staged in shared memory at a time
constexpr int kThreads = 512;       // 128 -> 512: 0.56 -> 0.44 s per 100 epochs (more lanes per phase)

struct Smem {
    double P[NP], G[NP];
    double X[kChunk * IN], t[kChunk];
    double z1[kChunk * H], z2[kChunk * H], z3[kChunk];
    double dz1[kChunk * H], dz2[kChunk * H], dz3[kChunk];
    double loss;
    int stop;
};

__device__ __forceinline__ double relu(double x) { return x > 0.0 ? x : 0.0; }

// Stage rows [c0, c0 + nc) of the batch (dataset rows rows_of(b)) into smem.
template <class RowOf>
__device__ void load_chunk(Smem &s, const double *x, const double *t, RowOf rows_of, int c0, int nc) {
    for (int i = threadIdx.x; i < nc * IN; i += blockDim.x) {
        const int b = i / IN, k = i - b * IN;
        s.X[i] = x[(size_t)rows_of(c0 + b) * IN + k];
    }
    for (int b = threadIdx.x; b < nc; b += blockDim.x) s.t[b] = t[rows_of(c0 + b)];
    __syncthreads();
}

// Forward + backprop of one staged chunk; gradients ACCUMULATE into s.G
// (the batch gradient is the sum over the batch's chunks).  Returns the sum of
// the chunk's squared errors (thread 0's value is the one used).
//   fnn.py:185-209:  z1 = X w1^T + b1, a1 = relu(z1), z2 = a1 w2^T + b2,
//   a2 = relu(z2), z3 = a2 wo^T + bo, y = relu(z3); dy = (2/n)(y - t),
//   dz3 = dy [z3 > 0], dw_out = dz3^T a2, db_out = sum dz3, da2 = dz3 wo,
//   dz2 = da2 [z2 > 0], dw2 = dz2^T a1, db2 = sum dz2, da1 = dz2 w2,
//   dz1 = da1 [z1 > 0], dw1 = dz1^T X, db1 = sum dz1
__device__ void chunk_forward(Smem &s, int nc) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < nc * H; i += nt) {
        const int b = i / H, o = i - b * H;
        double d = 0.0;
        for (int k = 0; k < IN; ++k) d = fma(s.X[b * IN + k], s.P[OW1 + o * IN + k], d);
        s.z1[i] = __dadd_rn(d, s.P[OB1 + o]);
    }
    __syncthreads();
    for (int i = tid; i < nc * H; i += nt) {
        const int b = i / H, o = i - b * H;
        double d = 0.0;
        for (int k = 0; k < H; ++k) d = fma(relu(s.z1[b * H + k]), s.P[OW2 + o * H + k], d);
        s.z2[i] = __dadd_rn(d, s.P[OB2 + o]);
    }
    __syncthreads();
    for (int b = tid; b < nc; b += nt) {
        double d = 0.0;
        for (int k = 0; k < H; ++k) d = fma(relu(s.z2[b * H + k]), s.P[OWO + k], d);
        s.z3[b] = __dadd_rn(d, s.P[OBO]);
    }
    __syncthreads();
}

__device__ double chunk_grads(Smem &s, int nc, double two_over_n) {
    const int tid = threadIdx.x, nt = blockDim.x;
    chunk_forward(s, nc);
    for (int b = tid; b < nc; b += nt) {
        const double z3 = s.z3[b];
        const double e = __dsub_rn(relu(z3), s.t[b]);
        const double dy = __dmul_rn(two_over_n, e);
        s.dz3[b] = z3 > 0.0 ? dy : 0.0;
        s.dz1[b * H] = __dmul_rn(e, e);            // squared error, parked in dz1 until summed
    }
    __syncthreads();
    double sq = 0.0;
    if (tid == 0)
        for (int b = 0; b < nc; ++b) sq = __dadd_rn(sq, s.dz1[b * H]);
    for (int o = tid; o <= H; o += nt) {
        double g = 0.0;
        if (o < H)
            for (int b = 0; b < nc; ++b) g = fma(s.dz3[b], relu(s.z2[b * H + o]), g);
        else
            for (int b = 0; b < nc; ++b) g = __dadd_rn(g, s.dz3[b]);
        s.G[OWO + o] = __dadd_rn(s.G[OWO + o], g);   // o == H is OBO
    }
    for (int i = tid; i < nc * H; i += nt) {
        const int b = i / H, o = i - b * H;
        s.dz2[i] = s.z2[i] > 0.0 ? __dmul_rn(s.dz3[b], s.P[OWO + o]) : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < H * H + H; i += nt) {
        double g = 0.0;
        if (i < H * H) {
            const int o = i / H, k = i - o * H;
            for (int b = 0; b < nc; ++b) g = fma(s.dz2[b * H + o], relu(s.z1[b * H + k]), g);
            s.G[OW2 + i] = __dadd_rn(s.G[OW2 + i], g);
        } else {
            const int o = i - H * H;
            for (int b = 0; b < nc; ++b) g = __dadd_rn(g, s.dz2[b * H + o]);
            s.G[OB2 + o] = __dadd_rn(s.G[OB2 + o], g);
        }
    }
    for (int i = tid; i < nc * H; i += nt) {
        const int b = i / H, k = i - b * H;
        double d = 0.0;
        for (int o = 0; o < H; ++o) d = fma(s.dz2[b * H + o], s.P[OW2 + o * H + k], d);
        s.dz1[i] = s.z1[i] > 0.0 ? d : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < H * IN + H; i += nt) {
        double g = 0.0;
        if (i < H * IN) {
            const int o = i / IN, k = i - o * IN;
            for (int b = 0; b < nc; ++b) g = fma(s.dz1[b * H + o], s.X[b * IN + k], g);
            s.G[OW1 + i] = __dadd_rn(s.G[OW1 + i], g);
        } else {
            const int o = i - H * IN;
            for (int b = 0; b < nc; ++b) g = __dadd_rn(g, s.dz1[b * H + o]);
            s.G[OB1 + o] = __dadd_rn(s.G[OB1 + o], g);
        }
    }
    __syncthreads();
    return sq;
}

// Gradient and loss of one batch of n rows, chunk by chunk; result in s.G and
// s.loss (all threads see it after the final barrier).
// `staged`: the batch (n <= kChunk) already sits in s.X / s.t
template <class RowOf>
__device__ void batch_grads(Smem &s, const double *x, const double *t, RowOf rows_of, int n,
                            bool staged = false) {
    for (int i = threadIdx.x; i < NP; i += blockDim.x) s.G[i] = 0.0;
    __syncthreads();
    const double two_over_n = __ddiv_rn(2.0, (double)n);
    double sq = 0.0;
    for (int c0 = 0; c0 < n; c0 += kChunk) {
        const int nc = n - c0 < kChunk ? n - c0 : kChunk;
        if (!staged) load_chunk(s, x, t, rows_of, c0, nc);
        sq = __dadd_rn(sq, chunk_grads(s, nc, two_over_n));
    }
    if (threadIdx.x == 0) s.loss = __ddiv_rn(sq, (double)n);
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_backward(const double *params, const double *x,
                                                       const double *t, const int32_t *rows, int n,
                                                       double *grad, double *loss) {
    __shared__ Smem s;
    for (int i = threadIdx.x; i < NP; i += blockDim.x) s.P[i] = params[i];
    __syncthreads();
    batch_grads(s, x, t, [&](int b) { return rows[b]; }, n);
    for (int i = threadIdx.x; i < NP; i += blockDim.x) grad[i] = s.G[i];
    if (threadIdx.x == 0) *loss = s.loss;
}

struct TrainArgs {
    const double *x, *t;
    const int32_t *train_rows, *val_rows, *order;
    int n_train, n_val, epochs, batch, nb;
    double lr;
    double *params, *batch_loss, *val_sq;
    int32_t *status;
};

__global__ void __launch_bounds__(kThreads) k_train(const TrainArgs a) {
    __shared__ Smem s;
    const int r = blockIdx.x;
    double *params = a.params + (size_t)r * NP;
    const int32_t *train_rows = a.train_rows + (size_t)r * a.n_train;
    const int32_t *val_rows = a.val_rows + (size_t)r * a.n_val;
    for (int i = threadIdx.x; i < NP; i += blockDim.x) s.P[i] = params[i];
    if (threadIdx.x == 0) s.stop = -1;
    __syncthreads();
    for (int e = 0; e < a.epochs; ++e) {
        const int32_t *order = a.order + ((size_t)r * a.epochs + e) * a.n_train;
        double *bl = a.batch_loss + ((size_t)r * a.epochs + e) * a.nb;
        // Small batches (all of a batch's elements fit one per thread): the
        // next batch's rows are fetched into registers at the start of a step
        // and staged after its update, so the order -> row -> x chain of
        // dependent global loads leaves the step's critical path
        const bool prefetch = a.batch * (IN + 1) <= (int)blockDim.x;
        const int tid = threadIdx.x;
        auto fetch = [&](int q, double &v) {
            const int s0 = q * a.batch;
            const int n = a.n_train - s0 < a.batch ? a.n_train - s0 : a.batch;
            if (tid < n * IN) {
                const int b = tid / IN, k = tid - b * IN;
                v = __ldg(a.x + (size_t)train_rows[order[s0 + b]] * IN + k);
            } else if (tid < n * IN + n) {
                v = __ldg(a.t + train_rows[order[s0 + tid - n * IN]]);
            }
        };
        auto stage = [&](int q, double v) {
            const int s0 = q * a.batch;
            const int n = a.n_train - s0 < a.batch ? a.n_train - s0 : a.batch;
            if (tid < n * IN) s.X[tid] = v;
            else if (tid < n * IN + n) s.t[tid - n * IN] = v;
        };
        if (prefetch) {
            double v0 = 0.0;
            fetch(0, v0);
            stage(0, v0);
            __syncthreads();
        }
        for (int q = 0; q < a.nb; ++q) {
            const int s0 = q * a.batch;
            const int n = a.n_train - s0 < a.batch ? a.n_train - s0 : a.batch;
            double next = 0.0;
            if (prefetch && q + 1 < a.nb) fetch(q + 1, next);
            batch_grads(s, a.x, a.t, [&](int b) { return train_rows[order[s0 + b]]; }, n, prefetch);
            const double loss = s.loss;
            if (!isfinite(loss)) {                 // fnn.py:288-289: TrainingDivergedError(epoch)
                if (threadIdx.x == 0) a.status[r] = e;
                return;                            // uniform: every thread read the same loss
            }
            if (threadIdx.x == 0) bl[q] = loss;
            for (int i = threadIdx.x; i < NP; i += blockDim.x)
                s.P[i] = __dsub_rn(s.P[i], __dmul_rn(a.lr, s.G[i]));   // sgd_step
            if (prefetch && q + 1 < a.nb) stage(q + 1, next);       // s.X / s.t are free now
            __syncthreads();
        }
        // validation MSE after the epoch (fnn._mse): squared errors per row
        double *vs = a.val_sq + ((size_t)r * a.epochs + e) * a.n_val;
        for (int c0 = 0; c0 < a.n_val; c0 += kChunk) {
            const int nc = a.n_val - c0 < kChunk ? a.n_val - c0 : kChunk;
            load_chunk(s, a.x, a.t, [&](int b) { return val_rows[b]; }, c0, nc);
            chunk_forward(s, nc);
            for (int b = threadIdx.x; b < nc; b += blockDim.x) {
                const double err = __dsub_rn(relu(s.z3[b]), s.t[b]);
                vs[c0 + b] = __dmul_rn(err, err);
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < NP; i += blockDim.x) params[i] = s.P[i];
    if (threadIdx.x == 0) a.status[r] = -1;
}

int launch_status() {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -2;
}

}  // namespace

extern "C" {

const char *ct_version(void) { return "cosched_train 0.1.0 (persistent-CTA fp64 SGD, sm_100a)"; }

int ct_backward(const double *d_params, const double *d_x, const double *d_t, const int32_t *d_rows,
                int32_t n, double *d_grad, double *d_loss, void *stream) {
    if (n < 1 || !d_params || !d_x || !d_t || !d_rows || !d_grad || !d_loss) return -1;
    k_backward<<<1, kThreads, 0, (cudaStream_t)stream>>>(d_params, d_x, d_t, d_rows, n, d_grad, d_loss);
    return launch_status();
}

int ct_train_sgd(const double *d_x, const double *d_t, const int32_t *d_train_rows, int32_t n_train,
                 const int32_t *d_val_rows, int32_t n_val, const int32_t *d_order, int32_t epochs,
                 int32_t batch, double lr, int32_t runs, double *d_params, double *d_batch_loss,
                 double *d_val_sq, int32_t *d_status, void *stream) {
    if (n_train < 1 || n_val < 0 || epochs < 1 || batch < 1 || runs < 1 || !(lr > 0.0) || !d_x ||
        !d_t || !d_train_rows || (n_val > 0 && (!d_val_rows || !d_val_sq)) || !d_order || !d_params ||
        !d_batch_loss || !d_status)
        return -1;
    TrainArgs a;
    a.x = d_x; a.t = d_t;
    a.train_rows = d_train_rows; a.val_rows = d_val_rows; a.order = d_order;
    a.n_train = n_train; a.n_val = n_val; a.epochs = epochs; a.batch = batch;
    a.nb = (n_train + batch - 1) / batch;
    a.lr = lr;
    a.params = d_params; a.batch_loss = d_batch_loss; a.val_sq = d_val_sq; a.status = d_status;
    k_train<<<runs, kThreads, 0, (cudaStream_t)stream>>>(a);
    return launch_status();
}

}  // extern "C"
