// sweep.cu -- sm_100a kernels + C ABI for the pair x knob sweep (include/cosched_b200.h).
//
// Pipeline per build_graph (scheduler.py:52-78), all stream-ordered:
//   k_tables   factored layer-1 partials (fp64 + fp32 copies), one thread per row
//   k_solo     per (budget, app) best exclusive split (estimator.py:139-180), fp64
//   k_sweep    per (pair, config-slice) fp32 screen of every co-run config:
//              z1 = (A_i + B_j) + K_c  ->  ReLU -> W2 (parameter bank) -> ReLU ->
//              head -> floor 0.5 (estimator.py:98-109) -> x base_time -> max over
//              members (estimator.py:127-129) -> per-budget (min, first index,
//              runner-up) -> shuffle merge across slices -> fp64 re-evaluation of
//              the winner -> co-run/solo decision (hwopt.py:77-87).  Raw
//              predictions never leave registers.
//   k_resolve  exact fp64 first-index argmin for the (rare) pairs whose fp32
//              runner-up is within rel_eps of the minimum (hwopt.py:59 ties).
//   k_scatter  symmetric N x N weights for PairGraph (scheduler.py:73-77).
//
// fp64 arithmetic uses explicit fma() in the same order as oracle/cosched_oracle.c,
// so fp64 outputs are bit-identical to the C restatement of the reference.
#include "cosched_b200.h"

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstddef>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace {

constexpr int NF = CS_NUM_FEATURES;
constexpr int HD = CS_HIDDEN;
constexpr int IN = CS_INPUT_DIM;
constexpr int ROW32 = 20;                  // fp32 table row: 18 + 2 pad (80 B, float4-aligned)
constexpr int KROW32 = 2 * ROW32;          // row stride of the interleaved K1|K2 fp32 knob table
constexpr int W2_TILE_ELEMS = 4 * 32 * 16; // fp16 B operands: 4 K-slices of W2 (tcgen05_util.cuh)
constexpr double FLOOR = 0.5;              // estimator.py:33
constexpr int kSweepThreads = 128;

// ---- kernel-parameter-bank network images ---------------------------------
struct Net64P {          // 9.1 KB: needs the >4 KB kernel-parameter space (CUDA >= 12.1)
    double w1[HD * IN];
    double b1[HD];
    double w2[HD * HD];
    double b2[HD];
    double wo[HD];
    double bo;
    double bounds[2 * NF];
    double pad_;          // 16-B multiple: the image's w1t / w2t copies stay bulk-copyable
};

struct Net32P {          // fp32 screen: W2 as FFMA constant-bank operands
    float w2[HD * HD];
    float b2[HD];
    float wo[HD];
    float bo;
};

struct GridP {
    const double *knob1, *knob2, *solo_knob;
    const uint32_t *mask;
    int32_t G, L, S;
    int32_t solo_off[CS_MAX_BUDGETS + 1];
};

GridP grid_params(const cs_grid *g) {
    GridP p;
    p.knob1 = g->knob1; p.knob2 = g->knob2; p.solo_knob = g->solo_knob; p.mask = g->mask;
    p.G = g->n_grid; p.L = g->n_budgets; p.S = g->solo_offsets[g->n_budgets];
    for (int l = 0; l <= CS_MAX_BUDGETS; ++l) p.solo_off[l] = l <= g->n_budgets ? g->solo_offsets[l] : p.S;
    return p;
}

bool net64_from(const cs_network *net, Net64P *p) {
    if (!net || !net->w1 || !net->b1 || !net->w2 || !net->b2 || !net->w_out || !net->b_out ||
        !net->feature_bounds)
        return false;
    memcpy(p->w1, net->w1, sizeof(p->w1));
    memcpy(p->b1, net->b1, sizeof(p->b1));
    memcpy(p->w2, net->w2, sizeof(p->w2));
    memcpy(p->b2, net->b2, sizeof(p->b2));
    memcpy(p->wo, net->w_out, sizeof(p->wo));
    p->bo = net->b_out[0];
    memcpy(p->bounds, net->feature_bounds, sizeof(p->bounds));
    p->pad_ = 0.0;
    return true;
}

// ---- pair index <-> (i, j), row-major i < j (scheduler.py:61) -------------
__host__ __device__ __forceinline__ int64_t row_start(int64_t i, int64_t n) {
    return i * (2 * n - i - 1) / 2;
}

__device__ __forceinline__ void pair_of(int64_t p, int n, int &i, int &j) {
    double b = 2.0 * n - 1.0;
    double disc = b * b - 8.0 * (double)p;
    int ii = (int)floor((b - sqrt(fmax(disc, 0.0))) * 0.5);
    ii = max(0, min(ii, n - 2));
    while (ii > 0 && row_start(ii, n) > p) --ii;
    while (ii < n - 2 && row_start(ii + 1, n) <= p) ++ii;
    i = ii;
    j = (int)(p - row_start(ii, n)) + ii + 1;
}

// ---- fp64 exact path (mirrors orc_head in oracle/cosched_oracle.c) --------
// The fp64 head weights ride in the kernel parameter bank (DFMA constant
// operands, no loads).  Loop order k-outer / o-inner keeps 18 independent
// accumulation chains in flight while every chain still sums over k in the
// oracle's order, so results stay bit-identical to it.
struct __align__(16) Head64P {   // 16 B: read with ld.shared.v2.f64
    double w2[HD * HD];
    double b2[HD];
    double wo[HD];
    double bo;
};

Head64P head64_from(const Net64P &n) {
    Head64P h;
    memcpy(h.w2, n.w2, sizeof(h.w2));
    memcpy(h.b2, n.b2, sizeof(h.b2));
    memcpy(h.wo, n.wo, sizeof(h.wo));
    h.bo = n.bo;
    return h;
}

// Two fp64 weights from shared memory (16 B, broadcast across the warp).
// Volatile so that the prefetches below stay where they are written:
// ptxas otherwise sinks each load next to its use at high register pressure
// and every DFMA then waits out a full LDS latency.
__device__ __forceinline__ double2 lds_f64x2(const double *p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

// Layer 2 + head in fp64, the oracle's fma order (per output: k ascending,
// then + b2; y: o ascending).  `net` MUST live in shared memory (every
// caller stages it there).  Two output rows at a time, their weights
// prefetched one double2 step ahead.
__device__ __forceinline__ double head64_lean(const Head64P &net, const double (&z)[HD]) {
    double h1[HD];
#pragma unroll
    for (int k = 0; k < HD; ++k) h1[k] = z[k] > 0.0 ? z[k] : 0.0;
    double y = 0.0;
#pragma unroll 1
    for (int o = 0; o < HD; o += 2) {
        const double *r0 = net.w2 + o * HD, *r1 = r0 + HD;
        double acc0 = 0.0, acc1 = 0.0;
        double2 w0 = lds_f64x2(r0), w1 = lds_f64x2(r1);
#pragma unroll
        for (int k = 0; k < HD; k += 2) {
            double2 n0 = w0, n1 = w1;
            if (k + 2 < HD) { n0 = lds_f64x2(r0 + k + 2); n1 = lds_f64x2(r1 + k + 2); }
            acc0 = fma(h1[k], w0.x, acc0);
            acc1 = fma(h1[k], w1.x, acc1);
            acc0 = fma(h1[k + 1], w0.y, acc0);
            acc1 = fma(h1[k + 1], w1.y, acc1);
            w0 = n0;
            w1 = n1;
        }
        const double2 b = lds_f64x2(net.b2 + o), wo = lds_f64x2(net.wo + o);
        acc0 = acc0 + b.x;
        acc1 = acc1 + b.y;
        y = fma(acc0 > 0.0 ? acc0 : 0.0, wo.x, y);
        y = fma(acc1 > 0.0 ? acc1 : 0.0, wo.y, y);
    }
    y = y + net.bo;
    return y > 0.0 ? y : 0.0;
}

// k_resolve's head: k-outer / o-inner, 18 independent fp64 chains (each
// still sums over k in the oracle's order), weights read as double2 along o
// from a k-major shared-memory copy `w2t` (w2t[k*18 + o] = w2[o*18 + k]).
__device__ __forceinline__ double head64t(const Head64P &net, const double *w2t,
                                          const double (&z)[HD]) {
    double acc[HD];
#pragma unroll
    for (int o = 0; o < HD; ++o) acc[o] = 0.0;
#pragma unroll
    for (int k = 0; k < HD; ++k) {
        const double hk = z[k] > 0.0 ? z[k] : 0.0;
#pragma unroll
        for (int o = 0; o < HD; o += 2) {
            const double2 w = lds_f64x2(w2t + k * HD + o);
            acc[o] = fma(hk, w.x, acc[o]);
            acc[o + 1] = fma(hk, w.y, acc[o + 1]);
        }
    }
    double y = 0.0;
#pragma unroll
    for (int o = 0; o < HD; ++o) {
        const double a2 = acc[o] + net.b2[o];
        y = fma(a2 > 0.0 ? a2 : 0.0, net.wo[o], y);
    }
    y = y + net.bo;
    return y > 0.0 ? y : 0.0;
}

// Stage the fp64 head weights in shared memory: 324+ distinct fp64 constants
// overflow the per-SM constant cache, while a shared-memory copy is read with
// broadcast LDS (every lane of a warp reads the same address).
// The device network image (cs_tables_set_network): Net64P, then w1
// transposed (w1t[k][h]); Head64P = {w2, b2, wo, bo} is a contiguous slice of
// Net64P.
constexpr int kImgHeadOff = (HD * IN + HD);                  // doubles before Net64P::w2
constexpr int kImgW1tOff = (int)(sizeof(Net64P) / 8);
constexpr int kImgW2tOff = kImgW1tOff + IN * HD;              // w2 k-major (w2t[k][o])
constexpr int kImgDoubles = kImgW2tOff + HD * HD;
static_assert(sizeof(Net64P) % 16 == 0 && (IN * HD * 8) % 16 == 0, "bulk-copy granules");

__device__ __forceinline__ const Head64P &stage_head64(const double *__restrict__ img, Head64P &sm) {
    const double *src = img + kImgHeadOff;
    double *dst = reinterpret_cast<double *>(&sm);
    for (int i = threadIdx.x; i < (int)(sizeof(Head64P) / sizeof(double)); i += blockDim.x)
        dst[i] = __ldg(src + i);
    __syncthreads();
    return sm;
}

// The fp64 tables are chunk-major so that a warp's gather is coalesced: the
// 18 values of a row are 9 double2 chunks, and chunk q of every row is
// stored together.  App rows: [9][N] double2 -- lanes reading consecutive
// apps (the j's of a pair block) hit consecutive 16 B.  Knob rows: [9][G][2]
// double2, member 0 (K1) and member 1 (K2) of a config side by side;
// knob2_64 = knob1_64 + 2, both indexed with member 0's index.
__host__ __device__ __forceinline__ size_t app64_at(int n, int r, int h) {
    return ((size_t)(h >> 1) * n + r) * 2 + (h & 1);
}
__host__ __device__ __forceinline__ size_t knob64_at(int G, int c, int member, int h) {
    return (((size_t)(h >> 1) * G + c) * 2 + member) * 2 + (h & 1);
}

// z = (A_self + B_other) + K_c in fp64, the oracle's sum order (16 B loads)
__device__ __forceinline__ void z64_row(const cs_tables &t, int self, int other, int c, int member,
                                        double (&z)[HD]) {
    const double2 *as = reinterpret_cast<const double2 *>(t.app_a64) + self;
    const double2 *bo = reinterpret_cast<const double2 *>(t.app_b64) + other;
    const double2 *kk = reinterpret_cast<const double2 *>(t.knob1_64) + 2 * (size_t)c + member;
    const size_t sn = (size_t)t.n_apps, sg = 2 * (size_t)t.n_grid;
#pragma unroll
    for (int q = 0; q < HD / 2; ++q) {
        const double2 a = __ldg(as + q * sn), b = __ldg(bo + q * sn), k = __ldg(kk + q * sg);
        z[2 * q] = (a.x + b.x) + k.x;
        z[2 * q + 1] = (a.y + b.y) + k.y;
    }
}

// floor(pred) x T of one member of pair (self, other) under config c
// (member 0: K1 / view hc, member 1: K2 / reversed partitions)
__device__ __forceinline__ double member_time64(const cs_tables &t, const Head64P &net,
                                                const double *w2t,
                                                const double *__restrict__ base_time, int self,
                                                int other, int c, int member) {
    double z[HD];
    z64_row(t, self, other, c, member, z);
    const double y = head64t(net, w2t, z);
    return (y < FLOOR ? FLOOR : y) * __ldg(base_time + self);
}

__device__ __forceinline__ double member_time64_lean(const cs_tables &t, const Head64P &net,
                                                     const double *__restrict__ base_time,
                                                     int self, int other, int c, int member) {
    double z[HD];
    z64_row(t, self, other, c, member, z);
    const double y = head64_lean(net, z);
    return (y < FLOOR ? FLOOR : y) * __ldg(base_time + self);
}

// fp64 floor test of one member's prediction (estimator.py:106-109): 1 if clamped
__device__ __forceinline__ int member_floor64(const cs_tables &t, const Head64P &net, int self,
                                              int other, int c, int member) {
    double z[HD];
    z64_row(t, self, other, c, member, z);
    return head64_lean(net, z) < FLOOR ? 1 : 0;
}

// CoRunTime of one config for pair (i, j): max over members (estimator.py:127-129)
__device__ __forceinline__ double corun64(const cs_tables &t, const Head64P &net,
                                          const double *w2t,
                                          const double *__restrict__ base_time, int i, int j,
                                          int c) {
    const double t1 = member_time64(t, net, w2t, base_time, i, j, c, 0);
    const double t2 = member_time64(t, net, w2t, base_time, j, i, c, 1);
    return t1 > t2 ? t1 : t2;
}

// ---- screened record -------------------------------------------------------
// The screens leave, per (pair, budget), either the winner (index + its fp64
// CoRunTime) or CS_SCREEN_AMBIGUOUS plus a queue entry for k_resolve.
constexpr int32_t CS_SCREEN_AMBIGUOUS = -2;
// ---- shared by both screens ----------------------------------------------
struct SweepArgs {
    cs_tables t;
    GridP g;
    const double *base_time, *solo_time;
    const int32_t *solo_clamps;
    int32_t n, log2s;
    int64_t p_begin, P;
    float eps;               // ambiguity band: runner-up within eps -> exact re-scan
    float near;              // runner-up within near (> eps): a sample of these pairs is
    int64_t vstride;         // (every vstride-th pair) fully re-scanned by k_resolve
    float tau;               // a row with a prediction within tau of the 0.5 floor
                             // has its floor clamps re-counted in fp64
    cs_pair_out out;
    int64_t *queue;          // (L + 2) P slots: [0, L P) re-scan / verify queue, then
                             // the queue of rows whose clamps k_resolve re-counts
    cs_counters *cnt;
    unsigned long long *clamps;
    uint32_t *trace;         // debug builds (CS_TC_TRACE): per-thread progress, host-mapped
    // fused tail (k_sweep_tc3 via cs_pair_sweep_fused): ambiguous pairs are
    // re-scanned in fp64 inside the kernel, and every (pair, budget) is
    // decided against solo_time and scattered into W (L x N x N, optional)
    int fused;
    double *W;
};

__device__ __forceinline__ bool screen_ambiguous(const SweepArgs &a, float best, float second) {
    return !(second > best * (1.0f + a.eps));
}
// non-ambiguous but close: the runner-up gets an fp64 re-evaluation as well
__device__ __forceinline__ bool screen_near(const SweepArgs &a, float best, float second) {
    return !(second > best * (1.0f + a.near));
}

// ambiguous (pair, budget): leave it to k_resolve
__device__ __forceinline__ void push_ambiguous(const SweepArgs &a, int l, int64_t pl) {
    const int64_t o = (int64_t)l * a.P + pl;
    a.out.corun_grid_index[o] = CS_SCREEN_AMBIGUOUS;
    const uint32_t q = atomicAdd(&a.cnt->queue_len, 1u);
    a.queue[q] = (pl << 4) | l;
}

// a (pair, member) row with a screened prediction within tau of the floor:
// k_resolve re-counts its clamps in fp64 (the screen does not count them)
__device__ __forceinline__ void push_row(const SweepArgs &a, int64_t pl, int member) {
    const uint32_t q = atomicAdd(&a.cnt->exact_rows, 1u);
    a.queue[(int64_t)a.g.L * a.P + q] = (pl << 1) | member;
}

// a certain winner whose runner-up is near (eps < gap <= near): every
// vstride-th such pair is re-scanned in fp64 by k_resolve as a check of the
// screen's order (a disagreement flags the sweep; the host then redoes it
// with a wider band).  Entries share the re-scan queue, tagged by bit 3.
__device__ __forceinline__ void maybe_verify(const SweepArgs &a, int l, int64_t pl, float best,
                                             float second) {
    if (!screen_near(a, best, second) || (a.p_begin + pl) % a.vstride) return;
    const uint32_t q = atomicAdd(&a.cnt->queue_len, 1u);
    a.queue[q] = (pl << 4) | 8 | l;
}

// the screen-error monitor: relative gap between a screened time and its fp64 value
__device__ __forceinline__ void monitor(const SweepArgs &a, double exact, float screened) {
    atomicMax(&a.cnt->screen_err_bits, __float_as_uint((float)(fabs(exact - (double)screened) / exact)));
}

// certain winner: its exact fp64 CoRunTime (+ the screen-error monitor)
__device__ __forceinline__ void write_winner(const SweepArgs &a, int l, int64_t pl, int idx,
                                             double co, float best) {
    const int64_t o = (int64_t)l * a.P + pl;
    a.out.corun_grid_index[o] = idx;
    a.out.corun_time[o] = co;
    monitor(a, co, best);
}

// co-run vs time-share for one (pair, budget) (hwopt.py:77-87) with the solo
// pair sum (0.0 + t_i) + t_j (estimator.py:168-178); writes the flag and the
// winning time, scatters it into W, and returns the solo-split floor clamps the
// reference counts for this pair (its two solorun_time calls)
template <class Args>
__device__ __forceinline__ int decide_write(const Args &a, int l, int64_t pl, int i, int j,
                                            int idx, double co) {
    const int64_t o = (int64_t)l * a.P + pl;
    const double *st = a.solo_time + (size_t)l * a.n;
    const double solo = (0.0 + st[i]) + st[j];
    const bool chosen = idx >= 0 && co <= solo;
    const double w = chosen ? co : solo;
    a.out.corun_chosen[o] = chosen;
    a.out.weight[o] = w;
    if (a.W) {
        double *Wl = a.W + (size_t)l * a.n * a.n;
        Wl[(size_t)i * a.n + j] = w;
        Wl[(size_t)j * a.n + i] = w;
    }
    return a.solo_clamps ? a.solo_clamps[(size_t)l * a.n + i] + a.solo_clamps[(size_t)l * a.n + j] : 0;
}

__device__ __forceinline__ float head32(const Net32P &net, const float (&z)[HD]) {
    float h[HD];
#pragma unroll
    for (int k = 0; k < HD; ++k) h[k] = fmaxf(z[k], 0.f);
    float y = net.bo;
#pragma unroll
    for (int o = 0; o < HD; ++o) {
        float acc = net.b2[o];
#pragma unroll
        for (int k = 0; k < HD; ++k) acc = fmaf(h[k], net.w2[o * HD + k], acc);
        y = fmaf(fmaxf(acc, 0.f), net.wo[o], y);
    }
    return y;
}

__device__ __forceinline__ void load_row20(const float *__restrict__ p, float (&r)[HD]) {
    const float4 *q = reinterpret_cast<const float4 *>(p);
    float4 v0 = __ldg(q), v1 = __ldg(q + 1), v2 = __ldg(q + 2), v3 = __ldg(q + 3), v4 = __ldg(q + 4);
    r[0] = v0.x; r[1] = v0.y; r[2] = v0.z; r[3] = v0.w;
    r[4] = v1.x; r[5] = v1.y; r[6] = v1.z; r[7] = v1.w;
    r[8] = v2.x; r[9] = v2.y; r[10] = v2.z; r[11] = v2.w;
    r[12] = v3.x; r[13] = v3.y; r[14] = v3.z; r[15] = v3.w;
    r[16] = v4.x; r[17] = v4.y;
}

#include "tcgen05_util.cuh"
#include "tc3_sweep.cuh"

// ---- k_tables: factored layer 1 (core.py:367-377 + fnn.py:163) ------------
__device__ __forceinline__ double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// The network is staged in shared memory once per block: the kernel parameter
// bank serializes lane-divergent reads (lane h reading w1[h][k] is 18
// different addresses), shared memory serves them in one wavefront; w1 is
// also kept transposed (w1t[k][h]) so lane h's reads are consecutive.
struct __align__(16) TablesSmem {
    Net64P net;                  // net | w1t | w2t: one image slice + the head, bulk-copied
    double w1t[IN][HD];
    double w2t[HD * HD];         // k-major W2: the solo heads as 18 independent chains
    Head64P head;
    double xs[4][2 * NF];        // per warp: the app's normalized counters
};

// Best split of budget l for this warp's app from the splits evaluated by
// lanes [s0, s1) (value `tt`, INFINITY outside): first index wins ties
// (estimator.py:175), clamps counted over the budget's splits.
__device__ __forceinline__ void solo_reduce(double tt, int clamp, int lane, int s0, int s1,
                                            int64_t w, cs_solo_out out) {
    const bool in = lane >= s0 && lane < s1;
    double best = in ? tt : INFINITY;
    int arg = in ? lane - s0 : INT_MAX;
    for (int off = 16; off; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, arg, off);
        if (ob < best || (ob == best && oi < arg)) { best = ob; arg = oi; }
    }
    const int cl = __reduce_add_sync(0xffffffffu, in ? clamp : 0);
    if (lane == 0) {
        out.solo_time[w] = arg == INT_MAX ? nan("") : best;
        out.solo_split[w] = arg == INT_MAX ? -1 : arg;
        if (out.solo_clamps) out.solo_clamps[w] = cl;
    }
}

// One warp per row -- the N apps (A and B partials), then the G configs (K1,
// K2, b1 folded), then the S solo splits (KS) -- with lane h < 18 producing
// hidden unit h; for app rows lane k first normalizes counter k (the fp64
// divisions happen once per app).  With `do_solo` (S <= 32) an app's warp
// then also evaluates its S exclusive splits (lane s = split s, the exact fp64
// head of k_solo) and reduces them per budget, so the solo step needs no
// launch of its own.  Threads below W2_TILE_ELEMS also write the fp16 B
// operands of the tensor-core screens.
__global__ void __launch_bounds__(128) k_tables(const __grid_constant__ Net64P net_unused,
                                                const double *__restrict__ feats, int n,
                                                const GridP g, const cs_tables t,
                                                const double *__restrict__ base_time,
                                                cs_solo_out solo, int do_solo,
                                                cs_counters *reset_cnt,
                                                unsigned long long *reset_clamps) {
    __shared__ TablesSmem sm;
    // let a programmatically dependent sweep start its prologue now (it still
    // waits for this grid to finish before reading the tables)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the device image (Net64P | w1t) and the head slice, staged by two TMA
    // bulk copies (the parameter bank would serialize these lane-divergent
    // reads; per-thread load/store loops left the block waiting on a chain of
    // global-load latencies)
    __shared__ uint64_t staged;
    if (threadIdx.x == 0) {
        tc::mbar_init(&staged, 1);
        tc::fence_mbar_init();
        constexpr uint32_t kNetW1t = (uint32_t)(sizeof(Net64P) + sizeof(double) * (IN * HD + HD * HD));
        static_assert(offsetof(TablesSmem, w1t) == sizeof(Net64P), "image order");
        static_assert(offsetof(TablesSmem, w2t) == sizeof(double) * kImgW2tOff, "image order");
        tc::mbar_expect_tx(&staged, kNetW1t + (uint32_t)sizeof(Head64P));
        tc::bulk_g2s(&sm.net, t.net_image, kNetW1t, &staged);
        tc::bulk_g2s(&sm.head, t.net_image + kImgHeadOff, (uint32_t)sizeof(Head64P), &staged);
    }
    __syncthreads();
    tc::mbar_wait(&staged, 0);
    // the image predates the previous kernel; the features may come from it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // fresh counters for the screen (it reads them only after this grid completes)
    if (blockIdx.x == 0) {
        if (reset_cnt && threadIdx.x < (int)(sizeof(cs_counters) / 4))
            reinterpret_cast<uint32_t *>(reset_cnt)[threadIdx.x] = 0u;
        if (reset_clamps && threadIdx.x < g.L) reset_clamps[threadIdx.x] = 0ull;
        for (int i = threadIdx.x; i < t.split_slots; i += blockDim.x) t.split_cnt[i] = 0u;
    }
    __syncthreads();
    const Net64P &net = sm.net;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < W2_TILE_ELEMS) write_b_slices(net, t.w2_tile, (int)tid);
    const int lane = threadIdx.x & 31;
    const int h = lane < HD ? lane : HD - 1;
    const int64_t rows = (int64_t)n + g.G + g.S;
    for (int64_t r = tid >> 5; r < rows; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        if (r < n) {
            const double f = lane < NF ? feats[r * NF + lane] : 0.0;
            // normalized counters through shared memory: the FMA chains below
            // then read them with independent broadcast loads instead of a
            // latency-bound shuffle per step
            double *xs = sm.xs[threadIdx.x >> 5];
            if (lane < NF) {
                xs[lane] = clip01(f / net.bounds[lane]);
                xs[NF + lane] = clip01(f / net.bounds[NF + lane]);
            }
            __syncwarp();
            double sa = 0.0, sb = 0.0;
#pragma unroll
            for (int k = 0; k < NF; ++k) {
                sa = fma(xs[k], sm.w1t[4 + k][h], sa);
                sb = fma(xs[NF + k], sm.w1t[4 + NF + k][h], sb);
            }
            __syncwarp();
            if (lane < HD) {
                t.app_a64[app64_at(n, (int)r, h)] = sa;
                t.app_b64[app64_at(n, (int)r, h)] = sb;
                t.app_a32[r * ROW32 + h] = (float)sa;
                t.app_b32[r * ROW32 + h] = (float)sb;
            } else if (lane < ROW32) {
                t.app_a32[r * ROW32 + lane] = 0.f;
                t.app_b32[r * ROW32 + lane] = 0.f;
            }
            if (do_solo) {
                // lane s: split s (all budgets' splits stacked, S <= 32); its
                // KS row exactly as the solo-row branch below computes it
                const int s = lane < g.S ? lane : 0;
                double z[HD];
#pragma unroll
                for (int hh = 0; hh < HD; ++hh) {
                    double ks = 0.0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) ks = fma(g.solo_knob[s * 4 + k], sm.w1t[k][hh], ks);
                    ks = ks + net.b1[hh];
                    z[hh] = __shfl_sync(0xffffffffu, sa, hh) + ks;
                }
                double y = head64t(sm.head, sm.w2t, z);
                int clamp = 0;
                if (y < FLOOR) { clamp = 1; y = FLOOR; }
                const double tt = y * base_time[r];
                for (int l = 0; l < g.L; ++l)
                    solo_reduce(tt, clamp, lane, g.solo_off[l], g.solo_off[l + 1], (int64_t)l * n + r, solo);
            }
        } else if (r < (int64_t)n + g.G) {
            const int64_t c = r - n;
            double s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                s1 = fma(g.knob1[c * 4 + k], sm.w1t[k][h], s1);
                s2 = fma(g.knob2[c * 4 + k], sm.w1t[k][h], s2);
            }
            s1 = s1 + net.b1[h];
            s2 = s2 + net.b1[h];
            if (lane < HD) {
                t.knob1_64[knob64_at(g.G, (int)c, 0, h)] = s1;
                t.knob1_64[knob64_at(g.G, (int)c, 1, h)] = s2;
                t.knob1_32[c * KROW32 + h] = (float)s1;
                t.knob2_32[c * KROW32 + h] = (float)s2;
            } else if (lane < ROW32) {
                t.knob1_32[c * KROW32 + lane] = 0.f;
                t.knob2_32[c * KROW32 + lane] = 0.f;
            }
        } else {
            const int64_t c = r - n - g.G;
            double s1 = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) s1 = fma(g.solo_knob[c * 4 + k], sm.w1t[k][h], s1);
            if (lane < HD) t.solo64[c * HD + h] = s1 + net.b1[h];
        }
    }
}

// ---- k_solo: per (budget, app) best split, fp64 (estimator.py:160-180) ----
// One warp per (budget, app); lane s evaluates split s (a budget has <= 32
// splits: 17 on the 6.25 W grid), then a first-index argmin over the warp.
__global__ void k_solo(const cs_tables t, const GridP g, const double *__restrict__ base_time,
                       int n, cs_solo_out out, const __grid_constant__ Head64P net_param) {
    __shared__ Head64P net_sm;
    const Head64P &net = stage_head64(t.net_image, net_sm);
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= (int64_t)n * g.L) return;
    const int l = (int)(w / n), a = (int)(w % n);
    const int s0 = g.solo_off[l], ns = g.solo_off[l + 1] - s0;
    double best = INFINITY;
    int arg = INT_MAX, clamp = 0;
    for (int s = lane; s < ns; s += 32) {
        double z[HD];
#pragma unroll
        for (int h = 0; h < HD; ++h) z[h] = t.app_a64[app64_at(n, a, h)] + t.solo64[(size_t)(s0 + s) * HD + h];
        double y = head64_lean(net, z);
        if (y < FLOOR) { ++clamp; y = FLOOR; }
        const double tt = y * base_time[a];
        if (tt < best) { best = tt; arg = s; }
    }
    for (int off = 16; off; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, arg, off);
        if (ob < best || (ob == best && oi < arg)) { best = ob; arg = oi; }
    }
    clamp = __reduce_add_sync(0xffffffffu, clamp);
    if (lane == 0) {
        out.solo_time[w] = arg == INT_MAX ? nan("") : best;
        out.solo_split[w] = arg == INT_MAX ? -1 : arg;
        if (out.solo_clamps) out.solo_clamps[w] = clamp;
    }
}

template <int L>
__global__ void __launch_bounds__(kSweepThreads) k_sweep(const SweepArgs a,
                                                         const __grid_constant__ Net32P net,
                                                         const __grid_constant__ Head64P net_param) {
    __shared__ Head64P net_sm;
    const Head64P &net64 = stage_head64(a.t.net_image, net_sm);
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int S = 1 << a.log2s;
    const int64_t pl = gt >> a.log2s;          // local pair index
    const int s = (int)(gt & (S - 1));         // config slice
    const bool live = pl < a.P;
    int i = 0, j = 1;
    if (live) pair_of(a.p_begin + pl, a.n, i, j);

    float best[L], second[L];
    int idx[L];
#pragma unroll
    for (int l = 0; l < L; ++l) { best[l] = FLT_MAX; second[l] = FLT_MAX; idx[l] = INT_MAX; }
    float miny1 = FLT_MAX, miny2 = FLT_MAX;   // smallest screened prediction per member

    if (live) {
        float p1[HD], p2[HD], tmp[HD];
        load_row20(a.t.app_a32 + (size_t)i * ROW32, p1);
        load_row20(a.t.app_b32 + (size_t)j * ROW32, tmp);
#pragma unroll
        for (int h = 0; h < HD; ++h) p1[h] += tmp[h];
        load_row20(a.t.app_a32 + (size_t)j * ROW32, p2);
        load_row20(a.t.app_b32 + (size_t)i * ROW32, tmp);
#pragma unroll
        for (int h = 0; h < HD; ++h) p2[h] += tmp[h];
        const float ti = (float)a.base_time[i], tj = (float)a.base_time[j];

        for (int c = s; c < a.g.G; c += S) {
            const uint32_t m = L == 1 ? 1u : __ldg(a.g.mask + c);
            float z[HD];
            load_row20(a.t.knob1_32 + (size_t)c * KROW32, z);
#pragma unroll
            for (int h = 0; h < HD; ++h) z[h] += p1[h];
            const float y1 = head32(net, z);
            load_row20(a.t.knob2_32 + (size_t)c * KROW32, z);
#pragma unroll
            for (int h = 0; h < HD; ++h) z[h] += p2[h];
            const float y2 = head32(net, z);
            miny1 = fminf(miny1, y1);
            miny2 = fminf(miny2, y2);
            const float tt = fmaxf(fmaxf(y1, 0.5f) * ti, fmaxf(y2, 0.5f) * tj);
#pragma unroll
            for (int l = 0; l < L; ++l) {
                if (L == 1 || ((m >> l) & 1u)) {
                    if (tt < best[l]) { second[l] = best[l]; best[l] = tt; idx[l] = c; }
                    else second[l] = fminf(second[l], tt);
                }
            }
        }
    }

    // Floor clamps (estimator.py:106-109) are never counted from the screen:
    // a member whose screened predictions (over every slice of the pair) all
    // lie above 0.5 + tau has none; any other member row is queued and
    // k_resolve re-counts it in fp64
    {
        float m1 = miny1, m2 = miny2;
        for (int off = 1; off < S; off <<= 1) {
            m1 = fminf(m1, __shfl_xor_sync(0xffffffffu, m1, off));
            m2 = fminf(m2, __shfl_xor_sync(0xffffffffu, m2, off));
        }
        if (live && s == 0) {
            if (!(m1 > 0.5f + a.tau)) push_row(a, pl, 0);
            if (!(m2 > 0.5f + a.tau)) push_row(a, pl, 1);
        }
    }

    // merge the S slices of a pair (adjacent lanes): lexicographic (value, index)
#pragma unroll
    for (int l = 0; l < L; ++l) {
        for (int off = 1; off < S; off <<= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best[l], off);
            const float os = __shfl_xor_sync(0xffffffffu, second[l], off);
            const int oi = __shfl_xor_sync(0xffffffffu, idx[l], off);
            const bool other = ob < best[l] || (ob == best[l] && oi < idx[l]);
            const float loser = other ? best[l] : ob;
            second[l] = fminf(fminf(second[l], os), loser);
            if (other) { best[l] = ob; idx[l] = oi; }
        }
    }

    if (!live || s != 0) return;
#pragma unroll 1
    for (int l = 0; l < L; ++l) {
        if (screen_ambiguous(a, best[l], second[l])) { push_ambiguous(a, l, pl); continue; }
        const double co = fmax(member_time64_lean(a.t, net64, a.base_time, i, j, idx[l], 0),
                               member_time64_lean(a.t, net64, a.base_time, j, i, idx[l], 1));
        write_winner(a, l, pl, idx[l], co, best[l]);
        maybe_verify(a, l, pl, best[l], second[l]);
    }
}

// ---- k_resolve: exact fp64 argmin for queued (pair, budget) ---------------
struct ResolveArgs {
    cs_tables t;
    GridP g;
    const double *base_time, *solo_time;
    int32_t n;
    int64_t p_begin, P;
    cs_pair_out out;
    const int64_t *queue;
    cs_counters *cnt;
    // fused (cs_pair_sweep_fused): also decide + scatter each resolved entry
    int fused;
    const int32_t *solo_clamps;
    unsigned long long *clamps;
    double *W;
};

__global__ void __launch_bounds__(128) k_resolve(const ResolveArgs a,
                                                 const __grid_constant__ Head64P net_param) {
    // One block per queued (pair, budget); thread c evaluates configs c,
    // c+128, ... in fp64, then a block-wide first-index argmin (ties ->
    // smallest index).
    __shared__ Head64P net_sm;
    __shared__ double red_v[4];
    __shared__ int red_i[4];
    // the weights do not depend on the screen: staged before the
    // programmatic-dependency wait (a no-op without a PDL launch)
    // (the k-major W2 is a slice of the device image, like the head: two TMA
    // bulk copies)
    __shared__ __align__(16) double w2t[HD * HD];
    __shared__ uint64_t staged;
    if (threadIdx.x == 0) {
        tc::mbar_init(&staged, 1);
        tc::fence_mbar_init();
        tc::mbar_expect_tx(&staged, (uint32_t)(sizeof(w2t) + sizeof(Head64P)));
        tc::bulk_g2s(w2t, a.t.net_image + kImgW2tOff, (uint32_t)sizeof(w2t), &staged);
        tc::bulk_g2s(&net_sm, a.t.net_image + kImgHeadOff, (uint32_t)sizeof(Head64P), &staged);
    }
    __syncthreads();
    tc::mbar_wait(&staged, 0);
    const Head64P &net64 = net_sm;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // blocks past both (device-side) queue lengths leave
    const uint32_t count = a.cnt->queue_len, rows = a.cnt->exact_rows;
    if (blockIdx.x >= count && blockIdx.x >= rows) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t q = blockIdx.x; q < count; q += gridDim.x) {
        const int64_t e = a.queue[q];
        const int64_t pl = e >> 4;
        const int l = (int)(e & 7);
        const bool verify = (e & 8) != 0;   // a certain winner re-scanned as a check
        int i, j;
        pair_of(a.p_begin + pl, a.n, i, j);
        double best = INFINITY;
        int arg = INT_MAX;
        for (int c = threadIdx.x; c < a.g.G; c += blockDim.x) {
            if (!((__ldg(a.g.mask + c) >> l) & 1u)) continue;
            const double tt = corun64(a.t, net64, w2t, a.base_time, i, j, c);
            if (tt < best) { best = tt; arg = c; }          // ascending c per thread
        }
        for (int off = 16; off; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, arg, off);
            if (ob < best || (ob == best && oi < arg)) { best = ob; arg = oi; }
        }
        if (lane == 0) { red_v[warp] = best; red_i[warp] = arg; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (red_v[w] < best || (red_v[w] == best && red_i[w] < arg)) { best = red_v[w]; arg = red_i[w]; }
            const int64_t o = (int64_t)l * a.P + pl;
            if (verify) {
                // the screen's winner (index and fp64 time) must be the exact one
                if (a.out.corun_grid_index[o] != arg || a.out.corun_time[o] != best)
                    atomicAdd(&a.cnt->verify_fail, 1u);
            } else {
            a.out.corun_grid_index[o] = arg == INT_MAX ? -1 : arg;
            a.out.corun_time[o] = arg == INT_MAX ? INFINITY : best;
            if (a.fused) {
                const int cl = decide_write(a, l, pl, i, j, arg == INT_MAX ? -1 : arg,
                                            arg == INT_MAX ? INFINITY : best);
                if (cl) atomicAdd(a.clamps + l, (unsigned long long)cl);
            }
            }
        }
        __syncthreads();
    }
    // rows whose floor clamps the screen could not count: all their co-run
    // predictions re-counted in fp64 (estimator.py:106-109)
    __shared__ unsigned int red_c[4][CS_MAX_BUDGETS];
    for (int64_t q = blockIdx.x; q < rows; q += gridDim.x) {
        const int64_t e = a.queue[(int64_t)a.g.L * a.P + q];
        const int64_t pl = e >> 1;
        const int member = (int)(e & 1);
        int i, j;
        pair_of(a.p_begin + pl, a.n, i, j);
        unsigned int cl[CS_MAX_BUDGETS] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = threadIdx.x; c < a.g.G; c += blockDim.x) {
            double z[HD];
            z64_row(a.t, member ? j : i, member ? i : j, c, member, z);
            if (head64t(net64, w2t, z) < FLOOR) {
                const uint32_t m = __ldg(a.g.mask + c);
#pragma unroll
                for (int l = 0; l < CS_MAX_BUDGETS; ++l) cl[l] += (m >> l) & 1u;
            }
        }
        for (int l = 0; l < a.g.L; ++l) {
            const unsigned int v = __reduce_add_sync(0xffffffffu, cl[l]);
            if (lane == 0) red_c[warp][l] = v;
        }
        __syncthreads();
        if (threadIdx.x < a.g.L) {
            unsigned long long v = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red_c[w][threadIdx.x];
            if (v) atomicAdd(a.clamps + threadIdx.x, v);
        }
        __syncthreads();
    }
}

// ---- k_decide: co-run vs time-share per (pair, budget) (hwopt.py:77-87) ----
// corun_time is final here (screen winner re-evaluated in fp64, or k_resolve);
// the solo pair sum is (0.0 + t_i) + t_j (estimator.py:168-178).  Also adds the
// solo-split clamps the reference counts per pair and, when W is given,
// scatters the winning time into the symmetric N x N matrix of budget l.
struct DecideArgs {
    const double *solo_time;
    const int32_t *solo_clamps;
    int32_t n, L;
    int64_t p_begin, P;
    cs_pair_out out;
    unsigned long long *clamps;
    double *W;               // L x N x N or null
};

__global__ void __launch_bounds__(256) k_decide(const DecideArgs a) {
    const int64_t total = (int64_t)a.L * a.P;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long cl[CS_MAX_BUDGETS] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int l = (int)(e / a.P);
        const int64_t pl = e - (int64_t)l * a.P;
        int i, j;
        pair_of(a.p_begin + pl, a.n, i, j);
        const double *st = a.solo_time + (size_t)l * a.n;
        const double solo = (0.0 + st[i]) + st[j];
        const double co = a.out.corun_time[e];
        const bool chosen = a.out.corun_grid_index[e] >= 0 && co <= solo;   // hwopt.py:86
        const double w = chosen ? co : solo;
        a.out.corun_chosen[e] = chosen;
        a.out.weight[e] = w;
        if (a.W) {
            double *Wl = a.W + (size_t)l * a.n * a.n;
            Wl[(size_t)i * a.n + j] = w;
            Wl[(size_t)j * a.n + i] = w;
        }
        if (a.solo_clamps) {
#pragma unroll
            for (int b = 0; b < CS_MAX_BUDGETS; ++b)
                if (b == l) cl[b] += a.solo_clamps[(size_t)l * a.n + i] + a.solo_clamps[(size_t)l * a.n + j];
        }
    }
    if (!a.solo_clamps) return;
#pragma unroll
    for (int b = 0; b < CS_MAX_BUDGETS; ++b) {
        if (b >= a.L) break;
        unsigned long long v = cl[b];
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(a.clamps + b, v);
    }
}

// ---- k_scatter: symmetric weight matrix ----------------------------------
__global__ void k_scatter(const double *__restrict__ weight, int n, int64_t p_begin, int64_t P,
                          double *__restrict__ W) {
    for (int64_t pl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pl < P;
         pl += (int64_t)gridDim.x * blockDim.x) {
        int i, j;
        pair_of(p_begin + pl, n, i, j);
        const double w = weight[pl];
        W[(size_t)i * n + j] = w;
        W[(size_t)j * n + i] = w;
    }
}

// ---- multi-GPU wire records (cs_pack_records / cs_unpack_gathered) --------
struct WireLayout {
    size_t time, idx, flag, total;
};
__host__ __device__ __forceinline__ size_t wire_align(size_t v) { return (v + 255) & ~(size_t)255; }
__host__ __device__ __forceinline__ WireLayout wire_layout(int64_t cap, int L) {
    WireLayout w;
    const size_t n = (size_t)cap * L;
    w.time = 0;
    w.idx = wire_align(8 * n);
    w.flag = w.idx + wire_align(2 * n);
    w.total = w.flag + wire_align(n);
    return w;
}

__global__ void k_pack_records(const cs_pair_out shard, int64_t P, int L, int64_t cap,
                               uint8_t *__restrict__ wire) {
    const WireLayout w = wire_layout(cap, L);
    double *t = reinterpret_cast<double *>(wire + w.time);
    uint16_t *ix = reinterpret_cast<uint16_t *>(wire + w.idx);
    uint8_t *fl = wire + w.flag;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)L * P;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = e / P, p = e - l * P, o = l * cap + p;
        const int32_t g = shard.corun_grid_index[e];
        t[o] = shard.corun_time[e];
        ix[o] = g < 0 ? (uint16_t)0xFFFF : (uint16_t)g;
        fl[o] = shard.corun_chosen[e];
    }
}

// One thread per global pair: owner rank of pair p, its wire slot, the
// decision record and (optionally) the two matrix entries, every budget.
__global__ void k_unpack_gathered(const uint8_t *__restrict__ gathered, int world, int64_t wire_bytes,
                                  int64_t P, int n, int L, int64_t cap,
                                  const double *__restrict__ solo_time, const cs_pair_out full,
                                  double *__restrict__ W) {
    const int64_t base = P / world, extra = P % world;
    const WireLayout wl = wire_layout(cap, L);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        // owner rank of pair p: the first `extra` ranks hold base + 1 pairs
        const int64_t cut = extra * (base + 1);
        const int64_t r = p < cut ? p / (base + 1) : extra + (p - cut) / base;
        const int64_t b = r * base + (r < extra ? r : extra);
        const uint8_t *blk = gathered + r * wire_bytes;
        const double *t = reinterpret_cast<const double *>(blk + wl.time);
        const uint16_t *ix = reinterpret_cast<const uint16_t *>(blk + wl.idx);
        const uint8_t *fl = blk + wl.flag;
        int i, j;
        pair_of(p, n, i, j);
        for (int l = 0; l < L; ++l) {
            const int64_t s = (int64_t)l * cap + (p - b), o = (int64_t)l * P + p;
            const double co = t[s];
            const uint16_t g = ix[s];
            const bool chosen = fl[s] != 0;
            const double *st = solo_time + (size_t)l * n;
            const double w = chosen ? co : (0.0 + st[i]) + st[j];     // hwopt.py:39-41
            full.corun_grid_index[o] = g == 0xFFFF ? -1 : (int32_t)g;
            full.corun_time[o] = co;
            full.corun_chosen[o] = chosen;
            full.weight[o] = w;
            if (W) {
                double *Wl = W + (size_t)l * n * n;
                Wl[(size_t)i * n + j] = w;
                Wl[(size_t)j * n + i] = w;
            }
        }
    }
}

// ---- k_analytic: the simenv analytic oracle as the model (analytic.py) ----
// Per pair, per config: slowdown_k = (resource*power)[view k][config][self] *
// contention(self, other) (simenv.py:182-218, host-built products), floor
// 0.5, x base time, max over members, per-budget first-index argmin, then the
// co-run / time-share decision and the scatter.  fp64 with explicit _rn
// intrinsics: no FMA contraction, so every value equals the reference's.
struct AnalyticArgs {
    const double *rp1, *rp2;        // G x N, config-major
    const double *compute, *memory; // N
    double cc, mm, cm;
    const double *base_time, *solo_time;   // N ; L x N
    const uint32_t *mask;           // G
    int32_t n, G, L;
    int64_t P;
    cs_pair_out out;
    double *W;
    unsigned long long *clamps;
};

__device__ __forceinline__ double contention64(double cc, double mm, double cm, double ca, double ma,
                                               double cb, double mb) {
    // 1.0 + (cc*a.c*b.c + mm*a.m*b.m + cm*(a.c*b.m + a.m*b.c))   (simenv.py:175-179)
    const double t1 = __dmul_rn(__dmul_rn(cc, ca), cb);
    const double t2 = __dmul_rn(__dmul_rn(mm, ma), mb);
    const double t3 = __dmul_rn(cm, __dadd_rn(__dmul_rn(ca, mb), __dmul_rn(ma, cb)));
    return __dadd_rn(1.0, __dadd_rn(__dadd_rn(t1, t2), t3));
}

__global__ void __launch_bounds__(256) k_analytic(const AnalyticArgs a) {
    unsigned long long cl[CS_MAX_BUDGETS] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.P;
         p += (int64_t)gridDim.x * blockDim.x) {
        int i, j;
        pair_of(p, a.n, i, j);
        const double ci = a.compute[i], mi = a.memory[i], cj = a.compute[j], mj = a.memory[j];
        const double c12 = contention64(a.cc, a.mm, a.cm, ci, mi, cj, mj);
        const double c21 = contention64(a.cc, a.mm, a.cm, cj, mj, ci, mi);
        const double Ti = a.base_time[i], Tj = a.base_time[j];
        double best[CS_MAX_BUDGETS];
        int idx[CS_MAX_BUDGETS];
        for (int l = 0; l < CS_MAX_BUDGETS; ++l) { best[l] = INFINITY; idx[l] = -1; }
        for (int c = 0; c < a.G; ++c) {
            double s1 = __dmul_rn(a.rp1[(size_t)c * a.n + i], c12);
            double s2 = __dmul_rn(a.rp2[(size_t)c * a.n + j], c21);
            const int k1 = s1 < FLOOR, k2 = s2 < FLOOR;
            s1 = k1 ? FLOOR : s1;
            s2 = k2 ? FLOOR : s2;
            const double t1 = __dmul_rn(s1, Ti), t2 = __dmul_rn(s2, Tj);
            const double tt = t1 >= t2 ? t1 : t2;                 // max([t1, t2])
            const uint32_t m = a.mask[c];
            for (int l = 0; l < a.L; ++l)
                if ((m >> l) & 1u) {
                    cl[l] += k1 + k2;
                    if (tt < best[l]) { best[l] = tt; idx[l] = c; }   // hwopt.py:59
                }
        }
        for (int l = 0; l < a.L; ++l) {
            const int64_t o = (int64_t)l * a.P + p;
            const double *st = a.solo_time + (size_t)l * a.n;
            const double solo = (0.0 + st[i]) + st[j];
            const bool chosen = idx[l] >= 0 && best[l] <= solo;
            const double w = chosen ? best[l] : solo;
            a.out.corun_grid_index[o] = idx[l];
            a.out.corun_time[o] = best[l];
            a.out.corun_chosen[o] = chosen;
            a.out.weight[o] = w;
            if (a.W) {
                double *Wl = a.W + (size_t)l * a.n * a.n;
                Wl[(size_t)i * a.n + j] = w;
                Wl[(size_t)j * a.n + i] = w;
            }
        }
    }
    for (int l = 0; l < a.L; ++l) {
        unsigned long long v = cl[l];
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(a.clamps + l, v);
    }
}

// ---- k_forward_rows: fnn.forward_batch, fp64 (fnn.py:161-165) -------------
__global__ void k_forward_rows(const __grid_constant__ Net64P net, const double *__restrict__ x,
                               int64_t rows, double *__restrict__ y) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const double *xr = x + r * IN;
        double h1[HD];
        for (int h = 0; h < HD; ++h) {
            double acc = 0.0;
            for (int k = 0; k < IN; ++k) acc = fma(xr[k], net.w1[h * IN + k], acc);
            acc = acc + net.b1[h];
            h1[h] = acc > 0.0 ? acc : 0.0;
        }
        double out = 0.0;
        for (int o = 0; o < HD; ++o) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < HD; ++k) acc = fma(h1[k], net.w2[o * HD + k], acc);
            acc = acc + net.b2[o];
            out = fma(acc > 0.0 ? acc : 0.0, net.wo[o], out);
        }
        out = out + net.bo;
        y[r] = out > 0.0 ? out : 0.0;
    }
}

#ifdef CS_TC_TRACE
void *getenv_ptr(const char *name) {
    const char *v = getenv(name);
    return v ? (void *)strtoull(v, nullptr, 0) : nullptr;
}
#endif

int sm_count() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

// stream-K split scratch of the tcgen05 screen: one slot per (CTA, group) of
// a full-device grid, two pieces per slot, 3L+1 fields (L <= 8) x 128 threads
constexpr int kMaxSplitSlots = 4 * 256;
int split_slots() {
    const int s = 4 * sm_count();
    return s < kMaxSplitSlots ? s : kMaxSplitSlots;
}
size_t split_scratch_floats() { return (size_t)split_slots() * 2 * (3 * CS_MAX_BUDGETS + 1) * 128; }

int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "cosched_b200: CUDA error: %s\n", cudaGetErrorString(e));
        return CS_ERR_CUDA;
    }
    return CS_OK;
}

int check_grid(const cs_grid *g) {
    // (a config index fits 13 bits of a clamp-queue entry)
    if (!g || g->n_grid < 0 || g->n_grid >= 8192 || g->n_budgets < 1 || g->n_budgets > CS_MAX_BUDGETS)
        return CS_ERR_ARG;
    if (g->n_grid > 0 && (!g->knob1 || !g->knob2 || !g->mask)) return CS_ERR_ARG;
    // Empty budgets are legal here (the reference's optimize_corun works on a
    // budget without solo splits and optimize_solo_pair on one without co-run
    // configs); their records come out as index -1 / NaN and the host raises
    // CS_ERR_NO_CONFIG / CS_ERR_UNREACHABLE semantics only for what it reads.
    for (int l = 0; l < g->n_budgets; ++l) {
        if (g->solo_offsets[l + 1] < g->solo_offsets[l] || g->n_configs[l] < 0) return CS_ERR_ARG;
    }
    if (g->solo_offsets[0] != 0 || (g->solo_offsets[g->n_budgets] > 0 && !g->solo_knob)) return CS_ERR_ARG;
    return CS_OK;
}

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

int choose_log2_slices(int64_t P, int G) {
    // enough (pair, slice) threads to fill the SMs about twice over, but
    // keep >= ~4 configs per slice so the per-thread prologue stays amortized
    const int64_t target = (int64_t)sm_count() * 2048;
    int l2 = 0;
    while (l2 < 3 && P * (1LL << l2) < target && (G >> (l2 + 1)) >= 4) ++l2;
    return l2;
}

template <int L>
int launch_sweep(const SweepArgs &a, const Net32P &net, const Head64P &h64, int kind,
                 cudaStream_t st) {
    if (kind == CS_KERNEL_SIMT) {
        const int64_t threads = a.P << a.log2s;
        const int64_t blocks = (threads + kSweepThreads - 1) / kSweepThreads;
        k_sweep<L><<<(unsigned)blocks, kSweepThreads, 0, st>>>(a, net, h64);
        return CS_OK;
    }
    const int64_t nblocks = (a.P + tc::kPairsPerBlock - 1) / tc::kPairsPerBlock;
    if (kind != CS_KERNEL_TCGEN05 && (kind & 0xF00) != 0x300) return CS_ERR_ARG;
    // default: 4 compute groups x 2 TMEM stages, per-group issuer warps,
    // elected a_ready arrives, issuer registers handed to the compute warps
    // by setmaxnreg, whole items round-robin (0x203342); the stream-K schedule
    // (0xA03342) measured slower (the extra fp64 tails of split items cost
    // more than the idle SMs it fills); other 0xV3GS kinds select
    // the measured alternatives below and the timing-probe instances compiled
    // with -DCS_TIMING_PROBES (tools/build_probes.sh, never the product)
    if (kind == CS_KERNEL_TCGEN05) {
        // Fewer work items than half the device's group slots (N <~ 180), or a
        // few rounds whose last one is less than half full (N ~ 400-700): the
        // stream-K schedule spreads the configs over every group slot
        // (tools/time_steps.py: N=20 49 -> 32 us, N=128 58 -> 38 us, N=512
        // 195 -> 181 us).  Otherwise whole items round-robin (at N=256 and
        // N=4,096 the split items' refills and extra tails cost more than
        // the idle slots they fill).
        const int64_t slots = (int64_t)sm_count() * 4;
        const int64_t rounds = (nblocks + slots - 1) / slots;
        const bool few = 2 * nblocks <= slots;
        const bool ragged = rounds >= 2 && rounds <= 8 && 2 * (nblocks - (rounds - 1) * slots) < slots;
        kind = (few || ragged) ? 0xA03342 : 0x203342;
    }
    const int G = (kind >> 4) & 0xF, S = kind & 0xF;
    int V = (kind >> 12) & 0xFFF;
    // stream-K keeps its schedule arithmetic in 32 bits
    if ((V & 2048) && nblocks * (int64_t)a.g.G >= ((int64_t)1 << 31)) V &= ~2048;
    const size_t smem = tc3_smem_bytes(a.g.G);
    if (smem > 227 * 1024) return CS_ERR_ARG;   // grid too large for the staged K tables
    auto go3 = [&](auto kern, int groups, int threads) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return CS_ERR_CUDA;
        int64_t c = (nblocks + groups - 1) / groups;
        if (V & 2048) {
            // stream-K: every SM, as long as a group slot keeps >= 32 configs
            const int64_t work = nblocks * (int64_t)a.g.G;
            c = (work + (int64_t)groups * 32 - 1) / ((int64_t)groups * 32);
            if (c * groups > a.t.split_slots) c = a.t.split_slots / groups;
        }
        if (c > sm_count()) c = sm_count();
        if (c < 1) c = 1;
        // programmatic dependent launch: the CTAs' prologue (TMEM allocation,
        // mbarrier init) overlaps the tail of k_tables; the kernel waits on
        // griddepcontrol.wait before it reads anything k_tables wrote
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)c);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, a, net, h64) != cudaSuccess) {
            cudaGetLastError();
            kern<<<(unsigned)c, threads, smem, st>>>(a, net, h64);
        }
        return CS_OK;
    };
#define CS_TC3(GG, SS, VV) \
    if (G == GG && S == SS && V == VV) \
        return go3(k_sweep_tc3<L, GG, SS, VV>, GG, tc3::Cfg<GG, SS, VV>::kThreads);
    CS_TC3(4, 2, 515)    // default: setmaxnreg, round-robin whole items
    CS_TC3(4, 2, 2563)   // setmaxnreg + stream-K
    CS_TC3(4, 2, 3)      // round-robin, no register rebalancing
#ifdef CS_TIMING_PROBES
    CS_TC3(4, 2, 531) CS_TC3(4, 2, 579) CS_TC3(4, 2, 595)
    CS_TC3(4, 2, 1539)   // single-term screen (bit 10)
#endif
#undef CS_TC3
    return CS_ERR_ARG;
}

}  // namespace

// =========================================================================
// C ABI
// =========================================================================
extern "C" {

const char *cs_version(void) { return "cosched_b200 0.1.0 (sm_100a)"; }

#ifdef CS_TC_CLOCKS
// DEBUG BUILDS ONLY: the screen's clock trace (tools/clock_trace.sh)
int cs_debug_clocks(unsigned long long *h, int count) {
    const int cap = (int)(sizeof(g_tc_clk) / sizeof(g_tc_clk[0]));
    return cudaMemcpyFromSymbol(h, g_tc_clk, sizeof(unsigned long long) * (count < cap ? count : cap)) ==
                   cudaSuccess ? 0 : CS_ERR_CUDA;
}
#endif

const char *cs_error_string(int code) {
    switch (code) {
        case CS_OK: return "ok";
        case CS_ERR_ARG: return "invalid argument";
        case CS_ERR_NO_CONFIG: return "no co-run configs exist for a requested budget";
        case CS_ERR_UNREACHABLE: return "budget is unreachable on the cap grids (no solo split)";
        case CS_ERR_CUDA: return "CUDA runtime error";
        case CS_ERR_PRECISION: return "fp32 screen error too large for an exact argmin";
        case CS_ERR_WORKSPACE: return "workspace too small";
        default: return "unknown error";
    }
}

size_t cs_tables_bytes(int32_t n_apps, int32_t n_grid, int32_t n_solo) {
    if (n_apps < 0 || n_grid < 0 || n_solo < 0) return 0;
    size_t b = 0;
    b += align256(sizeof(uint16_t) * W2_TILE_ELEMS);
    b += 2 * align256(sizeof(float) * (size_t)n_apps * ROW32);
    b += 2 * align256(sizeof(double) * (size_t)n_apps * HD);
    b += 2 * align256(sizeof(float) * (size_t)n_grid * ROW32);
    b += 2 * align256(sizeof(double) * (size_t)n_grid * HD);
    b += align256(sizeof(double) * (size_t)n_solo * HD);
    b += align256(sizeof(double) * (size_t)kImgDoubles);
    b += align256(sizeof(float) * split_scratch_floats());
    b += align256(sizeof(uint32_t) * (size_t)split_slots());
    return b;
}

int cs_tables_bind(void *d_base, size_t bytes, int32_t n_apps, int32_t n_grid, int32_t n_solo,
                   cs_tables *out) {
    if (!d_base || !out || ((uintptr_t)d_base & 255)) return CS_ERR_ARG;
    if (bytes < cs_tables_bytes(n_apps, n_grid, n_solo)) return CS_ERR_WORKSPACE;
    char *p = (char *)d_base;
    auto take = [&p](size_t sz) { char *r = p; p += align256(sz); return (void *)r; };
    out->n_apps = n_apps; out->n_grid = n_grid; out->n_solo = n_solo;
    out->w2_tile = (uint16_t *)take(sizeof(uint16_t) * W2_TILE_ELEMS);
    out->app_a32 = (float *)take(sizeof(float) * (size_t)n_apps * ROW32);
    out->app_b32 = (float *)take(sizeof(float) * (size_t)n_apps * ROW32);
    out->app_a64 = (double *)take(sizeof(double) * (size_t)n_apps * HD);
    out->app_b64 = (double *)take(sizeof(double) * (size_t)n_apps * HD);
    // fp32 knob rows of both members interleaved per config ([G][2][20]), so
    // the screen stages the whole table with one bulk (TMA) copy
    out->knob1_32 = (float *)take(2 * sizeof(float) * (size_t)n_grid * ROW32);
    out->knob2_32 = out->knob1_32 + ROW32;
    // fp64 knob rows of both members interleaved per chunk (see knob64_at)
    out->knob1_64 = (double *)take(2 * sizeof(double) * (size_t)n_grid * HD);
    out->knob2_64 = out->knob1_64 + 2;
    out->solo64 = (double *)take(sizeof(double) * (size_t)n_solo * HD);
    out->net_image = (double *)take(sizeof(double) * (size_t)kImgDoubles);
    out->split_scratch = (float *)take(sizeof(float) * split_scratch_floats());
    out->split_cnt = (uint32_t *)take(sizeof(uint32_t) * (size_t)split_slots());
    out->split_slots = split_slots();
    return CS_OK;
}

int cs_tables_set_network(const cs_network *net, const cs_tables *tables, void *stream) {
    Net64P np;
    if (!net64_from(net, &np) || !tables || !tables->net_image) return CS_ERR_ARG;
    static_assert(offsetof(Net64P, w2) == sizeof(double) * kImgHeadOff, "image layout");
    double img[kImgDoubles];
    memcpy(img, &np, sizeof(Net64P));
    for (int h = 0; h < HD; ++h)
        for (int k = 0; k < IN; ++k) img[kImgW1tOff + k * HD + h] = np.w1[h * IN + k];
    for (int o = 0; o < HD; ++o)
        for (int k = 0; k < HD; ++k) img[kImgW2tOff + k * HD + o] = np.w2[o * HD + k];
    // pageable source: returns once the bytes are staged, so `img` may go out of scope
    if (cudaMemcpyAsync(tables->net_image, img, sizeof(img), cudaMemcpyHostToDevice,
                        (cudaStream_t)stream) != cudaSuccess) {
        cudaGetLastError();
        return CS_ERR_CUDA;
    }
    return CS_OK;
}

namespace {
int launch_tables(const cs_network *net, const double *d_features, int32_t n_apps,
                  const cs_grid *d_grid, const cs_tables *tables, const double *d_base_time,
                  cs_solo_out solo, int do_solo, cs_counters *reset_cnt,
                  unsigned long long *reset_clamps, void *stream) {
    Net64P np;
    if (!net64_from(net, &np) || !tables || n_apps < 2 || !d_features) return CS_ERR_ARG;
    int rc = check_grid(d_grid);
    if (rc) return rc;
    GridP g = grid_params(d_grid);
    if (tables->n_apps != n_apps || tables->n_grid != g.G || tables->n_solo < g.S) return CS_ERR_ARG;
    const int64_t items = ((int64_t)n_apps + g.G + g.S) * 32;
    int64_t threads = items > W2_TILE_ELEMS ? items : W2_TILE_ELEMS;
    int blocks = (int)((threads + 127) / 128);
    if (blocks > sm_count() * 16) blocks = sm_count() * 16;
    // programmatic dependent launch: the blocks stage the network image
    // while the previous kernel (the host call's input prologue) finishes
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(128);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_tables, np, d_features, n_apps, g, *tables, d_base_time, solo,
                           do_solo, reset_cnt, reset_clamps) != cudaSuccess) {
        cudaGetLastError();
        k_tables<<<blocks, 128, 0, (cudaStream_t)stream>>>(np, d_features, n_apps, g, *tables,
                                                            d_base_time, solo, do_solo, reset_cnt,
                                                            reset_clamps);
    }
    return check_launch();
}
}  // namespace

int cs_build_tables(const cs_network *net, const double *d_features, int32_t n_apps,
                    const cs_grid *d_grid, const cs_tables *tables, void *stream) {
    return launch_tables(net, d_features, n_apps, d_grid, tables, nullptr, cs_solo_out{}, 0, nullptr,
                         nullptr, stream);
}

int cs_prepare(const cs_network *net, const double *d_features, const double *d_base_time,
               int32_t n_apps, const cs_grid *d_grid, const cs_tables *tables, cs_solo_out out,
               cs_counters *d_counters, unsigned long long *d_clamps, void *stream) {
    int rc = check_grid(d_grid);
    if (rc) return rc;
    if (!d_base_time || !out.solo_time || !out.solo_split) return CS_ERR_ARG;
    const int S = d_grid->solo_offsets[d_grid->n_budgets];
    if (S <= 32)   // one warp per app evaluates all its splits
        return launch_tables(net, d_features, n_apps, d_grid, tables, d_base_time, out, 1, d_counters,
                             d_clamps, stream);
    rc = launch_tables(net, d_features, n_apps, d_grid, tables, nullptr, cs_solo_out{}, 0, d_counters,
                       d_clamps, stream);
    if (rc) return rc;
    return cs_solo(net, tables, d_grid, d_base_time, out, stream);
}

int cs_solo(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
            const double *d_base_time, cs_solo_out out, void *stream) {
    Net64P n64;
    if (!net64_from(net, &n64)) return CS_ERR_ARG;
    int rc = check_grid(d_grid);
    if (rc) return rc;
    if (!tables || !d_base_time || !out.solo_time || !out.solo_split) return CS_ERR_ARG;
    GridP g = grid_params(d_grid);
    const int64_t threads = (int64_t)tables->n_apps * g.L * 32;
    k_solo<<<(unsigned)((threads + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        *tables, g, d_base_time, tables->n_apps, out, head64_from(n64));
    return check_launch();
}

namespace {
int pair_screen_impl(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                     const double *d_base_time, int64_t pair_begin, int64_t pair_end,
                     double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                     unsigned long long *d_clamps, int kernel_kind, const double *d_solo_time,
                     const int32_t *d_solo_clamps, double *d_w, int fused, void *stream);
}

int cs_pair_screen(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                   const double *d_base_time, int64_t pair_begin, int64_t pair_end,
                   double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                   unsigned long long *d_clamps, int kernel_kind, void *stream) {
    return pair_screen_impl(net, tables, d_grid, d_base_time, pair_begin, pair_end, rel_eps, out,
                            d_queue, d_counters, d_clamps, kernel_kind, nullptr, nullptr,
                            nullptr, 0, stream);
}

namespace {
int resolve_impl(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                 const double *d_base_time, int64_t pair_begin, int64_t pair_end, cs_pair_out out,
                 const int64_t *d_queue, cs_counters *d_counters, const double *d_solo_time,
                 const int32_t *d_solo_clamps, unsigned long long *d_clamps, double *d_w,
                 int fused, void *stream);
}

int cs_pair_screen_fused(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                         const double *d_base_time, const double *d_solo_time,
                         const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                         double rel_eps, cs_pair_out out, int64_t *d_queue,
                         cs_counters *d_counters, unsigned long long *d_clamps, double *d_w,
                         int kernel_kind, void *stream) {
    if (!d_solo_time || !out.corun_chosen || !out.weight || !d_queue) return CS_ERR_ARG;
    if (kernel_kind == CS_KERNEL_AUTO) kernel_kind = CS_KERNEL_TCGEN05;
    if (kernel_kind != CS_KERNEL_TCGEN05 && (kernel_kind & 0xF00) != 0x300) return CS_ERR_ARG;
    return pair_screen_impl(net, tables, d_grid, d_base_time, pair_begin, pair_end, rel_eps, out,
                            d_queue, d_counters, d_clamps, kernel_kind, d_solo_time,
                            d_solo_clamps, d_w, 1, stream);
}

int cs_resolve_fused(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                     const double *d_base_time, const double *d_solo_time,
                     const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                     cs_pair_out out, const int64_t *d_queue, cs_counters *d_counters,
                     unsigned long long *d_clamps, double *d_w, void *stream) {
    if (!d_solo_time || !out.corun_chosen || !out.weight || !d_clamps) return CS_ERR_ARG;
    return resolve_impl(net, tables, d_grid, d_base_time, pair_begin, pair_end, out, d_queue,
                        d_counters, d_solo_time, d_solo_clamps, d_clamps, d_w, 1, stream);
}

namespace {
// the tensor-core screen's fp16 operands must hold |z1| and |W2|, |b2|
bool fp16_screen_safe(const cs_network *net) {
    Net64P n64;
    if (!net64_from(net, &n64)) return false;
    double zmax = 0.0, wmax = 0.0;
    for (int h = 0; h < HD; ++h) {
        double r = fabs(n64.b1[h]);
        for (int k = 0; k < IN; ++k) r += fabs(n64.w1[h * IN + k]);
        zmax = fmax(zmax, r);
        wmax = fmax(wmax, fabs(n64.b2[h]));
        for (int k = 0; k < HD; ++k) wmax = fmax(wmax, fabs(n64.w2[h * HD + k]));
    }
    return zmax < 30000.0 && wmax < 30000.0;
}
}  // namespace

int cs_pair_sweep_fused(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                        const double *d_base_time, const double *d_solo_time,
                        const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                        double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                        unsigned long long *d_clamps, double *d_w, int kernel_kind, void *stream) {
    if (kernel_kind == CS_KERNEL_AUTO && !fp16_screen_safe(net)) {
        // beyond the fp16 range: the fp32 SIMT screen, then resolve + decide
        // (+ scatter) as separate steps -- identical results
        int rc = cs_pair_screen(net, tables, d_grid, d_base_time, pair_begin, pair_end, rel_eps,
                                out, d_queue, d_counters, d_clamps, CS_KERNEL_SIMT, stream);
        if (rc) return rc;
        rc = cs_resolve(net, tables, d_grid, d_base_time, pair_begin, pair_end, out, d_queue,
                        d_counters, d_clamps, stream);
        if (rc) return rc;
        return cs_pair_decide(d_grid, d_solo_time, d_solo_clamps, tables->n_apps, pair_begin,
                              pair_end, out, d_clamps, d_w, stream);
    }
    int rc = cs_pair_screen_fused(net, tables, d_grid, d_base_time, d_solo_time, d_solo_clamps,
                                  pair_begin, pair_end, rel_eps, out, d_queue, d_counters,
                                  d_clamps, d_w, kernel_kind, stream);
    if (rc) return rc;
    return cs_resolve_fused(net, tables, d_grid, d_base_time, d_solo_time, d_solo_clamps,
                            pair_begin, pair_end, out, d_queue, d_counters, d_clamps, d_w,
                            stream);
}

namespace {
int pair_screen_impl(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                     const double *d_base_time, int64_t pair_begin, int64_t pair_end,
                     double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                     unsigned long long *d_clamps, int kernel_kind, const double *d_solo_time,
                     const int32_t *d_solo_clamps, double *d_w, int fused, void *stream) {
    Net64P n64;
    if (!net64_from(net, &n64)) return CS_ERR_ARG;
    int rc = check_grid(d_grid);
    if (rc) return rc;
    if (!tables || !d_base_time || !d_clamps || !out.corun_grid_index || !out.corun_time ||
        !d_queue || !d_counters)
        return CS_ERR_ARG;
    const int64_t n = tables->n_apps;
    const int64_t P_all = n * (n - 1) / 2;
    if (pair_begin < 0 || pair_end > P_all || pair_begin > pair_end) return CS_ERR_ARG;
    if (!(rel_eps > 0.0 && rel_eps < 0.1)) return CS_ERR_ARG;
    if (pair_begin == pair_end) return CS_OK;

    Net32P n32;
    for (int k = 0; k < HD * HD; ++k) n32.w2[k] = (float)n64.w2[k];
    for (int k = 0; k < HD; ++k) { n32.b2[k] = (float)n64.b2[k]; n32.wo[k] = (float)n64.wo[k]; }
    n32.bo = (float)n64.bo;

    SweepArgs a{};
    a.t = *tables;
    a.g = grid_params(d_grid);
    a.base_time = d_base_time;
    a.n = (int32_t)n;
    a.p_begin = pair_begin;
    a.P = pair_end - pair_begin;
    a.log2s = choose_log2_slices(a.P, a.g.G);
    a.eps = (float)rel_eps;
    a.near = (float)fmin(64.0 * rel_eps, 0.05);
    // verify ~1/8 of the near pairs, at most a few hundred per sweep (one wave
    // of k_resolve blocks)
    a.vstride = a.P >> 14 > 8 ? a.P >> 14 : 8;
    a.tau = (float)(0.5 * rel_eps);
    a.out = out;
    a.queue = d_queue;
    a.cnt = d_counters;
    a.clamps = d_clamps;
    a.trace = nullptr;
    a.fused = fused;
    a.W = d_w;
    a.solo_time = d_solo_time;
    a.solo_clamps = d_solo_clamps;
#ifdef CS_TC_TRACE
    a.trace = (uint32_t *)getenv_ptr("CS_TC_TRACE_PTR");
#endif
    cudaStream_t st = (cudaStream_t)stream;
    const Head64P h64 = head64_from(n64);
    if (kernel_kind == CS_KERNEL_AUTO) {
        // the fp16 split needs |h| and |W2|, |b2| inside the fp16 range; a
        // pathological network falls back to the fp32 SIMT screen
        double zmax = 0.0, wmax = 0.0;
        for (int h = 0; h < HD; ++h) {
            double r = fabs(n64.b1[h]);
            for (int k = 0; k < IN; ++k) r += fabs(n64.w1[h * IN + k]);
            zmax = fmax(zmax, r);
            wmax = fmax(wmax, fabs(n64.b2[h]));
            for (int k = 0; k < HD; ++k) wmax = fmax(wmax, fabs(n64.w2[h * HD + k]));
        }
        kernel_kind = (zmax < 30000.0 && wmax < 30000.0) ? CS_KERNEL_TCGEN05 : CS_KERNEL_SIMT;
    }
    if (kernel_kind != CS_KERNEL_TCGEN05 && kernel_kind != CS_KERNEL_SIMT &&
        (kernel_kind & 0xF00) != 0x300)
        return CS_ERR_ARG;
    int lrc;
    switch (a.g.L) {
        case 1: lrc = launch_sweep<1>(a, n32, h64, kernel_kind, st); break;
        case 2: lrc = launch_sweep<2>(a, n32, h64, kernel_kind, st); break;
        case 3: lrc = launch_sweep<3>(a, n32, h64, kernel_kind, st); break;
        case 4: lrc = launch_sweep<4>(a, n32, h64, kernel_kind, st); break;
        case 5: lrc = launch_sweep<5>(a, n32, h64, kernel_kind, st); break;
        case 6: lrc = launch_sweep<6>(a, n32, h64, kernel_kind, st); break;
        case 7: lrc = launch_sweep<7>(a, n32, h64, kernel_kind, st); break;
        case 8: lrc = launch_sweep<8>(a, n32, h64, kernel_kind, st); break;
        default: return CS_ERR_ARG;
    }
    if (lrc) return lrc;
    return check_launch();
}
}  // namespace

int cs_pair_decide(const cs_grid *d_grid, const double *d_solo_time, const int32_t *d_solo_clamps,
                   int32_t n_apps, int64_t pair_begin, int64_t pair_end, cs_pair_out out,
                   unsigned long long *d_clamps, double *d_w, void *stream) {
    int rc = check_grid(d_grid);
    if (rc) return rc;
    if (!d_solo_time || n_apps < 2 || !out.corun_grid_index || !out.corun_time ||
        !out.corun_chosen || !out.weight || (d_solo_clamps && !d_clamps))
        return CS_ERR_ARG;
    if (pair_begin < 0 || pair_end > (int64_t)n_apps * (n_apps - 1) / 2 || pair_begin > pair_end)
        return CS_ERR_ARG;
    if (pair_begin == pair_end) return CS_OK;
    DecideArgs d{};
    d.solo_time = d_solo_time;
    d.solo_clamps = d_solo_clamps;
    d.n = n_apps;
    d.L = d_grid->n_budgets;
    d.p_begin = pair_begin;
    d.P = pair_end - pair_begin;
    d.out = out;
    d.clamps = d_clamps;
    d.W = d_w;
    const int64_t total = d.P * d.L;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
    k_decide<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d);
    return check_launch();
}

int cs_pair_sweep(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                  const double *d_base_time, const double *d_solo_time,
                  const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                  double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                  unsigned long long *d_clamps, void *stream) {
    return cs_pair_sweep_ex(net, tables, d_grid, d_base_time, d_solo_time, d_solo_clamps,
                            pair_begin, pair_end, rel_eps, out, d_queue, d_counters, d_clamps,
                            CS_KERNEL_AUTO, stream);
}

int cs_pair_sweep_ex(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                     const double *d_base_time, const double *d_solo_time,
                     const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                     double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                     unsigned long long *d_clamps, int kernel_kind, void *stream) {
    int rc = cs_pair_screen(net, tables, d_grid, d_base_time, pair_begin, pair_end, rel_eps, out,
                            d_queue, d_counters, d_clamps, kernel_kind, stream);
    if (rc) return rc;
    rc = cs_resolve(net, tables, d_grid, d_base_time, pair_begin, pair_end, out, d_queue,
                    d_counters, d_clamps, stream);
    if (rc) return rc;
    return cs_pair_decide(d_grid, d_solo_time, d_solo_clamps, tables->n_apps, pair_begin,
                          pair_end, out, d_clamps, nullptr, stream);
}

namespace {
int resolve_impl(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                 const double *d_base_time, int64_t pair_begin, int64_t pair_end, cs_pair_out out,
                 const int64_t *d_queue, cs_counters *d_counters, const double *d_solo_time,
                 const int32_t *d_solo_clamps, unsigned long long *d_clamps, double *d_w,
                 int fused, void *stream) {
    Net64P n64;
    if (!net64_from(net, &n64)) return CS_ERR_ARG;
    int rc = check_grid(d_grid);
    if (rc) return rc;
    if (!tables || !d_base_time || !d_queue || !d_counters) return CS_ERR_ARG;
    if (pair_begin == pair_end) return CS_OK;
    ResolveArgs a{};
    a.t = *tables;
    a.g = grid_params(d_grid);
    a.base_time = d_base_time;
    a.n = tables->n_apps;
    a.p_begin = pair_begin;
    a.P = pair_end - pair_begin;
    a.out = out;
    a.queue = d_queue;
    a.cnt = d_counters;
    a.fused = fused;
    a.solo_time = d_solo_time;
    a.solo_clamps = d_solo_clamps;
    a.clamps = d_clamps;
    a.W = d_w;
    // the queue length lives on the device: one resident wave of blocks that
    // stride over it (an oversized grid costs a launch wave per 148 x 16 blocks)
    // programmatic dependent launch behind the screen (see k_sweep_tc3)
    const Head64P h64 = head64_from(n64);
    cudaLaunchConfig_t cfg = {};
    // 2 blocks per SM at k_resolve's register count: one wave
    cfg.gridDim = dim3((unsigned)(sm_count() * 2));
    cfg.blockDim = dim3(128);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_resolve, a, h64) != cudaSuccess) {
        cudaGetLastError();
        k_resolve<<<sm_count() * 2, 128, 0, (cudaStream_t)stream>>>(a, h64);
    }
    return check_launch();
}
}  // namespace

int cs_resolve(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
               const double *d_base_time, int64_t pair_begin, int64_t pair_end,
               cs_pair_out out, const int64_t *d_queue, cs_counters *d_counters,
               unsigned long long *d_clamps, void *stream) {
    if (!d_clamps) return CS_ERR_ARG;
    return resolve_impl(net, tables, d_grid, d_base_time, pair_begin, pair_end, out, d_queue,
                        d_counters, nullptr, nullptr, d_clamps, nullptr, 0, stream);
}

int cs_scatter_weights(const double *d_weight, int32_t n_apps, int64_t pair_begin,
                       int64_t pair_end, double *d_w, void *stream) {
    if (!d_weight || !d_w || n_apps < 2 || pair_begin < 0 || pair_end < pair_begin ||
        pair_end > (int64_t)n_apps * (n_apps - 1) / 2)
        return CS_ERR_ARG;
    const int64_t P = pair_end - pair_begin;
    if (!P) return CS_OK;
    int64_t blocks = (P + 255) / 256;
    if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
    k_scatter<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_weight, n_apps, pair_begin, P, d_w);
    return check_launch();
}

size_t cs_wire_records_bytes(int64_t cap, int32_t n_budgets) {
    if (cap < 0 || n_budgets < 1 || n_budgets > CS_MAX_BUDGETS) return 0;
    return wire_layout(cap, n_budgets).total;
}

int cs_pack_records(cs_pair_out shard, int64_t n_pairs, int32_t n_budgets, int64_t cap,
                    void *d_wire, void *stream) {
    if (!d_wire || n_pairs < 0 || cap < n_pairs || n_budgets < 1 || n_budgets > CS_MAX_BUDGETS ||
        !shard.corun_grid_index || !shard.corun_time || !shard.corun_chosen || ((uintptr_t)d_wire & 255))
        return CS_ERR_ARG;
    if (!n_pairs) return CS_OK;
    int64_t blocks = ((int64_t)n_budgets * n_pairs + 255) / 256;
    if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
    k_pack_records<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(shard, n_pairs, n_budgets, cap,
                                                                       (uint8_t *)d_wire);
    return check_launch();
}

int cs_unpack_gathered(const void *d_gathered, int32_t world, size_t wire_bytes, int32_t n_apps,
                       int32_t n_budgets, const double *d_solo_time, cs_pair_out full,
                       double *d_w, void *stream) {
    if (!d_gathered || world < 1 || n_apps < 2 || n_budgets < 1 || n_budgets > CS_MAX_BUDGETS ||
        !d_solo_time || !full.corun_grid_index || !full.corun_time || !full.corun_chosen ||
        !full.weight)
        return CS_ERR_ARG;
    const int64_t P = (int64_t)n_apps * (n_apps - 1) / 2;
    const int64_t cap = (P + world - 1) / world;
    if (wire_bytes != wire_layout(cap, n_budgets).total) return CS_ERR_ARG;
    int64_t blocks = (P + 255) / 256;
    if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
    k_unpack_gathered<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        (const uint8_t *)d_gathered, world, (int64_t)wire_bytes, P, n_apps, n_budgets, cap,
        d_solo_time, full, d_w);
    return check_launch();
}

int cs_analytic_sweep(const double *d_rp1, const double *d_rp2, const double *d_compute,
                      const double *d_memory, const double *coef, const double *d_base_time,
                      const double *d_solo_time, const uint32_t *d_mask, int32_t n_apps,
                      int32_t n_grid, int32_t n_budgets, cs_pair_out out, double *d_w,
                      unsigned long long *d_clamps, void *stream) {
    if (!d_rp1 || !d_rp2 || !d_compute || !d_memory || !coef || !d_base_time || !d_solo_time ||
        !d_mask || n_apps < 2 || n_grid < 1 || n_budgets < 1 || n_budgets > CS_MAX_BUDGETS ||
        !out.corun_grid_index || !out.corun_time || !out.corun_chosen || !out.weight || !d_clamps)
        return CS_ERR_ARG;
    AnalyticArgs a{};
    a.rp1 = d_rp1; a.rp2 = d_rp2; a.compute = d_compute; a.memory = d_memory;
    a.cc = coef[0]; a.mm = coef[1]; a.cm = coef[2];
    a.base_time = d_base_time; a.solo_time = d_solo_time; a.mask = d_mask;
    a.n = n_apps; a.G = n_grid; a.L = n_budgets;
    a.P = (int64_t)n_apps * (n_apps - 1) / 2;
    a.out = out; a.W = d_w; a.clamps = d_clamps;
    int64_t blocks = (a.P + 255) / 256;
    if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
    k_analytic<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a);
    return check_launch();
}

int cs_forward_rows(const cs_network *net, const double *d_x, int64_t rows, double *d_y,
                    void *stream) {
    Net64P np;
    if (!net64_from(net, &np) || rows < 0 || (rows > 0 && (!d_x || !d_y))) return CS_ERR_ARG;
    if (!rows) return CS_OK;
    int64_t blocks = (rows + 127) / 128;
    if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
    k_forward_rows<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(np, d_x, rows, d_y);
    return check_launch();
}

// ---- host-buffer build_graph ---------------------------------------------
namespace {
struct GraphLayout {
    size_t feats, bt, knob1, knob2, mask, solo_knob, tables, solo_time, solo_split, solo_clamps,
        corun_idx, corun_time, chosen, weight, queue, qcount, clamps, W, total;
};

GraphLayout graph_layout(int32_t n, const cs_grid *g) {
    GraphLayout L{};
    const int64_t P = (int64_t)n * (n - 1) / 2;
    const int64_t nb = g->n_budgets, G = g->n_grid, S = g->solo_offsets[g->n_budgets];
    size_t off = 0;
    auto put = [&off](size_t sz) { size_t r = off; off += align256(sz); return r; };
    L.feats = put(sizeof(double) * (size_t)n * NF);
    L.bt = put(sizeof(double) * (size_t)n);
    L.knob1 = put(sizeof(double) * (size_t)G * 4);
    L.knob2 = put(sizeof(double) * (size_t)G * 4);
    L.mask = put(sizeof(uint32_t) * (size_t)G);
    L.solo_knob = put(sizeof(double) * (size_t)S * 4);
    L.tables = put(cs_tables_bytes(n, (int32_t)G, (int32_t)S));
    L.solo_time = put(sizeof(double) * (size_t)(nb * n));
    L.solo_split = put(sizeof(int32_t) * (size_t)(nb * n));
    L.solo_clamps = put(sizeof(int32_t) * (size_t)(nb * n));
    L.corun_idx = put(sizeof(int32_t) * (size_t)(nb * P));
    L.corun_time = put(sizeof(double) * (size_t)(nb * P));
    L.chosen = put(sizeof(uint8_t) * (size_t)(nb * P));
    L.weight = put(sizeof(double) * (size_t)(nb * P));
    L.queue = put(sizeof(int64_t) * (size_t)((nb + 2) * P));
    L.qcount = put(sizeof(cs_counters));
    L.clamps = put(sizeof(unsigned long long) * (size_t)nb);
    L.W = put(sizeof(double) * (size_t)n * n * nb);
    L.total = off;
    return L;
}
}  // namespace

int cs_device_alloc(size_t bytes, void **d_out) {
    if (!d_out || !bytes) return CS_ERR_ARG;
    *d_out = nullptr;
    if (cudaMalloc(d_out, bytes) != cudaSuccess) {
        cudaGetLastError();
        return CS_ERR_CUDA;
    }
    return CS_OK;
}

int cs_device_free(void *d_ptr) {
    // a workspace retained for cs_build_graph_host loses its state first, so a
    // later allocation at the same address can never inherit it
    cs_workspace_release(d_ptr);
    if (d_ptr && cudaFree(d_ptr) != cudaSuccess) return CS_ERR_CUDA;
    return CS_OK;
}

size_t cs_build_graph_workspace_bytes(int32_t n_apps, const cs_grid *h_grid) {
    if (n_apps < 2 || check_grid(h_grid) != CS_OK) return 0;
    return graph_layout(n_apps, h_grid).total;
}

namespace {
// Host-call prologue when the caller's inputs sit in pinned (device-mapped)
// memory: read them over PCIe straight into the workspace -- one launch
// instead of two H2D copies.
__global__ void k_call_begin(const double *__restrict__ hf, const double *__restrict__ hbt,
                             double *__restrict__ df, double *__restrict__ dbt, int n) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // k_tables may stage now
    const int64_t nf = (int64_t)n * NF, total = nf + n;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (k < nf) df[k] = hf[k];
        else dbt[k - nf] = hbt[k - nf];
    }
}

// Host-call epilogue: every output straight into pinned host memory -- the
// N x N matrix, the per-pair records, the solo results, the clamp counts and
// the counters -- by one launch of coalesced 16-byte stores over PCIe instead
// of up to eleven D2H copies (each a DMA setup on the call's critical path).
// Segments whose ends are not 16-byte aligned are copied bytewise.
constexpr int kCallSegs = 12;
struct CallEndArgs {
    const uint8_t *src[kCallSegs];
    uint8_t *dst[kCallSegs];
    int64_t bytes[kCallSegs];
    int64_t start16[kCallSegs + 1];   // prefix sums of the segments' 16-byte chunks
    uint32_t aligned;                 // bit g: segment g's src and dst are 16-byte aligned
    int n;
};
__device__ __forceinline__ void copy_segments(const CallEndArgs &a, int64_t k0, int64_t stride) {
    const int64_t total = a.start16[a.n];
    for (int64_t k = k0; k < total; k += stride) {
        int g = 0;
        while (k >= a.start16[g + 1]) ++g;
        const int64_t off = (k - a.start16[g]) * 16;
        const int64_t rem = a.bytes[g] - off;
        if (rem >= 16 && ((a.aligned >> g) & 1u)) {
            *reinterpret_cast<uint4 *>(a.dst[g] + off) =
                __ldcg(reinterpret_cast<const uint4 *>(a.src[g] + off));
        } else {
            const int m = rem < 16 ? (int)rem : 16;
            for (int b = 0; b < m; ++b) a.dst[g][off + b] = a.src[g][off + b];
        }
    }
}
__global__ void k_call_end(const CallEndArgs a) {
    copy_segments(a, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// After a bulk copy of the matrix and records that ran concurrently with
// k_resolve: re-copy what k_resolve may have changed -- the records and the
// two matrix entries of every resolved (pair, budget) -- then the small
// outputs.  Stream order puts these writes after the bulk copy's.
struct CallFixArgs {
    CallEndArgs small;
    const int64_t *queue;
    const cs_counters *cnt;
    cs_pair_out dev, host;            // host: device-visible pinned pointers (null: not requested)
    const double *W;
    double *hW;                       // null: no matrix requested
    int64_t P;
    int n;
};
__global__ void k_call_fixup(const CallFixArgs a) {
    const int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    const uint32_t q = a.cnt->queue_len;
    for (int64_t k = k0; k < q; k += stride) {
        const int64_t e = a.queue[k];
        if (e & 8) continue;          // sampled re-scans of certain winners change nothing
        const int64_t pl = e >> 4;
        const int l = (int)(e & 7);
        const int64_t o = (int64_t)l * a.P + pl;
        // bytewise: the caller's host arrays need not be aligned
        auto put = [](void *dst, const void *src, int bytes) {
            for (int b = 0; b < bytes; ++b) ((uint8_t *)dst)[b] = ((const uint8_t *)src)[b];
        };
        if (a.host.corun_grid_index) put(a.host.corun_grid_index + o, a.dev.corun_grid_index + o, 4);
        if (a.host.corun_time) put(a.host.corun_time + o, a.dev.corun_time + o, 8);
        if (a.host.corun_chosen) put(a.host.corun_chosen + o, a.dev.corun_chosen + o, 1);
        if (a.host.weight) put(a.host.weight + o, a.dev.weight + o, 8);
        if (a.hW) {
            int i, j;
            pair_of(pl, a.n, i, j);
            const size_t b = (size_t)l * a.n * a.n;
            put(a.hW + b + (size_t)i * a.n + j, a.W + b + (size_t)i * a.n + j, 8);
            put(a.hW + b + (size_t)j * a.n + i, a.W + b + (size_t)j * a.n + i, 8);
        }
    }
    copy_segments(a.small, k0, stride);
}

// device-visible address of a pinned host buffer, or null (pageable / unknown)
void *mapped_v(const void *p) {
    if (!p) return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}
}  // namespace

namespace {
// The per-call part of cs_build_graph_host (everything after the cached
// uploads): enqueue only, no synchronization -- so it can be captured.
int enqueue_graph_call(const cs_network *net, const cs_grid *h_grid, const double *h_features,
                       const double *h_base_time, int32_t n_apps, double rel_eps, char *ws,
                       const GraphLayout &L, double *h_weights, cs_pair_out h_pairs,
                       cs_solo_out h_solo, unsigned long long *h_clamps, uint32_t *h_counters,
                       cudaStream_t st);

struct HostCallKey {
    const void *f, *bt, *w, *p0, *p1, *p2, *p3, *s0, *s1, *s2, *cl, *stream;
    int32_t n;
    double eps;
    bool operator==(const HostCallKey &o) const { return memcmp(this, &o, sizeof(*this)) == 0; }
};
struct HostCallGraph {
    HostCallKey key;
    cudaGraphExec_t exec = nullptr;
    int hits = 0;            // identical calls seen; capture on the second
    bool failed = false;     // capture failed once: this key stays on the direct path
    uint64_t used = 0;       // LRU stamp
};
constexpr size_t kMaxGraphsPerWorkspace = 4;

// State of a workspace the caller declared persistent (cs_workspace_retain):
// what was last uploaded into it, one pinned counter slot, and the CUDA
// graphs of its repeated calls.  Freed by cs_workspace_release (which
// cs_device_free calls), so no state outlives the allocation.
struct WorkspaceState {
    size_t bytes = 0;
    std::vector<uint8_t> key;      // grid + network + sizes of the resident uploads; empty = none
    uint32_t *h_counters = nullptr;
    std::vector<HostCallGraph> graphs;
    uint64_t clock = 0;
    std::mutex mu;                 // one call at a time per workspace
};
std::mutex g_ws_mu;
std::unordered_map<const void *, std::shared_ptr<WorkspaceState>> g_ws;

void drop_graphs(WorkspaceState &w) {
    for (auto &g : w.graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    w.graphs.clear();
}
}  // namespace

int cs_workspace_retain(void *d_workspace, size_t workspace_bytes) {
    if (!d_workspace || ((uintptr_t)d_workspace & 255) || !workspace_bytes) return CS_ERR_ARG;
    auto st = std::make_shared<WorkspaceState>();
    st->bytes = workspace_bytes;
    if (cudaHostAlloc((void **)&st->h_counters, sizeof(cs_counters), cudaHostAllocDefault) !=
        cudaSuccess) {
        cudaGetLastError();
        return CS_ERR_CUDA;
    }
    std::shared_ptr<WorkspaceState> old;
    {
        std::lock_guard<std::mutex> lock(g_ws_mu);
        auto &slot = g_ws[d_workspace];
        old.swap(slot);
        slot = st;
    }
    if (old) {
        std::lock_guard<std::mutex> lock(old->mu);
        drop_graphs(*old);
        cudaFreeHost(old->h_counters);
        old->h_counters = nullptr;
    }
    return CS_OK;
}

int cs_workspace_release(void *d_workspace) {
    if (!d_workspace) return CS_OK;
    std::shared_ptr<WorkspaceState> st;
    {
        std::lock_guard<std::mutex> lock(g_ws_mu);
        auto it = g_ws.find(d_workspace);
        if (it == g_ws.end()) return CS_OK;
        st = it->second;
        g_ws.erase(it);
    }
    std::lock_guard<std::mutex> lock(st->mu);   // waits out a call in flight on it
    drop_graphs(*st);
    if (st->h_counters) cudaFreeHost(st->h_counters);
    st->h_counters = nullptr;
    st->key.clear();
    return CS_OK;
}

int cs_build_graph_host(const cs_network *net, const cs_grid *h_grid, const double *h_features,
                        const double *h_base_time, int32_t n_apps, double rel_eps,
                        void *d_workspace, size_t workspace_bytes, double *h_weights,
                        cs_pair_out h_pairs, cs_solo_out h_solo,
                        unsigned long long *h_clamps, void *stream) {
    if (!net || !h_features || !h_base_time || n_apps < 2 || !d_workspace) return CS_ERR_ARG;
    int rc = check_grid(h_grid);
    if (rc) return rc;
    const GraphLayout L = graph_layout(n_apps, h_grid);
    if (workspace_bytes < L.total) return CS_ERR_WORKSPACE;
    if ((uintptr_t)d_workspace & 255) return CS_ERR_ARG;
    Net64P np;
    if (!net64_from(net, &np)) return CS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    char *ws = (char *)d_workspace;
    const int nb = h_grid->n_budgets, G = h_grid->n_grid, S = h_grid->solo_offsets[nb];
    const size_t n = (size_t)n_apps;
#define CS_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { cudaGetLastError(); \
        fprintf(stderr, "cosched_b200: %s\n", cudaGetErrorString(_e)); return CS_ERR_CUDA; } } while (0)
#define CS_RC(x) do { int _r = (x); if (_r) return _r; } while (0)
    // A retained workspace (cs_workspace_retain) keeps the knob grid, the
    // network image and the zeroed matrix between calls and re-uploads only
    // what changed; any other workspace is uploaded into on every call.
    std::shared_ptr<WorkspaceState> state;
    {
        std::lock_guard<std::mutex> lock(g_ws_mu);
        auto it = g_ws.find(d_workspace);
        if (it != g_ws.end() && it->second->bytes == workspace_bytes) state = it->second;
    }
    std::unique_lock<std::mutex> call_lock;
    if (state) call_lock = std::unique_lock<std::mutex>(state->mu);
    if (state && !state->h_counters) state.reset();   // released while we waited
    thread_local std::vector<uint8_t> key_buf;      // no allocation per call once grown
    std::vector<uint8_t> &key = key_buf;
    key.clear();
    {
        auto put = [&key](const void *p, size_t bytes) {
            const uint8_t *b = (const uint8_t *)p;
            key.insert(key.end(), b, b + bytes);
        };
        const int32_t dims[4] = {n_apps, nb, G, S};
        put(dims, sizeof(dims));
        if (G) {
            put(h_grid->knob1, sizeof(double) * G * 4);
            put(h_grid->knob2, sizeof(double) * G * 4);
            put(h_grid->mask, sizeof(uint32_t) * G);
        }
        if (S) put(h_grid->solo_knob, sizeof(double) * S * 4);
        put(&np, sizeof(np));
    }
    const bool fresh = !state || state->key != key;
    if (fresh) {
        if (state) {
            state->key.clear();       // recorded again only once the uploads went through
            drop_graphs(*state);      // captured graphs carry the old grid / network
        }
        if (G) {
            CS_TRY(cudaMemcpyAsync(ws + L.knob1, h_grid->knob1, sizeof(double) * G * 4, cudaMemcpyHostToDevice, st));
            CS_TRY(cudaMemcpyAsync(ws + L.knob2, h_grid->knob2, sizeof(double) * G * 4, cudaMemcpyHostToDevice, st));
            CS_TRY(cudaMemcpyAsync(ws + L.mask, h_grid->mask, sizeof(uint32_t) * G, cudaMemcpyHostToDevice, st));
        }
        if (S) CS_TRY(cudaMemcpyAsync(ws + L.solo_knob, h_grid->solo_knob, sizeof(double) * S * 4, cudaMemcpyHostToDevice, st));
        // the sweep writes every off-diagonal entry each call; the diagonal stays 0
        CS_TRY(cudaMemsetAsync(ws + L.W, 0, sizeof(double) * n * n * nb, st));
        // network image into the workspace's tables (pageable copy, outside any graph)
        cs_tables t;
        CS_RC(cs_tables_bind(ws + L.tables, cs_tables_bytes(n_apps, G, S), n_apps, G, S, &t));
        CS_RC(cs_tables_set_network(net, &t, stream));
    }
    uint32_t *h_counters = state ? state->h_counters : nullptr;
    // Per-call work: replayed as a CUDA graph once the same call (retained
    // workspace, pinned host buffers, same non-default stream) repeats -- one
    // launch instead of ~15 API calls.  Pageable inputs or the legacy stream
    // never try a capture.
    HostCallKey key2{h_features, h_base_time, h_weights,
                     h_pairs.corun_grid_index, h_pairs.corun_time, h_pairs.corun_chosen,
                     h_pairs.weight, h_solo.solo_time, h_solo.solo_split, h_solo.solo_clamps,
                     h_clamps, stream, n_apps, rel_eps};
    const bool capturable = state && stream && mapped_v(h_features) && mapped_v(h_base_time);
    cudaGraphExec_t exec = nullptr;
    bool try_capture = false;
    HostCallGraph *entry = nullptr;
    if (capturable) {
        for (auto &g : state->graphs)
            if (g.key == key2) entry = &g;
        if (!entry) {
            if (state->graphs.size() >= kMaxGraphsPerWorkspace) {
                auto lru = state->graphs.begin();
                for (auto it = state->graphs.begin(); it != state->graphs.end(); ++it)
                    if (it->used < lru->used) lru = it;
                if (lru->exec) cudaGraphExecDestroy(lru->exec);
                state->graphs.erase(lru);
            }
            state->graphs.push_back(HostCallGraph{key2});
            entry = &state->graphs.back();
        }
        entry->used = ++state->clock;
        if (entry->exec) exec = entry->exec;
        else if (!entry->failed && ++entry->hits >= 2) try_capture = true;
    }
    auto fail = [&](int code) {
        if (state) state->key.clear();   // the workspace contents are unknown now
        return code;
    };
    static const bool dbg = getenv("CS_DEBUG_HOSTCALL") != nullptr;
    if (dbg) fprintf(stderr, "cs_build_graph_host: %s (capturable %d)\n",
                     exec ? "graph replay" : try_capture ? "capture" : "eager", (int)capturable);
    if (exec) {
        if (cudaGraphLaunch(exec, st) != cudaSuccess) { cudaGetLastError(); return fail(CS_ERR_CUDA); }
    } else if (try_capture) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t ge = nullptr;
        bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        int erc = ok ? enqueue_graph_call(net, h_grid, h_features, h_base_time, n_apps, rel_eps, ws, L,
                                          h_weights, h_pairs, h_solo, h_clamps, h_counters, st)
                     : CS_ERR_CUDA;
        if (ok) ok = cudaStreamEndCapture(st, &graph) == cudaSuccess && erc == CS_OK;
        if (ok) ok = cudaGraphInstantiate(&ge, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        entry->exec = ok ? ge : nullptr;
        entry->failed = !ok;
        int lrc = CS_OK;
        if (ok) lrc = cudaGraphLaunch(ge, st) == cudaSuccess ? CS_OK : CS_ERR_CUDA;
        else lrc = enqueue_graph_call(net, h_grid, h_features, h_base_time, n_apps, rel_eps, ws, L,
                                      h_weights, h_pairs, h_solo, h_clamps, h_counters, st);
        if (lrc) { cudaGetLastError(); return fail(lrc); }
    } else {
        const int lrc = enqueue_graph_call(net, h_grid, h_features, h_base_time, n_apps, rel_eps, ws,
                                           L, h_weights, h_pairs, h_solo, h_clamps, h_counters, st);
        if (lrc) return fail(lrc);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) { cudaGetLastError(); return fail(CS_ERR_CUDA); }
    if (fresh && state) state->key = key;
    // The screen's certain winners carry the observed fp32-vs-fp64 gap; argmin
    // parity needs it well inside rel_eps.  Otherwise (a network far outside
    // the trained range) redo the call with a wider ambiguity band -- more
    // pairs go to the exact fp64 resolve, the results stay identical.
    cs_counters counters;
    auto read_counters = [&]() -> bool {
        if (h_counters) { memcpy(&counters, h_counters, sizeof(counters)); return true; }
        return cudaMemcpy(&counters, ws + L.qcount, sizeof(counters), cudaMemcpyDeviceToHost) == cudaSuccess;
    };
    for (double eps = rel_eps;;) {
        if (!read_counters()) { cudaGetLastError(); return fail(CS_ERR_CUDA); }
        float err;
        memcpy(&err, &counters.screen_err_bits, sizeof(err));
        // a sampled exact re-scan disagreeing with the screen counts like an
        // error at the band itself
        if (counters.verify_fail) err = fmaxf(err, (float)eps);
        if (!(err > 0.25 * eps)) break;
        eps = fmax(16.0 * eps, 16.0 * (double)err);
        if (!(eps < 0.1)) return CS_ERR_PRECISION;
        const int lrc = enqueue_graph_call(net, h_grid, h_features, h_base_time, n_apps, eps, ws, L,
                                           h_weights, h_pairs, h_solo, h_clamps, h_counters, st);
        if (lrc) return fail(lrc);
        if (cudaStreamSynchronize(st) != cudaSuccess) { cudaGetLastError(); return fail(CS_ERR_CUDA); }
    }
#undef CS_TRY
#undef CS_RC
    return CS_OK;
}

namespace {
// A second stream (and events) per host thread for the chunked call below:
// the D2H copies of finished row blocks run on it while the next chunk
// computes.  Thread-local, so concurrent callers (and their graph captures)
// never share a stream.
constexpr int kMaxCallChunks = 16;
struct CopyLane {
    int device = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[kMaxCallChunks + 1] = {};
};
CopyLane *copy_lane() {
    thread_local CopyLane lane;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    if (lane.s && lane.device == dev) return &lane;
    if (lane.s) {            // another device: the old lane's stream / events belong there
        lane.s = nullptr;
        for (auto &e : lane.ev) e = nullptr;
    }
    if (cudaStreamCreateWithFlags(&lane.s, cudaStreamNonBlocking) != cudaSuccess) { lane.s = nullptr; return nullptr; }
    for (auto &e : lane.ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) { lane.s = nullptr; return nullptr; }
    lane.device = dev;
    return &lane;
}

int enqueue_graph_call(const cs_network *net, const cs_grid *h_grid, const double *h_features,
                       const double *h_base_time, int32_t n_apps, double rel_eps, char *ws,
                       const GraphLayout &L, double *h_weights, cs_pair_out h_pairs,
                       cs_solo_out h_solo, unsigned long long *h_clamps, uint32_t *h_counters,
                       cudaStream_t st) {
    void *stream = st;
    const int64_t P = (int64_t)n_apps * (n_apps - 1) / 2;
    const int nb = h_grid->n_budgets, G = h_grid->n_grid, S = h_grid->solo_offsets[nb];
    const size_t n = (size_t)n_apps;
#define CS_TRY(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { \
        fprintf(stderr, "cosched_b200: %s\n", cudaGetErrorString(_e)); return CS_ERR_CUDA; } } while (0)
#define CS_RC(x) do { int _r = (x); if (_r) return _r; } while (0)
    // (the queue / clamp counters are zeroed by k_tables, cs_prepare below)
    const double *zf = (const double *)mapped_v(h_features), *zb = (const double *)mapped_v(h_base_time);
    if (zf && zb) {
        const int64_t items = (int64_t)n * NF + n;
        int blocks = (int)((items + 255) / 256);
        if (blocks > sm_count()) blocks = sm_count();
        k_call_begin<<<blocks, 256, 0, st>>>(zf, zb, (double *)(ws + L.feats), (double *)(ws + L.bt),
                                             n_apps);
        CS_TRY(cudaGetLastError());
    } else {
        CS_TRY(cudaMemcpyAsync(ws + L.feats, h_features, sizeof(double) * n * NF, cudaMemcpyHostToDevice, st));
        CS_TRY(cudaMemcpyAsync(ws + L.bt, h_base_time, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    }

    cs_grid dg = *h_grid;
    dg.knob1 = (const double *)(ws + L.knob1);
    dg.knob2 = (const double *)(ws + L.knob2);
    dg.mask = (const uint32_t *)(ws + L.mask);
    dg.solo_knob = (const double *)(ws + L.solo_knob);
    cs_tables t;
    CS_RC(cs_tables_bind(ws + L.tables, cs_tables_bytes(n_apps, G, S), n_apps, G, S, &t));
    cs_solo_out so{(double *)(ws + L.solo_time), (int32_t *)(ws + L.solo_split),
                   (int32_t *)(ws + L.solo_clamps)};
    CS_RC(cs_prepare(net, (const double *)(ws + L.feats), (const double *)(ws + L.bt), n_apps, &dg,
                     &t, so, (cs_counters *)(ws + L.qcount), (unsigned long long *)(ws + L.clamps),
                     stream));
    cs_pair_out po{(int32_t *)(ws + L.corun_idx), (double *)(ws + L.corun_time),
                   (uint8_t *)(ws + L.chosen), (double *)(ws + L.weight)};
    cs_counters *dcnt = (cs_counters *)(ws + L.qcount);
    const size_t LP = (size_t)nb * P, LN = (size_t)nb * n;
    // Large graphs: the pairs are swept in K chunks of whole
    // matrix rows (rows [r_k, r_k+1) = the pairs (i, j) with r_k <= i < r_k+1,
    // a contiguous pair range), and the host copies of what a chunk made final
    // (its rows' upper part and its columns' lower part) and of its records
    // run on a second stream while the next chunk computes.  The
    // re-scan queue is per chunk (its counters are reset in between); the
    // screen-error monitor, the sampled re-scan disagreements and the clamp
    // counts accumulate over the chunks.
    // (pinned destinations only: a pageable D2H would block the host thread
    // and serialize the chunks)
    // Chunking pays once the D2H bytes outweigh its fixed cost (8 launches,
    // ragged rounds): measured crossover ~14 MB (N ~ 1,000 with records,
    // ~1,400 without; tools/e2e_breakdown.py).  Below it the single sweep and
    // the one-kernel zero-copy epilogue win.
    static const double min_chunk_bytes =
        getenv("CS_HOSTCALL_CHUNK_BYTES") ? atof(getenv("CS_HOSTCALL_CHUNK_BYTES")) : 14e6;
    const double d2h_bytes = (h_weights ? 8.0 * n * n * nb : 0.0) +
                             (double)LP * ((h_pairs.corun_grid_index ? 4 : 0) + (h_pairs.corun_time ? 8 : 0) +
                                           (h_pairs.corun_chosen ? 1 : 0) + (h_pairs.weight ? 8 : 0));
    const bool big_mapped = (!h_weights || mapped_v(h_weights)) &&
                            (!h_pairs.corun_grid_index || mapped_v(h_pairs.corun_grid_index)) &&
                            (!h_pairs.corun_time || mapped_v(h_pairs.corun_time)) &&
                            (!h_pairs.corun_chosen || mapped_v(h_pairs.corun_chosen)) &&
                            (!h_pairs.weight || mapped_v(h_pairs.weight));
    const bool all_mapped = big_mapped && (!h_solo.solo_time || mapped_v(h_solo.solo_time)) &&
                            (!h_solo.solo_split || mapped_v(h_solo.solo_split)) &&
                            (!h_solo.solo_clamps || mapped_v(h_solo.solo_clamps)) &&
                            (!h_clamps || mapped_v(h_clamps)) && h_counters && mapped_v(h_counters);
    CopyLane *lane = (d2h_bytes >= min_chunk_bytes && h_weights && big_mapped) ? copy_lane() : nullptr;
    CopyLane *fork = nullptr;     // the small-graph path's second stream (below)
    if (lane) {
        const int K = 8;
        int64_t rows[K + 1];
        rows[0] = 0;
        rows[K] = n_apps;
        // shrinking chunks: a chunk's copies (29 B per pair with records)
        // take about half its compute time, so each chunk's copies hide
        // behind the next, smaller chunk, and only the last (4% of the pairs)
        // is copied after the sweep
        static const double cum[K] = {0.0, 0.25, 0.45, 0.61, 0.74, 0.84, 0.91, 0.96};
        for (int k = 1; k < K; ++k) {
            const int64_t target = (int64_t)(cum[k] * (double)P);
            int64_t r = rows[k - 1];
            while (r < n_apps - 1 && row_start(r + 1, n_apps) <= target) ++r;
            rows[k] = r > rows[k - 1] ? r : rows[k - 1];
        }
        for (int k = 0; k < K; ++k) {
            const int64_t r0 = rows[k], r1 = rows[k + 1];
            if (r1 <= r0) continue;
            const int64_t p0 = row_start(r0, n_apps), p1 = r1 >= n_apps - 1 ? P : row_start(r1, n_apps);
            if (k > 0) {       // a fresh re-scan queue (its entries are chunk-relative)
                CS_TRY(cudaMemsetAsync(&dcnt->queue_len, 0, sizeof(uint32_t), st));
                CS_TRY(cudaMemsetAsync(&dcnt->exact_rows, 0, sizeof(uint32_t), st));
            }
            // a chunk's records sit budget-major inside its own slice of the
            // workspace arrays, [nb p0, nb p1): the kernels index them with
            // the chunk's pair count as the budget stride
            const size_t np = (size_t)(p1 - p0), q0 = (size_t)nb * (size_t)p0;
            if (p1 > p0) {
                cs_pair_out pk{po.corun_grid_index + q0, po.corun_time + q0, po.corun_chosen + q0,
                               po.weight + q0};
                CS_RC(cs_pair_sweep_fused(net, &t, &dg, (const double *)(ws + L.bt), so.solo_time,
                                          so.solo_clamps, p0, p1, rel_eps, pk, (int64_t *)(ws + L.queue),
                                          dcnt, (unsigned long long *)(ws + L.clamps),
                                          (double *)(ws + L.W), CS_KERNEL_AUTO, stream));
            }
            CS_TRY(cudaEventRecord(lane->ev[k], st));
            CS_TRY(cudaStreamWaitEvent(lane->s, lane->ev[k], 0));
            // the entries chunk k made final: rows [r0, r1) from column r0 on,
            // and the column strip [r0, r1) of the rows below (W[a][b] with
            // min(a, b) in [r0, r1)) -- the columns left of r0 went with
            // earlier chunks, so the copy after the last chunk is only its
            // diagonal block
            for (int l = 0; l < nb; ++l) {
                const double *dW = (const double *)(ws + L.W) + (size_t)l * n * n;
                double *hW = h_weights + (size_t)l * n * n;
                CS_TRY(cudaMemcpy2DAsync(hW + r0 * n + r0, sizeof(double) * n, dW + r0 * n + r0,
                                         sizeof(double) * n, sizeof(double) * (n - r0), (size_t)(r1 - r0),
                                         cudaMemcpyDeviceToHost, lane->s));
                if ((size_t)r1 < n)
                    CS_TRY(cudaMemcpy2DAsync(hW + r1 * n + r0, sizeof(double) * n, dW + r1 * n + r0,
                                             sizeof(double) * n, sizeof(double) * (r1 - r0), n - (size_t)r1,
                                             cudaMemcpyDeviceToHost, lane->s));
                if (!np) continue;
                const size_t src = q0 + (size_t)l * np, dst = (size_t)l * (size_t)P + (size_t)p0;
                if (h_pairs.corun_grid_index) CS_TRY(cudaMemcpyAsync(h_pairs.corun_grid_index + dst, po.corun_grid_index + src, 4 * np, cudaMemcpyDeviceToHost, lane->s));
                if (h_pairs.corun_time) CS_TRY(cudaMemcpyAsync(h_pairs.corun_time + dst, po.corun_time + src, 8 * np, cudaMemcpyDeviceToHost, lane->s));
                if (h_pairs.corun_chosen) CS_TRY(cudaMemcpyAsync(h_pairs.corun_chosen + dst, po.corun_chosen + src, np, cudaMemcpyDeviceToHost, lane->s));
                if (h_pairs.weight) CS_TRY(cudaMemcpyAsync(h_pairs.weight + dst, po.weight + src, 8 * np, cudaMemcpyDeviceToHost, lane->s));
            }
        }
        CS_TRY(cudaEventRecord(lane->ev[K], lane->s));     // join the copies back
        CS_TRY(cudaStreamWaitEvent(st, lane->ev[K], 0));
    } else if (fp16_screen_safe(net) && all_mapped && (fork = copy_lane()) != nullptr) {
        // the screen, then the bulk copy of the matrix and records on a second
        // stream WHILE k_resolve re-scans the few queued pairs; k_call_fixup
        // (below) re-copies those pairs once both are done
        double *dW = h_weights ? (double *)(ws + L.W) : nullptr;
        CS_RC(cs_pair_screen_fused(net, &t, &dg, (const double *)(ws + L.bt), so.solo_time,
                                   so.solo_clamps, 0, P, rel_eps, po, (int64_t *)(ws + L.queue), dcnt,
                                   (unsigned long long *)(ws + L.clamps), dW, CS_KERNEL_TCGEN05, stream));
        CS_TRY(cudaEventRecord(fork->ev[0], st));
        CS_TRY(cudaStreamWaitEvent(fork->s, fork->ev[0], 0));
        CallEndArgs bulk{};
        auto add = [&bulk](void *h_dst, const void *d_src, size_t bytes) {
            if (!h_dst || !bytes) return;
            void *m = mapped_v(h_dst);
            bulk.src[bulk.n] = (const uint8_t *)d_src;
            bulk.dst[bulk.n] = (uint8_t *)m;
            bulk.bytes[bulk.n] = (int64_t)bytes;
            if ((((uintptr_t)d_src | (uintptr_t)m) & 15) == 0) bulk.aligned |= 1u << bulk.n;
            bulk.start16[bulk.n + 1] = bulk.start16[bulk.n] + (int64_t)((bytes + 15) / 16);
            ++bulk.n;
        };
        if (h_weights) add(h_weights, ws + L.W, sizeof(double) * n * n * nb);
        add(h_pairs.corun_grid_index, po.corun_grid_index, 4 * LP);
        add(h_pairs.corun_time, po.corun_time, 8 * LP);
        add(h_pairs.corun_chosen, po.corun_chosen, LP);
        add(h_pairs.weight, po.weight, 8 * LP);
        if (bulk.n) {
            int blocks = (int)((bulk.start16[bulk.n] + 255) / 256);
            if (blocks > 2 * sm_count()) blocks = 2 * sm_count();
            k_call_end<<<blocks, 256, 0, fork->s>>>(bulk);
            CS_TRY(cudaGetLastError());
        }
        CS_TRY(cudaEventRecord(fork->ev[1], fork->s));
        CS_RC(cs_resolve_fused(net, &t, &dg, (const double *)(ws + L.bt), so.solo_time, so.solo_clamps,
                               0, P, po, (int64_t *)(ws + L.queue), dcnt, (unsigned long long *)(ws + L.clamps),
                               dW, stream));
        CS_TRY(cudaStreamWaitEvent(st, fork->ev[1], 0));
    } else {
        CS_RC(cs_pair_sweep_fused(net, &t, &dg, (const double *)(ws + L.bt), so.solo_time,
                                  so.solo_clamps, 0, P, rel_eps, po, (int64_t *)(ws + L.queue), dcnt,
                                  (unsigned long long *)(ws + L.clamps),
                                  h_weights ? (double *)(ws + L.W) : nullptr, CS_KERNEL_AUTO, stream));
    }
    // the outputs (+ the queue length / screen-error monitor the caller checks
    // after the sync): one epilogue kernel when every destination is pinned,
    // else plain copies
    CallEndArgs e{};
    bool zc_out = true;
    auto seg = [&](void *h_dst, const void *d_src, size_t bytes) {
        if (!h_dst || !bytes || !zc_out) return;
        void *m = mapped_v(h_dst);
        if (!m || e.n == kCallSegs) { zc_out = false; return; }
        e.src[e.n] = (const uint8_t *)d_src;
        e.dst[e.n] = (uint8_t *)m;
        e.bytes[e.n] = (int64_t)bytes;
        if ((((uintptr_t)d_src | (uintptr_t)m) & 15) == 0) e.aligned |= 1u << e.n;
        e.start16[e.n + 1] = e.start16[e.n] + (int64_t)((bytes + 15) / 16);
        ++e.n;
    };
    if (!lane && !fork) {
        if (h_weights) seg(h_weights, ws + L.W, sizeof(double) * n * n * nb);
        seg(h_pairs.corun_grid_index, po.corun_grid_index, 4 * LP);
        seg(h_pairs.corun_time, po.corun_time, 8 * LP);
        seg(h_pairs.corun_chosen, po.corun_chosen, LP);
        seg(h_pairs.weight, po.weight, 8 * LP);
    }
    seg(h_solo.solo_time, so.solo_time, 8 * LN);
    seg(h_solo.solo_split, so.solo_split, 4 * LN);
    seg(h_solo.solo_clamps, so.solo_clamps, 4 * LN);
    seg(h_clamps, ws + L.clamps, 8 * (size_t)nb);
    seg(h_counters, ws + L.qcount, sizeof(cs_counters));
    if (fork) {
        CallFixArgs fx{};
        fx.small = e;
        fx.queue = (const int64_t *)(ws + L.queue);
        fx.cnt = dcnt;
        fx.dev = po;
        fx.host = cs_pair_out{(int32_t *)mapped_v(h_pairs.corun_grid_index), (double *)mapped_v(h_pairs.corun_time),
                              (uint8_t *)mapped_v(h_pairs.corun_chosen), (double *)mapped_v(h_pairs.weight)};
        fx.W = (const double *)(ws + L.W);
        fx.hW = h_weights ? (double *)mapped_v(h_weights) : nullptr;
        fx.P = P;
        fx.n = n_apps;
        k_call_fixup<<<sm_count(), 256, 0, st>>>(fx);
        CS_TRY(cudaGetLastError());
    } else if (zc_out) {
        const int64_t items = e.start16[e.n];
        int blocks = (int)((items + 255) / 256);
        if (blocks > 2 * sm_count()) blocks = 2 * sm_count();
        if (blocks < 1) blocks = 1;
        k_call_end<<<blocks, 256, 0, st>>>(e);
        CS_TRY(cudaGetLastError());
    } else {
        if (!lane) {
            if (h_weights)
                CS_TRY(cudaMemcpyAsync(h_weights, ws + L.W, sizeof(double) * n * n * nb,
                                       cudaMemcpyDeviceToHost, st));
            if (h_pairs.corun_grid_index) CS_TRY(cudaMemcpyAsync(h_pairs.corun_grid_index, po.corun_grid_index, 4 * LP, cudaMemcpyDeviceToHost, st));
            if (h_pairs.corun_time) CS_TRY(cudaMemcpyAsync(h_pairs.corun_time, po.corun_time, 8 * LP, cudaMemcpyDeviceToHost, st));
            if (h_pairs.corun_chosen) CS_TRY(cudaMemcpyAsync(h_pairs.corun_chosen, po.corun_chosen, LP, cudaMemcpyDeviceToHost, st));
            if (h_pairs.weight) CS_TRY(cudaMemcpyAsync(h_pairs.weight, po.weight, 8 * LP, cudaMemcpyDeviceToHost, st));
        }
        if (h_solo.solo_time) CS_TRY(cudaMemcpyAsync(h_solo.solo_time, so.solo_time, 8 * LN, cudaMemcpyDeviceToHost, st));
        if (h_solo.solo_split) CS_TRY(cudaMemcpyAsync(h_solo.solo_split, so.solo_split, 4 * LN, cudaMemcpyDeviceToHost, st));
        if (h_solo.solo_clamps) CS_TRY(cudaMemcpyAsync(h_solo.solo_clamps, so.solo_clamps, 4 * LN, cudaMemcpyDeviceToHost, st));
        if (h_clamps) CS_TRY(cudaMemcpyAsync(h_clamps, ws + L.clamps, 8 * (size_t)nb, cudaMemcpyDeviceToHost, st));
        if (h_counters) CS_TRY(cudaMemcpyAsync(h_counters, ws + L.qcount, sizeof(cs_counters), cudaMemcpyDeviceToHost, st));
    }
#undef CS_TRY
#undef CS_RC
    return CS_OK;
}
}  // namespace


}  // extern "C"
