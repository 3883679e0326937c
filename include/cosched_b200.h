/*
 * cosched_b200.h -- C ABI of the B200 pair x knob sweep.
 *
 * The reference (arXiv 2405.03831, package `cosched`, pure Python) has no
 * native boundary; the entry points below are what its optimizer/scheduler
 * layer binds (ctypes stub in INTEGRATION.md) to replace, for a trained-FNN
 * model, the per-pair Python loops:
 *
 *   cs_build_tables   replaces core.normalize_input (core.py:334-377) + the
 *                     first layer of fnn.forward_batch (fnn.py:163) by factored
 *                     per-app / per-knob partials computed once per sweep.
 *   cs_solo           replaces estimator.solorun_time (estimator.py:139-180)
 *                     via hwopt.optimize_solo_pair (hwopt.py:68-74), hoisted
 *                     to one evaluation per (app, split).
 *   cs_pair_sweep     replaces scheduler.build_graph's per-pair loop
 *   + cs_resolve      (scheduler.py:52-78) over hwopt.decide_pair
 *                     (hwopt.py:77-87) -> optimize_corun (hwopt.py:44-65) ->
 *                     estimator.corun_time (estimator.py:112-129) ->
 *                     slowdown floor (estimator.py:98-109).
 *   cs_scatter_weights fills the symmetric N x N matrix handed to
 *                     matcher.PairGraph (matcher.py:28-63; scheduler.py:73-77).
 *   cs_forward_rows   replaces fnn.forward / forward_batch (fnn.py:146-165) for
 *                     scalar queries (FnnSlowdownModel.predict_slowdown,
 *                     estimator.py:59-67).
 *   cs_build_graph_host  the whole build_graph with HOST buffers (H2D, tables,
 *                     solo, sweep, resolve, scatter, D2H) in one call.
 *
 * Conventions: every `d_` pointer is device memory owned by the caller; every
 * `h_` pointer is host memory (pinned for overlap, pageable works).  Only
 * cs_device_alloc and cs_workspace_retain allocate; calls are stream-ordered on `stream` (a cudaStream_t, NULL =
 * legacy default stream) and only cs_build_graph_host synchronizes.  The only
 * state kept between calls is that of workspaces the caller explicitly
 * retains (cs_workspace_retain); calls are re-entrant across host threads
 * and devices.
 * Return value: 0 on success, a negative CS_ERR_* code otherwise.
 *
 * Pairs are unordered (i < j) in row-major order, linear index
 *   p(i, j) = i*(2N - i - 1)/2 + (j - i - 1)          (scheduler.py:61)
 * and a shard is a contiguous range [pair_begin, pair_end).
 */
#ifndef COSCHED_B200_H
#define COSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_NUM_FEATURES 18   /* core.py:18  */
#define CS_INPUT_DIM 40      /* core.py:21  */
#define CS_HIDDEN 18         /* fnn.py:19   */
#define CS_MAX_BUDGETS 8     /* budgets swept in one call */

enum {
    CS_OK = 0,
    CS_ERR_ARG = -1,          /* bad shape/size/pointer                -> ValidationError */
    CS_ERR_NO_CONFIG = -2,    /* a budget admits no co-run config      (hwopt.py:62-64)   */
    CS_ERR_UNREACHABLE = -3,  /* a budget admits no solo split         (estimator.py:165) */
    CS_ERR_CUDA = -4,         /* CUDA launch/runtime failure           -> RuntimeError    */
    CS_ERR_WORKSPACE = -5,    /* workspace smaller than required       -> ValueError      */
    CS_ERR_PRECISION = -6     /* screen error beyond any usable rel_eps -> RuntimeError   */
};

/* Screen kernels of cs_pair_sweep_ex (results are identical: both feed the same
 * exact fp64 re-evaluation / re-scan). */
enum {
    CS_KERNEL_AUTO = 0,          /* tcgen05 on sm_100a                                    */
    CS_KERNEL_TCGEN05 = 1,       /* layer 2 on tensor cores, A operand in TMEM, fp16 3-term
                                    split, fp32 accumulate                                */
    CS_KERNEL_SIMT = 2           /* layer 2 as fp32 FFMA with W2 in the parameter bank
                                    (also the fallback for networks beyond fp16 range)   */
};

/* NetworkWeights (fnn.py:42-68), HOST fp64, row-major exactly as the
 * reference's JSON v1 document (fnn.py:311-324).  Copied by value into the
 * kernel parameter bank at each launch. */
typedef struct {
    const double *w1;             /* 18 x 40 */
    const double *b1;             /* 18      */
    const double *w2;             /* 18 x 18 */
    const double *b2;             /* 18      */
    const double *w_out;          /* 1 x 18  */
    const double *b_out;          /* 1       */
    const double *feature_bounds; /* 36      */
} cs_network;

/* The knob grid of L budgets (core.py:380-407).  Configs are the union of
 * each budget's co-run list, in the reference's lexicographic enumeration
 * order (so first-index tie-breaking per budget is preserved).  knob rows are
 * the normalized model inputs [cores/32, gpcs/8, cpu_cap/250, gpu_cap/250]
 * (core.py:368-371) of the member-1 view and of the reversed-partition
 * member-2 view (core.py:152-159).  mask[c] bit l = config c is legal in
 * budget l.  Solo splits of budget l are rows [solo_offsets[l],
 * solo_offsets[l+1]) of solo_knob ([1, 1, c/250, g/250]).
 * Pointers are device memory for the device-level calls, host memory for
 * cs_build_graph_host. */
typedef struct {
    int32_t n_grid;               /* G */
    const double *knob1;          /* G x 4 */
    const double *knob2;          /* G x 4 */
    const uint32_t *mask;         /* G     */
    int32_t n_budgets;            /* L, 1..CS_MAX_BUDGETS */
    int32_t n_configs[CS_MAX_BUDGETS];         /* host: configs legal in budget l */
    int32_t solo_offsets[CS_MAX_BUDGETS + 1];  /* host: solo rows of budget l */
    const double *solo_knob;      /* solo_offsets[L] x 4 */
} cs_grid;

/* Device tables carved from one caller buffer by cs_tables_bind. */
typedef struct {
    int32_t n_apps, n_grid, n_solo;
    uint16_t *w2_tile;            /* fp16 [W2hi|W2hi|W2lo|b2] B operand of the tcgen05 screen */
    float *app_a32, *app_b32;     /* N x 20 (18 + pad): primary / co-runner partials */
    double *app_a64, *app_b64;    /* 18 x N, chunk-major: [9][N] double2 */
    float *knob1_32, *knob2_32;   /* b1 folded; [G][2][20], K1|K2 interleaved (row stride 40), knob2_32 = knob1_32 + 20 */
    double *knob1_64, *knob2_64;  /* b1 folded; [9][G][2] double2, K1|K2 interleaved, knob2_64 = knob1_64 + 2 */
    double *solo64;               /* S x 18, b1 folded */
    double *net_image;            /* the network in device memory (cs_tables_set_network) */
    float *split_scratch;         /* tcgen05 screen, stream-K: partial argmins of work items
                                     cut between group slots, [slots][2][3L+1][128] */
    uint32_t *split_cnt;          /* per slot: pieces of its split item seen so far (zeroed
                                     by cs_prepare, left zero by the screen) */
    int32_t split_slots;          /* capacity of the two arrays above (group slots) */
} cs_tables;

/* Per-pair outputs of one shard, budget-major: element [l * P + (p - pair_begin)]. */
typedef struct {
    int32_t *corun_grid_index;    /* best config, index into the grid (-1: none) */
    double *corun_time;           /* CoRunTime of that config, fp64 re-evaluated */
    uint8_t *corun_chosen;        /* corun_time <= solo pair time (hwopt.py:86) */
    double *weight;               /* winning_time (hwopt.py:39-41) */
} cs_pair_out;

/* Per-app solo results, budget-major [l * N + a]. */
typedef struct {
    double *solo_time;            /* best exclusive time at the budget */
    int32_t *solo_split;          /* index within the budget's solo list */
    int32_t *solo_clamps;         /* floor clamps over that app's splits */
} cs_solo_out;

const char *cs_version(void);
const char *cs_error_string(int code);

/* --- device-level, stream-ordered -------------------------------------- */
size_t cs_tables_bytes(int32_t n_apps, int32_t n_grid, int32_t n_solo);
int cs_tables_bind(void *d_base, size_t bytes, int32_t n_apps, int32_t n_grid, int32_t n_solo,
                   cs_tables *out);
/* Copy the network into the tables' device image.  Call once after binding
 * (and whenever the weights change) BEFORE any kernel call that takes these
 * tables: the kernels read the weights from device memory (coalesced) instead
 * of the kernel parameter bank, whose lane-divergent reads serialize.  The
 * copy is issued on `stream` from pageable host memory (the call returns once
 * the host data is staged), so it must not be captured into a CUDA graph. */
int cs_tables_set_network(const cs_network *net, const cs_tables *tables, void *stream);

int cs_build_tables(const cs_network *net, const double *d_features, int32_t n_apps,
                    const cs_grid *d_grid, const cs_tables *tables, void *stream);

int cs_solo(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
            const double *d_base_time, cs_solo_out out, void *stream);

/* Counters of one screen (cs_pair_screen[_fused] -> cs_resolve[_fused]);
 * the caller zeroes them before each sweep (cs_prepare can). */
typedef struct {
    uint32_t queue_len;          /* (pair, budget)s queued for the exact fp64 re-scan        */
    uint32_t screen_err_bits;    /* float bits: largest relative gap seen between a screened
                                    time and its fp64 value (winners and near-tie runner-ups) */
    uint32_t exact_rows;         /* (pair, member) rows queued for an fp64 re-count of their
                                    floor clamps (a screened prediction within tau of 0.5)    */
    uint32_t verify_fail;        /* sampled near-tie pairs whose exact fp64 re-scan disagreed
                                    with the screen's winner (0 expected; the host redoes the
                                    sweep with a wider band otherwise)                        */
} cs_counters;

/* cs_build_tables + cs_solo in ONE launch (each app's warp also evaluates its
 * exclusive splits; falls back to two launches when a grid stacks more than 32
 * solo splits).  Results identical to the two calls.  d_counters and d_clamps
 * (L x u64), when not NULL, are zeroed by the same launch -- ready for the
 * screen that follows (no separate memsets in the sweep's CUDA graph). */
int cs_prepare(const cs_network *net, const double *d_features, const double *d_base_time,
               int32_t n_apps, const cs_grid *d_grid, const cs_tables *tables, cs_solo_out out,
               cs_counters *d_counters, unsigned long long *d_clamps, void *stream);

/* The pair sweep is three stream-ordered steps (cs_solo may run concurrently
 * with the first two; only cs_pair_decide reads the solo results):
 *
 *   cs_pair_screen  screens every (pair, config) of the shard -- on the tensor
 *                   cores by default (CS_KERNEL_*) -- keeping per (pair,
 *                   budget) the first-index minimum and the runner-up (value
 *                   and index).  When the runner-up is more than rel_eps above
 *                   the minimum the winner is re-evaluated in fp64
 *                   (corun_grid_index / corun_time final); a sample of the
 *                   pairs whose runner-up is within 64 rel_eps is queued for a
 *                   full fp64 re-scan as a check (d_counters->verify_fail).
 *                   Ambiguous (pair, budget)s get
 *                   corun_grid_index = -2 and an entry in d_queue, which needs
 *                   (L + 2) * P int64 slots.  Co-run floor clamps accumulate
 *                   in d_clamps (L x u64, zeroed): counted from the screen,
 *                   except for a (pair, member) row with a screened
 *                   prediction within tau = rel_eps / 2 of the 0.5 floor,
 *                   which is queued (d_queue[L P ...], d_counters->exact_rows).
 *   cs_resolve      exact fp64 first-index argmin for every queued (pair,
 *                   budget); fp64 re-count of the floor clamps of every
 *                   queued row into d_clamps.
 *   cs_pair_decide  co-run vs time-share per (pair, budget) against the solo
 *                   pair sum, adds the solo clamps the reference counts per
 *                   pair (so d_clamps ends equal to clamp_stats over
 *                   build_graph, estimator.py:98-109), and optionally scatters
 *                   the winning times into d_w (L x N x N, zeroed by the caller).
 *
 * `net` (host) is passed to the kernels that need it by value (parameter
 * bank).  cs_pair_sweep[_ex] = screen + resolve + decide without d_w. */
int cs_pair_screen(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                   const double *d_base_time, int64_t pair_begin, int64_t pair_end,
                   double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                   unsigned long long *d_clamps, int kernel_kind, void *stream);

int cs_resolve(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
               const double *d_base_time, int64_t pair_begin, int64_t pair_end,
               cs_pair_out out, const int64_t *d_queue, cs_counters *d_counters,
               unsigned long long *d_clamps, void *stream);

int cs_pair_decide(const cs_grid *d_grid, const double *d_solo_time, const int32_t *d_solo_clamps,
                   int32_t n_apps, int64_t pair_begin, int64_t pair_end, cs_pair_out out,
                   unsigned long long *d_clamps, double *d_w, void *stream);

/* The pair sweep in TWO launches (tcgen05 screen only: CS_KERNEL_AUTO /
 * CS_KERNEL_TCGEN05): the screen decides every
 * unambiguous (pair, budget) itself -- co-run vs time-share against
 * d_solo_time (cs_prepare / cs_solo, stream-ordered before) and the scatter
 * into d_w (L x N x N, zeroed once by the caller; NULL to skip) -- and k_resolve
 * does the same for the queued ones after their exact fp64 re-scan.  Same
 * results and counters as cs_pair_screen + cs_resolve + cs_pair_decide. */
int cs_pair_sweep_fused(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                        const double *d_base_time, const double *d_solo_time,
                        const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                        double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                        unsigned long long *d_clamps, double *d_w, int kernel_kind, void *stream);
/* Its two launches separately (cs_pair_sweep_fused = screen_fused + resolve_fused). */
int cs_pair_screen_fused(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                         const double *d_base_time, const double *d_solo_time,
                         const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                         double rel_eps, cs_pair_out out, int64_t *d_queue,
                         cs_counters *d_counters, unsigned long long *d_clamps, double *d_w,
                         int kernel_kind, void *stream);
int cs_resolve_fused(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                     const double *d_base_time, const double *d_solo_time,
                     const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                     cs_pair_out out, const int64_t *d_queue, cs_counters *d_counters,
                     unsigned long long *d_clamps, double *d_w, void *stream);

int cs_pair_sweep(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                  const double *d_base_time, const double *d_solo_time,
                  const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                  double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                  unsigned long long *d_clamps, void *stream);

int cs_pair_sweep_ex(const cs_network *net, const cs_tables *tables, const cs_grid *d_grid,
                     const double *d_base_time, const double *d_solo_time,
                     const int32_t *d_solo_clamps, int64_t pair_begin, int64_t pair_end,
                     double rel_eps, cs_pair_out out, int64_t *d_queue, cs_counters *d_counters,
                     unsigned long long *d_clamps, int kernel_kind, void *stream);

/* W[i*N+j] = W[j*N+i] = weight of budget `budget`; the caller zeroes W. */
int cs_scatter_weights(const double *d_weight, int32_t n_apps, int64_t pair_begin,
                       int64_t pair_end, double *d_w, void *stream);

/* --- multi-GPU record exchange (dist.py) -------------------------------- *
 * The wire format of one rank's shard: 11 bytes per (pair, budget) --
 * corun_time f64 | corun_grid_index u16 (0xFFFF: none) | corun_chosen u8 --
 * each field budget-major with `cap` slots per budget, 256-B aligned.  The
 * winning weight is not sent: rank 0 re-derives it exactly as the sweep does
 * (co-run time if chosen, else (0.0 + t_i) + t_j, hwopt.py:39-41).  Every
 * rank's buffer has the same size, so one NCCL gather to rank 0 moves them
 * all (rank r owns pairs dist.shard_range(P, r, world)). */
size_t cs_wire_records_bytes(int64_t cap, int32_t n_budgets);
/* shard records (cs_pair_out with row stride n_pairs) -> wire buffer */
int cs_pack_records(cs_pair_out shard, int64_t n_pairs, int32_t n_budgets, int64_t cap,
                    void *d_wire, void *stream);
/* rank 0: the `world` gathered wire buffers (wire_bytes each, rank order) ->
 * the full record set `full` (L x P, P = N(N-1)/2; weight re-derived from
 * d_solo_time, L x N) and, when d_w is not NULL, the symmetric L x N x N
 * matrix (diagonal left untouched: zero it once). */
int cs_unpack_gathered(const void *d_gathered, int32_t world, size_t wire_bytes, int32_t n_apps,
                       int32_t n_budgets, const double *d_solo_time, cs_pair_out full,
                       double *d_w, void *stream);

/* The pair sweep with the reference's ANALYTIC oracle as the model
 * (simenv.py:154-233) instead of the FNN.  The caller
 * passes, config-major (G x N), the products resource*power of every app for
 * the member-1 view (d_rp1) and the reversed-partition view (d_rp2), the apps'
 * compute / memory intensities, coef = {compute_compute, memory_memory,
 * compute_memory}, and the solo times (L x N).  Outputs as cs_pair_out
 * (exact: fp64 without contraction); d_w (L x N x N, zeroed) optional;
 * d_clamps (L, zeroed) counts co-run floor clamps. */
int cs_analytic_sweep(const double *d_rp1, const double *d_rp2, const double *d_compute,
                      const double *d_memory, const double *coef, const double *d_base_time,
                      const double *d_solo_time, const uint32_t *d_mask, int32_t n_apps,
                      int32_t n_grid, int32_t n_budgets, cs_pair_out out, double *d_w,
                      unsigned long long *d_clamps, void *stream);

/* fnn.forward_batch on rows x 40 normalized inputs (fp64, unfloored). */
int cs_forward_rows(const cs_network *net, const double *d_x, int64_t rows, double *d_y,
                    void *stream);

/* --- host-buffer convenience: the whole build_graph --------------------- */
/* Device workspace for callers without their own allocator (the ctypes binding
 * in INTEGRATION.md): cudaMalloc / cudaFree on the current device, 256-byte
 * aligned.  These are the only allocating calls of the ABI. */
int cs_device_alloc(size_t bytes, void **d_out);
int cs_device_free(void *d_ptr);

size_t cs_build_graph_workspace_bytes(int32_t n_apps, const cs_grid *h_grid);
/* Optional persistence of a cs_build_graph_host workspace.  After
 * cs_workspace_retain the library keeps the knob grid, the network image and
 * the zeroed matrix resident in d_workspace, re-uploads only what changed, and
 * replays repeated identical calls (pinned host buffers, non-default stream)
 * as a CUDA graph (at most 4 per workspace, LRU).  The caller must not write
 * the workspace between calls and must call cs_workspace_release before
 * freeing it (cs_device_free does so).  A workspace that was never retained
 * is uploaded into on every call and carries no state between calls.  One
 * call at a time per workspace (calls on one retained workspace serialize). */
int cs_workspace_retain(void *d_workspace, size_t workspace_bytes);
int cs_workspace_release(void *d_workspace);
/* h_weights: L x N x N (NULL to skip); h_pairs members: L x P host arrays
 * (NULL members skipped); h_solo members: L x N host arrays (NULL skipped);
 * h_clamps: L (NULL to skip).  Full graph (all P pairs).  Synchronizes
 * `stream` before returning.  Transfers: pinned inputs are read by a
 * zero-copy kernel; when every destination is pinned, kernels write the
 * outputs into them over PCIe -- the matrix and records on a second stream
 * beside k_resolve, then a fixup of the resolved pairs and the small
 * outputs (else cudaMemcpyAsync per array);
 * calls with >= 14 MB of pinned outputs sweep in 8 row chunks
 * and copy each finished row block while the next one computes. */
int cs_build_graph_host(const cs_network *net, const cs_grid *h_grid, const double *h_features,
                        const double *h_base_time, int32_t n_apps, double rel_eps,
                        void *d_workspace, size_t workspace_bytes, double *h_weights,
                        cs_pair_out h_pairs, cs_solo_out h_solo,
                        unsigned long long *h_clamps, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* COSCHED_B200_H */
