// tc3_sweep.cuh -- the tcgen05 screen (k_sweep_tc3): pair x knob tiles through
// layer 2 of the network on the tensor cores, fused with the floor, the
// objective, the per-budget argmin and the exact fp64 winner.
//
// Per CTA: G = 4 compute warpgroups ("groups", 128 threads: TMEM lane r = pair
// r/2 of the group's 64-pair work item, member r%2) and one MMA-issuer warp
// per group.  Per config the group's threads build their A rows (layer-1
// ReLU, fp16 hi/lo split) straight into TMEM, the issuer warp's elected lane
// issues 4 x tcgen05.mma M128 N24 K16 (A in TMEM, B = the W2 split in SMEM),
// and the epilogue reads D back with tcgen05.ld for the head and the argmin.
// S = 2 TMEM stages pipeline build(c) against epilogue(c - 1).
//
// Instruction diet (CUDA-core issue is the binding limit, profiles/r2*):
//   * the config loop is unrolled over the S stages, so every TMEM address,
//     mbarrier address and phase bit is a compile-time offset;
//   * one elected arrive per warp on a_ready; the issuer warps sleep in
//     mbarrier.try_wait with a suspend-time hint;
//   * the K1/K2 rows of a config are interleaved ([c][member][20], one TMA
//     bulk copy) so both member lanes of a warp read one 160-byte line;
//   * setmaxnreg moves the issuer warpgroup's registers to the compute
//     warpgroups (32 / 112).
//
// Work schedule (V bit 11, "stream-K"): the G x gridDim group slots split the
// flattened (work item, config) space into equal contiguous ranges, so every
// SM gets the same number of config steps even when there are fewer work
// items than slots (256 apps: 510 items for 592 slots).  An item cut between
// slots is finished by the LAST of its pieces to arrive: each piece leaves its
// partial (min, first index, runner-up, smallest prediction) per thread in
// the split scratch (cs_tables.split_scratch), bumps the item's counter, and
// the last one merges the pieces in config order -- the same first-index
// argmin -- then runs the exact tail.  Without bit 11 each slot takes whole
// items round-robin.
#pragma once

#ifdef CS_TC_CLOCKS
// DEBUG BUILDS ONLY (tools/clock_trace.sh): per-config timestamps of block 0's
// first work item, configs [kClk0, kClk0 + 32), read back by cs_debug_clocks
__device__ unsigned long long g_tc_clk[4 * 4 * 4 * 32 + 4 * 2 * 32];
constexpr int kClk0 = 20;
#define TC_CLK(slot) (g_tc_clk[slot] = clock64())
#endif

namespace tc3 {

// V bit 0: one elected arrive per warp on a_ready (count 4);
// V bit 1: one MMA-issuer warp per group;
// V bit 9: setmaxnreg register rebalancing (issuers 32, compute 112);
// V bit 10: single-term screen -- A = fp16 RN(ReLU(z1)) only (no lo split),
//           3 MMAs (A W2hi + A W2lo + tail); needs a wider ambiguity band;
// V bit 11: stream-K work schedule (above).
// Timing probes (tools/build_probes.sh, -DCS_TIMING_PROBES; WRONG results by
// design, never in the product .so): bit 4 no MMAs / waits, bit 6 no fp64
// winner re-evaluation, bit 7 no record / matrix writes.
template <int G, int S, int V = 0>
struct Cfg {
    static constexpr bool kMaxNReg = (V & 512) != 0;
    static constexpr bool kStreamK = (V & 2048) != 0;
    static constexpr bool kOneTerm = (V & 1024) != 0;
#ifdef CS_TIMING_PROBES
    static constexpr bool kNoTensor = (V & 16) != 0;
    static constexpr bool kNoExact = (V & 64) != 0;
    static constexpr bool kNoWrite = (V & 128) != 0;
#else
    static constexpr bool kNoTensor = false, kNoExact = false, kNoWrite = false;
#endif
    static_assert((V & 3) == 3, "elected arrives and per-group issuer warps");
    static_assert(!kMaxNReg || G == 4, "warpgroup-aligned roles for setmaxnreg");
    static constexpr int kThreads = G * tc::kGroupThreads + G * 32;
    static_assert(G * S * 56 <= 512, "TMEM holds 512 columns");
    __device__ static constexpr uint32_t d_col(int g, int s) { return (uint32_t)((g * S + s) * 32); }
    __device__ static constexpr uint32_t a_col(int g, int s) {
        return (uint32_t)(G * S * 32 + (g * S + s) * 24);
    }
};

// try_wait with a suspend-time hint: the warp sleeps in the barrier unit
// instead of re-issuing the probe (used by the MMA-issuer warps)
__device__ __forceinline__ bool mbar_try_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    if (mbar_try_sleep(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_sleep(bar, parity)) {
        if (clock64() - t0 > 4000000000LL) __trap();
    }
}

// warp-uniform wait: the exit test is a warp vote, so the warp leaves the
// loop converged and the .sync.aligned tcgen05 ops that follow need no
// __syncwarp (bounded like tc::mbar_wait)
__device__ __forceinline__ void mbar_wait_warp(uint64_t *bar, uint32_t parity) {
    if (__all_sync(0xffffffffu, tc::mbar_try(bar, parity))) return;
    const long long t0 = clock64();
    while (!__all_sync(0xffffffffu, tc::mbar_try(bar, parity))) {
        if (clock64() - t0 > 4000000000LL) __trap();
    }
}

// tcgen05.st of the 20 live A columns as 8 + 8 + 4 (smaller register blocks
// than one x16 leave ptxas room to store the conversions in place)
__device__ __forceinline__ void tmem_st20_848(uint32_t taddr, const uint32_t (&w)[20]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr + 8),
                 "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
                 "r"(w[15])
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + 16),
                 "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19])
                 : "memory");
}

// The 4 MMAs of one (group, config) plus the commit, issued by ONE elected
// lane inside a single asm block that the whole (converged) warp executes:
// no divergent branch around tcgen05.mma, so ptxas does not wrap every MMA in
// a uniformization loop.  tools/mma_bench.cu measured 29 cycles/MMA issued
// this way against 75+ for a `lane == 0` branch (the tensor pipe itself
// sustains one M128 N32 K16 MMA per ~16 cycles per SM).
//   z2 = A_s0 q0 + A_s1 q0 + A_s2 q1 + A_s0 q2
template <bool kOneTerm>
__device__ __forceinline__ void issue_config(uint32_t d_t, uint32_t a_t, uint64_t bq0, uint64_t bq1,
                                             uint64_t bq2, uint64_t *bar) {
    if constexpr (kOneTerm) {
        // z2 = A_s0 q0 + A_s2 q1 + A_s0 q2 (A_s2 column 17 holds zeros)
        asm volatile(
            "{\n\t.reg .pred e, pf, pt;\n\t"
            "setp.ne.b32 pf, %6, %6;\n\t"
            "setp.eq.b32 pt, %6, %6;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %6, pf;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %4, %6, pt;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %6, pt;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%2];\n}"
            ::"r"(d_t), "r"(a_t), "r"(tc::smem_u32(bar)), "l"(bq0), "l"(bq1), "l"(bq2), "r"(tc::kIdesc),
              "r"(a_t + 16)
            : "memory");
        return;
    }
    asm volatile(
        "{\n\t.reg .pred e, pf, pt;\n\t"
        "setp.ne.b32 pf, %6, %6;\n\t"
        "setp.eq.b32 pt, %6, %6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %6, pf;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %3, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %4, %6, pt;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %6, pt;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%2];\n}"
        ::"r"(d_t), "r"(a_t), "r"(tc::smem_u32(bar)), "l"(bq0), "l"(bq1), "l"(bq2), "r"(tc::kIdesc),
          "r"(a_t + 8), "r"(a_t + 16)
        : "memory");
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds2(uint32_t a) {
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}

// this thread's A row of one config (20 live 32-bit TMEM columns, layout of
// tcgen05_util.cuh), stored into its TMEM lane.  krow: 32-bit shared-window
// address of this member's K row (a plain integer, so ptxas never re-derives
// the generic->shared mapping in the loop)
template <bool kOneTerm>
__device__ __forceinline__ void build_row(const float2 (&p2)[9], uint32_t krow, uint32_t taddr) {
    const float4 q0 = lds4(krow), q1 = lds4(krow + 16), q2 = lds4(krow + 32), q3 = lds4(krow + 48);
    const float2 q4 = lds2(krow + 64);
    const float2 kr[9] = {make_float2(q0.x, q0.y), make_float2(q0.z, q0.w),
                          make_float2(q1.x, q1.y), make_float2(q1.z, q1.w),
                          make_float2(q2.x, q2.y), make_float2(q2.z, q2.w),
                          make_float2(q3.x, q3.y), make_float2(q3.z, q3.w), q4};
    uint32_t w[20];
    if constexpr (kOneTerm) {
        // hi only, rounded to nearest; columns 8-15 are never read
#pragma unroll
        for (int v = 0; v < 9; ++v) {
            const float2 z = tc2::add2(p2[v], kr[v]);
            const uint32_t hw = tc2::cvt_rn_relu(z.x, z.y);
            if (v < 8) w[v] = hw;
            else w[16] = hw;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + 16),
                     "r"(w[16]), "r"(0u), "r"(0x3C003C00u), "r"(w[16])
                     : "memory");
        tc2::tmem_st_wait();
        tc::fence_before();
        return;
    }
#pragma unroll
    for (int v = 0; v < 9; ++v) {
        const float2 z = tc2::add2(p2[v], kr[v]);
        const uint32_t hw = tc2::cvt_rz_relu(z.x, z.y);
        // the residual z - hi straight from the packed halves: one mixed
        // f16*f16+f32 FMA (FHFMA) per element, no f16->f32 unpack
        const float2 lo = tc2::residual_h2(hw, z);
        const uint32_t lw = tc2::cvt_rn_relu(lo.x, lo.y);
        if (v < 8) { w[v] = hw; w[8 + v] = lw; }
        else { w[16] = hw; w[17] = lw; }
    }
    w[18] = 0x3C003C00u;   // (1.0h, 1.0h): carries b2
    w[19] = w[16];         // (hi16, hi17) again: carries W2lo[:, 16:18]
    tmem_st20_848(taddr, w);
    tc2::tmem_st_wait();
    tc::fence_before();
}

__device__ __forceinline__ float2 lds_f32x2(const float *p) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                 : "=f"(v.x), "=f"(v.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

__device__ __forceinline__ void group_sync(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(tc::kGroupThreads) : "memory");
}

// The work of one group slot: contiguous segments (work item, [c0, c1)).
// All stream-K arithmetic is 32-bit (the launcher keeps W = items x configs
// below 2^31): 64-bit divisions compile to calls that spill the live state.
struct Schedule {
    int64_t nblocks, T64, blk;    // round-robin: items, slots, next item
    uint32_t T, k, n_cfg;         // slots, this slot, configs per item
    uint32_t W, q, r;             // stream-K: W = items * n_cfg = q * T + r
    uint32_t pos, end;
    bool stream_k;
    // start of slot kk's range: floor(kk * W / T) exactly, as kk q + kk r / T
    __device__ uint32_t bound(uint32_t kk) const { return kk * q + (kk * r) / T; }
    // the slot whose range holds flattened position x
    __device__ uint32_t slot_of(uint32_t x) const {
        uint32_t kk = (uint32_t)((float)x * ((float)T / (float)W));
        if (kk >= T) kk = T - 1;
        while (kk + 1 < T && bound(kk + 1) <= x) ++kk;
        while (kk > 0 && bound(kk) > x) --kk;
        return kk;
    }
    __device__ void init() {
        if (stream_k) { pos = bound(k); end = bound(k + 1); }
        else blk = k;
    }
    __device__ bool next(int64_t &item, int &c0, int &c1) {
        if (stream_k) {
            if (pos >= end) return false;
            const uint32_t it = pos / n_cfg;
            item = it;
            c0 = (int)(pos - it * n_cfg);
            c1 = (int)(c0 + (end - pos) < n_cfg ? c0 + (end - pos) : n_cfg);
            pos += (uint32_t)(c1 - c0);
            return true;
        }
        if (blk >= nblocks) return false;
        item = blk;
        c0 = 0;
        c1 = (int)n_cfg;
        blk += T64;
        return true;
    }
    // which of slot kk's two scratch sides holds its piece of `item`:
    // 0 = the first segment of its range, 1 = the last
    __device__ int side(uint32_t kk, uint32_t item) const { return bound(kk) / n_cfg == item ? 0 : 1; }
};

}  // namespace tc3

template <int L, int G, int S, int V>
__global__ void __launch_bounds__(tc3::Cfg<G, S, V>::kThreads, 1)
    k_sweep_tc3(const SweepArgs a, const __grid_constant__ Net32P net,
                const __grid_constant__ Head64P net_param) {
    using C = tc3::Cfg<G, S, V>;
    constexpr int kThreads = C::kThreads;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ int s_last[G];                 // stream-K: this group finishes the item
    // carve: [B slices 4 KB][K12: G_cfg x 2 x 20 fp32][mask G_cfg][d_ready G*S][a_ready G*S]
    //        [staged][tmem slot][Head64P][wo, bo fp32]
    uint8_t *b_tile = smem;
    float *k12 = reinterpret_cast<float *>(b_tile + tc2::kBBytes);
    uint32_t *masks = reinterpret_cast<uint32_t *>(k12 + (size_t)a.g.G * 2 * ROW32);
    uint64_t *d_ready = reinterpret_cast<uint64_t *>(
        smem + ((reinterpret_cast<uint8_t *>(masks + a.g.G) - smem + 7) & ~ptrdiff_t(7)));
    uint64_t *a_ready = d_ready + G * S;
    uint64_t *staged = a_ready + G * S;        // completion of the prologue's bulk copies
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(staged + 1);
    Head64P *net64 = reinterpret_cast<Head64P *>(
        smem + ((reinterpret_cast<uint8_t *>(staged + 3) - smem + 15) & ~ptrdiff_t(15)));
    float *wo_s = reinterpret_cast<float *>(net64 + 1);          // wo[18], bo
    static_assert(sizeof(Head64P) % 16 == 0, "bulk-copy granule");

    const int tid = threadIdx.x;
    const int g = tid / tc::kGroupThreads;     // == G: the MMA-issuer warpgroup
    const int t = tid % tc::kGroupThreads;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    // prologue that reads nothing of k_tables' output: barriers + TMEM first
    if (tid == 0) {
        for (int i = 0; i < G * S; ++i) {
            tc::mbar_init(&d_ready[i], 1);
            tc::mbar_init(&a_ready[i], tc::kGroupThreads / 32);
        }
        tc::mbar_init(staged, 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
    // programmatic dependent launch: wait for k_tables' results to be visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // a programmatically dependent k_resolve may be scheduled now: its blocks
    // take SMs this grid leaves free and stage their weights, then wait for
    // this grid to finish before reading the queue
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the per-sweep tables k_tables wrote -- the fp16 B operand (W2 split), the
    // interleaved K1|K2 knob rows and the fp64 head -- are staged by TMA bulk
    // copies issued by one thread, completing on `staged`
    if (tid == 0) {
        const uint32_t kbytes = (uint32_t)a.g.G * 2 * ROW32 * sizeof(float);
        tc::mbar_expect_tx(staged, tc2::kBBytes + kbytes + (uint32_t)sizeof(Head64P));
        tc::bulk_g2s(b_tile, a.t.w2_tile, tc2::kBBytes, staged);
        tc::bulk_g2s(k12, a.t.knob1_32, kbytes, staged);
        tc::bulk_g2s(net64, a.t.net_image + kImgHeadOff, (uint32_t)sizeof(Head64P), staged);
    }
    for (int i = tid; i < a.g.G; i += kThreads) masks[i] = L == 1 ? 1u : a.g.mask[i];
    // 0.5 wo (the |z2| half of the ReLU, see `math`) and bo
    if (tid <= HD) wo_s[tid] = tid < HD ? 0.5f * net.wo[tid] : net.bo;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    tc::mbar_wait(staged, 0);
    const uint32_t tmem_base = *tmem_slot;
    const int n_cfg = a.g.G;
    tc3::Schedule sched;
    sched.nblocks = (a.P + tc::kPairsPerBlock - 1) / tc::kPairsPerBlock;
    sched.T = gridDim.x * G;
    sched.T64 = sched.T;
    sched.k = blockIdx.x * G + (g < G ? g : warp - G * (tc::kGroupThreads / 32));
    sched.n_cfg = (uint32_t)n_cfg;
    sched.W = (uint32_t)(sched.nblocks * n_cfg);        // < 2^31 (launcher)
    sched.q = sched.W / sched.T;
    sched.r = sched.W - sched.q * sched.T;
    sched.stream_k = C::kStreamK;
    sched.init();

    // setmaxnreg sits at the head of each role's branch: code after it that
    // both roles share would be register-allocated for the smaller budget
    if (g >= G) {
        // ===== MMA-issuer warp q serves group q: the same segments, in order =====
        if (C::kMaxNReg) asm volatile("setmaxnreg.dec.sync.aligned.u32 32;" ::: "memory");
        const uint32_t b_addr = tc::smem_u32(b_tile);
        const uint64_t bq0 = tc2::slice_desc(b_addr), bq1 = tc2::slice_desc(b_addr + 1024),
                       bq2 = tc2::slice_desc(b_addr + 2048);
        if (C::kNoTensor) {
            // timing probe: CUDA-core work only (results are garbage)
        } else {
            const int q = warp - G * (tc::kGroupThreads / 32);
            uint32_t ph = 0;                           // bit s: parity of a_ready[q][s]
            int64_t item;
            int c0, c1;
            while (sched.next(item, c0, c1)) {
                int st = 0;                            // stages restart per segment
                for (int c = c0; c < c1; ++c) {
                    const int b = q * S + st;
                    tc3::mbar_wait_sleep(&a_ready[b], (ph >> st) & 1u);
#ifdef CS_TC_CLOCKS
                    const bool clk = blockIdx.x == 0 && item == (int64_t)q && lane == 0 &&
                                     c >= kClk0 && c < kClk0 + 32;
                    if (clk) TC_CLK(4 * 4 * 4 * 32 + (q * 2 + 0) * 32 + (c - kClk0));
#endif
                    ph ^= 1u << st;
                    __syncwarp();
                    tc::fence_after();
                    tc3::issue_config<C::kOneTerm>(tmem_base + C::d_col(q, st), tmem_base + C::a_col(q, st),
                                      bq0, bq1, bq2, &d_ready[b]);
#ifdef CS_TC_CLOCKS
                    if (clk) TC_CLK(4 * 4 * 4 * 32 + (q * 2 + 1) * 32 + (c - kClk0));
#endif
                    st = st + 1 == S ? 0 : st + 1;
                }
            }
        }
    } else {
        if (C::kMaxNReg) asm volatile("setmaxnreg.inc.sync.aligned.u32 112;" ::: "memory");
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        uint32_t ta[S], td[S], ph[S];
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
            ta[s2] = tmem_base + lane_off + C::a_col(g, s2);
            td[s2] = tmem_base + lane_off + C::d_col(g, s2);
            ph[s2] = 0;
            tc2::tmem_st_zero4(ta[s2] + 20);      // never-written tail (columns 20-23)
        }
        tc2::tmem_st_wait();
        uint64_t *ar = &a_ready[g * S], *dr = &d_ready[g * S];

        int clamps[L];
#pragma unroll
        for (int l = 0; l < L; ++l) clamps[l] = 0;
        const int member = t & 1;

        int64_t blk;
        int cb, ce;
        while (sched.next(blk, cb, ce)) {
            const int64_t pl = blk * tc::kPairsPerBlock + (t >> 1);
            const bool live = pl < a.P;
            int i = 0, j = 1;
            if (live) pair_of(a.p_begin + pl, a.n, i, j);
            const int self = member ? j : i, other = member ? i : j;
            float2 p2[9];
            {
                float p[HD], tmp[HD];
                load_row20(a.t.app_a32 + (size_t)self * ROW32, p);
                load_row20(a.t.app_b32 + (size_t)other * ROW32, tmp);
#pragma unroll
                for (int w = 0; w < 9; ++w)
                    p2[w] = make_float2(p[2 * w] + tmp[2 * w], p[2 * w + 1] + tmp[2 * w + 1]);
            }
            const float T_self = (float)a.base_time[self];
            // head weights from shared memory (the fp32 copy staged above),
            // re-read per work item (volatile: not hoisted out of the item
            // loop) so their 19 registers are free in the fp64 tail
            float2 wo2[9];
#pragma unroll
            for (int o = 0; o < 9; ++o) wo2[o] = tc3::lds_f32x2(wo_s + 2 * o);
            const float bo = tc3::lds_f32x2(wo_s + HD).x;
            const uint32_t krow = tc::smem_u32(k12 + member * ROW32);   // + c * 2 * ROW32 * 4

            float best[L], second[L];
            float miny = FLT_MAX;          // smallest screened prediction of this row
            int idx[L];
#pragma unroll
            for (int l = 0; l < L; ++l) { best[l] = FLT_MAX; second[l] = FLT_MAX; idx[l] = INT_MAX; }

            // epilogue of config c from stage s (s compile-time after unrolling)
            // y = wo . ReLU(z2) + bo with ReLU(x) = (x + |x|) / 2: the linear
            // half 0.5 wo . z2 is TMEM column 18 (B row 18 = 0.5 wo^T W2, its
            // bias 0.5 wo . b2), the other half an FFMA2 chain on |z2| (the
            // abs is a free operand modifier) -- no FMNMX per element
            auto math = [&](int c, const float (&z)[HD + 2]) {
                float2 y2 = make_float2(z[HD], bo);
#pragma unroll
                for (int o = 0; o < 9; ++o)
                    y2 = tc2::fma2(make_float2(fabsf(z[2 * o]), fabsf(z[2 * o + 1])), wo2[o], y2);
                const float y = y2.x + y2.y;
                miny = fminf(miny, y);
                const float tm = fmaxf(y, 0.5f) * T_self;
                const float tt = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
                if (L == 1) {
                    if (tt < best[0]) { second[0] = best[0]; best[0] = tt; idx[0] = c; }
                    else second[0] = fminf(second[0], tt);
                } else {
                    // branch-free per budget: a config outside budget l enters as +max
                    const uint32_t m = masks[c];
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        const float v = ((m >> l) & 1u) ? tt : FLT_MAX;
                        const bool lt = v < best[l];
                        second[l] = lt ? best[l] : fminf(second[l], v);
                        best[l] = lt ? v : best[l];
                        idx[l] = lt ? c : idx[l];
                    }
                }
            };
#ifdef CS_TC_CLOCKS
            const bool clk_item = blockIdx.x == 0 && blk == (int64_t)g && lane == 0;
            auto clk_at = [&](int c, int ev) {
                if (clk_item && c >= kClk0 && c < kClk0 + 32)
                    TC_CLK(((g * 4 + (warp & 3)) * 4 + ev) * 32 + (c - kClk0));
            };
#endif
            auto epilogue = [&](int c, int s) {
                float z[HD + 2];
#ifdef CS_TC_CLOCKS
                clk_at(c, 2);
#endif
                if (!C::kNoTensor) tc3::mbar_wait_warp(&dr[s], ph[s]);
#ifdef CS_TC_CLOCKS
                clk_at(c, 3);
#endif
                ph[s] ^= 1u;
                tc::fence_after();
                tc::tmem_ld20(td[s], z);
                math(c, z);
            };
            auto build = [&](int c, int s) {
#ifdef CS_TC_CLOCKS
                clk_at(c, 0);
#endif
                tc3::build_row<C::kOneTerm>(p2, krow + (uint32_t)c * (2 * ROW32 * 4), ta[s]);
                __syncwarp();
                if (lane == 0) tc2::mbar_arrive(&ar[s]);
#ifdef CS_TC_CLOCKS
                clk_at(c, 1);
#endif
                asm volatile("" ::: "memory");   // keep build / epilogue phases apart
            };

            // software pipeline over this segment's configs [cb, ce), stage of
            // config cb + u = u % S:
            //   build(0 .. S-2); [build(u), epilogue(u-S+1)] for u >= S-1; drain
            const int n = ce - cb;
#pragma unroll
            for (int u = 0; u < S - 1; ++u)
                if (u < n) build(cb + u, u);
            int c = S - 1;                               // c % S == S - 1 throughout
            for (; c + S <= n; c += S) {
#pragma unroll
                for (int u = 0; u < S; ++u) {
                    build(cb + c + u, (S - 1 + u) % S);
                    epilogue(cb + c + u - (S - 1), u % S);
                }
            }
#pragma unroll
            for (int u = 0; u < 2 * S - 1; ++u) {
                const int cc = c + u, x = cc - (S - 1);
                if (cc < n) build(cb + cc, (S - 1 + u) % S);
                if (x >= 0 && x < n) epilogue(cb + x, u % S);
            }

            if (cb != 0 || ce != n_cfg) {
                // ---- a piece of a split item: park it; the last piece merges ----
                const uint32_t k = sched.k, item = (uint32_t)blk;
                const int nf = 3 * L + 1;
                float *mine = a.t.split_scratch +
                              ((size_t)(k * 2 + sched.side(k, item)) * nf) * tc::kGroupThreads + t;
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    mine[(size_t)l * tc::kGroupThreads] = best[l];
                    mine[(size_t)(L + l) * tc::kGroupThreads] = second[l];
                    mine[(size_t)(2 * L + l) * tc::kGroupThreads] = __int_as_float(idx[l]);
                }
                mine[(size_t)(3 * L) * tc::kGroupThreads] = miny;
                __threadfence();
                tc3::group_sync(g);
                const uint32_t kf = sched.slot_of(item * sched.n_cfg);
                const uint32_t kl = sched.slot_of(item * sched.n_cfg + sched.n_cfg - 1);
                if (t == 0) {
                    const uint32_t old = atomicAdd(a.t.split_cnt + kf, 1u);
                    const bool last = old == (uint32_t)(kl - kf);
                    if (last) a.t.split_cnt[kf] = 0u;    // ready for the next launch
                    s_last[g] = last;
                }
                tc3::group_sync(g);
                if (!s_last[g]) continue;
                __threadfence();
                // merge the pieces in config order: first index of the minimum,
                // runner-up = the smallest value that is not the winner
#pragma unroll
                for (int l = 0; l < L; ++l) { best[l] = FLT_MAX; second[l] = FLT_MAX; idx[l] = INT_MAX; }
                miny = FLT_MAX;
                for (uint32_t kk = kf; kk <= kl; ++kk) {
                    const float *pc = a.t.split_scratch +
                                      ((size_t)(kk * 2 + sched.side(kk, item)) * nf) * tc::kGroupThreads + t;
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        const float pb = __ldcg(pc + (size_t)l * tc::kGroupThreads);
                        const float ps = __ldcg(pc + (size_t)(L + l) * tc::kGroupThreads);
                        const int pi = __float_as_int(__ldcg(pc + (size_t)(2 * L + l) * tc::kGroupThreads));
                        const bool lt = pb < best[l];
                        second[l] = fminf(fminf(second[l], ps), lt ? best[l] : pb);
                        idx[l] = lt ? pi : idx[l];
                        best[l] = lt ? pb : best[l];
                    }
                    miny = fminf(miny, __ldcg(pc + (size_t)(3 * L) * tc::kGroupThreads));
                }
            }

            // Floor clamps (estimator.py:106-109) are never counted from the
            // screen: a row whose screened predictions all lie above 0.5 + tau
            // has none, any other row is re-counted in fp64 by k_resolve
            if (live && !(miny > 0.5f + a.tau)) push_row(a, pl, member);

            // ---- per (pair, budget): queue it (k_resolve), or re-evaluate the
            //      winner in fp64 and, fused, decide + scatter it right here ----
#pragma unroll 1
            for (int l = 0; l < L; ++l) {
                const bool ambiguous = screen_ambiguous(a, best[l], second[l]);
                const double tm64 = ambiguous ? 0.0
                    : C::kNoExact ? (double)best[l]
                    : member_time64_lean(a.t, *net64, a.base_time, self, other, idx[l], member);
                const double co = fmax(tm64, __shfl_xor_sync(0xffffffffu, tm64, 1));
                if (live && member == 0 && !C::kNoWrite) {
                    if (ambiguous) {
                        push_ambiguous(a, l, pl);
                    } else {
                        write_winner(a, l, pl, idx[l], co, best[l]);
                        maybe_verify(a, l, pl, best[l], second[l]);
                        if (a.fused) clamps[l] += decide_write(a, l, pl, i, j, idx[l], co);
                    }
                }
            }
        }
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const int tot = __reduce_add_sync(0xffffffffu, clamps[l]);
            if (lane == 0 && tot) atomicAdd(a.clamps + l, (unsigned long long)tot);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

inline size_t tc3_smem_bytes(int n_grid) {
    size_t b = (size_t)tc2::kBBytes;
    b += 2 * (size_t)n_grid * ROW32 * sizeof(float) + (size_t)n_grid * sizeof(uint32_t);
    b = (b + 7) & ~(size_t)7;
    b += 2 * 16 * sizeof(uint64_t) + 3 * sizeof(uint64_t) + 16 + sizeof(Head64P) + 20 * sizeof(float);
    return b;
}
