// tc4_sweep.cuh -- tcgen05 screen, v5: warp-specialized builder / epilogue warps.
//
// Same math, TMEM layout and result contract as k_sweep_tc3.  v4 measured its
// CUDA-core work alone at ~70% of the kernel time (a probe without MMAs / waits)
// with 58-67% issue-slot use: every compute warp alternated "build A(c+1)" and
// "epilogue of c" and stalled on the MMA round trip in between.  Here the two
// halves run in DIFFERENT warps over the SAME TMEM lane quadrant (warp % 4 picks
// the quadrant, so a builder warp and an epilogue warp own the same 32 rows):
//   builder warp   : K row -> A(c) in TMEM (tcgen05.st) -> arrive a_ready
//   issuer warp    : a_ready(c) + d_free(previous use of the stage) -> 4 MMAs -> commit d_ready
//   epilogue warp  : d_ready(c) -> tcgen05.ld D -> arrive d_free -> head, floor, max, argmin
// so a group has 8 compute warps and S stages in flight, and each warp holds
// only its half of the state (fewer registers -> more resident warps).
// A builder reuses stage s once MMA(previous use of s) completed (d_ready);
// the issuer reuses D(s) once the epilogue warps have read it (d_free).
#pragma once

namespace tc4 {

template <int G, int S>
struct Cfg {
    static constexpr int kWarpsPerGroup = 8;                 // 4 builders + 4 epilogue
    static constexpr int kThreads = G * kWarpsPerGroup * 32 + G * 32;
    static_assert(G * S * 56 <= 512, "TMEM holds 512 columns");
    static_assert(kThreads <= 1024, "CTA size");
    __device__ static constexpr uint32_t d_col(int g, int s) { return (uint32_t)((g * S + s) * 32); }
    __device__ static constexpr uint32_t a_col(int g, int s) {
        return (uint32_t)(G * S * 32 + (g * S + s) * 24);
    }
};

}  // namespace tc4

template <int L, int G, int S>
__global__ void __launch_bounds__(tc4::Cfg<G, S>::kThreads, 1)
    k_sweep_tc4(const SweepArgs a, const __grid_constant__ Net32P net,
                const __grid_constant__ Head64P net_param) {
    using C = tc4::Cfg<G, S>;
    constexpr int kThreads = C::kThreads;
    extern __shared__ __align__(1024) uint8_t smem[];
    // carve: [B slices 4 KB][K12][mask][d_ready G*S][a_ready G*S][d_free G*S][tmem slot][Head64P][wo, bo]
    uint8_t *b_tile = smem;
    float *k12 = reinterpret_cast<float *>(smem + tc2::kBBytes);
    uint32_t *masks = reinterpret_cast<uint32_t *>(k12 + (size_t)a.g.G * 2 * ROW32);
    uint64_t *d_ready = reinterpret_cast<uint64_t *>(
        smem + ((reinterpret_cast<uint8_t *>(masks + a.g.G) - smem + 7) & ~ptrdiff_t(7)));
    uint64_t *a_ready = d_ready + G * S;
    uint64_t *d_free = a_ready + G * S;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(d_free + G * S);
    Head64P *net64 = reinterpret_cast<Head64P *>(
        smem + ((reinterpret_cast<uint8_t *>(d_free + G * S + 2) - smem + 15) & ~ptrdiff_t(15)));
    float *wo_s = reinterpret_cast<float *>(net64 + 1);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int g = warp / C::kWarpsPerGroup;          // == G: issuer warps
    const int wg = warp % C::kWarpsPerGroup;         // 0-3 builders, 4-7 epilogue
    const int q = wg & 3;                            // TMEM lane quadrant (== warp % 4)
    const int t = q * 32 + lane;                     // row within the group's tile

    if (tid == 0) {
        for (int i = 0; i < G * S; ++i) {
            tc::mbar_init(&d_ready[i], 1);
            tc::mbar_init(&a_ready[i], 4);
            tc::mbar_init(&d_free[i], 4);
        }
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = tid; i < tc2::kBBytes / 16; i += kThreads)
        reinterpret_cast<uint4 *>(b_tile)[i] =
            reinterpret_cast<const uint4 *>(a.t.w2_tile + tc::kBBytes / 2)[i];
    for (int i = tid; i < a.g.G * ROW32; i += kThreads) {
        const int c = i / ROW32, h = i - c * ROW32;
        k12[(2 * c) * ROW32 + h] = a.t.knob1_32[i];
        k12[(2 * c + 1) * ROW32 + h] = a.t.knob2_32[i];
    }
    for (int i = tid; i < a.g.G; i += kThreads) masks[i] = L == 1 ? 1u : a.g.mask[i];
    if (tid <= HD) wo_s[tid] = tid < HD ? net.wo[tid] : net.bo;
    for (int i = tid; i < (int)(sizeof(Head64P) / 8); i += kThreads)
        reinterpret_cast<double *>(net64)[i] = __ldg(a.t.net_image + kImgHeadOff + i);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int64_t nblocks = (a.P + tc::kPairsPerBlock - 1) / tc::kPairsPerBlock;
    const int64_t total_groups = (int64_t)gridDim.x * G;
    const int n_cfg = a.g.G;

    if (g >= G) {
        // ===== MMA issuer warp for group qg =====
        const int qg = warp - G * C::kWarpsPerGroup;
        const uint32_t b_addr = tc::smem_u32(b_tile);
        const uint64_t bq0 = tc2::slice_desc(b_addr), bq1 = tc2::slice_desc(b_addr + 1024),
                       bq2 = tc2::slice_desc(b_addr + 2048);
        uint32_t aph = 0, fph = 0, used = 0;           // per-stage bits
        int st = 0;
        for (int64_t blk = (int64_t)blockIdx.x * G + qg; blk < nblocks; blk += total_groups) {
            for (int k = 0; k < n_cfg; ++k) {
                const int b = qg * S + st;
                tc3::mbar_wait_sleep(&a_ready[b], (aph >> st) & 1u);
                aph ^= 1u << st;
                if ((used >> st) & 1u) {                // D(st) read by the epilogue warps?
                    tc3::mbar_wait_sleep(&d_free[b], (fph >> st) & 1u);
                    fph ^= 1u << st;
                }
                used |= 1u << st;
                __syncwarp();
                tc::fence_after();
                tc3::issue_config(tmem_base + C::d_col(qg, st), tmem_base + C::a_col(qg, st),
                                  bq0, bq1, bq2, &d_ready[b]);
                st = st + 1 == S ? 0 : st + 1;
            }
        }
    } else if (wg < 4) {
        // ===== builder warp: A rows of this quadrant =====
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t ta0 = tmem_base + lane_off + C::a_col(g, 0);
        for (int s2 = 0; s2 < S; ++s2) tc2::tmem_st_zero4(ta0 + s2 * 24 + 20);
        tc2::tmem_st_wait();
        uint32_t bph = 0, used = 0;
        int st = 0;
        const int member = t & 1;
        const uint32_t krow0 = tc::smem_u32(k12 + member * ROW32);
        for (int64_t blk = (int64_t)blockIdx.x * G + g; blk < nblocks; blk += total_groups) {
            const int64_t pl = blk * tc::kPairsPerBlock + (t >> 1);
            int i = 0, j = 1;
            if (pl < a.P) pair_of(a.p_begin + pl, a.n, i, j);
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
            for (int c = 0; c < n_cfg; ++c) {
                if ((used >> st) & 1u) {               // MMA of the stage's last use done
                    tc3::mbar_wait_warp(&d_ready[g * S + st], (bph >> st) & 1u);
                    bph ^= 1u << st;
                }
                used |= 1u << st;
                tc3::build_row(p2, krow0 + (uint32_t)c * (2 * ROW32 * 4), ta0 + st * 24);
                __syncwarp();
                if (lane == 0) tc2::mbar_arrive(&a_ready[g * S + st]);
                st = st + 1 == S ? 0 : st + 1;
            }
        }
    } else {
        // ===== epilogue warp: D rows of this quadrant =====
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t td0 = tmem_base + lane_off + C::d_col(g, 0);
        float2 wo2[9];
#pragma unroll
        for (int o = 0; o < 9; ++o) wo2[o] = make_float2(wo_s[2 * o], wo_s[2 * o + 1]);
        const float bo = wo_s[HD];
        int clamps[L];
#pragma unroll
        for (int l = 0; l < L; ++l) clamps[l] = 0;
        uint32_t eph = 0;
        int st = 0;
        const int member = t & 1;
        for (int64_t blk = (int64_t)blockIdx.x * G + g; blk < nblocks; blk += total_groups) {
            const int64_t pl = blk * tc::kPairsPerBlock + (t >> 1);
            const bool live = pl < a.P;
            int i = 0, j = 1;
            if (live) pair_of(a.p_begin + pl, a.n, i, j);
            const int self = member ? j : i, other = member ? i : j;
            const float T_self = (float)a.base_time[self];
            float best[L], second[L];
            int idx[L], bcl[L];
#pragma unroll
            for (int l = 0; l < L; ++l) { best[l] = FLT_MAX; second[l] = FLT_MAX; idx[l] = INT_MAX; bcl[l] = 0; }
            for (int c = 0; c < n_cfg; ++c) {
                float z[HD];
                tc3::mbar_wait_warp(&d_ready[g * S + st], (eph >> st) & 1u);
                eph ^= 1u << st;
                tc::fence_after();
                tc::tmem_ld18(td0 + st * 32, z);
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc2::mbar_arrive(&d_free[g * S + st]);
                st = st + 1 == S ? 0 : st + 1;
                float2 y2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int o = 0; o < 9; ++o)
                    y2 = tc2::fma2(make_float2(fmaxf(z[2 * o], 0.f), fmaxf(z[2 * o + 1], 0.f)),
                                   wo2[o], y2);
                const float y = (y2.x + y2.y) + bo;
                const int cl = y < 0.5f;
                const float tm = fmaxf(y, 0.5f) * T_self;
                const float tt = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
                const uint32_t m = L == 1 ? 1u : masks[c];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    if (L == 1 || ((m >> l) & 1u)) {
                        bcl[l] += cl;
                        if (tt < best[l]) { second[l] = best[l]; best[l] = tt; idx[l] = c; }
                        else second[l] = fminf(second[l], tt);
                    }
                }
            }
#pragma unroll
            for (int l = 0; l < L; ++l) clamps[l] += live ? bcl[l] : 0;
#pragma unroll 1
            for (int l = 0; l < L; ++l) {
                const bool ambiguous = screen_ambiguous(a, best[l], second[l]);
                const double tm64 = ambiguous ? 0.0
                    : member_time64_lean(a.t, *net64, a.base_time, self, other, idx[l], member);
                const double co = fmax(tm64, __shfl_xor_sync(0xffffffffu, tm64, 1));
                if (live && member == 0) {
                    if (ambiguous) {
                        push_ambiguous(a, l, pl);
                    } else {
                        write_winner(a, l, pl, idx[l], co, best[l]);
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

inline size_t tc4_smem_bytes(int n_grid) {
    size_t b = (size_t)tc2::kBBytes;
    b += 2 * (size_t)n_grid * ROW32 * sizeof(float) + (size_t)n_grid * sizeof(uint32_t);
    b = (b + 7) & ~(size_t)7;
    b += 3 * 16 * sizeof(uint64_t) + 32 + sizeof(Head64P) + 20 * sizeof(float);
    return b;
}
