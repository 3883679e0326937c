// tc2_sweep.cuh -- tcgen05 screen, v3: A operand written straight into TMEM.
//
// Same math and result contract as k_sweep_tc (tc_sweep.cuh); what changes is
// where the A operand lives.  Profiling v2 (profiles/) showed the SMEM port
// bound: every 128-row tile was written to shared memory (16 KB of STS) and
// read back by each of the 4 MMAs (16 KB of A reads).  Here each thread
// stores its fp16 row into its own TMEM lane with two tcgen05.st
// (32x32b.x16 + .x4), the MMAs take A from TMEM ("[a_tmem]" form), and shared
// memory only feeds B (1 KB per MMA) and the broadcast K rows.
//
// K layout of a row (20 live 32-bit columns of 24, halves in pairs):
//   cols 0-7   hi(h_0..h_15)          slice 0
//   cols 8-15  lo(h_0..h_15)          slice 1
//   col 16     hi(h_16), hi(h_17)     slice 2 ...
//   col 17     lo(h_16), lo(h_17)
//   col 18     1.0, 1.0               (carries b2 = b2hi + b2lo)
//   cols 19-23 0
// B is held as four 16-wide K slices (N = 32 rows each, canonical layout):
//   q0 = W2hi[:, 0:16]   q1 = [W2hi16 W2hi17 W2hi16 W2hi17 b2hi b2lo W2lo16 W2lo17 0..]
//   q2 = W2lo[:, 0:16]   q3 = [W2lo16 W2lo17 0..]
// and z2 = A_s0 q0 + A_s1 q0 + A_s2 q1 + A_s0 q2 + A_s2 q3 (5 MMAs, K = 16):
// (hi + lo) W2hi + hi W2lo + b2, the same 3-term split as v2.
#pragma once

namespace tc2 {

constexpr int kBSliceBytes = 32 * 16 * 2;     // N=32 rows x 16 halves
constexpr int kBBytes = 4 * kBSliceBytes;     // 4 KB

// canonical no-swizzle K-major slice: 8x16 B core matrices, LBO 128 B, SBO 256 B
__host__ __device__ __forceinline__ uint32_t slice_off(int row, int chunk) {
    return (uint32_t)((row >> 3) * 256 + chunk * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint64_t slice_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)(256u >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(accumulate), "r"(tc::kIdesc));
}

__device__ __forceinline__ void tmem_st20(uint32_t taddr, const uint32_t (&w)[20]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
        "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
        "r"(w[15])
        : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + 16),
                 "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19])
                 : "memory");
}

__device__ __forceinline__ void tmem_st_zero4(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(taddr), "r"(0u)
                 : "memory");
}

__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// {lo half = a, hi half = b}: round toward zero with ReLU / round to nearest with ReLU
__device__ __forceinline__ uint32_t cvt_rz_relu(float a, float b) {
    uint32_t r;
    asm("cvt.rz.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}
__device__ __forceinline__ uint32_t cvt_rn_relu(float a, float b) {
    uint32_t r;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long r, x = *reinterpret_cast<unsigned long long *>(&a),
                          y = *reinterpret_cast<unsigned long long *>(&b);
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    return *reinterpret_cast<float2 *>(&r);
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long r, x = *reinterpret_cast<unsigned long long *>(&a),
                          y = *reinterpret_cast<unsigned long long *>(&b);
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    return *reinterpret_cast<float2 *>(&r);
}

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long r, x = *reinterpret_cast<unsigned long long *>(&a),
                          y = *reinterpret_cast<unsigned long long *>(&b),
                          z = *reinterpret_cast<unsigned long long *>(&c);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(y), "l"(z));
    return *reinterpret_cast<float2 *>(&r);
}

}  // namespace tc2

// fp16 B slices of v3 (written by k_tables next to the v2 tile)
__device__ void write_b_slices(const Net64P &net, uint16_t *tile, int idx) {
    // idx in [0, 4 * 32 * 16)
    const int q = idx / 512, rem = idx % 512, n = rem / 16, kk = rem % 16;
    auto hi_of = [](double x) { return (double)__half2float(__double2half(x)); };
    double v = 0.0;
    if (n < HD) {
        const double *w = net.w2 + n * HD;
        if (q == 0) v = hi_of(w[kk]);
        else if (q == 2) v = w[kk] - hi_of(w[kk]);
        else if (q == 1) {
            if (kk == 0 || kk == 2) v = hi_of(w[16]);
            else if (kk == 1 || kk == 3) v = hi_of(w[17]);
            else if (kk == 4) v = hi_of(net.b2[n]);
            else if (kk == 5) v = net.b2[n] - hi_of(net.b2[n]);
            // k 6-7 meet A column 19: zero in this kernel, (hi16, hi17) in
            // k_sweep_tc3, which so folds the q3 term into this slice
            else if (kk == 6) v = w[16] - hi_of(w[16]);
            else if (kk == 7) v = w[17] - hi_of(w[17]);
        } else {  // q == 3
            if (kk == 0) v = w[16] - hi_of(w[16]);
            else if (kk == 1) v = w[17] - hi_of(w[17]);
        }
    }
    __half h = __double2half(v);
    const uint32_t off = q * tc2::kBSliceBytes + tc2::slice_off(n, kk >> 3) + (kk & 7) * 2;
    tile[off / 2] = *reinterpret_cast<uint16_t *>(&h);
}

// TMEM map (columns): all D stages first (32 columns each, 32-aligned), then all
// A stages (24 columns each): D(g, s) = (g*S + s)*32, A(g, s) = G*S*32 + (g*S + s)*24.
template <int G, int S>
struct Tc2Cfg {
    static constexpr int kThreads = G * tc::kGroupThreads + G * 32;   // + one issuer warp per group
    static constexpr int kCols = G * S * 56;
    static_assert(kCols <= 512, "TMEM holds 512 columns");
    __device__ static constexpr uint32_t d_col(int g, int s) { return (uint32_t)((g * S + s) * 32); }
    __device__ static constexpr uint32_t a_col(int g, int s) {
        return (uint32_t)(G * S * 32 + (g * S + s) * 24);
    }
};

template <int L, int G, int S>
__global__ void __launch_bounds__(Tc2Cfg<G, S>::kThreads, 1)
    k_sweep_tc2(const SweepArgs a, const __grid_constant__ Net32P net,
                const __grid_constant__ Head64P net_param) {
    using Cfg = Tc2Cfg<G, S>;
    extern __shared__ __align__(1024) uint8_t smem[];
    // carve: [B slices 4 KB][K1 | K2 fp32 G x 20][mask G][d_ready G*S][a_ready G*S][tmem slot]
    uint8_t *b_tile = smem;
    float *k1s = reinterpret_cast<float *>(smem + tc2::kBBytes);
    float *k2s = k1s + (size_t)a.g.G * ROW32;
    uint32_t *masks = reinterpret_cast<uint32_t *>(k2s + (size_t)a.g.G * ROW32);
    // d_ready[g*S+s]: MMA -> epilogue (tcgen05.commit, count 1)
    // a_ready[g*S+s]: A rows in TMEM -> MMA issuer (one arrive per compute warp, count 4)
    uint64_t *d_ready = reinterpret_cast<uint64_t *>(
        smem + ((reinterpret_cast<uint8_t *>(masks + a.g.G) - smem + 7) & ~ptrdiff_t(7)));
    uint64_t *a_ready = d_ready + G * S;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_ready + G * S);
    Head64P *net64 = reinterpret_cast<Head64P *>(
        smem + ((reinterpret_cast<uint8_t *>(a_ready + G * S + 2) - smem + 15) & ~ptrdiff_t(15)));

    const int tid = threadIdx.x;
    const int g = tid / tc::kGroupThreads;     // >= G: the MMA-issuer warps
    const int t = tid % tc::kGroupThreads;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    for (int i = tid; i < tc2::kBBytes / 16; i += Cfg::kThreads)
        reinterpret_cast<uint4 *>(b_tile)[i] =
            reinterpret_cast<const uint4 *>(a.t.w2_tile + tc::kBBytes / 2)[i];
    for (int i = tid; i < a.g.G * ROW32; i += Cfg::kThreads) {
        k1s[i] = a.t.knob1_32[i];
        k2s[i] = a.t.knob2_32[i];
    }
    for (int i = tid; i < a.g.G; i += Cfg::kThreads) masks[i] = L == 1 ? 1u : a.g.mask[i];
    for (int i = tid; i < (int)(sizeof(Head64P) / 8); i += Cfg::kThreads)
        reinterpret_cast<double *>(net64)[i] = __ldg(a.t.net_image + kImgHeadOff + i);
    if (tid == 0) {
        for (int i = 0; i < G * S; ++i) {
            tc::mbar_init(&d_ready[i], 1);
            tc::mbar_init(&a_ready[i], 4);
        }
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int64_t nblocks = (a.P + tc::kPairsPerBlock - 1) / tc::kPairsPerBlock;
    const int64_t total_groups = (int64_t)gridDim.x * G;

    if (g >= G) {
        // ===== MMA issuer warps: warp 4G + q serves group q =====
        const int q = warp - G * (tc::kGroupThreads / 32);
        const uint32_t b_addr = tc::smem_u32(b_tile);
        const uint64_t bq0 = tc2::slice_desc(b_addr), bq1 = tc2::slice_desc(b_addr + 1024),
                       bq2 = tc2::slice_desc(b_addr + 2048), bq3 = tc2::slice_desc(b_addr + 3072);
        uint32_t aph = 0;                              // bit s: parity of a_ready[q][s]
        int st = 0;
        for (int64_t blk = (int64_t)blockIdx.x * G + q; blk < nblocks; blk += total_groups) {
            for (int k = 0; k < a.g.G; ++k) {
                tc::mbar_wait(&a_ready[q * S + st], (aph >> st) & 1u);
                aph ^= 1u << st;
                __syncwarp();
                tc::fence_after();
                if (lane == 0) {
                    const uint32_t a_t = tmem_base + Cfg::a_col(q, st);
                    const uint32_t d_t = tmem_base + Cfg::d_col(q, st);
                    tc2::mma_ts(d_t, a_t + 0, bq0, 0);
                    tc2::mma_ts(d_t, a_t + 8, bq0, 1);
                    tc2::mma_ts(d_t, a_t + 16, bq1, 1);
                    tc2::mma_ts(d_t, a_t + 0, bq2, 1);
                    tc2::mma_ts(d_t, a_t + 16, bq3, 1);
                    tc::mma_commit(&d_ready[q * S + st]);
                }
                __syncwarp();
                st = st + 1 == S ? 0 : st + 1;
            }
        }
    } else {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    // zero the never-written tail (columns 20-23) of every A stage of this lane
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) tc2::tmem_st_zero4(tmem_base + lane_off + Cfg::a_col(g, s2) + 20);
    tc2::tmem_st_wait();

    float2 wo2[9];
#pragma unroll
    for (int o = 0; o < 9; ++o) wo2[o] = make_float2(net.wo[2 * o], net.wo[2 * o + 1]);
    uint32_t phase = 0;                        // bit s: parity of d_ready[g][s]
    int clamps[L];
#pragma unroll
    for (int l = 0; l < L; ++l) clamps[l] = 0;
    const int member = t & 1;
    int st_build = 0, st_epi = 0;              // stage of the next build / epilogue

    for (int64_t blk = (int64_t)blockIdx.x * G + g; blk < nblocks; blk += total_groups) {
        const int64_t pl = blk * tc::kPairsPerBlock + (t >> 1);
        const bool live = pl < a.P;
        const int live_i = live ? 1 : 0;
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
        const float *kt = member ? k2s : k1s;

        float best[L], second[L];
        int idx[L];
#pragma unroll
        for (int l = 0; l < L; ++l) { best[l] = FLT_MAX; second[l] = FLT_MAX; idx[l] = INT_MAX; }

        for (int k = 0; k < a.g.G + S - 1; ++k) {
            if (k < a.g.G) {
                // ---- 1. this lane's A row for config k, straight into TMEM ----
                const float4 *kq = reinterpret_cast<const float4 *>(kt + (size_t)k * ROW32);
                const float4 q0 = kq[0], q1 = kq[1], q2 = kq[2], q3 = kq[3], q4 = kq[4];
                const float2 kr[9] = {make_float2(q0.x, q0.y), make_float2(q0.z, q0.w),
                                      make_float2(q1.x, q1.y), make_float2(q1.z, q1.w),
                                      make_float2(q2.x, q2.y), make_float2(q2.z, q2.w),
                                      make_float2(q3.x, q3.y), make_float2(q3.z, q3.w),
                                      make_float2(q4.x, q4.y)};
                // ReLU + split in three packed steps per pair: hi = rz(relu z) <= relu z,
                // so lo = z - hi is >= 0 whenever z >= 0 and is clamped to 0 by the
                // second relu conversion when z < 0 (then hi = 0 as well).
                uint32_t w[20];
#pragma unroll
                for (int v = 0; v < 9; ++v) {
                    const float2 z = tc2::add2(p2[v], kr[v]);
                    const uint32_t hw = tc2::cvt_rz_relu(z.x, z.y);
                    const float2 lo = tc2::sub2(z, tc::unpack_half2(hw));
                    const uint32_t lw = tc2::cvt_rn_relu(lo.x, lo.y);
                    if (v < 8) { w[v] = hw; w[8 + v] = lw; }
                    else { w[16] = hw; w[17] = lw; }
                }
                w[18] = 0x3C003C00u;   // (1.0h, 1.0h)
                w[19] = 0u;
                tc2::tmem_st20(tmem_base + lane_off + Cfg::a_col(g, st_build), w);
                tc2::tmem_st_wait();
                // order this warp's TMEM stores (and its earlier TMEM loads of the
                // same D stage) before the issuer's MMA, then signal A(k) ready
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc2::mbar_arrive(&a_ready[g * S + st_build]);
                st_build = st_build + 1 == S ? 0 : st_build + 1;
            }
            // ---- 2. epilogue of config k-(S-1) ----
            if (k >= S - 1) {
                const int c = k - (S - 1);
                tc::mbar_wait(&d_ready[g * S + st_epi], (phase >> st_epi) & 1u);
                __syncwarp();
                phase ^= 1u << st_epi;
                tc::fence_after();
                float z[HD];
                tc::tmem_ld18(tmem_base + lane_off + Cfg::d_col(g, st_epi), z);
                st_epi = st_epi + 1 == S ? 0 : st_epi + 1;
                float2 y2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int o = 0; o < 9; ++o)
                    y2 = tc2::fma2(make_float2(fmaxf(z[2 * o], 0.f), fmaxf(z[2 * o + 1], 0.f)),
                                   wo2[o], y2);
                const float y = (y2.x + y2.y) + net.bo;
                const int cl = y < 0.5f;
                const float tm = fmaxf(y, 0.5f) * T_self;
                const float tt = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
                const uint32_t m = masks[c];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    if (L == 1 || ((m >> l) & 1u)) {
                        clamps[l] += cl & live_i;
                        if (tt < best[l]) { second[l] = best[l]; best[l] = tt; idx[l] = c; }
                        else second[l] = fminf(second[l], tt);
                    }
                }
            }
        }
        // ---- per (pair, budget): queue it, or re-evaluate the winner in fp64
        //      (member m's thread computes member m's time; one shuffle) ----
#pragma unroll 1
        for (int l = 0; l < L; ++l) {
            const bool ambiguous = screen_ambiguous(a, best[l], second[l]);
            // every lane reaches the shuffle (ambiguity differs across the warp's pairs)
            const double tm64 = ambiguous ? 0.0
                : member_time64_lean(a.t, *net64, a.base_time, self, other, idx[l], member);
            const double co = fmax(tm64, __shfl_xor_sync(0xffffffffu, tm64, 1));
            if (live && member == 0) {
                if (ambiguous) push_ambiguous(a, l, pl);
                else write_winner(a, l, pl, idx[l], co, best[l]);
            }
        }
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int tot = __reduce_add_sync(0xffffffffu, clamps[l]);
        if (lane == 0 && tot) atomicAdd(a.clamps + l, (unsigned long long)tot);
    }
    }   // compute groups
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

inline size_t tc2_smem_bytes(int n_grid) {
    size_t b = (size_t)tc2::kBBytes;
    b += 2 * (size_t)n_grid * ROW32 * sizeof(float) + (size_t)n_grid * sizeof(uint32_t);
    b = (b + 7) & ~(size_t)7;
    b += 2 * 16 * sizeof(uint64_t) + 32 + sizeof(Head64P);
    return b;
}
