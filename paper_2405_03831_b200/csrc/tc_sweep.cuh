// tc_sweep.cuh -- tcgen05 (5th-gen tensor core) variant of the pair x knob screen.
//
// Included by sweep.cu (shares its types: cs_tables, GridP, Net32P, SweepArgs,
// head64c, corun-member fp64 evaluation).
//
// Mapping.  A CTA of 512 threads = 4 independent *groups* of 128 threads
// (4 warps each, warp w owns TMEM lanes 32*(w%4)..+31).  A group sweeps a block
// of 64 pairs: row r = 2*u + m is pair u's member m (m = 0: job i with view hc,
// m = 1: job j with the reversed-partition view, estimator.py:112-129).  For
// every co-run config c the group
//   1. builds A(c) in shared memory: thread r computes h = ReLU(P_r + K_m(c))
//      in fp32 (P_r = A_i + B_j or A_j + B_i, K with b1 folded) and stores
//      the fp16 split [hi | lo | hi | 1 1 | 0...] (K = 64) of its row in the
//      canonical no-swizzle K-major layout (8x16 B core matrices);
//   2. one elected thread issues 4 x tcgen05.mma.kind::f16 (M=128, N=32, K=16)
//      against B = [W2hi; W2hi; W2lo; b2hi; b2lo] (also fp16, staged once),
//      accumulating z2 = W2 h + b2 in fp32 in TMEM, and commits to an mbarrier;
//   3. the 128 threads tcgen05.ld their row of z2 (18 columns), finish
//      ReLU -> head -> floor -> x base_time in fp32, take the max over the two
//      members with one shuffle and update the pair's (min, first index,
//      runner-up) per budget.
// A and D are double-buffered, so the build of c+1 and the epilogue of c-1
// overlap the MMA of c.  The 3-term fp16 split keeps the screen at fp32-level
// error (3e-7 relative, measured in emulation and at run time via
// SweepArgs.qcount[1]); the exact fp64 re-evaluation / re-scan downstream is
// shared with the SIMT kernel, so results are identical.
#pragma once

#ifdef CS_TC_TRACE
#define TC_TRACE(stage, k) \
    do { if (a.trace) ((volatile uint32_t *)a.trace)[blockIdx.x * tc::kThreads + threadIdx.x] = \
             ((uint32_t)(k) << 8) | (stage); } while (0)
#else
#define TC_TRACE(stage, k) do { } while (0)
#endif

namespace tc {

constexpr int kGroups = 4;
constexpr int kGroupThreads = 128;
constexpr int kThreads = kGroups * kGroupThreads;
constexpr int kPairsPerBlock = 64;
constexpr int kK = 64;                    // fp16 K extent of A / B rows
constexpr int kTileBytes = 128 * kK * 2;  // 16 KB A tile
constexpr int kBBytes = 32 * kK * 2;      // 4 KB B tile (N = 32)
constexpr int kTmemColsPerGroup = 64;     // 2 D buffers x 32 fp32 columns
constexpr uint32_t kIdesc = (1u << 4)            // D = f32
                          | (0u << 7) | (0u << 10)  // A, B = f16
                          | (0u << 15) | (0u << 16) // both K-major
                          | ((32u >> 3) << 17)      // N = 32
                          | ((128u >> 4) << 24);    // M = 128

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// byte offset of (row, 16-byte chunk j) in a no-swizzle K-major tile whose
// core matrices are 8 rows x 16 B: LBO (next chunk along K) = 128 B,
// SBO (next 8-row group) = 1024 B
__device__ __forceinline__ uint32_t tile_off(int row, int chunk) {
    return (uint32_t)((row >> 3) * 1024 + chunk * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)(128u >> 4) << 16;     // leading byte offset (K direction)
    d |= (uint64_t)(1024u >> 4) << 32;    // stride byte offset (M/N direction)
    d |= (uint64_t)1 << 46;               // descriptor version for sm_100
    return d;                              // base offset 0, no swizzle
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Bounded wait: a lost MMA completion traps (kernel error) after ~2 s of
// SM clock instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try(bar, parity)) {
        if (clock64() - t0 > 4000000000LL) __trap();
    }
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kGroupThreads) : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 18 fp32 columns of this thread's TMEM lane (x16 + x2)
__device__ __forceinline__ void tmem_ld18(uint32_t taddr, float (&v)[18]) {
    uint32_t r[18];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(r[16]), "=r"(r[17])
                 : "r"(taddr + 16));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 18; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ float2 unpack_half2(uint32_t w) {
    __half2 h = *reinterpret_cast<__half2 *>(&w);
    return __half22float2(h);
}

}  // namespace tc

// B tile (W2 split, fp16, canonical layout) written by k_tables:
// row n < 18: [W2hi(n,0..17) | W2hi(n,0..17) | W2lo(n,0..17) | b2hi(n) b2lo(n) | 0 x 8]
__device__ void write_b_tile(const Net64P &net, uint16_t *tile, int idx) {
    // idx in [0, 32 * 64): one fp16 element
    const int n = idx / tc::kK, k = idx % tc::kK;
    double v = 0.0;
    if (n < HD) {
        if (k < 54) {
            const int kk = k % 18, seg = k / 18;
            const double w = net.w2[n * HD + kk];
            const double hi = (double)__half2float(__double2half(w));
            v = seg < 2 ? hi : w - hi;
        } else if (k == 54) {
            v = (double)__half2float(__double2half(net.b2[n]));
        } else if (k == 55) {
            v = net.b2[n] - (double)__half2float(__double2half(net.b2[n]));
        }
    }
    __half h = __double2half(v);
    const uint32_t off = tc::tile_off(n, k >> 3) + (k & 7) * 2;
    tile[off / 2] = *reinterpret_cast<uint16_t *>(&h);
}

template <int L>
__global__ void __launch_bounds__(tc::kThreads, 1)
    k_sweep_tc(const SweepArgs a, const __grid_constant__ Net32P net,
               const __grid_constant__ Head64P net_param) {
    extern __shared__ __align__(1024) uint8_t smem[];
    // carve: [A tiles: 4 groups x 2 x 16 KB][B tile 4 KB][K1 | K2 fp32 G x 20][mask G][mbar 8][tmem slot]
    uint8_t *a_tiles = smem;
    uint8_t *b_tile = smem + tc::kGroups * 2 * tc::kTileBytes;
    float *k1s = reinterpret_cast<float *>(b_tile + tc::kBBytes);
    float *k2s = k1s + (size_t)a.g.G * ROW32;
    uint32_t *masks = reinterpret_cast<uint32_t *>(k2s + (size_t)a.g.G * ROW32);
    uint64_t *mbars = reinterpret_cast<uint64_t *>(
        smem + ((reinterpret_cast<uint8_t *>(masks + a.g.G) - smem + 7) & ~ptrdiff_t(7)));
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbars + 2 * tc::kGroups);
    Head64P *net64 = reinterpret_cast<Head64P *>(
        smem + ((reinterpret_cast<uint8_t *>(mbars + 2 * tc::kGroups + 2) - smem + 15) & ~ptrdiff_t(15)));

    const int tid = threadIdx.x;
    const int g = tid / tc::kGroupThreads;        // group
    const int t = tid % tc::kGroupThreads;        // row within the group's tile
    const int warp = tid >> 5;

    // ---- one-time CTA setup ----
    for (int i = tid; i < tc::kGroups * 2 * tc::kTileBytes / 16; i += tc::kThreads)
        reinterpret_cast<uint4 *>(a_tiles)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < tc::kBBytes / 16; i += tc::kThreads)
        reinterpret_cast<uint4 *>(b_tile)[i] = reinterpret_cast<const uint4 *>(a.t.w2_tile)[i];
    for (int i = tid; i < a.g.G * ROW32; i += tc::kThreads) {
        k1s[i] = a.t.knob1_32[i];
        k2s[i] = a.t.knob2_32[i];
    }
    for (int i = tid; i < a.g.G; i += tc::kThreads) masks[i] = L == 1 ? 1u : a.g.mask[i];
    for (int i = tid; i < (int)(sizeof(Head64P) / 8); i += tc::kThreads)
        reinterpret_cast<double *>(net64)[i] = __ldg(a.t.net_image + kImgHeadOff + i);
    if (tid == 0) {
        for (int i = 0; i < 2 * tc::kGroups; ++i) tc::mbar_init(&mbars[i], 1);
        tc::fence_mbar_init();
    }
    TC_TRACE(1, 0);
    if (warp == 0) tc::tmem_alloc(tmem_slot, tc::kGroups * tc::kTmemColsPerGroup);
    TC_TRACE(2, 0);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t d_col0 = tmem_base + g * tc::kTmemColsPerGroup;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint8_t *my_tiles = a_tiles + g * 2 * tc::kTileBytes;
    uint32_t phase[2] = {0u, 0u};
    int clamps[L];
#pragma unroll
    for (int l = 0; l < L; ++l) clamps[l] = 0;

    const int64_t nblocks = (a.P + tc::kPairsPerBlock - 1) / tc::kPairsPerBlock;
    const int64_t total_groups = (int64_t)gridDim.x * tc::kGroups;
    const int member = t & 1;

    for (int64_t blk = (int64_t)blockIdx.x * tc::kGroups + g; blk < nblocks; blk += total_groups) {
        const int64_t pl = blk * tc::kPairsPerBlock + (t >> 1);
        const bool live = pl < a.P;
        int i = 0, j = 1;
        if (live) pair_of(a.p_begin + pl, a.n, i, j);
        const int self = member ? j : i, other = member ? i : j;
        float p[HD], tmp[HD];
        load_row20(a.t.app_a32 + (size_t)self * ROW32, p);
        load_row20(a.t.app_b32 + (size_t)other * ROW32, tmp);
#pragma unroll
        for (int h = 0; h < HD; ++h) p[h] += tmp[h];
        const float T_self = (float)a.base_time[self];
        const float *kt = member ? k2s : k1s;

        float best[L], second[L];
        int idx[L];
#pragma unroll
        for (int l = 0; l < L; ++l) { best[l] = FLT_MAX; second[l] = FLT_MAX; idx[l] = INT_MAX; }

        for (int k = 0; k <= a.g.G; ++k) {
            if (k < a.g.G) {
                // ---- 1. build this thread's A row for config k ----
                float kr[HD];
                const float4 *kq = reinterpret_cast<const float4 *>(kt + (size_t)k * ROW32);
                float4 q0 = kq[0], q1 = kq[1], q2 = kq[2], q3 = kq[3], q4 = kq[4];
                kr[0] = q0.x; kr[1] = q0.y; kr[2] = q0.z; kr[3] = q0.w;
                kr[4] = q1.x; kr[5] = q1.y; kr[6] = q1.z; kr[7] = q1.w;
                kr[8] = q2.x; kr[9] = q2.y; kr[10] = q2.z; kr[11] = q2.w;
                kr[12] = q3.x; kr[13] = q3.y; kr[14] = q3.z; kr[15] = q3.w;
                kr[16] = q4.x; kr[17] = q4.y;
                uint32_t hw[9], lw[9];
#pragma unroll
                for (int w = 0; w < 9; ++w) {
                    const float h0 = fmaxf(p[2 * w] + kr[2 * w], 0.f);
                    const float h1 = fmaxf(p[2 * w + 1] + kr[2 * w + 1], 0.f);
                    hw[w] = tc::pack_half2(h0, h1);
                    const float2 back = tc::unpack_half2(hw[w]);
                    lw[w] = tc::pack_half2(h0 - back.x, h1 - back.y);
                }
                uint8_t *tile = my_tiles + (k & 1) * tc::kTileBytes;
                const uint32_t ones = 0x3C003C00u;   // (1.0h, 1.0h)
                // words: [hw0..8 | lw0..8 | hw0..8 | ones | 0 0 0 0]
                const uint32_t row[28] = {hw[0], hw[1], hw[2], hw[3], hw[4], hw[5], hw[6],
                                          hw[7], hw[8], lw[0], lw[1], lw[2], lw[3], lw[4],
                                          lw[5], lw[6], lw[7], lw[8], hw[0], hw[1], hw[2],
                                          hw[3], hw[4], hw[5], hw[6], hw[7], hw[8], ones};
#pragma unroll
                for (int c = 0; c < 7; ++c)
                    *reinterpret_cast<uint4 *>(tile + tc::tile_off(t, c)) =
                        make_uint4(row[4 * c], row[4 * c + 1], row[4 * c + 2], row[4 * c + 3]);
            }
            tc::fence_proxy_async();
            tc::fence_before();
            __syncwarp();
            TC_TRACE(3, k);
            tc::group_bar(g);
            TC_TRACE(4, k);
            // ---- 2. one thread issues the MMAs of config k ----
            if (k < a.g.G && t == 0) {
                tc::fence_after();
                const uint32_t a_addr = tc::smem_u32(my_tiles + (k & 1) * tc::kTileBytes);
                const uint32_t b_addr = tc::smem_u32(b_tile);
#pragma unroll
                for (int s = 0; s < tc::kK / 16; ++s)
                    tc::mma_f16(d_col0 + (k & 1) * 32, tc::smem_desc(a_addr + s * 256),
                                tc::smem_desc(b_addr + s * 256), s > 0);
                tc::mma_commit(&mbars[2 * g + (k & 1)]);
            }
            __syncwarp();
            TC_TRACE(5, k);
            // ---- 3. epilogue of config k-1 ----
            if (k >= 1) {
                const int c = k - 1, b = c & 1;
                tc::mbar_wait(&mbars[2 * g + b], phase[b]);
                __syncwarp();
                TC_TRACE(6, k);
                phase[b] ^= 1u;
                tc::fence_after();
                float z[HD];
                tc::tmem_ld18(d_col0 + b * 32 + lane_off, z);
                float y = net.bo;
#pragma unroll
                for (int o = 0; o < HD; ++o) y = fmaf(fmaxf(z[o], 0.f), net.wo[o], y);
                const int cl = y < 0.5f;
                const float tm = fmaxf(y, 0.5f) * T_self;
                const float tt = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 1));
                const uint32_t m = masks[c];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    if (L == 1 || ((m >> l) & 1u)) {
                        clamps[l] += live ? cl : 0;
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
    // clamp counters: one atomic per warp and budget
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int tot = __reduce_add_sync(0xffffffffu, clamps[l]);
        if ((tid & 31) == 0 && tot) atomicAdd(a.clamps + l, (unsigned long long)tot);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem_base, tc::kGroups * tc::kTmemColsPerGroup);
    }
    TC_TRACE(8, 0);
}

inline size_t tc_smem_bytes(int G) {
    size_t b = (size_t)tc::kGroups * 2 * tc::kTileBytes + tc::kBBytes;
    b += 2 * (size_t)G * ROW32 * sizeof(float) + (size_t)G * sizeof(uint32_t);
    b = (b + 7) & ~(size_t)7;
    b += 2 * tc::kGroups * sizeof(uint64_t) + 32 + sizeof(Head64P);
    return b;
}
