// tcgen05_util.cuh -- PTX helpers of the tcgen05 screen (k_sweep_tc3): TMEM
// allocation and loads/stores, mbarriers, fences, the fp16 B-operand slices
// of W2 and the packed f32x2 / f16x2 conversions the A-row build uses.
//
// Included by sweep.cu (shares Net64P, HD).
#pragma once

#ifdef CS_TC_TRACE
#define TC_TRACE(stage, k) \
    do { if (a.trace) ((volatile uint32_t *)a.trace)[blockIdx.x * blockDim.x + threadIdx.x] = \
             ((uint32_t)(k) << 8) | (stage); } while (0)
#else
#define TC_TRACE(stage, k) do { } while (0)
#endif

namespace tc {

constexpr int kGroups = 4;               // compute groups per CTA
constexpr int kGroupThreads = 128;
constexpr int kThreads = kGroups * kGroupThreads;
constexpr int kPairsPerBlock = 64;
constexpr uint32_t kIdesc = (1u << 4)            // D = f32
                          | (0u << 7) | (0u << 10)  // A, B = f16
                          | (0u << 15) | (0u << 16) // both K-major
                          | ((24u >> 3) << 17)      // N = 24: z2[0:18] + the head column
                          | ((128u >> 4) << 24);    // M = 128

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
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

// TMA bulk copy global -> shared (cp.async.bulk, the 1-D form of the tensor
// memory accelerator): completion is signalled on `bar` as transaction bytes.
// dst / src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
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

// 20 fp32 columns of this thread's TMEM lane (x16 + x4)
__device__ __forceinline__ void tmem_ld20(uint32_t taddr, float (&v)[20]) {
    uint32_t r[20];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19])
                 : "r"(taddr + 16));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 20; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ float2 unpack_half2(uint32_t w) {
    __half2 h = *reinterpret_cast<__half2 *>(&w);
    return __half22float2(h);
}

}  // namespace tc

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

// z - float(h) for the two halves of h (lo half <-> z.x): fma.rn.f32.f16
// (FHFMA), h * -1 + z, exact when h is z truncated to fp16
__device__ __forceinline__ float2 residual_h2(uint32_t h, float2 z) {
    float2 r;
    asm("{\n\t.reg .f16 a, b, m;\n\t"
        "mov.b32 {a, b}, %2;\n\t"
        "mov.b16 m, 0xBC00;\n\t"
        "fma.rn.f32.f16 %0, a, m, %3;\n\t"
        "fma.rn.f32.f16 %1, b, m, %4;\n}"
        : "=f"(r.x), "=f"(r.y) : "r"(h), "f"(z.x), "f"(z.y));
    return r;
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

// fp16 B slices of W2 (written once per sweep by k_tables into cs_tables.w2_tile):
//   q0 = W2hi[:, 0:16]   q1 = [W2hi16 W2hi17 W2hi16 W2hi17 b2hi b2lo W2lo16 W2lo17 0..]
//   q2 = W2lo[:, 0:16]   q3 = [W2lo16 W2lo17 0..] (unused by k_sweep_tc3)
__device__ void write_b_slices(const Net64P &net, uint16_t *tile, int idx) {
    // idx in [0, 4 * 32 * 16)
    const int q = idx / 512, rem = idx % 512, n = rem / 16, kk = rem % 16;
    auto hi_of = [](double x) { return (double)__half2float(__double2half(x)); };
    double v = 0.0;
    // row 18: 0.5 wo^T W2 (and bias 0.5 wo . b2) -- D column 18 is then the
    // linear half of the head, 0.5 wo . z2 (see k_sweep_tc3's epilogue)
    double row[HD], bias;
    if (n < HD) {
        for (int k = 0; k < HD; ++k) row[k] = net.w2[n * HD + k];
        bias = net.b2[n];
    } else {
        bias = 0.0;
        for (int k = 0; k < HD; ++k) row[k] = 0.0;
        for (int o = 0; o < HD; ++o) {
            for (int k = 0; k < HD; ++k) row[k] += 0.5 * net.wo[o] * net.w2[o * HD + k];
            bias += 0.5 * net.wo[o] * net.b2[o];
        }
    }
    if (n <= HD) {
        const double *w = row;
        if (q == 0) v = hi_of(w[kk]);
        else if (q == 2) v = w[kk] - hi_of(w[kk]);
        else if (q == 1) {
            if (kk == 0 || kk == 2) v = hi_of(w[16]);
            else if (kk == 1 || kk == 3) v = hi_of(w[17]);
            else if (kk == 4) v = hi_of(bias);
            else if (kk == 5) v = bias - hi_of(bias);
            // k 6-7 meet A column 19 = (hi16, hi17): k_sweep_tc3 so folds the
            // W2lo[:, 16:18] term into this slice
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
