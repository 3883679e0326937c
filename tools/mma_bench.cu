// mma_bench.cu -- cost model of small tcgen05.mma (kind::f16, M=128, K=16) on sm_100a.
//
// For the pair sweep the MMAs are tiny (N=32) and chained per config, so what
// matters is (a) issue throughput of back-to-back MMAs from one thread, (b) how
// it scales with the number of issuing warps per CTA, (c) the round trip
// issue -> commit -> mbarrier -> waiter, and (d) whether N or the A source
// (TMEM vs SMEM) changes any of it.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_bench.cu -o tools/mma_bench
// Run:   tools/mma_bench            (one line per case: cycles per MMA, per round)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)(256u >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}
// whole warp executes; one elected lane issues (no divergent branch around the MMA)
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "elect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t *bar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                     smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t *bar, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t ph) {
    const long long t0 = clock64();
    while (!try_wait(bar, ph))
        if (clock64() - t0 > 2000000000LL) __trap();
}

// mode 0: throughput (commit per round, wait only at the end), the round's
//         MMAs accumulate into ONE D (a dependent chain, as in the sweep)
// mode 1: latency (wait for each round's commit before issuing the next)
// mode 2: throughput, the round's MMAs go to `per_round` different D (acc = 0)
// mode 3: throughput, `chains` D accumulators interleaved: MMA k of the round
//         goes to D[k % chains] (dependency distance = chains)
// mode 4: mode 2 plus `chains` x 32 independent FFMAs after every MMA in the
//         issuing thread (is the issuing warp blocked while the MMA issues?)
// mode 5: mode 2 issued by TWO lanes of each issuer warp (per-warp or per-thread?)
__global__ void bench(int issuers, int n, int a_tmem, int per_round, int rounds, int mode,
                      int chains, long long *out) {
    __shared__ __align__(1024) uint8_t a_s[128 * 16 * 2];   // one K=16 slice
    __shared__ __align__(1024) uint8_t b_s[256 * 16 * 2];
    __shared__ __align__(8) uint64_t bars[32];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (int)sizeof(a_s) / 4; i += blockDim.x) ((uint32_t *)a_s)[i] = 0x3c003c00u;
    for (int i = threadIdx.x; i < (int)sizeof(b_s) / 4; i += blockDim.x) ((uint32_t *)b_s)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 32; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    long long t0 = 0, t1 = 0;
    float facc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (warp < issuers && (lane == 0 || (mode == 5 && lane == 16))) {
        // issuer w: D at columns [w * 128 / issuers ...), A (TMEM) at 384 + 32 w
        // D: 64 columns per issuer (<= 4 issuers), 32 (8 issuers, mode 2 uses one D)
        const uint32_t d = tmem + (uint32_t)(issuers > 4 ? warp * 32 : warp * (n <= 64 ? 64 : 128)) +
                           (lane == 16 ? 32u : 0u);
        const uint32_t at = tmem + (issuers > 4 ? 256 + (warp & 7) * 24 : 384 + warp * 32);
        const uint64_t ad = desc(smem_u32(a_s)), bd = desc(smem_u32(b_s));
        const uint32_t id = idesc(n);
        uint32_t ph = 0;
        t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            for (int k = 0; k < per_round; ++k) {
                uint32_t dk = d, acc = k > 0;
                if (mode == 2) { dk = issuers > 4 ? d : d + 32 * (k & 1); acc = 0; }
                if (mode == 3) { dk = d + 32 * (k % chains); acc = k >= chains; }
                if (mode >= 4) { dk = d; acc = 0; }
                if (a_tmem) mma_ts(dk, at + 8 * (k % 3), bd, id, acc);
                else mma_ss(dk, ad, bd, id, acc);
                if (mode == 4)
                    for (int f = 0; f < chains * 4; ++f)
#pragma unroll
                        for (int q = 0; q < 8; ++q) facc[q] = fmaf(facc[q], 1.0001f, 0.5f);
            }
            commit(&bars[warp + (lane == 16 ? 8 : 0)]);
            if (mode == 1) { wait(&bars[warp], ph); ph ^= 1; }
        }
        if (mode != 1) {
            // a final commit on a second barrier tracks every MMA issued so far
            commit(&bars[16 + warp + (lane == 16 ? 8 : 0)]);
            wait(&bars[16 + warp + (lane == 16 ? 8 : 0)], 0);
        }
        t1 = clock64();
        if (blockIdx.x == 0 && lane == 0) out[warp] = t1 - t0;
        if (facc[0] + facc[3] + facc[7] == 1234.5f) out[15] = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// tight issue loops: 4 MMAs per round into 4 D (acc=0) or one D (acc chain),
// compile-time offsets; style 0: lane 0 branch, style 1: whole warp + elect.sync
template <int STYLE, bool CHAIN>
__global__ void tight(int issuers, int rounds, long long *out) {
    __shared__ __align__(1024) uint8_t b_s[32 * 16 * 2];
    __shared__ __align__(8) uint64_t bars[32];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (int)sizeof(b_s) / 4; i += blockDim.x) ((uint32_t *)b_s)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 32; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (warp < issuers) {
        const uint32_t d = tmem + (uint32_t)(warp * 32);            // 8 issuers x 32 cols (CHAIN)
        const uint32_t at = tmem + 256 + (uint32_t)(warp & 7) * 24;
        const uint64_t bd = desc(smem_u32(b_s));
        const uint32_t id = idesc(32);
        long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (STYLE == 0) {
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_ts(CHAIN ? d : d + 8 * k, at + 8 * (k % 3), bd, id, CHAIN ? (k > 0) : 0);
                    commit(&bars[warp]);
                }
                __syncwarp();
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    mma_ts_elect(CHAIN ? d : d + 8 * k, at + 8 * (k % 3), bd, id, CHAIN ? (k > 0) : 0);
                commit_elect(&bars[warp]);
            }
        }
        if (lane == 0) {
            commit(&bars[16 + warp]);
            wait(&bars[16 + warp], 0);
        }
        __syncwarp();
        long long t1 = clock64();
        if (blockIdx.x == 0 && lane == 0) out[warp] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int STYLE, bool CHAIN>
void run_tight(int sms, long long *d_out, int issuers) {
    long long h_out[16];
    const int rounds = 4000;
    cudaMemset(d_out, 0, 16 * sizeof(long long));
    tight<STYLE, CHAIN><<<sms, 256>>>(issuers, 10, d_out);
    tight<STYLE, CHAIN><<<sms, 256>>>(issuers, rounds, d_out);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); exit(1); }
    cudaMemcpy(h_out, d_out, sizeof(h_out), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < issuers; ++w) mx = h_out[w] > mx ? h_out[w] : mx;
    const double pr = (double)mx / rounds;
    printf("tight style=%s chain=%d issuers=%d | %7.1f cycles/round  %6.1f cycles/MMA/issuer  %6.1f cycles/MMA/SM\n",
           STYLE ? "elect" : "lane0", (int)CHAIN, issuers, pr, pr / 4, pr / 4 / issuers);
}

int main() {
    long long *d_out, h_out[16];
    cudaMalloc(&d_out, 16 * sizeof(long long));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int rounds = 2000;
    printf("mode issuers N a_src per_round chains | cycles/round (max over issuers) cycles/MMA/issuer "
           "cycles/MMA/SM | ms\n");
    struct Case { int mode, issuers, n, a_tmem, per_round, chains; };
    const Case cases[] = {
        {2, 1, 32, 1, 4, 1}, {2, 4, 32, 1, 4, 1},
        {4, 1, 32, 1, 4, 0}, {4, 1, 32, 1, 4, 1}, {4, 1, 32, 1, 4, 2}, {4, 1, 32, 1, 4, 4},
        {4, 1, 32, 1, 4, 8}, {4, 4, 32, 1, 4, 2},
        {5, 1, 32, 1, 4, 1}, {5, 4, 32, 1, 4, 1},
    };
    for (int is : {1, 2, 4, 8}) {
        run_tight<0, true>(sms, d_out, is);
        run_tight<0, false>(sms, d_out, is);
        run_tight<1, true>(sms, d_out, is);
        run_tight<1, false>(sms, d_out, is);
    }
    for (const Case &c : cases) {
        cudaMemset(d_out, 0, sizeof(h_out));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        bench<<<sms, 512>>>(c.issuers, c.n, c.a_tmem, c.per_round, 10, c.mode, c.chains, d_out);
        cudaEventRecord(e0);
        bench<<<sms, 512>>>(c.issuers, c.n, c.a_tmem, c.per_round, rounds, c.mode, c.chains, d_out);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h_out, d_out, sizeof(h_out), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int w = 0; w < c.issuers; ++w) mx = h_out[w] > mx ? h_out[w] : mx;
        const double per_round_c = (double)mx / rounds;
        printf("%s %d %3d %s %2d ch%d | %8.1f %7.1f %7.1f | %.3f\n",
               c.mode == 0 ? "thr-chain" : c.mode == 1 ? "latency  " : c.mode == 2 ? "thr-indep" : "thr-inter",
               c.issuers, c.n, c.a_tmem ? "tmem" : "smem", c.per_round, c.chains, per_round_c,
               per_round_c / c.per_round, per_round_c / c.per_round / c.issuers, ms);
    }
    return 0;
}
