// tc_probe.cu -- isolated check of the tcgen05 building blocks used by k_sweep_tc:
// canonical no-swizzle K-major smem layout + descriptors, kind::f16 MMA M128 N32 K16 x4,
// commit -> mbarrier, tcgen05.ld 32x32b.  Bounded waits: traps instead of hanging.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../include tc_probe.cu -o tc_probe
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t tile_off(int row, int chunk) { return (uint32_t)((row >> 3) * 1024 + chunk * 128 + (row & 7) * 16); }

__device__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int version_bit) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    if (version_bit) d |= (uint64_t)1 << 46;
    return d;
}

__global__ void probe(const __half *A, const __half *B, float *D, int *status, uint32_t idesc,
                      uint32_t lbo, uint32_t sbo, int version_bit) {
    __shared__ __align__(1024) uint8_t a_s[128 * 64 * 2];
    __shared__ __align__(1024) uint8_t b_s[32 * 64 * 2];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    // row t of A (64 halves) -> canonical layout
    for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4 *>(a_s + tile_off(t, c)) = reinterpret_cast<const uint4 *>(A + t * 64)[c];
    if (t < 32)
        for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4 *>(b_s + tile_off(t, c)) = reinterpret_cast<const uint4 *>(B + t * 64)[c];
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (t == 0) {
        for (int s = 0; s < 4; ++s) {
            uint64_t ad = make_desc(smem_u32(a_s) + s * 256, lbo, sbo, version_bit);
            uint64_t bd = make_desc(smem_u32(b_s) + s * 256, lbo, sbo, version_bit);
            uint32_t acc = s > 0;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                         :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)) : "memory");
    }
    // bounded wait
    uint32_t done = 0;
    for (long it = 0; it < (1L << 22) && !done; ++it) {
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n}"
                     : "=r"(done) : "r"(smem_u32(&mbar)) : "memory");
    }
    if (!done) { if (t == 0) atomicExch(status, -1); }
    else {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)((t / 32) * 32) << 16);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(taddr));
        uint32_t r2[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r2[0]), "=r"(r2[1]), "=r"(r2[2]), "=r"(r2[3]), "=r"(r2[4]), "=r"(r2[5]), "=r"(r2[6]), "=r"(r2[7]),
                       "=r"(r2[8]), "=r"(r2[9]), "=r"(r2[10]), "=r"(r2[11]), "=r"(r2[12]), "=r"(r2[13]), "=r"(r2[14]), "=r"(r2[15])
                     : "r"(taddr + 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int k = 0; k < 16; ++k) { D[t * 32 + k] = __uint_as_float(r[k]); D[t * 32 + 16 + k] = __uint_as_float(r2[k]); }
        if (t == 0) atomicExch(status, 1);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tmem));
}

int main(int argc, char **argv) {
    __half hA[128 * 64], hB[32 * 64];
    double ref[128 * 32];
    srand(1);
    for (int i = 0; i < 128 * 64; ++i) hA[i] = __float2half((float)((rand() % 17) - 8) / 8.0f);
    for (int i = 0; i < 32 * 64; ++i) hB[i] = __float2half((float)((rand() % 13) - 6) / 4.0f);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32; ++n) {
            double s = 0;
            for (int k = 0; k < 64; ++k) s += (double)__half2float(hA[m * 64 + k]) * (double)__half2float(hB[n * 64 + k]);
            ref[m * 32 + n] = s;
        }
    __half *dA, *dB; float *dD; int *dS;
    cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, 128 * 32 * 4); cudaMalloc(&dS, 4);
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    const uint32_t idesc_base = (1u << 4) | ((32u >> 3) << 17);
    struct V { const char *name; uint32_t idesc, lbo, sbo; int ver; } vs[] = {
        {"m@24 lbo128 sbo1024 v1", idesc_base | ((128u >> 4) << 24), 128, 1024, 1},
        {"m@24 lbo1024 sbo128 v1", idesc_base | ((128u >> 4) << 24), 1024, 128, 1},
        {"m@23 lbo128 sbo1024 v1", idesc_base | ((128u >> 4) << 23), 128, 1024, 1},
        {"m@23 lbo1024 sbo128 v1", idesc_base | ((128u >> 4) << 23), 1024, 128, 1},
    };
    for (auto &v : vs) {
        float hD[128 * 32];
        int st = 0;
        cudaMemset(dS, 0, 4);
        cudaMemset(dD, 0, 128 * 32 * 4);
        probe<<<1, 128>>>(dA, dB, dD, dS, v.idesc, v.lbo, v.sbo, v.ver);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: CUDA error %s\n", v.name, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int i = 0; i < 128 * 32; ++i) maxerr = fmax(maxerr, fabs(hD[i] - ref[i]));
        printf("%-26s status %d  max|D-ref| %.3g  D[0]=%g ref[0]=%g D[33]=%g ref[33]=%g\n", v.name, st, maxerr,
               hD[0], ref[0], hD[33], ref[33]);
    }
    return 0;
}
