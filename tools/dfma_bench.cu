// FP64 FMA throughput and latency on this GPU (tools/dfma_bench.cu).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dfma_bench.cu -o tools/dfma_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) x[u] = threadIdx.x * 1e-9 + u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < ILP; ++u) x[u] = fma(x[u], a, b);
    }
    double s = 0;
#pragma unroll
    for (int u = 0; u < ILP; ++u) s += x[u];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int ILP>
void run(int blocks, int threads, int iters) {
    double *d;
    cudaMalloc(&d, 8 * 1024);
    k_dfma<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_dfma<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int dev; cudaGetDevice(&dev);
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double fmas = (double)blocks * threads * iters * ILP;
    double per_sm_clk = fmas / (ms * 1e-3) / sms / (clk * 1e3);
    printf("ILP %d, %d blocks x %d threads: %.3f ms, %.2f TFMA/s = %.1f DFMA/clk/SM (clock %d MHz)\n",
           ILP, blocks, threads, ms, fmas / (ms * 1e-3) / 1e12, per_sm_clk, clk / 1000);
    cudaFree(d);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(sms, 32, 20000);        // one warp per SM: latency
    run<4>(sms, 32, 20000);
    run<8>(sms * 4, 256, 4000);
    run<8>(sms * 8, 256, 4000);
    run<3>(sms * 5, 128, 8000);
    return 0;
}
