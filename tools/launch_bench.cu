// launch_bench.cu -- cost of kernel launches vs parameter size (direct and CUDA-graph replay).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/launch_bench.cu -o tools/launch_bench
#include <cuda_runtime.h>
#include <cstdio>
template <int N> struct P { double v[N]; };
template <int N> __global__ void k(const __grid_constant__ P<N> p, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.v[0] == 12345.0) out[0] = p.v[N - 1];
}
template <int N> void run(cudaStream_t st, double *out, int blocks) {
    P<N> p{};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 10; ++i) k<N><<<blocks, 128, 0, st>>>(p, out);
    cudaEventRecord(e0, st);
    const int reps = 200;
    for (int i = 0; i < reps; ++i) k<N><<<blocks, 128, 0, st>>>(p, out);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // graph of `reps` launches
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < reps; ++i) k<N><<<blocks, 128, 0, st>>>(p, out);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float gms; cudaEventElapsedTime(&gms, e0, e1);
    printf("param %6zu B  blocks %5d : direct %.2f us/launch   graph %.2f us/launch\n", sizeof(P<N>), blocks,
           ms * 1e3 / reps, gms * 1e3 / reps);
}
int main() {
    cudaStream_t st; cudaStreamCreate(&st);
    double *out; cudaMalloc(&out, 8);
    for (int b : {1, 148, 592, 1184}) {
        run<1>(st, out, b); run<128>(st, out, b); run<512>(st, out, b); run<1200>(st, out, b);
    }
    return 0;
}
