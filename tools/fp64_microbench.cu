// FP64-pipe microbenchmark for the roofline denominator.
// Measures, on the whole GPU, the sustained rate of DFMA, DADD, DMUL and of IEEE double
// division (a/b, the sequence used by the solver) with 8 independent chains per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fp64_microbench fp64_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void k_dfma(double *out, int iters, double b, double c) {
    double a[kChains];
#pragma unroll
    for (int q = 0; q < kChains; q++) a[q] = threadIdx.x * 1e-3 + q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int q = 0; q < kChains; q++) a[q] = __fma_rn(a[q], b, c);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < kChains; q++) s += a[q];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_dadd(double *out, int iters, double b) {
    double a[kChains];
#pragma unroll
    for (int q = 0; q < kChains; q++) a[q] = threadIdx.x * 1e-3 + q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int q = 0; q < kChains; q++) a[q] = __dadd_rn(a[q], b);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < kChains; q++) s += a[q];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_ddiv(double *out, int iters, double b) {
    double a[kChains];
#pragma unroll
    for (int q = 0; q < kChains; q++) a[q] = 1.0 + threadIdx.x * 1e-3 + q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int q = 0; q < kChains; q++) a[q] = b / a[q];
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < kChains; q++) s += a[q];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    auto run = [&](const char *name, auto launch, int it_used) {
        const double lanes = (double)blocks * threads * kChains * it_used;
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(s);
            launch();
            cudaEventRecord(e);
            cudaEventSynchronize(e);
            float ms;
            cudaEventElapsedTime(&ms, s, e);
            if (ms < best) best = ms;
        }
        double ops = lanes / (best / 1e3);
        printf("{\"op\": \"%s\", \"ops_per_s\": %.6e, \"per_sm_per_clk_at_max\": %.3f, \"ms\": %.3f}\n", name, ops,
               ops / sms / (clk * 1e3), best);
    };
    run("dfma", [&] { k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9); }, iters);
    run("dadd", [&] { k_dadd<<<blocks, threads>>>(out, iters, 1e-9); }, iters);
    run("ddiv", [&] { k_ddiv<<<blocks, threads>>>(out, iters / 8, 1.0000001); }, iters / 8);
    printf("{\"sms\": %d, \"clock_khz_max\": %d}\n", sms, clk);
    return 0;
}
