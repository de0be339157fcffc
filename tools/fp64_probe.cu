// FP64 pipe probe: throughput of DFMA / DADD / DMUL and dependent-chain latency on
// the box it runs on. Used to pin the FP64 roofline denominator (MEASURED_PEAKS.json
// has no FP64 figure). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int CH>
__global__ void tput(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) x[c] = __fma_rn(x[c], a, b);
            if (OP == 1) x[c] = __dadd_rn(x[c], b);
            if (OP == 2) x[c] = __dmul_rn(x[c], a);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

template <int OP>
__global__ void lat(double* out, int iters, double a, double b, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) x = __fma_rn(x, a, b);
        if (OP == 1) x = __dadd_rn(x, b);
        if (OP == 2) x = __dmul_rn(x, a);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

template <int OP>
double run_tput(double* d, int blocks, int threads, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    tput<OP, 8><<<blocks, threads>>>(d, iters / 10, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    tput<OP, 8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(blocks) * threads * iters * 8;
    return ops / (ms * 1e-3);  // instructions (lane-ops) per second
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    int sms = p.multiProcessorCount;
    double* d; cudaMalloc(&d, 64);
    long long* cyc; cudaMalloc(&cyc, 8);
    const char* names[3] = {"DFMA", "DADD", "DMUL"};
    double r[3];
    for (int rep = 0; rep < 2; ++rep) {
        r[0] = run_tput<0>(d, sms * 8, 256, 20000);
        r[1] = run_tput<1>(d, sms * 8, 256, 20000);
        r[2] = run_tput<2>(d, sms * 8, 256, 20000);
    }
    int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", p.name, sms, clk_khz);
    for (int o = 0; o < 3; ++o) printf(", \"%s_lane_ops_per_s\": %.4e", names[o], r[o]);
    printf(", \"fp64_peak_tflops_dfma\": %.3f", 2 * r[0] / 1e12);
    long long c;
    lat<0><<<1, 32>>>(d, 10000, 1.0000001, 1e-9, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"DFMA_latency_clk\": %.2f", c / 10000.0);
    lat<1><<<1, 32>>>(d, 10000, 1.0000001, 1e-9, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"DADD_latency_clk\": %.2f", c / 10000.0);
    lat<2><<<1, 32>>>(d, 10000, 1.0000001, 1e-9, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"DMUL_latency_clk\": %.2f}\n", c / 10000.0);
    return 0;
}
