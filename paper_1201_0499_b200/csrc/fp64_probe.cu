// FP64 roofline denominator, measured on the running device: DFMA throughput with 8
// independent chains per thread over a full grid (2 flops per DFMA), and the FP64 pipe's issue
// rate per operation (DFMA / DADD / DMUL lane operations per second, 16 chains per thread). Not
// part of the reference surface; bench.py calls them so the roofline fraction uses the same box
// and clocks.
#include <cuda_runtime.h>

#include "../../include/polyjac_b200.h"

namespace {
__global__ void dfma_chains(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = __fma_rn(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}
template <int OP>
__global__ void pipe_chains(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            if (OP == 0) x[c] = __fma_rn(x[c], a, b);
            if (OP == 1) x[c] = __dadd_rn(x[c], b);
            if (OP == 2) x[c] = __dmul_rn(x[c], a);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}
}  // namespace

extern "C" int pj_fp64_pipe_probe(int device, double* lane_ops_per_s) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return PJ_ECUDA;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, device);
    double* d = nullptr;
    cudaMalloc(&d, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 8000;
    void (*kern[3])(double*, int, double, double) = {pipe_chains<0>, pipe_chains<1>, pipe_chains<2>};
    for (int op = 0; op < 3; ++op) {
        kern[op]<<<blocks, threads>>>(d, iters / 10, 1.0000001, 1e-9);
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            kern[op]<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        lane_ops_per_s[op] = double(blocks) * threads * iters * 16 / (best * 1e-3);
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    cudaSetDevice(prev);
    return e == cudaSuccess ? PJ_OK : PJ_ECUDA;
}

extern "C" int pj_fp64_peak_probe(int device, double* tflops) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return PJ_ECUDA;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, device);
    double* d = nullptr;
    cudaMalloc(&d, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
    dfma_chains<<<blocks, threads>>>(d, iters / 10, 1.0000001, 1e-9);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        dfma_chains<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return PJ_ECUDA;
    *tflops = 2.0 * double(blocks) * threads * iters * 8 / (best * 1e-3) / 1e12;
    return PJ_OK;
}
