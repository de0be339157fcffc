// Developer microbenchmark: FP64 dependent-issue latency and per-SM-subpartition throughput on
// this GPU (DADD / DFMA chains; CH independent chains per thread, W warps per CTA, one CTA per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, bool FMA>
__global__ void chain(double* out, long long iters, long long* cyc) {
    double v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3 + c;
    const double a = 1.0000001, b = 1e-9;
    long long t0 = clock64();
    for (long long i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) v[c] = FMA ? __fma_rn(v[c], a, b) : __dadd_rn(v[c], b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH, bool FMA>
void run(int warps, int sms) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * sms * warps * 32);
    cudaMalloc(&cyc, sizeof(long long));
    const long long iters = 2000;
    chain<CH, FMA><<<sms, warps * 32>>>(out, iters, cyc);
    chain<CH, FMA><<<sms, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double ops = double(iters) * 8 * CH;  // per thread
    printf("%s chains/thread %d warps/SM %2d: %.2f cycles per dependent op, %.3f warp-inst/clk per SM\n",
           FMA ? "DFMA" : "DADD", CH, warps, c / (double(iters) * 8), ops * warps / c);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {1, 4, 8, 16}) {
        run<1, false>(w, sms);
        run<2, false>(w, sms);
        run<4, false>(w, sms);
        run<8, false>(w, sms);
        run<1, true>(w, sms);
        run<4, true>(w, sms);
    }
    return 0;
}
