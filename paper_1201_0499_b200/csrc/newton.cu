// Newton corrector on device: the consumer of the evaluator's output.
//
// For every point b of a batch, given the evaluator's result [f_b | J_b] (EvaluationResult
// layout, ref include/polyjac/system.hpp:48-54: n values, then the row-major Jacobian), solve
//
//     J_b · dx = y_b − f_b          (y = optional target, 0 when absent)
//
// by Gaussian elimination with partial pivoting, and write x_new = x_b + dx. This is the step
// the paper evaluates systems for (Newton / path tracking); the reference lists
// it as out of scope, so its operation order is defined here and restated
// verbatim by the oracle (oracle/oracle.cpp: newton_one), which makes the device result
// bit-identical to the oracle in both precisions.
//
// Operation order (T = complex double or complex double-double):
//   rhs_i = y_i + (−f_i)                          (−f_i when y is absent)
//   for kk = 0..n−1:
//     piv = first i ≥ kk maximising |Re_hi A[i][kk]| + |Im_hi A[i][kk]| (strictly > 0, else
//           the point is singular: status 1, x_new = x)
//     swap rows kk, piv over columns kk..n (column n = rhs)
//     inv_kk = 1 / A[kk][kk]                       (cinv below)
//     l_i = A[i][kk] · inv_kk                     i > kk (normalised product)
//     A[i][j] = A[i][j] + (−(l_i · A[kk][j]))     i > kk, j = kk+1..n (dd: product left
//                                                  unnormalised, the addition renormalises)
//   for i = n−1..0:  dx_i = rhs_i · inv_i;  rhs_r = rhs_r + (−(A[r][i] · dx_i))  for r < i
//   x_new_i = x_i + dx_i
//
// B200 mapping: a CTA owns one point at a time (persistent grid over the batch). The
// augmented matrix [J | rhs] lives in shared memory as W planes of n × (n+1) doubles (row
// stride n+1: a warp's column walk hits every bank pair once); n ≤ 64 fits (133 KB in dd), larger
// systems use a per-CTA global scratch slab with the same code. Warp 0 does the pivot search
// (shuffle arg-max), the row swap, the pivot inverse and the multipliers; all warps then
// update the trailing block (one element per thread per pass); back substitution runs in warp
// 0 with the right-hand side in registers (a lane owns rows lane + 32q) and the solved
// component broadcast by shuffle. Several CTAs per SM overlap one CTA's serial phases with the
// others' trailing updates. The path is FP64-issue-bound like the evaluator.
#include <cuda_runtime.h>

#include <cmath>

#include "dd.cuh"
#include "eval_kernels.h"

namespace pjb {
namespace {

__device__ __forceinline__ CD nt_neg(CD a) { return {-a.re, -a.im}; }
__device__ __forceinline__ CDD nt_neg(CDD a) { return {-a.rh, -a.rl, -a.ih, -a.il}; }
// pivot magnitude: |Re| + |Im| of the high words (rounded once)
__device__ __forceinline__ double nt_mag1(CD a) { return __dadd_rn(fabs(a.re), fabs(a.im)); }
__device__ __forceinline__ double nt_mag1(CDD a) { return __dadd_rn(fabs(a.rh), fabs(a.ih)); }
// reported norms: max of |Re_hi|, |Im_hi|
__device__ __forceinline__ double nt_magmax(CD a) { return fmax(fabs(a.re), fabs(a.im)); }
__device__ __forceinline__ double nt_magmax(CDD a) { return fmax(fabs(a.rh), fabs(a.ih)); }
__device__ __forceinline__ bool nt_finite(CD a) { return isfinite(a.re) && isfinite(a.im); }
__device__ __forceinline__ bool nt_finite(CDD a) {
    return isfinite(a.rh) && isfinite(a.rl) && isfinite(a.ih) && isfinite(a.il);
}
// trailing-update product: dd leaves it unnormalised (the following addition renormalises)
__device__ __forceinline__ CD nt_umul(CD a, CD b) { return cd_mul(a, b); }
__device__ __forceinline__ CDD nt_umul(CDD a, CDD b) { return cdd_mul_u(a, b); }

// real dd product (FMA TwoProd, cross terms, Fast2Sum) and reciprocal
__device__ __forceinline__ DD nt_dd_mul(DD a, DD b) {
    double p = __dmul_rn(a.hi, b.hi);
    double e = __fma_rn(a.hi, b.hi, -p);
    e = __fma_rn(a.hi, b.lo, e);
    e = __fma_rn(a.lo, b.hi, e);
    return fast_two_sum(p, e);
}
// 1/a: q = RN(1/a.hi); t = 1 − a·q (the first FMA is exact); q + t·q
__device__ __forceinline__ DD nt_dd_rcp(DD a) {
    double q = __drcp_rn(a.hi);
    double t = __fma_rn(-a.hi, q, 1.0);
    t = __fma_rn(-a.lo, q, t);
    return fast_two_sum(q, __dmul_rn(t, q));
}
// complex inverse conj(a) / |a|^2
__device__ __forceinline__ CD nt_inv(CD a) {
    double den = __dadd_rn(__dmul_rn(a.re, a.re), __dmul_rn(a.im, a.im));
    double r = __drcp_rn(den);
    return {__dmul_rn(a.re, r), __dmul_rn(-a.im, r)};
}
__device__ __forceinline__ CDD nt_inv(CDD a) {
    DD re{a.rh, a.rl}, im{a.ih, a.il};
    DD den = dd_add(nt_dd_mul(re, re), nt_dd_mul(im, im));
    DD r = nt_dd_rcp(den);
    DD o = nt_dd_mul(re, r), p = nt_dd_mul({-a.ih, -a.il}, r);
    return {o.hi, o.lo, p.hi, p.lo};
}

template <class T>
__device__ __forceinline__ T shfl_idx(T v, int src);
template <>
__device__ __forceinline__ CD shfl_idx<CD>(CD v, int src) {
    return {__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src)};
}
template <>
__device__ __forceinline__ CDD shfl_idx<CDD>(CDD v, int src) {
    return {__shfl_sync(0xffffffffu, v.rh, src), __shfl_sync(0xffffffffu, v.rl, src),
            __shfl_sync(0xffffffffu, v.ih, src), __shfl_sync(0xffffffffu, v.il, src)};
}

// NQ: rows per lane in back substitution (n <= 32*NQ)
template <class T, int NQ>
__global__ void __launch_bounds__(256) newton_kernel(NewtonArgs a) {
    using S = Sc<T>;
    constexpr int W = S::W;
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_piv;
    const int n = a.n, ld = n + 1, P = n * ld;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    double* A = a.gscratch ? a.gscratch + size_t(blockIdx.x) * a.gstride : smem;
    double* INV = A + size_t(W) * P;  // [W][n] pivot inverses
    const size_t nout = size_t(n) * n + n;

    for (long long b = blockIdx.x; b < a.B; b += gridDim.x) {
        const double* ev = a.evals + size_t(b) * nout * W;
        // ---- load [J | y − f] into planes
        for (int t = tid; t < n * n; t += nt) {
            const int i = t / n, j = t - i * n;
            S::st_planes(A + i * ld + j, P, S::ld_aos(ev + size_t(n + t) * W));
        }
        if (warp == 0) {
            double rn = 0.0;
            for (int i = lane; i < n; i += 32) {
                T r = nt_neg(S::ld_aos(ev + size_t(i) * W));
                if (a.target) r = S::add(S::ld_aos(a.target + (size_t(b) * n + i) * W), r);
                S::st_planes(A + i * ld + n, P, r);
                rn = fmax(rn, nt_magmax(r));
            }
            for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
            if (lane == 0 && a.norms) a.norms[2 * b] = rn;
        }
        __syncthreads();

        // ---- elimination with partial pivoting
        bool singular = false;
        for (int kk = 0; kk < n; ++kk) {
            if (warp == 0) {
                double best = 0.0;
                int bi = -1;
                for (int i = kk + lane; i < n; i += 32) {
                    const double mg = nt_mag1(S::ld_planes(A + i * ld + kk, P));
                    if (mg > best) {
                        best = mg;
                        bi = i;
                    }
                }
                for (int o = 16; o; o >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) {
                        best = ob;
                        bi = oi;
                    }
                }
                if (bi >= 0) {
                    if (bi != kk)
                        for (int j = kk + lane; j <= n; j += 32) {
                            T u = S::ld_planes(A + kk * ld + j, P), v = S::ld_planes(A + bi * ld + j, P);
                            S::st_planes(A + kk * ld + j, P, v);
                            S::st_planes(A + bi * ld + j, P, u);
                        }
                    __syncwarp();
                    const T iv = nt_inv(S::ld_planes(A + kk * ld + kk, P));  // every lane, same value
                    if (lane == 0) S::st_planes(INV + kk, n, iv);
                    for (int i = kk + 1 + lane; i < n; i += 32)
                        S::st_planes(A + i * ld + kk, P, S::mul(S::ld_planes(A + i * ld + kk, P), iv));
                }
                if (lane == 0) s_piv = bi;
            }
            __syncthreads();
            if (s_piv < 0) {
                singular = true;
                break;
            }
            const int R = n - kk - 1, C = n - kk;
            for (int e = tid; e < R * C; e += nt) {
                const int r = e / C;
                const int i = kk + 1 + r, j = kk + 1 + (e - r * C);
                const T l = S::ld_planes(A + i * ld + kk, P);
                const T u = S::ld_planes(A + kk * ld + j, P);
                const T v = S::ld_planes(A + i * ld + j, P);
                S::st_planes(A + i * ld + j, P, S::add(v, nt_neg(nt_umul(l, u))));
            }
            __syncthreads();
        }

        // ---- back substitution (warp 0), rhs rows lane + 32q in registers
        if (warp == 0) {
            const double* x = a.points + size_t(b) * n * W;
            double* xo = a.points_out + size_t(b) * n * W;
            if (singular) {
                for (int i = lane; i < n; i += 32) S::st_aos(xo + size_t(i) * W, S::ld_aos(x + size_t(i) * W));
                if (lane == 0) {
                    if (a.norms) a.norms[2 * b + 1] = INFINITY;
                    if (a.status) a.status[b] = 1;
                }
            } else {
                T rr[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int r = lane + 32 * q;
                    rr[q] = r < n ? S::ld_planes(A + r * ld + n, P) : S::zero();
                }
                for (int i = n - 1; i >= 0; --i) {
                    const int owner = i & 31, qi = i >> 5;
                    T v = rr[0];
#pragma unroll
                    for (int q = 1; q < NQ; ++q)
                        if (q == qi) v = rr[q];
                    v = shfl_idx(v, owner);
                    const T dx = S::mul(v, S::ld_planes(INV + i, n));
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const int r = lane + 32 * q;
                        if (r < i) rr[q] = S::add(rr[q], nt_neg(nt_umul(S::ld_planes(A + r * ld + i, P), dx)));
                        if (r == i) rr[q] = dx;
                    }
                }
                double dn = 0.0;
                bool fin = true;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int r = lane + 32 * q;
                    if (r < n) {
                        const T xn = S::add(S::ld_aos(x + size_t(r) * W), rr[q]);
                        S::st_aos(xo + size_t(r) * W, xn);
                        dn = fmax(dn, nt_magmax(rr[q]));
                        fin = fin && nt_finite(xn);
                    }
                }
                for (int o = 16; o; o >>= 1) dn = fmax(dn, __shfl_xor_sync(0xffffffffu, dn, o));
                fin = __all_sync(0xffffffffu, fin);
                if (lane == 0) {
                    if (a.norms) a.norms[2 * b + 1] = dn;
                    if (a.status) a.status[b] = fin ? 0 : 2;
                }
            }
        }
        __syncthreads();  // the next point reuses the matrix storage
    }
}

template <class T>
const void* newton_fn(int nq) {
    switch (nq) {
        case 1: return (const void*)newton_kernel<T, 1>;
        case 2: return (const void*)newton_kernel<T, 2>;
        case 4: return (const void*)newton_kernel<T, 4>;
        default: return (const void*)newton_kernel<T, 8>;
    }
}
int nq_of(int n) { return n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8; }
const void* fn_of(int prec, int n) { return prec == 1 ? newton_fn<CD>(nq_of(n)) : newton_fn<CDD>(nq_of(n)); }

}  // namespace

size_t newton_matrix_bytes(int prec, int n) {
    const int W = prec == 1 ? 2 : 4;
    return (size_t(W) * n * (n + 1) + size_t(W) * n) * sizeof(double);
}

int newton_blocks_per_sm(int prec, int n, int threads, size_t smem) {
    const void* f = fn_of(prec, n);
    if (smem) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, threads, smem) != cudaSuccess) return 0;
    return nb;
}

cudaError_t launch_newton(int prec, const NewtonArgs& args, int blocks, int threads, size_t smem, cudaStream_t st) {
    if (args.B <= 0) return cudaSuccess;
    const void* f = fn_of(prec, args.n);
    if (smem) {
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e) return e;
    }
    const long long nb = blocks < args.B ? blocks : args.B;
    void* kargs[] = {const_cast<NewtonArgs*>(&args)};
    return cudaLaunchKernel(f, dim3(unsigned(nb)), dim3(threads), kargs, smem, st);
}

}  // namespace pjb
