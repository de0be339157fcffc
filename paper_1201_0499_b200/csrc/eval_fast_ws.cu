// Warp-specialised fast complex double-double kernel for d <= 2 and m <= 32 (one 32-monomial
// chunk per row): the C1/C2/C5 shapes. Same arithmetic, orders and contract as eval_fast.cu's
// d <= 2 path (suffix-product Speelpenning seeded with c*f, balanced segmented stage 3), but the
// CTA's warps split into two roles joined by a ring of staging buffers:
//   * producer warps run stages 1-2 (FP64-dense: the complex dd product chains) of a
//     (row p, point t) task into a free staging buffer and hand it over;
//   * consumer warps run stage 3 (shared-memory-latency-bound: the segmented sums, the
//     segment-partial adds and the HBM stores) on filled buffers and hand them back.
// In the fused kernel every warp alternates between the two phases, and the CTA's warps drift
// through them in step (same code, same task cost, one tile barrier): the FP64 pipe saturated
// while the warps run their chains and idled while they all sum. Split roles keep FP64-dense and
// latency-bound warps resident side by side on every scheduler at all times.
//
// Hand-off: buffer b of the ring (NB = number of warps) carries task tau with b = tau mod NB;
// full[b] / empty[b] count the rounds of buffer b produced / consumed (release stores by lane 0
// after a block fence and warp barrier, acquire loads by every waiting lane). Every warp takes
// its tasks in increasing tau and waits only on smaller tau, so the earliest unfinished task can
// always proceed (no deadlock for any producer : consumer split). The point tables belong to the producers:
// a named barrier over the producer warps guards each tile reload. Tasks are numbered in the
// order of the fused kernel (task = p * tp + t within a tile), producers take tau = w, w + P, ...,
// consumers tau = w', w' + C, ...
#include <cuda_runtime.h>

#include <cstdint>

#include "dd.cuh"
#include "eval_kernels.h"
#include "fast_common.cuh"

namespace pjb {

namespace {

// Ring hand-off through monotone per-buffer round counters in shared memory (not mbarrier
// parities: a buffer's rounds are produced and consumed by different warps, so a waiter can be a
// round ahead of the buffer, which a parity cannot tell apart from the round behind).
__device__ __forceinline__ unsigned ld_acquire(const unsigned* a) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(a)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* a, unsigned v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(a)), "r"(v) : "memory");
}
#ifndef PJB_WS_BACKOFF
#define PJB_WS_BACKOFF 256
#endif
// a waiting warp backs off between polls (nanosleep) so its spin does not take issue slots from
// the producers on the same scheduler
__device__ __forceinline__ void wait_at_least(const unsigned* a, unsigned v) {
    while (ld_acquire(a) < v) {
#if PJB_WS_BACKOFF
        __nanosleep(PJB_WS_BACKOFF);
#endif
    }
}
// every lane's shared-memory accesses to the buffer are ordered before lane 0's release
__device__ __forceinline__ void publish(unsigned* a, unsigned v, int lane) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) st_release(a, v);
}
__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace

// Stages 1-2 of one (row p, point table xt) task into the staging buffer stg (d <= 2, m <= 32):
// see eval_fast.cu (suffix products B_j staged in slot j, f = B_{k-1-c_g}, prefix chain seeded
// with c*f, L'_j = F'_j * B_j, power rule a_j * L'_j, value F'_{k-1} * v_{k-1}).
template <int K, int NS>
__device__ __forceinline__ void ws_stage12(const DevSystem& S, const double* xt, double* stg, int p, int lane,
                                           bool divf) {
    constexpr int W = 4;
    const CDD one = {1.0, 0.0, 0.0, 0.0};
    const int m = S.m;
    const int g = lane < m ? lane : m - 1;  // inactive lanes shadow a real monomial
    const int s = p * m + g;
    uint32_t pw[(K + 7) / 8 * 4];
    {
        const uint4* row = reinterpret_cast<const uint4*>(S.posexp + (size_t)s * S.kp);
#pragma unroll
        for (int q = 0; q < (K + 7) / 8; ++q) {
            const uint4 w = __ldg(row + q);
            pw[4 * q + 0] = w.x;
            pw[4 * q + 1] = w.y;
            pw[4 * q + 2] = w.z;
            pw[4 * q + 3] = w.w;
        }
    }
    auto POS = [&](int j) -> int { return (pw[j >> 1] >> ((j & 1) * 16)) & 255u; };
    auto EX1 = [&](int j) -> int { return (pw[j >> 1] >> ((j & 1) * 16 + 8)) & 255u; };
    const double* cf = S.coefT + (size_t)p * W * 32 + lane;
    auto SCALE = [&](int j, const CDD& x) -> CDD {
        const double a = EX1(j) ? 2.0 : 1.0;
        return {__dmul_rn(x.rh, a), __dmul_rn(x.rl, a), __dmul_rn(x.ih, a), __dmul_rn(x.il, a)};
    };
    auto X = [&](int j) -> CDD { return ld_hl(xt + 2 * POS(j), 2 * NS); };
    auto SLOT = [&](int j) -> double* { return stg + j * W * 32 + 2 * lane; };

    if (divf) {  // division form, as in eval_fast.cu (table rows x, x^2, 1/x)
        auto YP = [&](int j) -> CDD { return ld_hl(xt + EX1(j) * W * NS + 2 * POS(j), 2 * NS); };
        auto IV = [&](int j) -> CDD { return ld_hl(xt + 2 * W * NS + 2 * POS(j), 2 * NS); };
        CDD V = YP(0);
#pragma unroll
        for (int j = 1; j < K; ++j) V = cmul_n((j & 1) == 0, V, YP(j));
        const CDD cval = {__ldg(cf), __ldg(cf + 32), __ldg(cf + 64), __ldg(cf + 96)};
        const CDD cV = cdd_mul(V, cval);
        st_hl(SLOT(K), 64, cV);
#pragma unroll
        for (int j = 0; j < K; ++j) st_hl(SLOT(j), 64, SCALE(j, cdd_mul_u(cV, IV(j))));
        return;
    }
    // ---- stage 1 (ws): suffix products
    int cg = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) cg += EX1(j) & 1;
    st_hl(SLOT(K - 1), 64, one);
    CDD B0 = X(K - 1);
    st_hl(SLOT(K - 2), 64, B0);
#pragma unroll
    for (int j = K - 3; j >= 0; --j) {
        B0 = cmul_n(((K - 3 - j) & 1) != 0, B0, X(j + 1));
        st_hl(SLOT(j), 64, B0);
    }
    CDD f = ld_hl(SLOT(max(K - 1 - cg, 0)), 64);
    if (__any_sync(0xffffffffu, cg == K)) {
        const CDD fa = cdd_mul(B0, X(0));
        if (cg == K) f = fa;
    }
    // ---- stage 2 (ws): prefix chain seeded with c*f
    const CDD cval = {__ldg(cf), __ldg(cf + 32), __ldg(cf + 64), __ldg(cf + 96)};
    CDD Fp = cdd_mul(f, cval);
    st_hl(SLOT(0), 64, SCALE(0, cdd_mul_u(Fp, B0)));
#pragma unroll
    for (int j = 1; j < K; ++j) {
        Fp = cmul_n(((j - 1) & 1) != 0, Fp, X(j - 1));
        if (j < K - 1) {
            const CDD L = cdd_mul_u(Fp, ld_hl(SLOT(j), 64));
            st_hl(SLOT(j), 64, SCALE(j, L));
        }
    }
    st_hl(SLOT(K - 1), 64, SCALE(K - 1, Fp));
    st_hl(SLOT(K), 64, cdd_mul(Fp, X(K - 1)));
}

// Stage 3 of one task from the staging buffer stg (m <= 32: one chunk, results final):
// phase 1 balanced segmented sums with the partials left in the consumed slots, phase 2 the
// per-output partial adds and the HBM stores (see eval_fast.cu). codes / sq0: the (row, chunk)
// schedule, loaded by the caller before the buffer is ready.
template <int K>
__device__ __forceinline__ void ws_stage3(const DevSystem& S, double* stg, double* out, long long orow_pt, int p,
                                          int lane, const uint32_t (&codes)[K + 1], const uint4& sq0) {
    constexpr int R = K + 1;
    constexpr int W = 4;
    const int n = S.n;
    const CDD zero = {0.0, 0.0, 0.0, 0.0};
    // ---- stage 3, phase 1 (ws)
    {
        double sr = 0.0, lr = 0.0, si = 0.0, li = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t code = codes[r];
            if (code & kSchValid) {
                double* sl = stg + 2 * (code & 0x1fff);
                const CDD tv = ld_hl(sl, 64);
                const DD a = two_sum(sr, tv.rh), b = two_sum(si, tv.ih);
                sr = a.hi;
                si = b.hi;
                lr = __dadd_rn(lr, __dadd_rn(tv.rl, a.lo));
                li = __dadd_rn(li, __dadd_rn(tv.il, b.lo));
                if (code & kSchFlush) {
                    st_hl(sl, 64, CDD{sr, lr, si, li});
                    sr = lr = si = li = 0.0;
                }
            }
        }
    }
    __syncwarp();
    // ---- stage 3, phase 2 (ws)
    const long long nout = (long long)n * n + n;
    double* const orow = out + orow_pt * nout * W;
    const int npass = (n + 64) >> 6;
    for (int k2 = 0; k2 < npass; ++k2) {
        const size_t rec = ((size_t)p * npass + k2) * 32 + lane;
        const uint4 sq = k2 == 0 ? sq0 : __ldg(S.segq + rec);
        const int o1 = 64 * k2 + lane, o2 = sq.x >> 16;
        const int cnt1 = sq.x & 0xff, tot = cnt1 + ((sq.x >> 8) & 0xff);
        const bool has1 = o1 <= n, has2 = o2 != 0xffff;
        const uint32_t pk[3] = {sq.y, sq.z, sq.w};
        const uint16_t* xs = tot > 6 ? S.segcode + __ldg(S.seg + rec) : nullptr;
        auto CODE = [&](int qq) -> int {
            if (qq >= 6) return __ldg(xs + qq);
            const uint32_t w = qq < 2 ? pk[0] : qq < 4 ? pk[1] : pk[2];
            return (w >> (16 * (qq & 1))) & 0xffff;
        };
        auto LDE = [&](int e) -> CDD { return ld_hl(stg + 2 * e, 64); };
        auto FIN = [&](int o, const CDD& v) {
            const long long at = o == 0 ? p : n + (long long)p * n + (o - 1);
            st_aos(orow + at * W, cdd_renorm(v));
        };
        CDD r = zero;
#pragma unroll
        for (int qq = 0; qq < 6; ++qq) {
            if (qq < cnt1) {
                const CDD sv = LDE((pk[qq >> 1] >> (16 * (qq & 1))) & 0xffff);
                r = qq == 0 ? sv : cdd_add(r, sv);
            }
        }
        for (int qq = 6; qq < cnt1; ++qq) r = cdd_add(r, LDE(CODE(qq)));
        if (has1) FIN(o1, r);
        if (has2) {  // a secondary output without entries is a structural zero column
            CDD r2 = tot > cnt1 ? LDE(CODE(cnt1)) : zero;
            for (int qq = cnt1 + 1; qq < tot; ++qq) r2 = cdd_add(r2, LDE(CODE(qq)));
            FIN(o2, r2);
        }
    }
}

template <int K, int NS>
__global__ void __launch_bounds__(256, 3) fast_ws_kernel(DevSystem S, const double* __restrict__ pts,
                                                         double* __restrict__ out, long long B, int TP, int NP,
                                                         int* __restrict__ flag) {
    constexpr int W = 4;
    constexpr int R = K + 1;
    constexpr int stgW = (K + 1) * W * 32;
    extern __shared__ __align__(16) double smem_[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NB = nw, NC = nw - NP;
    const int n = S.n;
    const int tabPt = 3 * W * NS;  // rows x, x^2, 1/x (eval_fast.cu's tables for d <= 2)
    double* tab = smem_;
    double* ring = smem_ + TP * tabPt;
    unsigned* full = reinterpret_cast<unsigned*>(ring + NB * stgW);  // rounds produced, per buffer
    unsigned* empty = full + NB;                                      // rounds consumed, per buffer
    if (threadIdx.x < 2 * NB) full[threadIdx.x] = 0;
    __syncthreads();
    const long long ntiles = (B + TP - 1) / TP;
    long long tau0 = 0;  // first task number of the current tile
    if (warp < NP) {
        // ---------------------------------------------------------------- producers
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const long long b0 = tile * TP;
            const int tp = (int)min((long long)TP, B - b0);
            named_sync(1, NP * 32);  // every producer is done with the previous tile's table
            for (int i = threadIdx.x; i < tp * n; i += NP * 32) {
                const int t = i / n, v = i - t * n;
                CDD x = ld_aos(pts + ((b0 + t) * n + v) * W);
                if (!fin(x)) atomicOr(flag, 1);
                double* pb = tab + t * tabPt + 2 * v;
                st_hl(pb, 2 * NS, x);
                st_hl(pb + W * NS, 2 * NS, cdd_mul(x, x));
                st_hl(pb + 2 * W * NS, 2 * NS, cdd_inv(x));
            }
            named_sync(1, NP * 32);
            for (int task = warp; task < tp * n; task += NP) {
                const long long tau = tau0 + task;
                const int b = (int)(tau % NB);
                const unsigned rnd = (unsigned)(tau / NB);
                const int p = task / tp, t = task - p * tp;
                wait_at_least(empty + b, rnd);
                ws_stage12<K, NS>(S, tab + t * tabPt, ring + b * stgW, p, lane, div_form_ok(tab + t * tabPt, n, lane));
                publish(full + b, rnd + 1, lane);
            }
            tau0 += tp * n;
        }
    } else {
        // ---------------------------------------------------------------- consumers
        const int cw = warp - NP;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const long long b0 = tile * TP;
            const int tp = (int)min((long long)TP, B - b0);
            for (int task = cw; task < tp * n; task += NC) {
                const long long tau = tau0 + task;
                const int b = (int)(tau % NB);
                const unsigned rnd = (unsigned)(tau / NB);
                const int p = task / tp, t = task - p * tp;
                uint32_t codes[R];
                {
                    const uint32_t* sc = S.sch + (size_t)p * R * 32 + lane;
#pragma unroll
                    for (int r = 0; r < R; ++r) codes[r] = __ldg(sc + r * 32);
                }
                const uint4 sq0 = __ldg(S.segq + (size_t)p * ((n + 64) >> 6) * 32 + lane);
                wait_at_least(full + b, rnd + 1);
                ws_stage3<K>(S, ring + b * stgW, out, b0 + t, p, lane, codes, sq0);
                publish(empty + b, rnd + 1, lane);
            }
            tau0 += tp * n;
        }
    }
}

// ----------------------------------------------------------------------------- dispatch
namespace {

template <int K, int NS>
cudaError_t ws_launch_t(const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                        cudaStream_t st) {
    auto kern = fast_ws_kernel<K, NS>;
    if (L.smem_bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern));
        if (e != cudaSuccess) return e;
    }
    kern<<<L.blocks, L.threads, L.smem_bytes, st>>>(S, pts, out, B, L.tp, L.producers, L.flag);
    return cudaGetLastError();
}
template <int K, int NS>
int ws_occ_t(int threads, size_t smem) {
    auto kern = fast_ws_kernel<K, NS>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern)))
        return 0;
    int nb = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) == cudaSuccess ? nb : 0;
}

}  // namespace

#ifndef PJB_WS_KS
#define PJB_WS_KS(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)
#endif

bool fast_ws_supported(int k, int n, int m, int d) {
    if (d > 2 || m > 32 || n > 64) return false;
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return true;
        PJB_WS_KS(PJB_CASE)
#undef PJB_CASE
        default: return false;
    }
}

size_t fast_ws_smem(int n, int k, int nw, int tp) {
    const size_t ns = n <= 32 ? 32 : 64;
    return (size_t(tp) * 3 * 4 * ns + size_t(nw) * (k + 1) * 4 * 32) * sizeof(double) + 2 * size_t(nw) * sizeof(unsigned);
}

cudaError_t launch_fast_ws(int k, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                           cudaStream_t st) {
    const bool n32 = S.n <= 32;
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return n32 ? ws_launch_t<KK, 32>(L, S, pts, out, B, st) : ws_launch_t<KK, 64>(L, S, pts, out, B, st);
        PJB_WS_KS(PJB_CASE)
#undef PJB_CASE
        default: return cudaErrorInvalidValue;
    }
}

int fast_ws_blocks_per_sm(int k, int n, int threads, size_t smem) {
    const bool n32 = n <= 32;
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return n32 ? ws_occ_t<KK, 32>(threads, smem) : ws_occ_t<KK, 64>(threads, smem);
        PJB_WS_KS(PJB_CASE)
#undef PJB_CASE
        default: return 0;
    }
}

}  // namespace pjb
