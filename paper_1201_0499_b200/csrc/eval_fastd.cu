// Fast complex-double kernel in the REFERENCE operation order (PJ_PREC_D): bit-exact with the
// unmodified reference's EvaluationContext::evaluate, like the generic kernel, but specialised
// for throughput (SURVEY.md §8 config C4 and the drop-in's own precision).
//
// Reference path (ref = /root/reference/proj): stage1_powers / common factor
// ref/src/kernels.cpp:9-53, speelpenning_gradient + stage2_term ref/src/kernels.cpp:55-127,
// stage3_sum ref/src/kernels.cpp:139-146, transpose ref/src/engine.cpp:215-223. Every product and
// sum below is the reference's, in the reference's order and operand order, spelled with _rn
// intrinsics (no contraction) — only the assignment of work to threads differs.
//
// Mapping (same family as eval_kernels.cu / eval_fast.cu):
//   * a CTA owns a tile of TP points (coordinates and, for d > 2, the power table in shared
//     memory, plane layout);
//   * a warp owns one (row p, point PAIR) task: lane g evaluates monomial g of row p for two
//     points at once — two independent dependency chains per lane (in-order issue overlaps
//     them) and one set of coefficient / position loads for both;
//   * K (variables per monomial) is a template parameter: every chain is unrolled; a monomial's
//     fused position/exponent words arrive in one 16-byte load; its k+1 coefficients are
//     prefetched before stage 1 so their L2 latency hides behind the chains;
//   * stage 3 keeps the reference's ascending-g order per output (a sequential chain per
//     output), with one lane walking the gather list of a Jacobian column for both points
//     (columns grouped into quarter-warps by the host against bank conflicts) and lane 0 also
//     running the two m-term value chains in the same loop.
#include <cuda_runtime.h>

#include <cstdint>

#include "dd.cuh"
#include "eval_kernels.h"

namespace pjb {

namespace {

// (re, im) adjacent in shared memory: one 16-byte access per complex value
__device__ __forceinline__ CD ldv(const double* p) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    return {v.x, v.y};
}
__device__ __forceinline__ void stv(double* p, const CD& v) { *reinterpret_cast<double2*>(p) = make_double2(v.re, v.im); }
__device__ __forceinline__ CD sel(bool c, const CD& a, const CD& b) { return {c ? a.re : b.re, c ? a.im : b.im}; }

constexpr int kP = 2;  // points per lane
// staging swizzle of derivative row j (row K, the value terms, is not swizzled)
__host__ __device__ constexpr int fastd_swz(int j, int K) { return j < K ? (5 * j) & 7 : 0; }
#ifndef PJB_FASTD_VPER
#define PJB_FASTD_VPER 2
#endif
constexpr int kVPer = PJB_FASTD_VPER;  // value-chain terms per stage-3 loop iteration (measured: 2 beats 1, 4, 8)
#ifndef PJB_FASTD_MINB
#define PJB_FASTD_MINB(K) 2
#endif

}  // namespace

// Register budget: 2 CTAs of 256 threads (<= 128 registers; 3 CTAs spill at k = 8).
template <int K>
constexpr int fastd_min_blocks() { return PJB_FASTD_MINB(K); }

// SPLIT: the small-batch instantiation (a batch with fewer tiles than CTAs): SP CTAs share each
// tile's tasks (see eval_fast.cu). A separate instantiation, so the split's loop state never
// touches the register budget of the main kernel (128 registers, no room)
template <int K, bool D2, bool SPLIT = false>
__global__ void __launch_bounds__(256, fastd_min_blocks<K>()) fastd_kernel(DevSystem S, const double* __restrict__ pts,
                                                    double* __restrict__ out, long long B, int TP,
                                                    int* __restrict__ flag, int SP) {
    constexpr int W = 2;
    // staging: slot (j, point u) of lane g at ((j * kP + u) * 32 + g) * W (re, im adjacent)
    constexpr int stgW = (K + 1) * kP * W * 32;
    extern __shared__ __align__(16) double smem_[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = S.n, m = S.m, d = S.d, C = S.chunks, nm = S.nm;
    const int D1 = d > 2 ? d - 1 : 1;
    const int tabPt = D1 * W * n;
    const int accW = C > 1 ? (n + 1) * kP * W : 0;  // accumulator (output o, point u) at (o*kP + u)*W
    double* tab = smem_;
    double* stg = smem_ + TP * tabPt + warp * (stgW + accW);
    double* acc = stg + stgW;
    const long long ntiles = (B + TP - 1) / TP;
    const long long nout = (long long)n * n + n;
    const CD one = {1.0, 0.0};
    const CD zero = {0.0, 0.0};

    for (long long tile = SPLIT ? blockIdx.x / SP : blockIdx.x; tile < ntiles; tile += SPLIT ? gridDim.x / SP : gridDim.x) {
        const long long b0 = tile * TP;
        const int tp = (int)min((long long)TP, B - b0);
        for (int i = threadIdx.x; i < tp * n; i += blockDim.x) {
            const int t = i / n, v = i - t * n;
            const double2 xv = *reinterpret_cast<const double2*>(pts + ((b0 + t) * n + v) * W);
            if (!(isfinite(xv.x) && isfinite(xv.y))) atomicOr(flag, 1);
            stv(tab + t * tabPt + v * W, CD{xv.x, xv.y});
        }
        __syncthreads();
        if (!D2) {  // power table rows e = 2..d-1, ref kernels.cpp:16-24: row[e] = row[e-1] * x
            for (int i = threadIdx.x; i < tp * n; i += blockDim.x) {
                const int t = i / n, v = i - t * n;
                double* pb = tab + t * tabPt + v * W;  // power e of variable v at ((e-1) * n + v) * W
                const CD x = ldv(pb);
                CD r = x;
                for (int e = 2; e < d; ++e) {
                    r = cd_mul(r, x);
                    stv(pb + (e - 1) * W * n, r);
                }
            }
            __syncthreads();
        }
        const int npairs = (tp + 1) / 2;
        for (int task = SPLIT ? warp + (int)(blockIdx.x % SP) * nw : warp; task < npairs * n; task += SPLIT ? nw * SP : nw) {
            const int p = task / npairs, pair = task - p * npairs;
            const int t0 = 2 * pair;
            const bool has1 = t0 + 1 < tp;
            const double* xt[kP] = {tab + t0 * tabPt, tab + (has1 ? t0 + 1 : t0) * tabPt};
            CD vacc[kP] = {zero, zero};
            for (int c = 0; c < C; ++c) {
                const int graw = c * 32 + lane;
                const int g = graw < m ? graw : m - 1;  // inactive lanes shadow a real monomial
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
                auto EM1 = [&](int j) -> int { return (pw[j >> 1] >> ((j & 1) * 16 + 8)) & 255u; };
                // coefficients (pre-scaled a_j * c rounded as the reference, ref packing.cpp:46-49):
                // block j < K derivative coefficients, block K the value coefficient; loaded at use
                // (one load serves both points)
                const double* cfp = S.coef + s;
                auto COEF = [&](int j) -> CD { return {__ldg(cfp + (size_t)(2 * j) * nm), __ldg(cfp + (size_t)(2 * j + 1) * nm)}; };
                auto X = [&](int u, int j) -> CD { return ldv(xt[u] + POS(j) * W); };
                // powers[pos][a-1] (ref kernels.cpp:49-51): row 0 is 1, row 1 is x, row e the table
                auto PW = [&](int u, int j) -> CD {
                    const int e = EM1(j);
                    if constexpr (D2) {
                        return sel(e != 0, X(u, j), one);
                    } else {
                        return e == 0 ? one : ldv(xt[u] + ((e - 1) * n + POS(j)) * W);
                    }
                };
                // derivative rows j < K keep lane g's slot at g ^ swz(j) (a fixed per-row XOR that
                // spreads the stage-3 column walks over the bank quads); the value row is plain
                auto SLOT = [&](int j, int u) -> double* { return stg + ((j * kP + u) * 32 + (lane ^ fastd_swz(j, K))) * W; };

                // stage 1: common factor, ref kernels.cpp:45-53 (sequential from j = 0); for k >= 3 it
                // runs fused with the forward products below (one gather of x_j serves both chains)
                CD f[kP];
                if constexpr (K <= 2) {
#pragma unroll
                    for (int u = 0; u < kP; ++u) f[u] = PW(u, 0);
#pragma unroll
                    for (int j = 1; j < K; ++j)
#pragma unroll
                        for (int u = 0; u < kP; ++u) f[u] = cd_mul(f[u], PW(u, j));
                }

                // stage 2: speelpenning_gradient + stage2_term, ref kernels.cpp:55-127
                if constexpr (K == 1) {
#pragma unroll
                    for (int u = 0; u < kP; ++u) {
                        const CD L0 = cd_mul(one, f[u]);
                        const CD val = cd_mul(L0, X(u, 0));
                        stv(SLOT(0, u), cd_mul(L0, COEF(0)));
                        stv(SLOT(1, u), cd_mul(val, COEF(1)));
                    }
                } else if constexpr (K == 2) {
#pragma unroll
                    for (int u = 0; u < kP; ++u) {
                        const CD v0 = X(u, 0), v1 = X(u, 1);
                        const CD L0 = cd_mul(v1, f[u]), L1 = cd_mul(v0, f[u]);
                        const CD val = cd_mul(L1, v1);
                        stv(SLOT(0, u), cd_mul(L0, COEF(0)));
                        stv(SLOT(1, u), cd_mul(L1, COEF(1)));
                        stv(SLOT(2, u), cd_mul(val, COEF(2)));
                    }
                } else {
                    // forward products L[1] = v0, L[r+2] = L[r+1] * v[r+1] (kernels.cpp:69-73); the
                    // ones the backward pass consumes are parked in their staging slots
                    // powers[pos_j][a_j - 1] given the gathered x_j
                    auto PWv = [&](int u, int j, const CD& v) -> CD {
                        const int e = EM1(j);
                        if constexpr (D2) {
                            return sel(e != 0, v, one);
                        } else {
                            return e == 0 ? one : ldv(xt[u] + ((e - 1) * n + POS(j)) * W);
                        }
                    };
                    CD F[kP], vlast[kP];
                    // k <= 9: forward products L[1..k-2] kept in registers (compile-time indices); above,
                    // parked in the staging slots (registers would spill)
                    constexpr bool kFReg = K <= 9;  // measured k = 8: +4%; k >= 10 spills
                    CD Fs[kP][kFReg ? K : 1];
#pragma unroll
                    for (int u = 0; u < kP; ++u) {
                        const CD v0 = X(u, 0);
                        f[u] = PWv(u, 0, v0);
                        F[u] = v0;
                        if constexpr (kFReg) Fs[u][1] = v0;
                        else stv(SLOT(1, u), v0);
                    }
#pragma unroll
                    for (int j = 1; j < K; ++j)
#pragma unroll
                        for (int u = 0; u < kP; ++u) {
                            const CD v = X(u, j);
                            f[u] = cd_mul(f[u], PWv(u, j, v));
                            if (j <= K - 2) {  // forward step r = j - 1: L[j+1] = L[j] * v[j]
                                F[u] = cd_mul(F[u], v);
                                if (j + 1 < K - 1) {
                                    if constexpr (kFReg) Fs[u][j + 1] = F[u];
                                    else stv(SLOT(j + 1, u), F[u]);
                                }
                            } else {
                                vlast[u] = v;
                            }
                        }
                    // backward running product (kernels.cpp:76-89), each L[j] finished in place:
                    // L[j] * factor (:108-110), then * derivative coefficient (:115-116)
                    CD q[kP];
#pragma unroll
                    for (int u = 0; u < kP; ++u) {
                        q[u] = vlast[u];
                        CD L;
                        if constexpr (kFReg) L = cd_mul(Fs[u][K - 2], q[u]);
                        else L = cd_mul(ldv(SLOT(K - 2, u)), q[u]);
                        L = cd_mul(L, f[u]);
                        stv(SLOT(K - 2, u), cd_mul(L, COEF(K - 2)));
                    }
#pragma unroll
                    for (int r = 1; r <= K - 3; ++r)
#pragma unroll
                        for (int u = 0; u < kP; ++u) {
                            q[u] = cd_mul(q[u], X(u, K - 1 - r));
                            CD L;
                            if constexpr (kFReg) L = cd_mul(Fs[u][K - 2 - r], q[u]);
                            else L = cd_mul(ldv(SLOT(K - 2 - r, u)), q[u]);
                            L = cd_mul(L, f[u]);
                            stv(SLOT(K - 2 - r, u), cd_mul(L, COEF(K - 2 - r)));
                        }
#pragma unroll
                    for (int u = 0; u < kP; ++u) {
                        q[u] = cd_mul(q[u], X(u, 1));
                        const CD L0 = cd_mul(q[u], f[u]);
                        stv(SLOT(0, u), cd_mul(L0, COEF(0)));
                        // L[k-1] * factor, then the value L[k] = L[k-1] * v[k-1] (kernels.cpp:112)
                        const CD Lk1 = cd_mul(F[u], f[u]);
                        const CD val = cd_mul(Lk1, vlast[u]);
                        stv(SLOT(K - 1, u), cd_mul(Lk1, COEF(K - 1)));
                        stv(SLOT(K, u), cd_mul(val, COEF(K)));
                    }
                }
                __syncwarp();

                // stage 3 (kernels.cpp:139-146): ascending-g chains. Lane v: Jacobian column v of
                // both points over the gather list (structural zeros skipped: adding the reference's
                // exact +0 pads to an accumulator that starts at +0 never changes its bits); lane 0
                // additionally runs the two value chains over the chunk's monomials.
                const bool last = c + 1 == C;
                const int gl = min(32, m - c * 32);
                // lane slot vi handles the column the host assigned to it (columns grouped into
                // quarter-warps against bank conflicts; slot 0 is always column 0): one 8-byte
                // record {first entry, count | column << 16}
                for (int vi = lane; vi < n; vi += 32) {  // n >= 1: lane 0 always takes v = 0
                    const int2 cq = __ldg(S.colq + (size_t)(p * C + c) * n + vi);
                    const int v = cq.y >> 16;
                    const bool jac = v < n;
                    const int e0 = cq.x, len = cq.y & 0xffff;
                    CD a[kP];
#pragma unroll
                    for (int u = 0; u < kP; ++u) a[u] = c == 0 || !jac ? zero : ldv(acc + ((v + 1) * kP + u) * W);
                    // the value chains ride with column 0 (lane 0), kVPer terms per iteration (still
                    // one sequential chain: the loop trip count shrinks, not the order)
                    const int vlen = v == 0 ? gl : 0;
                    const int iters = max(len, (vlen + kVPer - 1) / kVPer);
                    for (int it = 0; it < iters; ++it) {
                        if (it < len) {
                            const int ent = __ldg(S.gm_ent + e0 + it);
                            const int jr = ent >> 5;
                            const double* sl = stg + (jr * kP * 32 + ((ent & 31) ^ ((5 * jr) & 7))) * W;
#pragma unroll
                            for (int u = 0; u < kP; ++u) a[u] = cd_add(a[u], ldv(sl + u * 32 * W));
                        }
#pragma unroll
                        for (int h = 0; h < kVPer; ++h) {
                            const int g2 = kVPer * it + h;
                            if (g2 < vlen) {
#pragma unroll
                                for (int u = 0; u < kP; ++u)
                                    vacc[u] = cd_add(vacc[u], ldv(stg + ((K * kP + u) * 32 + g2) * W));
                            }
                        }
                    }
                    if (jac) {
                        if (last) {
#pragma unroll
                            for (int u = 0; u < kP; ++u)
                                if (u == 0 || has1)
                                    *reinterpret_cast<double2*>(out + ((b0 + t0 + u) * nout + n + (long long)p * n + v) * W) =
                                        make_double2(a[u].re, a[u].im);
                        } else {
#pragma unroll
                            for (int u = 0; u < kP; ++u) stv(acc + ((v + 1) * kP + u) * W, a[u]);
                        }
                    }
                }
                if (last && lane == 0) {
#pragma unroll
                    for (int u = 0; u < kP; ++u)
                        if (u == 0 || has1)
                            *reinterpret_cast<double2*>(out + ((b0 + t0 + u) * nout + p) * W) =
                                make_double2(vacc[u].re, vacc[u].im);
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------- dispatch
namespace {

template <int K, bool D2>
cudaError_t launch_dt(const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                      cudaStream_t st) {
    auto kern = L.splits > 1 ? fastd_kernel<K, D2, true> : fastd_kernel<K, D2, false>;
    if (L.smem_bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern));
        if (e != cudaSuccess) return e;
    }
    kern<<<L.blocks, L.threads, L.smem_bytes, st>>>(S, pts, out, B, L.tp, L.flag, L.splits);
    return cudaGetLastError();
}
template <int K, bool D2>
int occ_dt(int threads, size_t smem) {
    auto kern = fastd_kernel<K, D2>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern)))
        return 0;
    int nb = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) == cudaSuccess ? nb : 0;
}

}  // namespace

#define PJB_FASTD_KS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

bool fastd_supported(int k) { return k >= 1 && k <= 16; }

size_t fastd_smem(int n, int m, int k, int d, int nw, int tp) {
    const size_t D1 = d > 2 ? d - 1 : 1;
    const size_t tab = D1 * 2 * size_t(n);
    const size_t chunks = (size_t(m) + 31) / 32;
    const size_t per_warp = size_t(k + 1) * kP * 2 * 32 + (chunks > 1 ? size_t(n + 1) * kP * 2 : 0);
    return (tp * tab + nw * per_warp) * sizeof(double);
}

cudaError_t launch_fastd(int k, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                         cudaStream_t st) {
    const bool d2 = S.d <= 2;
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return d2 ? launch_dt<KK, true>(L, S, pts, out, B, st) : launch_dt<KK, false>(L, S, pts, out, B, st);
        PJB_FASTD_KS(PJB_CASE)
#undef PJB_CASE
        default: return cudaErrorInvalidValue;
    }
}

int fastd_blocks_per_sm(int k, int d, int threads, size_t smem) {
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return d <= 2 ? occ_dt<KK, true>(threads, smem) : occ_dt<KK, false>(threads, smem);
        PJB_FASTD_KS(PJB_CASE)
#undef PJB_CASE
        default: return 0;
    }
}

}  // namespace pjb
