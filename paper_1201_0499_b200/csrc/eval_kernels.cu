// sm_100a kernels for the three-stage system + Jacobian evaluation (arXiv 1201.0499), batched
// over evaluation points.
//
// Reference path replaced (ref = /root/reference/proj):
//   EvaluationContext::evaluate_into  ref/src/engine.cpp:181-224 (3 pool launches + transpose)
//   stage1_powers / common factor     ref/src/kernels.cpp:9-53
//   speelpenning_gradient / stage2    ref/src/kernels.cpp:55-127
//   stage3_sum                        ref/src/kernels.cpp:139-146
//
// Mapping (B200-first):
//   * a CTA owns a tile of TP points; their coordinates (and for d > 2 the power table
//     x_v^e, e = 1..d-1, ref kernels.cpp:16-24) sit in shared memory in pair layout (ld_pr);
//   * a warp owns one (polynomial row p, point) task at a time; lane g evaluates monomial
//     g of row p (stages 1 and 2 in registers; the forward products of the Speelpenning
//     schedule are parked in the warp's staging area, which then receives the k+1 final
//     terms), chunks of 32 monomials when m > 32;
//   * stage 3 is an on-chip ordered gather: lane v walks the precomputed (row, column)
//     list of (g, j) contributions to Jacobian entry (p, v) in ascending g and sums them
//     (no padded Mons buffer, no HBM round trip; structural zeros are never touched and
//     stay exact +0). The value of row p is the m-term sum of the monomial values.
//   * results go straight to HBM in the reference's EvaluationResult order.
//
// ORDER = kRef keeps the reference's operation order everywhere (bit-exact with
// EvaluationContext::evaluate in complex double, and with the oracle's dd restatement in
// complex double-double). ORDER = kFast sums the row value with a warp-shuffle tree
// (documented order difference, tolerance-checked).
#include <cuda_runtime.h>

#include <cstdint>

#include "dd.cuh"
#include "eval_kernels.h"

namespace pjb {

// Pair layout (like the fast kernels): element e of an array of P elements keeps (re, im) at
// base + 2e (complex double) or (re_hi, im_hi) at base + 2e and (re_lo, im_lo) at base + 2P + 2e
// (complex dd) — one 16-byte shared access per pair.
__device__ __forceinline__ CD ld_pr(const double* base, int e, int, CD*) {
    const double2 v = *reinterpret_cast<const double2*>(base + 2 * e);
    return {v.x, v.y};
}
__device__ __forceinline__ CDD ld_pr(const double* base, int e, int P, CDD*) {
    const double2 h = *reinterpret_cast<const double2*>(base + 2 * e);
    const double2 l = *reinterpret_cast<const double2*>(base + 2 * P + 2 * e);
    return {h.x, l.x, h.y, l.y};
}
__device__ __forceinline__ void st_pr(double* base, int e, int, const CD& v) {
    *reinterpret_cast<double2*>(base + 2 * e) = make_double2(v.re, v.im);
}
__device__ __forceinline__ void st_pr(double* base, int e, int P, const CDD& v) {
    *reinterpret_cast<double2*>(base + 2 * e) = make_double2(v.rh, v.ih);
    *reinterpret_cast<double2*>(base + 2 * P + 2 * e) = make_double2(v.rl, v.il);
}

constexpr int kRef = 0;
constexpr int kFast = 1;

// RAG: ragged system: row p owns terms [row_off[p], row_off[p+1])
// and stage-3 chunks [row_chunk[p], row_chunk[p+1]); term s has term_k[s] <= k variables (k = the
// maximum). Per term the reference's stage-1/2 sequence for its own k_s; the value coefficient and
// value staging slot sit at block k (the uniform layout's block k), derivative j at block j.
template <class T, int ORDER, bool GSCR, bool RAG>
__global__ void __launch_bounds__(256) eval_kernel(DevSystem S, const double* __restrict__ pts,
                                                   double* __restrict__ out, long long B, int TP,
                                                   double* __restrict__ gscratch, int* __restrict__ flag) {
    using O = Sc<T>;
    constexpr int W = O::W;
    extern __shared__ __align__(16) double smem_[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = S.n, m = S.m, d = S.d;
    const int kv = S.k;  // value block / staging row (the maximum k of a ragged system)
    auto LD = [](const double* base, int e, int P) -> T { return ld_pr(base, e, P, static_cast<T*>(nullptr)); };
    const int D1 = d > 2 ? d - 1 : 1;  // stored powers e = 1..D1
    const int tabPt = D1 * W * n;      // doubles per point
    const int stgW = (kv + 1) * W * 32;  // staging doubles per warp
    const int accW = (n + 1) * W;      // accumulator doubles per warp
    double* base = GSCR ? gscratch + (size_t)blockIdx.x * (TP * tabPt + nw * (stgW + accW)) : smem_;
    double* tab = base;
    double* stg = base + TP * tabPt + warp * (stgW + accW);
    double* acc = stg + stgW;
    const long long ntiles = (B + TP - 1) / TP;
    const long long nout = (long long)n * n + n;
    const int nm = S.nm;

    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long b0 = tile * TP;
        const int tp = (int)min((long long)TP, B - b0);
        // coordinates of the tile's points -> power plane e = 1 (coalesced AoS reads)
        for (int i = threadIdx.x; i < tp * n; i += blockDim.x) {
            const int t = i / n, v = i - t * n;
            T x = O::ld_aos(pts + ((b0 + t) * n + v) * W);
            if (!O::finite(x)) atomicOr(flag, 1);
            st_pr(tab + t * tabPt, v, n, x);
        }
        __syncthreads();
        if (d > 2) {  // power chains, ref kernels.cpp:16-24: row[e] = row[e-1] * x
            for (int i = threadIdx.x; i < tp * n; i += blockDim.x) {
                const int t = i / n, v = i - t * n;
                double* pb = tab + t * tabPt;
                const T x = LD(pb, v, n);
                T r = x;
                for (int e = 2; e < d; ++e) {
                    r = O::mul(r, x);
                    st_pr(pb + (e - 1) * W * n, v, n, r);
                }
            }
            __syncthreads();
        }

        for (int task = warp; task < tp * n; task += nw) {
            const int p = task / tp, t = task - p * tp;
            const double* xt = tab + t * tabPt;
            double* orow = out + ((b0 + t) * nout) * W;
            T vacc = O::zero();
            // row p: its terms [s0, s0 + mrow) and stage-3 chunks [cb, cb + nch)
            const int s0 = RAG ? __ldg(S.row_off + p) : p * m;
            const int mrow = RAG ? __ldg(S.row_off + p + 1) - s0 : m;
            const int cb = RAG ? __ldg(S.row_chunk + p) : p * S.chunks;
            const int nch = RAG ? __ldg(S.row_chunk + p + 1) - cb : S.chunks;
            for (int c = 0; c < nch; ++c) {
                const int g = c * 32 + lane;
                T valterm = O::zero();
                if (g < mrow) {
                    const int s = s0 + g;
                    const int k = RAG ? int(__ldg(S.term_k + s)) : S.k;  // this term's variables
                    const uint16_t* pe = S.posexp + (size_t)s * S.kp;
                    const uint32_t* pe32 = S.posexp32 + (size_t)s * S.kp;
                    const bool wide = S.posexp32 != nullptr;  // uniform across the grid
                    const double* cf = S.coef + s;
                    auto POS = [&](int j) -> int { return wide ? int(__ldg(pe32 + j) & 0xffffu) : (__ldg(pe + j) & 255); };
                    auto EXP = [&](int j) -> int { return wide ? int(__ldg(pe32 + j) >> 16) : (__ldg(pe + j) >> 8); };
                    auto X = [&](int j) -> T { return LD(xt, POS(j), n); };
                    auto PW = [&](int j) -> T {
                        const int e = EXP(j);
                        if (e == 0) return O::one();
                        return LD(xt + (e - 1) * W * n, POS(j), n);
                    };
                    auto COEF = [&](int j) -> T {
                        const double* q = cf + (size_t)j * W * nm;
                        T r;
                        if constexpr (W == 2) {
                            r = T{__ldg(q), __ldg(q + nm)};
                        } else {
                            r = T{__ldg(q), __ldg(q + nm), __ldg(q + 2 * nm), __ldg(q + 3 * nm)};
                        }
                        return r;
                    };
                    auto SLOT = [&](int j) -> double* { return stg + j * W * 32; };  // slot j of this lane: element lane

                    // stage 1: common factor, ref kernels.cpp:45-53
                    T f = PW(0);
                    for (int j = 1; j < k; ++j) f = O::mul(f, PW(j));

                    // stage 2: ref kernels.cpp:55-127 (operation and operand order kept)
                    if (k == 1) {
                        T L0 = O::mul(O::one(), f);
                        T val = O::mul(L0, X(0));
                        st_pr(SLOT(0), lane, 32, O::mul(L0, COEF(0)));
                        valterm = O::mul(val, COEF(kv));
                    } else if (k == 2) {
                        const T v0 = X(0), v1 = X(1);
                        T L0 = O::mul(v1, f), L1 = O::mul(v0, f);
                        T val = O::mul(L1, v1);
                        st_pr(SLOT(0), lane, 32, O::mul(L0, COEF(0)));
                        st_pr(SLOT(1), lane, 32, O::mul(L1, COEF(1)));
                        valterm = O::mul(val, COEF(kv));
                    } else {
                        // forward products L[1] = v0, L[r+2] = L[r+1] * v[r+1]
                        T F = X(0);
                        st_pr(SLOT(1), lane, 32, F);
                        for (int r = 0; r + 2 <= k - 1; ++r) {
                            F = O::mul(F, X(r + 1));
                            if (r + 2 < k - 1) st_pr(SLOT(r + 2), lane, 32, F);
                        }
                        // F == L[k-1]; backward running product q
                        const T vlast = X(k - 1);
                        T q = vlast;
                        {
                            T L = O::mul(LD(SLOT(k - 2), lane, 32), q);
                            L = O::mul(L, f);
                            st_pr(SLOT(k - 2), lane, 32, O::mul(L, COEF(k - 2)));
                        }
                        for (int r = 1; r <= k - 3; ++r) {
                            q = O::mul(q, X(k - 1 - r));
                            T L = O::mul(LD(SLOT(k - 2 - r), lane, 32), q);
                            L = O::mul(L, f);
                            st_pr(SLOT(k - 2 - r), lane, 32, O::mul(L, COEF(k - 2 - r)));
                        }
                        q = O::mul(q, X(1));
                        {
                            T L = O::mul(q, f);
                            st_pr(SLOT(0), lane, 32, O::mul(L, COEF(0)));
                        }
                        T Lk1 = O::mul(F, f);
                        T val = O::mul(Lk1, vlast);
                        st_pr(SLOT(k - 1), lane, 32, O::mul(Lk1, COEF(k - 1)));
                        valterm = O::mul(val, COEF(kv));
                    }
                    if (ORDER == kRef) st_pr(SLOT(kv), lane, 32, valterm);
                }
                __syncwarp();
                // stage 3 (Jacobian): ascending-g ordered gather over the (row, column) map
                const bool last = c + 1 == nch;
                for (int v = lane; v < n; v += 32) {
                    const int li = (cb + c) * n + v;
                    const int e0 = __ldg(S.gm_off + li), e1 = __ldg(S.gm_off + li + 1);
                    T a = c == 0 ? O::zero() : LD(acc, v, n + 1);
                    for (int e = e0; e < e1; ++e) {
                        const int ent = __ldg(S.gm_ent + e);
                        a = O::add(a, LD(stg + (ent >> 5) * W * 32, ent & 31, 32));
                    }
                    if (last)
                        O::st_aos(orow + ((size_t)n + (size_t)p * n + v) * W, a);
                    else
                        st_pr(acc, v, n + 1, a);
                }
                // stage 3 (value)
                if (ORDER == kRef) {
                    if (lane == 0) {
                        const int gl = min(32, mrow - c * 32);
                        for (int gg = 0; gg < gl; ++gg) vacc = O::add(vacc, LD(stg + kv * W * 32, gg, 32));
                    }
                } else {
                    T r = valterm;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) r = O::add(r, O::shfl_xor(r, off));
                    vacc = c == 0 ? r : O::add(vacc, r);
                }
                if (last && lane == 0) O::st_aos(orow + (size_t)p * W, vacc);
                __syncwarp();
            }
        }
        __syncthreads();
    }
}

template <class T, int ORDER, bool GSCR, bool RAG>
static cudaError_t launch_one(const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                              cudaStream_t st) {
    auto kern = eval_kernel<T, ORDER, GSCR, RAG>;
    if (!GSCR && L.smem_bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern));
        if (e != cudaSuccess) return e;
    }
    kern<<<L.blocks, L.threads, GSCR ? 0 : L.smem_bytes, st>>>(S, pts, out, B, L.tp, L.gscratch, L.flag);
    return cudaGetLastError();
}

template <class T, int ORDER>
static cudaError_t launch_to(const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                             cudaStream_t st) {
    const bool g = L.gscratch != nullptr, r = S.row_off != nullptr;
    if (r) return g ? launch_one<T, ORDER, true, true>(L, S, pts, out, B, st) : launch_one<T, ORDER, false, true>(L, S, pts, out, B, st);
    return g ? launch_one<T, ORDER, true, false>(L, S, pts, out, B, st) : launch_one<T, ORDER, false, false>(L, S, pts, out, B, st);
}

cudaError_t launch_eval(int prec, int order, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out,
                        long long B, cudaStream_t st) {
    if (prec == 1) return order == kRef ? launch_to<CD, kRef>(L, S, pts, out, B, st) : launch_to<CD, kFast>(L, S, pts, out, B, st);
    return order == kRef ? launch_to<CDD, kRef>(L, S, pts, out, B, st) : launch_to<CDD, kFast>(L, S, pts, out, B, st);
}

template <class T, int ORDER, bool RAG>
static int occ_one(int threads, size_t smem) {
    int nb = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_kernel<T, ORDER, false, RAG>, threads, smem) == cudaSuccess ? nb : 0;
}

int max_blocks_per_sm(int prec, int order, int threads, size_t smem, bool ragged) {
    if (ragged) {
        if (prec == 1) return order == kRef ? occ_one<CD, kRef, true>(threads, smem) : occ_one<CD, kFast, true>(threads, smem);
        return order == kRef ? occ_one<CDD, kRef, true>(threads, smem) : occ_one<CDD, kFast, true>(threads, smem);
    }
    if (prec == 1) return order == kRef ? occ_one<CD, kRef, false>(threads, smem) : occ_one<CD, kFast, false>(threads, smem);
    return order == kRef ? occ_one<CDD, kRef, false>(threads, smem) : occ_one<CDD, kFast, false>(threads, smem);
}

int dyn_smem_limit(const void* f) {
    int dev = 0, v = 48 * 1024;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, f) == cudaSuccess) v -= int(fa.sharedSizeBytes);
    return v;
}

// Finiteness check of a point batch (pj_evaluate with PJ_VALIDATE, pj_newton_host): grid-stride
// 16-byte loads, one atomic per warp that saw a non-finite word. HBM-bound (one read of the
// points); the evaluation kernels keep their own flag for the asynchronous path.
__global__ void check_finite_kernel(const double2* __restrict__ p, long long count2, int* __restrict__ flag) {
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count2; i += (long long)gridDim.x * blockDim.x) {
        const double2 v = __ldg(p + i);
        bad |= !isfinite(v.x) || !isfinite(v.y);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t launch_check_finite(const double* pts, long long doubles, int* flag, int sms, cudaStream_t st) {
    const long long c2 = doubles / 2;  // W is 2 or 4: always an even number of doubles
    if (c2 <= 0) return cudaSuccess;
    const long long want = (c2 + 255) / 256;
    const int blocks = (int)(want < (long long)sms * 8 ? want : (long long)sms * 8);
    check_finite_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(pts), c2, flag);
    return cudaGetLastError();
}

// Prime the dynamic-smem attribute so the occupancy query sees the opt-in limit.
template <class T, int ORDER>
static cudaError_t set_attr_pair(int b) {
    cudaError_t e = cudaFuncSetAttribute(eval_kernel<T, ORDER, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e) return e;
    return cudaFuncSetAttribute(eval_kernel<T, ORDER, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}
cudaError_t set_smem_attr(size_t bytes) {
    const int b = (int)bytes;
    cudaError_t e;
    if ((e = set_attr_pair<CD, kRef>(b)) || (e = set_attr_pair<CD, kFast>(b)) || (e = set_attr_pair<CDD, kRef>(b))) return e;
    return set_attr_pair<CDD, kFast>(b);
}

}  // namespace pjb
