// Fast complex double-double kernel (default PJ_PREC_DD order), specialised on the number of
// variables per monomial K and on P points per lane.
//
// Same mapping as eval_kernels.cu (CTA = tile of points, warp = (row p, points) task, lane =
// monomial, on-chip ordered stage-3 gather), plus:
//   * K is a template parameter: every chain is unrolled, so the common-factor chain and the
//     forward-product chain interleave in program order (in-order issue sees two independent
//     dependency chains per point), and a monomial's K fused position/exponent words arrive in
//     one 16-byte load;
//   * coefficient planes tiled per (row, 32-monomial chunk) with the lane index fastest, and
//     the point tables with a compile-time plane stride: every load of a (j, component) pair
//     is one base register + an immediate offset;
//   * products inside a chain alternate between renormalised and unrenormalised (see cmul_n);
//   * stage 3 runs a balanced segmented reduction over a precomputed (row, chunk) schedule:
//     every lane sums k+1 consecutive terms of the output-major list, then each output adds
//     its few segment partials;
//   * the division form (points whose coordinates all lie in [2^-16, 2^16], checked per task):
//     V = prod x_j^a_j from the power table, value c*V, derivative j = a_j * (c*V) * (1/x_j) with
//     1/x in the table — 2k complex products per monomial; other points take the chains below;
//   * "back-fused" Speelpenning order: the common factor seeds the backward running product,
//     q = f, L'_j = F_j * q, q *= v_j — all k factor-scaled derivatives in 3k-4 complex
//     products instead of the reference's (3k-6) + k (ref src/kernels.cpp:55-110). Per monomial
//     5k-3 complex products instead of 6k-5 (37 vs 43 at k = 8). The value is L'_{k-1} * v_{k-1}
//     as in the reference (kernels.cpp:112).
// Results differ from the reference order only by rounding; the contract is
// |got - want| <= 1e-30 * sum|terms|, checked in tests/test_gpu_parity.py.
#include <cuda_runtime.h>

#include <cstdint>

#include "dd.cuh"
#include "eval_kernels.h"
#include "fast_common.cuh"

namespace pjb {


// NS: compile-time plane stride of the shared-memory point tables (>= n), so that the four
// component loads of a gather share one address register (immediate offsets).
#ifndef PJB_D2_SUFFIX
#define PJB_D2_SUFFIX 1
#endif
#ifndef PJB_FAST_DIV
#define PJB_FAST_DIV 1
#endif
// Register budget: 3 CTAs x 256 threads (<= 85 registers) for k <= 12, where the per-warp
// staging also fits three CTAs; 2 CTAs (<= 128 registers) above. Measured with tools/tune.py:
// k = 8: 0.853 (3 CTAs) vs 0.843 (2 CTAs); k = 16: 0.763 (2 CTAs) vs 0.723 (3 CTAs).
// k > 12: CTAs of up to 16 warps (one per SM when the staging of 8+ warps fills shared memory);
// (512, 1) keeps the 128-register budget of (256, 2).
template <int K>
constexpr int fast_min_blocks() { return K <= 12 ? 3 : 1; }  // re-measured r01z: (256, 2) -3.5%, (256, 4) -1.3%
template <int K>
constexpr int fast_max_threads() { return K <= 12 ? 256 : 512; }

template <int K, int NS, bool D2>
__global__ void __launch_bounds__(fast_max_threads<K>(), fast_min_blocks<K>()) fast_kernel(DevSystem S, const double* __restrict__ pts,
                                                   double* __restrict__ out, long long B, int TP,
                                                   int* __restrict__ flag, int SP) {
    constexpr int W = 4;
    constexpr int R = K + 1;                 // stage-3 schedule entries per lane
    constexpr int stgW = (K + 1) * W * 32;   // staging doubles per warp
    extern __shared__ __align__(16) double smem_[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = S.n, m = S.m, d = S.d, C = S.chunks;
    const int TR = fast_tab_rows(d), dm = TR - 1;  // rows x^1..x^dm, then 1/x (row dm)
    const int tabPt = TR * W * NS;
    const int accW = C > 1 ? (n + 1) * W : 0;
    double* tab = smem_;
    double* stg = smem_ + TP * tabPt + warp * (stgW + accW);
    double* acc = stg + stgW;
    const long long ntiles = (B + TP - 1) / TP;
    const long long nout = (long long)n * n + n;
    const CDD one = {1.0, 0.0, 0.0, 0.0};
    const CDD zero = {0.0, 0.0, 0.0, 0.0};

    // SP CTAs share each tile (SP > 1 only for batches with fewer tiles than CTAs; the host makes
    // the grid a multiple of SP): CTA blockIdx takes part blockIdx mod SP of the tile's tasks,
    // warp + part*nw with step SP*nw, so a single point's 32 rows still spread over the SM array
    for (long long tile = blockIdx.x / SP; tile < ntiles; tile += gridDim.x / SP) {
        const long long b0 = tile * TP;
        const int tp = (int)min((long long)TP, B - b0);
        // point tables: x, the power chains x^e (ref kernels.cpp:16-24, normalised products) up to
        // x^dm, and 1/x (the division form's; div_form_ok picks the form per point)
        for (int i = threadIdx.x; i < tp * n; i += blockDim.x) {
            const int t = i / n, v = i - t * n;
            const CDD x = ld_aos(pts + ((b0 + t) * n + v) * W);
            if (!fin(x)) atomicOr(flag, 1);
            double* pb = tab + t * tabPt + 2 * v;
            st_hl(pb, 2 * NS, x);
            CDD r = x;
            for (int e = 2; e <= dm; ++e) {
                r = cdd_mul(r, x);
                st_hl(pb + (e - 1) * W * NS, 2 * NS, r);
            }
#if PJB_FAST_DIV
            st_hl(pb + dm * W * NS, 2 * NS, cdd_inv(x));
#endif
        }
        __syncthreads();
#ifdef PJB_STAGGER
        if (warp & 1) __nanosleep(PJB_STAGGER);  // experiment: desynchronise the CTA's warps
#endif
        for (int task = warp + (int)(blockIdx.x % SP) * nw; task < tp * n; task += nw * SP) {
            const int p = task / tp, t = task - p * tp;
            const double* xt = tab + t * tabPt;
            const bool divf = PJB_FAST_DIV && div_form_ok(xt, n, lane);  // warp-uniform
            for (int c = 0; c < C; ++c) {
                const int graw = c * 32 + lane;
                const int g = graw < m ? graw : m - 1;  // inactive lanes shadow a real monomial
                const int s = p * m + g;
                // fused position/exponent words, kept packed (K/2 registers) and decoded on use:
                // the exponents are needed again at the end of the backward chain
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
                // prefetch the stage-3 schedule of this (row, chunk) into registers now, so its L2
                // latency hides behind stage 2 (in-order issue would otherwise stall on it)
                const size_t pc = (size_t)(p * C + c);
                uint32_t codes[R];
                {
                    const uint32_t* sc = S.sch + pc * R * 32 + lane;
#pragma unroll
                    for (int r = 0; r < R; ++r) codes[r] = __ldg(sc + r * 32);
                }
                const uint4 sq0 = __ldg(S.segq + pc * ((n + 64) >> 6) * 32 + lane);
                // the monomial's coefficient c (lane-minor tile of this (row, chunk))
                const double* cf = S.coefT + pc * W * 32 + lane;
                // power-rule scaling a_j * x: d <= 2 means a_j in {1, 2}, an exact scaling of every
                // word; otherwise TwoProd of the high word by the small integer, low word folded in
                auto SCALE = [&](int j, const CDD& x) -> CDD {
                    if constexpr (D2) {
                        const double a = EX1(j) ? 2.0 : 1.0;
                        return {__dmul_rn(x.rh, a), __dmul_rn(x.rl, a), __dmul_rn(x.ih, a), __dmul_rn(x.il, a)};
                    } else {
                        const double a = (double)(EX1(j) + 1);
                        const double pr = __dmul_rn(x.rh, a), pi = __dmul_rn(x.ih, a);
                        return {pr, __fma_rn(x.rl, a, __fma_rn(x.rh, a, -pr)), pi,
                                __fma_rn(x.il, a, __fma_rn(x.ih, a, -pi))};
                    }
                };
                auto X = [&](int j) -> CDD { return ld_hl(xt + 2 * POS(j), 2 * NS); };
                // x^(a_j - 1): branch-free. d <= 2 (D2): select between 1 and the gathered x;
                // otherwise a table load (row max(a_j - 2, 0)) and a select for a_j == 1
                auto PWsel = [&](int j, const CDD& v) -> CDD {
                    if constexpr (D2) {
                        return sel_cdd(EX1(j) != 0, v, one);
                    } else {
                        const int e1 = EX1(j);
                        const int e = e1 > 0 ? e1 - 1 : 0;
                        return sel_cdd(e1 != 0, ld_hl(xt + e * W * NS + 2 * POS(j), 2 * NS), one);
                    }
                };
                auto SLOT = [&](int j) -> double* { return stg + j * W * 32 + 2 * lane; };

                if (divf) {
                // ---- stages 1-2, division form: V = prod_j x_j^a_j (table rows, one chain of
                // k-1 products), value c*V, derivative j = a_j * (c*V) * (1/x_j) — the same
                // quantity as c * a_j * x_j^(a_j-1) * prod_{l != j} x_l^a_l, in 2k complex products
                // instead of 3k-2 (d <= 2) or 4k-3; the k closing products are independent.
                // Chain states as elsewhere: a product renormalises iff its input is not normalised.
                auto YP = [&](int j) -> CDD { return ld_hl(xt + EX1(j) * W * NS + 2 * POS(j), 2 * NS); };
                auto IV = [&](int j) -> CDD { return ld_hl(xt + dm * W * NS + 2 * POS(j), 2 * NS); };
                CDD V = YP(0);
#pragma unroll
                for (int j = 1; j < K; ++j) V = cmul_n((j & 1) == 0, V, YP(j));
                const CDD cval = {__ldg(cf), __ldg(cf + 32), __ldg(cf + 64), __ldg(cf + 96)};
                const CDD cV = cdd_mul(V, cval);
                st_hl(SLOT(K), 64, cV);
#pragma unroll
                for (int j = 0; j < K; ++j) st_hl(SLOT(j), 64, SCALE(j, cdd_mul_u(cV, IV(j))));
                } else {
#if PJB_D2_SUFFIX
                if constexpr (D2) {
                // ---- stage 1 (d <= 2): suffix products B_j = v_{j+1}...v_{k-1}, staged in slot j.
                // The host orders each monomial's variables with the a_j = 2 ones last
                // (order_variables), so the common factor f = prod over a_j = 2 of x_j is the suffix
                // product B_{k-1-c_g} (c_g = the number of a_j = 2): no separate factor chain —
                // 3k-2 complex products per monomial instead of 4k-3 (22 vs 29 at k = 8).
                // Chain states are compile-time: B_j is normalised iff k-2-j is even.
                int cg = 0;
#pragma unroll
                for (int j = 0; j < K; ++j) cg += EX1(j) & 1;
                // (registers are tight at 3 CTAs/SM: x values and B_0 are re-gathered from shared
                // memory at their second use rather than kept live)
                st_hl(SLOT(K - 1), 64, one);  // B_{k-1} = 1: f for c_g = 0
                CDD B0 = X(K - 1);
                st_hl(SLOT(K - 2), 64, B0);
#pragma unroll
                for (int j = K - 3; j >= 0; --j) {
                    B0 = cmul_n(((K - 3 - j) & 1) != 0, B0, X(j + 1));
                    st_hl(SLOT(j), 64, B0);
                }
                CDD f = ld_hl(SLOT(max(K - 1 - cg, 0)), 64);
                if (__any_sync(0xffffffffu, cg == K)) {  // every exponent 2: f = B_0 * v_0
                    const CDD fa = cdd_mul(B0, X(0));
                    if (cg == K) f = fa;
                }
                // ---- stage 2 (d <= 2): prefix chain seeded with the coefficient and the factor,
                // F'_0 = f*c, F'_{j+1} = F'_j * v_j; every derivative L'_j = F'_j * B_j (slot j)
                // carries c and f; power rule a_j * L'_j exact; value F'_{k-1} * v_{k-1}
                // (ref kernels.cpp:108-118 order: value after the factor). F'_j normalised iff j even.
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
                } else {
#endif
                // ---- stage 1 + forward products (interleaved chains); chain states are
                // compile-time after unrolling: F_j is normalised iff j is odd, f_j iff j is even;
                // a product renormalises iff its chain input is not normalised
                CDD Fc, f, vlast;
                {
                    const CDD v0 = X(0);
                    f = PWsel(0, v0);
                    Fc = v0;
                    st_hl(SLOT(1), 64, v0);
                }
#pragma unroll
                for (int j = 1; j < K; ++j) {
                    const CDD v = X(j);
                    f = cmul_n((j & 1) == 0, f, PWsel(j, v));
                    if (j < K - 1) {
                        Fc = cmul_n((j & 1) == 0, Fc, v);
                        if (j + 1 < K - 1) st_hl(SLOT(j + 1), 64, Fc);
                    } else {
                        vlast = v;
                    }
                }
                // ---- stage 2, back-fused and coefficient-seeded: q = f * c; L'_j = F_j * q;
                // q *= v_j. Every staged derivative then already carries c, and the power rule
                // is the cheap exact scaling a_j * L'_j (ref kernels.cpp:108-118 multiplies by the
                // pre-scaled a_j * c instead: k + 1 complex products, here 1 product + k scalings)
                constexpr bool f_norm = ((K - 1) & 1) == 0;
                CDD q;
                {
                    const CDD cval = {__ldg(cf), __ldg(cf + 32), __ldg(cf + 64), __ldg(cf + 96)};
                    const CDD q0 = cmul_n(!f_norm, f, cval);  // normalised iff f was not
                    const CDD L = cdd_mul_u(Fc, q0);
                    st_hl(SLOT(K - 1), 64, SCALE(K - 1, L));
                    st_hl(SLOT(K), 64, cdd_mul(L, vlast));
                    q = cmul_n(f_norm, q0, vlast);
                }
#pragma unroll
                for (int j = K - 2; j >= 1; --j) {
                    const bool q_norm = (((K - 2 - j) & 1) == 0) ? f_norm : !f_norm;  // state of q here
                    const CDD L = cdd_mul_u(ld_hl(SLOT(j), 64), q);
                    st_hl(SLOT(j), 64, SCALE(j, L));
                    q = cmul_n(!q_norm, q, X(j));
                }
                st_hl(SLOT(0), 64, SCALE(0, q));
#if PJB_D2_SUFFIX
                }
#endif
                }  // divf
                __syncwarp();
                // ---- stage 3, phase 1: balanced segmented sums. The (row, chunk) schedule
                // hands every lane R consecutive entries of the output-major, ascending-g list
                // of staged terms; a lane flushes its running sum at segment ends. The running
                // sum defers renormalisation: TwoSum of the high words, low words and the TwoSum
                // error accumulated (8 DADD per component instead of 11, and the high-word chain
                // is one dependent add per term); the partial is renormalised by the phase-2 add.
                // Error <= ~(c^3/6 + 3c) u^2 * sum|terms| for a segment of c <= k+1 terms.
                {
                    double sr = 0.0, lr = 0.0, si = 0.0, li = 0.0;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const uint32_t code = codes[r];
                        if (code & kSchValid) {
                            double* sl = stg + 2 * (code & 0x1fff);  // code: 16-byte unit
                            const CDD tv = ld_hl(sl, 64);
                            const DD a = two_sum(sr, tv.rh), b = two_sum(si, tv.ih);
                            sr = a.hi;
                            si = b.hi;
                            lr = __dadd_rn(lr, __dadd_rn(tv.rl, a.lo));
                            li = __dadd_rn(li, __dadd_rn(tv.il, b.lo));
                            if (code & kSchFlush) {
                                // the partial overwrites the staging slot this lane just consumed
                                // (each slot is read exactly once, by this lane): no extra smem
                                st_hl(sl, 64, CDD{sr, lr, si, li});
                                sr = lr = si = li = 0.0;
                            }
                        }
                    }
                }
                __syncwarp();
                // ---- stage 3, phase 2: every output adds its (few) segment partials in order.
                // Pass k2 covers outputs [64*k2, 64*k2 + 64): lane l owns o1 = 64*k2 + l and at
                // most one secondary output o2 from the upper half, paired by the host with a
                // lightly loaded lane (the lane's record lists o1's segment codes, then o2's);
                // n = 32: 33 outputs in one pass, the value keeps lane 0 to itself
                const bool last = c + 1 == C;
                auto INIT = [&](int o) -> CDD { return c == 0 ? zero : ld_hl(acc + 2 * o, 2 * (n + 1)); };
                // (k > 12: the point's output row and the row's Jacobian base hoisted out of the
                // stores — measured +1% at C3; the k <= 12 kernels keep the inline form, which
                // their register schedule prefers: -2% at C2 otherwise)
                double* const orow = out + (b0 + t) * nout * W;
                const int jb = n + p * n - 1;
                auto FIN = [&](int o, const CDD& v) {
                    if (last) {
                        if constexpr (K > 12) {
                            st_aos(orow + (o == 0 ? p : jb + o) * W, cdd_renorm(v));
                        } else if (t < tp) {
                            const long long at = o == 0 ? p : n + (long long)p * n + (o - 1);
                            st_aos(out + ((b0 + t) * nout + at) * W, cdd_renorm(v));
                        }
                    } else {
                        st_hl(acc + 2 * o, 2 * (n + 1), v);
                    }
                };
                const int npass = (n + 64) >> 6;
                for (int k2 = 0; k2 < npass; ++k2) {
                    const size_t rec = (pc * npass + k2) * 32 + lane;
                    const uint4 sq = k2 == 0 ? sq0 : __ldg(S.segq + rec);
                    const int o1 = 64 * k2 + lane, o2 = sq.x >> 16;
                    const int cnt1 = sq.x & 0xff, tot = cnt1 + ((sq.x >> 8) & 0xff);
                    const bool has1 = o1 <= n, has2 = o2 != 0xffff;
                    const uint32_t pk[3] = {sq.y, sq.z, sq.w};
                    const uint16_t* xs = tot > 6 ? S.segcode + __ldg(S.seg + rec) : nullptr;
                    auto CODE = [&](int qq) -> int {  // qq-th code of the lane's list (dynamic qq)
                        if (qq >= 6) return __ldg(xs + qq);
                        const uint32_t w = qq < 2 ? pk[0] : qq < 4 ? pk[1] : pk[2];
                        return (w >> (16 * (qq & 1))) & 0xffff;
                    };
                    auto LDE = [&](int e) -> CDD { return ld_hl(stg + 2 * e, 64); };  // e: 16-byte unit
                    CDD r = has1 ? INIT(o1) : zero;
#pragma unroll
                    for (int qq = 0; qq < 6; ++qq) {
                        if (qq < cnt1) {
                            const CDD sv = LDE((pk[qq >> 1] >> (16 * (qq & 1))) & 0xffff);
                            r = qq == 0 && c == 0 ? sv : cdd_add(r, sv);
                        }
                    }
                    for (int qq = 6; qq < cnt1; ++qq) r = cdd_add(r, LDE(CODE(qq)));  // rare
                    if (has1) FIN(o1, r);
                    if (has2) {  // the lane's secondary output (few lanes)
                        CDD r2;
                        if (tot == cnt1 + 1 && c == 0) {  // one segment (the host places it so)
                            r2 = LDE(CODE(cnt1));
                        } else {
                            r2 = INIT(o2);
                            for (int qq = cnt1; qq < tot; ++qq) {
                                const CDD sv = LDE(CODE(qq));
                                r2 = qq == cnt1 && c == 0 ? sv : cdd_add(r2, sv);
                            }
                        }
                        FIN(o2, r2);
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------- dispatch
namespace {

template <int K, int NS, bool D2>
cudaError_t launch_t(const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                     cudaStream_t st) {
    auto kern = fast_kernel<K, NS, D2>;
    if (L.smem_bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern));
        if (e != cudaSuccess) return e;
    }
    kern<<<L.blocks, L.threads, L.smem_bytes, st>>>(S, pts, out, B, L.tp, L.flag, L.splits);
    return cudaGetLastError();
}

template <int K, int NS, bool D2>
int occ_t(int threads, size_t smem) {
    auto kern = fast_kernel<K, NS, D2>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit((const void*)kern)))
        return 0;
    int nb = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) == cudaSuccess ? nb : 0;
}

template <int K, bool D2>
cudaError_t launch_kd(int ns, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                      cudaStream_t st) {
    if (ns == 32) return launch_t<K, 32, D2>(L, S, pts, out, B, st);
    if (ns == 64) return launch_t<K, 64, D2>(L, S, pts, out, B, st);
    return launch_t<K, 256, D2>(L, S, pts, out, B, st);
}
template <int K>
cudaError_t launch_k(int ns, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                     cudaStream_t st) {
    return S.d <= 2 ? launch_kd<K, true>(ns, L, S, pts, out, B, st) : launch_kd<K, false>(ns, L, S, pts, out, B, st);
}
template <int K, bool D2>
int occ_kd(int ns, int threads, size_t smem) {
    if (ns == 32) return occ_t<K, 32, D2>(threads, smem);
    if (ns == 64) return occ_t<K, 64, D2>(threads, smem);
    return occ_t<K, 256, D2>(threads, smem);
}
template <int K>
int occ_k(int ns, int d, int threads, size_t smem) {
    return d <= 2 ? occ_kd<K, true>(ns, threads, smem) : occ_kd<K, false>(ns, threads, smem);
}

}  // namespace

#ifndef PJB_FAST_KS
#define PJB_FAST_KS(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
#endif

bool fast_supported(int k) {
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return true;
        PJB_FAST_KS(PJB_CASE)
#undef PJB_CASE
        default: return false;
    }
}

int fast_plane_stride(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : 256; }

cudaError_t launch_fast(int k, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                        cudaStream_t st) {
    const int ns = fast_plane_stride(S.n);
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return launch_k<KK>(ns, L, S, pts, out, B, st);
        PJB_FAST_KS(PJB_CASE)
#undef PJB_CASE
        default: return cudaErrorInvalidValue;
    }
}

int fast_blocks_per_sm(int k, int n, int d, int threads, size_t smem) {
    const int ns = fast_plane_stride(n);
    switch (k) {
#define PJB_CASE(KK) \
    case KK: return occ_k<KK>(ns, d, threads, smem);
        PJB_FAST_KS(PJB_CASE)
#undef PJB_CASE
        default: return 0;
    }
}

}  // namespace pjb
