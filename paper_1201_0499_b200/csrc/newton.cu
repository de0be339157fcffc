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
// Operation order (T = complex double or complex double-double); pivoting is implicit (rows are
// never moved, the pivot sequence is recorded), the arithmetic is that of the row-swapping form:
//   rhs_i = y_i + (−f_i)                          (−f_i when y is absent)
//   active rows: all; for kk = 0..n−1:
//     piv_kk = the active row maximising |Re_hi A[i][kk]| + |Im_hi A[i][kk]| (ties: the smallest
//              row index; the maximum must be > 0, else the point is singular: status 1, x_new = x)
//     inv_kk = 1 / A[piv_kk][kk]                   (conj(a) / |a|², nt_inv below); piv_kk leaves
//              the active set
//     l_i = A[i][kk] · inv_kk                      active i (normalised product)
//     A[i][j] = A[i][j] + (−(l_i · A[piv_kk][j]))  active i, j = kk+1..n (column n = rhs; the dd
//                                                  product is left unnormalised, the addition
//                                                  renormalises)
//   for s = n−1..0:  dx_s = rhs[piv_s] · inv_s;  rhs[piv_t] = rhs[piv_t] + (−(A[piv_t][s] · dx_s)) for t < s
//   x_new_i = x_i + dx_i
//
// B200 mapping: a CTA owns one point at a time (persistent grid over the batch). The
// augmented matrix [J | rhs] lives in shared memory, n × (n+1) elements (row stride n+1) in the
// pair layout (NL below); n ≤ 64 fits (133 KB in dd), larger systems use a per-CTA global slab
// with the same code. Warp 0 runs one column ahead ("look-ahead"): during step kk it updates column
// kk+1 of the active rows (the values stay in its registers), picks piv_{kk+1} by a redux
// arg-max while every lane inverts its own candidates speculatively, broadcasts the winner's
// inverse and forms the multipliers of column kk+1 and the next active-row list — while warps 1.. update columns kk+2..n of step kk (a thread keeps one pivot-row element
// in registers and walks rows). One barrier per step. Back substitution runs in warp 0 with the
// right-hand side in registers (a lane owns rows lane + 32q) and each solved component
// broadcast by shuffle. Several CTAs per SM overlap one CTA's serial phases with the others'
// updates. The path is FP64-issue-bound like the evaluator.
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>
#include <set>

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
// |a|^2 in dd with a short dependency chain: the two squares are non-negative, so their high
// parts are summed with an exact Fast2Sum after ordering them by size (no TwoSum), and the square
// errors (x_hi^2 - p exactly, plus 2 x_hi x_lo) join the low word before one closing Fast2Sum
__device__ __forceinline__ DD nt_abs2(DD re, DD im) {
    const double p1 = __dmul_rn(re.hi, re.hi), p2 = __dmul_rn(im.hi, im.hi);
    double e1 = __fma_rn(re.hi, re.hi, -p1), e2 = __fma_rn(im.hi, im.hi, -p2);
    e1 = __fma_rn(__dadd_rn(re.hi, re.hi), re.lo, e1);
    e2 = __fma_rn(__dadd_rn(im.hi, im.hi), im.lo, e2);
    const DD s = fast_two_sum(fmax(p1, p2), fmin(p1, p2));
    return fast_two_sum(s.hi, __dadd_rn(s.lo, __dadd_rn(e1, e2)));
}
__device__ __forceinline__ CDD nt_inv(CDD a) {
    DD re{a.rh, a.rl}, im{a.ih, a.il};
    DD den = nt_abs2(re, im);
    DD r = nt_dd_rcp(den);
    DD o = nt_dd_mul(re, r), p = nt_dd_mul({-a.ih, -a.il}, r);
    return {o.hi, o.lo, p.hi, p.lo};
}

// Matrix storage ("pair" layout): element e of an array of P elements keeps (re, im) at base + 2e
// (complex double) or the high pair (re_hi, im_hi) at base + 2e and the low pair (re_lo, im_lo) at
// base + 2P + 2e (complex dd): one 16-byte access per pair.
template <class T>
struct NL;
template <>
struct NL<CD> {
    __device__ static CD ld(const double* A, int e, int) {
        const double2 v = *reinterpret_cast<const double2*>(A + 2 * e);
        return {v.x, v.y};
    }
    __device__ static void st(double* A, int e, int, const CD& v) {
        *reinterpret_cast<double2*>(A + 2 * e) = make_double2(v.re, v.im);
    }
    // offset of AoS component comp (re, im) of element e
    __device__ static int off(int e, int comp, int) { return 2 * e + comp; }
};
template <>
struct NL<CDD> {
    __device__ static CDD ld(const double* A, int e, int P) {
        const double2 h = *reinterpret_cast<const double2*>(A + 2 * e);
        const double2 l = *reinterpret_cast<const double2*>(A + 2 * P + 2 * e);
        return {h.x, l.x, h.y, l.y};
    }
    __device__ static void st(double* A, int e, int P, const CDD& v) {
        *reinterpret_cast<double2*>(A + 2 * e) = make_double2(v.rh, v.ih);
        *reinterpret_cast<double2*>(A + 2 * P + 2 * e) = make_double2(v.rl, v.il);
    }
    // offset of AoS component comp (re_hi, re_lo, im_hi, im_lo) of element e
    __device__ static int off(int e, int comp, int P) { return (comp & 1) * 2 * P + 2 * e + (comp >> 1); }
};

// dynamic shared memory ints (4 per row), rounded to whole 16-byte units, in doubles
__host__ __device__ __forceinline__ int newton_int_words(int n) { return (4 * n + 3) / 4 * 2; }

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

// ---- pieces shared by the two Newton kernels
// Load [J | y − f] of point b (all threads; role warp 0 the right-hand side, its norm, the identity
// row list). Shared-memory matrices: 8-byte cp.async copies straight into the pair layout (no
// registers, every copy in flight at once); global slabs: plain loads. The caller waits + syncs.
template <class T, bool GS = false>
__device__ __forceinline__ void nt_load(const NewtonArgs& a, long long b, double* A, int* list, int* sing,
                                        int warp) {
    using S = Sc<T>;
    constexpr int W = S::W;
    const int n = a.n, ld = n + 1, P = n * ld;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const double* ev = a.evals + size_t(b) * (size_t(n) * n + n) * W;
    if (!GS) {
        // word t = (element el = i * n + j, component t mod W); the thread's (i, j) advance by a fixed
        // stride (nt / W elements), so the loop carries no integer division (it used to dominate
        // the load phase: ~1.2k instructions per thread and point)
        const int es = nt / W, di = es / n, dj = es - di * n;
        int el = tid / W;
        const int comp = tid - el * W;
        int i = el / n, j = el - i * n;
        const double* src = ev + size_t(n) * W + tid;
#if PJB_NT_LDX == 1  // timing experiment: no matrix load at all (results wrong)
        if (0)
#elif PJB_NT_LDX == 2  // timing experiment: 16-byte copies into a wrong layout (results wrong)
        for (int t = 2 * tid; t < n * n * W; t += 2 * nt) {
            const unsigned dst = unsigned(__cvta_generic_to_shared(A + t));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(ev + size_t(n) * W + t));
        }
        if (0)
#endif
        for (int t = tid; t < n * n * W; t += nt, src += nt) {
            const unsigned dst = unsigned(__cvta_generic_to_shared(A + NL<T>::off(i * ld + j, comp, P)));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
            i += di;
            j += dj;
            if (j >= n) {
                j -= n;
                ++i;
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    } else {
        for (int t = tid; t < n * n; t += nt) {
            const int i = t / n, j = t - i * n;
            NL<T>::st(A, i * ld + j, P, S::ld_aos(ev + size_t(n + t) * W));
        }
    }
    if (warp == 0) {
        double rn = 0.0;
        for (int i = lane; i < n; i += 32) {
            T r = nt_neg(S::ld_aos(ev + size_t(i) * W));
            if (a.target) r = S::add(S::ld_aos(a.target + (size_t(b) * n + i) * W), r);
            NL<T>::st(A, i * ld + n, P, r);
            rn = fmax(rn, nt_magmax(r));
            list[i] = i;
        }
        for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
        if (lane == 0) {
            if (a.norms) a.norms[2 * b] = rn;
            *sing = 0;
        }
    }
}

// Back substitution (warp 0): rhs of physical rows lane + 32q in registers;
// dx_s = rhs[piv_s] * inv_s, then rhs[piv_t] -= A[piv_t][s] * dx_s for t < s; x_new = x + dx.
template <class T, int NQ>
__device__ __forceinline__ void nt_back_substitute(const NewtonArgs& a, long long b, const double* A,
                                                   const double* INV, double* DX, const int* s_piv,
                                                   const int* s_step, bool singular) {
    using S = Sc<T>;
    constexpr int W = S::W;
    const int n = a.n, ld = n + 1, P = n * ld, lane = threadIdx.x & 31;
    const double* x = a.points + size_t(b) * n * W;
    double* xo = a.points_out + size_t(b) * n * W;
    if (singular) {
        for (int i = lane; i < n; i += 32) S::st_aos(xo + size_t(i) * W, S::ld_aos(x + size_t(i) * W));
        if (lane == 0) {
            if (a.norms) a.norms[2 * b + 1] = INFINITY;
            if (a.status) a.status[b] = 1;
        }
        return;
    }
    T rr[NQ];
    int st[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int r = lane + 32 * q;
        rr[q] = r < n ? NL<T>::ld(A, r * ld + n, P) : S::zero();
        st[q] = r < n ? s_step[r] : -1;
    }
    for (int s = n - 1; s >= 0; --s) {
        const int pr = s_piv[s];
        const int owner = pr & 31, qi = pr >> 5;
        T xs = rr[0];
#pragma unroll
        for (int q = 1; q < NQ; ++q)
            if (q == qi) xs = rr[q];
        xs = shfl_idx(xs, owner);
        xs = S::mul(xs, NL<T>::ld(INV, s, n));
        if (lane == 0) NL<T>::st(DX, s, n, xs);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (st[q] >= 0 && st[q] < s)
                rr[q] = S::add(rr[q], nt_neg(nt_umul(NL<T>::ld(A, (lane + 32 * q) * ld + s, P), xs)));
    }
    __syncwarp();
    double dn = 0.0;
    bool fin = true;
    for (int i = lane; i < n; i += 32) {
        const T d = NL<T>::ld(DX, i, n);
        const T xn = S::add(S::ld_aos(x + size_t(i) * W), d);
        S::st_aos(xo + size_t(i) * W, xn);
        dn = fmax(dn, nt_magmax(d));
        fin = fin && nt_finite(xn);
    }
    for (int o = 16; o; o >>= 1) dn = fmax(dn, __shfl_xor_sync(0xffffffffu, dn, o));
    fin = __all_sync(0xffffffffu, fin);
    if (lane == 0) {
        if (a.norms) a.norms[2 * b + 1] = dn;
        if (a.status) a.status[b] = fin ? 0 : 2;
    }
}

// ---- mixed-precision solve (PJ_NEWTON_MIXED, complex dd input, n <= 32): the LU factorisation in
// complex double on the high words of J, then NIT steps of iterative refinement with the residual
// in complex dd. Operation order (restated by oracle/oracle.cpp: newton_one_mixed):
//   rhs = y + (-f) in dd (-f when y is absent); A = (Re hi, Im hi) of J, column n = hi words of rhs;
//   the complex-double elimination of newton_kernel<CD> on [A | rhs_hi]; dx = its back substitution
//   (in dd with zero low words); then NIT times:
//     partial residuals per row i and group g = 0..3: acc_g = sum over j = g, g+4, ... ascending of
//       cdd_mul_u(J_ij, dx_j) (cdd_add, starting from 0); r_i = rhs_i + (-((acc_0 + acc_1) + (acc_2 + acc_3)));
//     b = hi words of r; forward substitution with the stored multipliers (step order, the same
//     operations the elimination applied to the right-hand side column); back substitution with
//     the pivot inverses -> c (complex double); dx_j = dx_j + c_j (dd add, c's low words zero);
//   x_new = x + dx (dd). status 3 when the last correction is not below 2^-64 of |dx| (the
//   refinement has not converged to dd accuracy: J too ill-conditioned for the double factors).
constexpr int kMixedIters = 2;

__device__ __forceinline__ void nt_load_mixed(const NewtonArgs& a, long long b, double* A, int* list, int* sing,
                                              int warp) {
    const int n = a.n, ld = n + 1, P = n * ld;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const double* ev = a.evals + size_t(b) * (size_t(n) * n + n) * 4;
    // the high words (re_hi, im_hi) of every J element into the complex-double pair layout
    const int es = nt / 2, di = es / n, dj = es - di * n;
    int el = tid / 2;
    const int comp = tid - el * 2;
    int i = el / n, j = el - i * n;
    for (int t = tid; t < n * n * 2; t += nt) {
        const unsigned dst = unsigned(__cvta_generic_to_shared(A + NL<CD>::off(i * ld + j, comp, P)));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(ev + size_t(n) * 4 + 2 * t));
        i += di;
        j += dj;
        if (j >= n) {
            j -= n;
            ++i;
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (warp == 0) {
        double rn = 0.0;
        for (int r = lane; r < n; r += 32) {
            CDD v = nt_neg(Sc<CDD>::ld_aos(ev + size_t(r) * 4));
            if (a.target) v = cdd_add(Sc<CDD>::ld_aos(a.target + (size_t(b) * n + r) * 4), v);
            NL<CD>::st(A, r * ld + n, P, CD{v.rh, v.ih});
            rn = fmax(rn, nt_magmax(v));
            list[r] = r;
        }
        for (int o = 16; o; o >>= 1) rn = fmax(rn, __shfl_xor_sync(0xffffffffu, rn, o));
        if (lane == 0) {
            if (a.norms) a.norms[2 * b] = rn;
            *sing = 0;
        }
    }
}

// After the complex-double elimination (all threads; n <= 32, lanes = physical rows). DXD: the dd
// solution [4][n] (pair layout), PART: four dd partial residuals per row [4][4n], DXC: corrections.
__device__ __forceinline__ void nt_mixed_finish(const NewtonArgs& a, long long b, const double* A, const double* INV,
                                                double* DXD, double* PART, double* DXC, const int* s_piv,
                                                const int* s_step, bool singular, int warp, long long* phm = nullptr) {
    const int n = a.n, ld = n + 1, P = n * ld, lane = threadIdx.x & 31;
#ifdef PJB_NT_PHASES
    // developer instrumentation: phm[0..3] += initial solve, residual sums, refinement solves, update
    long long tm = clock64();
#define PJB_PHM(i)                      \
    {                                   \
        const long long t_ = clock64(); \
        phm[i] += t_ - tm;              \
        tm = t_;                        \
    }
#else
#define PJB_PHM(i)
#endif
    const double* x = a.points + size_t(b) * n * 4;
    double* xo = a.points_out + size_t(b) * n * 4;
    const double* ev = a.evals + size_t(b) * (size_t(n) * n + n) * 4;
    if (singular) {
        if (warp == 0) {
            for (int i = lane; i < n; i += 32) Sc<CDD>::st_aos(xo + size_t(i) * 4, Sc<CDD>::ld_aos(x + size_t(i) * 4));
            if (lane == 0) {
                if (a.norms) a.norms[2 * b + 1] = INFINITY;
                if (a.status) a.status[b] = 1;
            }
        }
        return;
    }
    const bool row = lane < n;
    const int st = row ? s_step[lane] : -1;  // the step this lane's physical row was pivoted at
    // complex-double triangular solves on the lane-held right-hand side b (physical rows): the
    // forward substitution repeats the elimination's updates of column n, then the back substitution
    // (each step's pivot row, inverse and matrix entry are loaded one step ahead: off the chain)
    auto back = [&](CD bb) {
        int pr = s_piv[n - 1];
        CD iv = NL<CD>::ld(INV, n - 1, n), av = row ? NL<CD>::ld(A, lane * ld + n - 1, P) : CD{0.0, 0.0};
        for (int s = n - 1; s >= 0; --s) {
            const int s1 = s > 0 ? s - 1 : 0;
            const int pr1 = s_piv[s1];
            const CD iv1 = NL<CD>::ld(INV, s1, n);
            const CD av1 = row ? NL<CD>::ld(A, lane * ld + s1, P) : CD{0.0, 0.0};
            CD xs = shfl_idx(bb, pr);
            xs = cd_mul(xs, iv);
            if (lane == 0) NL<CD>::st(DXC, s, n, xs);
            if (row && st < s) bb = cd_add(bb, nt_neg(cd_mul(av, xs)));
            pr = pr1;
            iv = iv1;
            av = av1;
        }
        __syncwarp();
    };
    double cmax = 0.0;
    CDD rhs{0.0, 0.0, 0.0, 0.0};  // warp 0: this lane's dd right-hand side, kept for the residuals
    if (warp == 0 && row) {
        rhs = nt_neg(Sc<CDD>::ld_aos(ev + size_t(lane) * 4));
        if (a.target) rhs = cdd_add(Sc<CDD>::ld_aos(a.target + (size_t(b) * n + lane) * 4), rhs);
    }
    if (warp == 0) {
        back(row ? NL<CD>::ld(A, lane * ld + n, P) : CD{0.0, 0.0});
        for (int i = lane; i < n; i += 32) {
            const CD c = NL<CD>::ld(DXC, i, n);
            NL<CDD>::st(DXD, i, n, CDD{c.re, 0.0, c.im, 0.0});
        }
    }
    PJB_PHM(0)
    for (int it = 0; it < kMixedIters; ++it) {
        __syncthreads();  // DXD complete
        // partial residual sums: warp g, lane = row i, columns j = g, g+4, ...
        if (row) {
            CDD acc{0.0, 0.0, 0.0, 0.0};
            const double* jr = ev + (size_t(n) + size_t(lane) * n) * 4;
            for (int j = warp; j < n; j += 4)
                acc = cdd_add(acc, cdd_mul_u(Sc<CDD>::ld_aos(jr + size_t(j) * 4), NL<CDD>::ld(DXD, j, n)));
            NL<CDD>::st(PART + warp * 4 * n, lane, n, acc);
        }
        __syncthreads();
        PJB_PHM(1)
        if (warp == 0) {
            CD bb{0.0, 0.0};
            CDD r{0.0, 0.0, 0.0, 0.0};
            if (row) {
                r = rhs;
                const CDD s01 = cdd_add(NL<CDD>::ld(PART, lane, n), NL<CDD>::ld(PART + 4 * n, lane, n));
                const CDD s23 = cdd_add(NL<CDD>::ld(PART + 8 * n, lane, n), NL<CDD>::ld(PART + 12 * n, lane, n));
                r = cdd_add(r, nt_neg(cdd_add(s01, s23)));
                bb = CD{r.rh, r.ih};
            }
            // forward substitution (the elimination's operations on column n, in step order)
            int pk = s_piv[0];
            CD lk = row ? NL<CD>::ld(A, lane * ld, P) : CD{0.0, 0.0};
            for (int kk = 0; kk < n; ++kk) {
                const int k1 = kk + 1 < n ? kk + 1 : kk;
                const int pk1 = s_piv[k1];
                const CD lk1 = row ? NL<CD>::ld(A, lane * ld + k1, P) : CD{0.0, 0.0};
                const CD bp = shfl_idx(bb, pk);
                if (row && st > kk) bb = cd_add(bb, nt_neg(cd_mul(lk, bp)));
                pk = pk1;
                lk = lk1;
            }
            back(bb);
            double cm = 0.0;
            for (int i = lane; i < n; i += 32) {
                const CD c = NL<CD>::ld(DXC, i, n);
                NL<CDD>::st(DXD, i, n, cdd_add(NL<CDD>::ld(DXD, i, n), CDD{c.re, 0.0, c.im, 0.0}));
                cm = fmax(cm, nt_magmax(c));
            }
            for (int o = 16; o; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
            cmax = cm;
        }
        PJB_PHM(2)
    }
    if (warp == 0) {
        __syncwarp();
        double dn = 0.0;
        bool fin = true;
        for (int i = lane; i < n; i += 32) {
            const CDD d = NL<CDD>::ld(DXD, i, n);
            const CDD xn = cdd_add(Sc<CDD>::ld_aos(x + size_t(i) * 4), d);
            Sc<CDD>::st_aos(xo + size_t(i) * 4, xn);
            dn = fmax(dn, nt_magmax(d));
            fin = fin && nt_finite(xn);
        }
        for (int o = 16; o; o >>= 1) dn = fmax(dn, __shfl_xor_sync(0xffffffffu, dn, o));
        fin = __all_sync(0xffffffffu, fin);
        if (lane == 0) {
            if (a.norms) a.norms[2 * b + 1] = dn;
            if (a.status) a.status[b] = !fin ? 2 : (cmax > ldexp(dn, -64) ? 3 : 0);
        }
    }
    PJB_PHM(3)
#undef PJB_PHM
}

// NQ: active-row slots per lane (look-ahead) and rows per lane (back substitution), n <= 32*NQ
// kRecip[c] = ceil(2^16 / c): floor(x / c) == (x * kRecip[c]) >> 16 for x, c <= 256
__constant__ unsigned kRecip[257];

#ifndef PJB_NT_ROTATE
#define PJB_NT_ROTATE 1
#endif
#ifndef PJB_NT_PREFETCH
#define PJB_NT_PREFETCH 1
#endif
#ifndef PJB_NT_MINB
#define PJB_NT_MINB 6
#endif
#ifndef PJB_NT_T1
#define PJB_NT_T1 128
#endif
// n <= 32 (NQ = 1) runs 128-thread CTAs, six per SM (the matrix is 36 KB in dd): 85 registers
template <int NQ>
struct NtBounds {
    // (measured: 160-thread CTAs, four per SM: n = 32 dd -2.7%, complex double +22% time)
    static constexpr int threads = NQ == 1 ? PJB_NT_T1 : 256, blocks = NQ == 1 ? PJB_NT_MINB : 1;
};
#ifndef PJB_NT_MINB_D
#define PJB_NT_MINB_D 8
#endif
// complex double at n <= 32 (18 KB of matrix): eight CTAs per SM, 64 registers (measured 2.35 ms vs
// 2.45 (7) and 2.60 (6) at C2)
#ifndef PJB_NT_MINB_MX
#define PJB_NT_MINB_MX 8
#endif
template <class T, int NQ, bool MX = false>
constexpr int nt_min_blocks() {
    return MX ? PJB_NT_MINB_MX : NQ == 1 && Sc<T>::W == 2 ? PJB_NT_MINB_D : NtBounds<NQ>::blocks;
}
// GS: the matrix lives in a per-CTA global slab (a.gscratch) instead of shared memory. A separate
// instantiation, so that in the shared-memory kernel the compiler sees every matrix access as a
// shared-memory access (LDS/STS, not generic LD/ST that must resolve the address space at run time)
// MX: the mixed-precision solve (T = CD, NQ = 1: complex-double factorisation of a complex-dd
// system, refined in dd; see nt_mixed_finish)
template <class T, int NQ, bool GS, bool MX = false>
__global__ void __launch_bounds__(NtBounds<NQ>::threads, nt_min_blocks<T, NQ, MX>()) newton_kernel(NewtonArgs a) {
    using S = Sc<T>;
    constexpr int W = S::W;
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_sing, s_la;
    const int n = a.n, ld = n + 1, P = n * ld;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    // Warp roles. A warp's SM sub-partition (scheduler) is its hardware warp slot mod 4, and a CTA's
    // warps occupy consecutive slots: with a fixed look-ahead warp every co-resident CTA would put
    // its latency-critical look-ahead chain (and the back substitution) on the same scheduler. The
    // role-0 warp is therefore the CTA's warp (slot group of warp 0) mod nw, which spreads the
    // chains of the CTAs sharing an SM over the schedulers.
    if (tid == 0) {
        unsigned wid = 0;
#if PJB_NT_ROTATE
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
#endif
        s_la = int((wid >> 2) % unsigned(blockDim.x >> 5));
    }
    __syncthreads();
    const int nw = nt >> 5, warp = ((tid >> 5) - s_la + nw) % nw;  // role index: 0 = look-ahead
    // dynamic shared memory: ints (pivot rows, pivot step of each row, two active-row lists), then
    // the matrix planes unless they live in a global slab
    int* s_piv = reinterpret_cast<int*>(smem);
    int* s_step = s_piv + n;
    int* s_list0 = s_step + n;
    int* s_list1 = s_list0 + n;
    double* A = GS ? a.gscratch + size_t(blockIdx.x) * a.gstride : smem + newton_int_words(n);
    double* INV = A + size_t(W) * P;  // [W][n] pivot inverses
    double* DX = INV + size_t(W) * n;   // [W][n] solution
    double* DXD = DX + size_t(W) * n;   // MX: the dd solution [4][n], then four partial residuals, corrections
    double* PART = DXD + 4 * size_t(n);
    double* DXC = PART + 16 * size_t(n);

#ifdef PJB_NT_TRACE
    long long* tsub = nullptr;  // look-ahead sub-phase clocks (developer instrumentation)
#define PJB_TSUB(c, k) \
    if (tsub && lane == 0) tsub[4 * (c) + (k)] = clock64();
#else
#define PJB_TSUB(c, k)
#endif
    // Warp-0 look-ahead for column c: rows list[0..R) (values v[] already in registers), pick the
    // pivot, store inv_c and the multipliers of column c, write the next list (R-1 rows).
    auto pivot_phase = [&](int c, const int* list, int R, const T* v, int* next) {
        PJB_TSUB(c, 0)
        // every lane inverts its own candidates speculatively, off the arg-max's critical path
        T ivq[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) ivq[q] = nt_inv(v[q]);
        double best = 0.0;
        int bi = -1, bq = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int idx = lane + 32 * q;
            if (idx < R) {
                const double mg = nt_mag1(v[q]);
                const int r = list[idx];
                if (mg > best || (mg == best && bi >= 0 && r < bi)) {
                    best = mg;
                    bi = r;
                    bq = idx;
                }
            }
        }
        // arg-max over the warp with redux: the largest magnitude (its bits are monotonic, high
        // word then low word), ties to the smallest row — the same rule as a sequential scan
        const unsigned long long bits = __double_as_longlong(best);
        const unsigned hi = unsigned(bits >> 32), lo = unsigned(bits);
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        const bool cand = bi >= 0 && hi == mh && lo == ml;
        const int rmin = __reduce_min_sync(0xffffffffu, cand ? bi : 0x7fffffff);
        PJB_TSUB(c, 1)
        if (rmin == 0x7fffffff) {
            if (lane == 0) s_sing = 1;
            return;
        }
        const int owner = __ffs(__ballot_sync(0xffffffffu, cand && bi == rmin)) - 1;
        bi = rmin;
        bq = __shfl_sync(0xffffffffu, bq, owner);
        T iv = ivq[0];
#pragma unroll
        for (int q = 1; q < NQ; ++q)
            if (q == (bq >> 5)) iv = ivq[q];
        iv = shfl_idx(iv, owner);
        PJB_TSUB(c, 2)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int idx = lane + 32 * q;
            if (idx < R) {
                const int r = list[idx];
                if (r != bi) NL<T>::st(A, r * ld + c, P, S::mul(v[q], iv));
                // next list: the pivot's slot takes the last row
                if (idx < R - 1) next[idx] = idx == bq ? list[R - 1] : r;
            }
        }
        if (lane == 0) {
            NL<T>::st(INV, c, n, iv);
            s_piv[c] = bi;
            s_step[bi] = c;
        }
        PJB_TSUB(c, 3)
    };
#ifdef PJB_NT_PHASES
    // developer instrumentation: per-CTA cycle totals of the load, elimination and back-substitution
    // phases over all of its points, after the B status words (status must hold B + 2 + 16 * grid; phases 4-7 break down the mixed refinement)
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tph = clock64();
#define PJB_PH(i)                      \
    {                                  \
        const long long t_ = clock64(); \
        ph[i] += t_ - tph;             \
        tph = t_;                      \
    }
#else
#define PJB_PH(i)
#endif
    for (long long b = blockIdx.x; b < a.B; b += gridDim.x) {
        if constexpr (MX)
            nt_load_mixed(a, b, A, s_list0, &s_sing, warp);
        else
            nt_load<T, GS>(a, b, A, s_list0, &s_sing, warp);
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
        PJB_PH(0)
#if PJB_NT_PREFETCH
        // complex-double factorisations (the d solve and the mixed solve) pull the CTA's next point
        // into L2 while this one is eliminated (measured: d 2.21 -> 2.18 ms; the dd solve, 0.5%
        // slower with it, does not; the mixed solve 4.23 -> 4.20 ms with the right element width:
        // profiles/r02_newton_l2prefetch_ab.log, r02_newton_prefetch_w.log, r02_newton_prefetch_w_ab.log)
        if (W == 2 && b + gridDim.x < a.B) {
            constexpr int WE = MX ? 4 : W;  // the evaluator output's element width
            const char* nx = reinterpret_cast<const char*>(a.evals + size_t(b + gridDim.x) * (size_t(n) * n + n) * WE);
            const int lines = int((size_t(n) * n + n) * WE * sizeof(double) / 128);
            for (int l = tid; l < lines; l += nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + size_t(l) * 128));
        }
#endif
        // ---- column 0: pivot, inverse, multipliers
        if (warp == 0) {
            T v[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int idx = lane + 32 * q;
                v[q] = idx < n ? NL<T>::ld(A, idx * ld, P) : S::zero();
            }
            pivot_phase(0, s_list0, n, v, s_list1);
        }
        __syncthreads();

        // ---- elimination: step kk updates the active rows (R of them) at columns kk+1..n; warp 0
        // takes column kk+1 and looks ahead, warps 1.. the rest.
        bool singular = s_sing != 0;
#ifdef PJB_NT_TRACE
        // developer instrumentation: per-step clocks of block 0's first point (warp 0 look-ahead
        // start/end, updater warp 1 end, barrier exit) into a.status (reinterpreted as long long)
        // (the trace lives after the B status words: status must have B + 2 + 8n entries)
        long long* trace = (blockIdx.x == 0 && b == 0 && a.status)
                               ? reinterpret_cast<long long*>(a.status + ((a.B + 1) & ~1LL)) : nullptr;
        tsub = trace ? trace + 4 * n : nullptr;
#endif
        for (int kk = 0; kk < n && !singular; ++kk) {
#ifdef PJB_NT_TRACE
            if (trace && lane == 0 && warp <= 1) trace[4 * kk + warp] = clock64();
#endif
            const int R = n - kk - 1;
            const int* list = (kk & 1) ? s_list0 : s_list1;
            int* next = (kk & 1) ? s_list1 : s_list0;
            const int pr = s_piv[kk];
            if (warp == 0) {
                if (kk + 1 < n) {
                    const int c = kk + 1;
                    const T u = NL<T>::ld(A, pr * ld + c, P);
                    T v[NQ];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const int idx = lane + 32 * q;
                        if (idx < R) {
                            const int r = list[idx];
                            v[q] = S::add(NL<T>::ld(A, r * ld + c, P),
                                          nt_neg(nt_umul(NL<T>::ld(A, r * ld + kk, P), u)));
                        } else {
                            v[q] = S::zero();
                        }
                    }
                    pivot_phase(c, list, R, v, next);
                }
#ifdef PJB_NT_TRACE
                if (trace && lane == 0) trace[4 * kk + 2] = clock64();
#endif
            } else {
                // columns kk+2..n (Cp of them) for R rows: a thread keeps u = A[pr][j] in registers
                // and walks rows rg, rg+G, ...
                const int Cp = n - kk - 1, Tp = nt - 32, tp = (warp - 1) * 32 + lane;
                // measured (tools/nt_quick.py, C2/C3): column pairs win for complex double and
                // n > 32 (n = 64 dd: 8.92 -> 8.40 ms), single columns for n <= 32 dd (7.80 vs 8.42 ms)
                constexpr bool kPairs = NQ >= 2 || W == 2;
                if constexpr (kPairs) {
                // column pairs (j, j + Ch): one multiplier load serves two independent chains
                const int Ch = (Cp + 1) >> 1;
                for (int c0 = 0; c0 < Ch; c0 += Tp) {
                    const int cw = min(Tp, Ch - c0);
                    const unsigned rc = kRecip[cw];
                    const int G = int((unsigned(Tp) * rc) >> 16), rg = int((unsigned(tp) * rc) >> 16);
                    if (rg >= G) continue;
                    const int ci = c0 + (tp - rg * cw);
                    const int j1 = kk + 2 + ci, j2 = j1 + Ch;
                    const bool two = ci + Ch < Cp;
                    const T u1 = NL<T>::ld(A, pr * ld + j1, P);
                    const T u2 = two ? NL<T>::ld(A, pr * ld + j2, P) : u1;
                    for (int idx = rg; idx < R; idx += G) {
                        const int r = list[idx];
                        const T l = NL<T>::ld(A, r * ld + kk, P);
                        const T v1 = NL<T>::ld(A, r * ld + j1, P);
                        const T v2 = two ? NL<T>::ld(A, r * ld + j2, P) : v1;
                        const T w1 = S::add(v1, nt_neg(nt_umul(l, u1)));
                        const T w2 = S::add(v2, nt_neg(nt_umul(l, u2)));
                        NL<T>::st(A, r * ld + j1, P, w1);
                        if (two) NL<T>::st(A, r * ld + j2, P, w2);
                    }
                }
                } else {
                for (int c0 = 0; c0 < Cp; c0 += Tp) {
                    const int cw = min(Tp, Cp - c0);
                    const unsigned rc = kRecip[cw];
                    const int G = int((unsigned(Tp) * rc) >> 16), rg = int((unsigned(tp) * rc) >> 16);
                    if (rg >= G) continue;
                    const int j = kk + 2 + c0 + (tp - rg * cw);
                    const T u = NL<T>::ld(A, pr * ld + j, P);
                    for (int idx = rg; idx < R; idx += G) {
                        const int r = list[idx];
                        const T l = NL<T>::ld(A, r * ld + kk, P);
                        const T v = NL<T>::ld(A, r * ld + j, P);
                        NL<T>::st(A, r * ld + j, P, S::add(v, nt_neg(nt_umul(l, u))));
                    }
                }
                }
            }
            __syncthreads();
#ifdef PJB_NT_TRACE
            if (trace && tid == 0) trace[4 * kk + 3] = clock64();
#endif
            singular = s_sing != 0;
        }

        PJB_PH(1)
        if constexpr (MX)
            nt_mixed_finish(a, b, A, INV, DXD, PART, DXC, s_piv, s_step, singular, warp
#ifdef PJB_NT_PHASES
                            , ph + 4
#endif
            );
        else if (warp == 0)
            nt_back_substitute<T, NQ>(a, b, A, INV, DX, s_piv, s_step, singular);
        __syncthreads();  // the next point reuses the matrix storage
        PJB_PH(2)
#ifdef PJB_NT_PHASES
        ++ph[3];
#endif
    }
#ifdef PJB_NT_PHASES
    if (tid == 0 && a.status) {
        long long* o = reinterpret_cast<long long*>(a.status + ((a.B + 1) & ~1LL)) + 8 * blockIdx.x;
        for (int i = 0; i < 8; ++i) o[i] = ph[i];
    }
#endif
#undef PJB_PH
}

// ---- blocked variant for n <= 32 (opt-in, pj_set_kernel_variant with PJ_OP_NEWTON): the
// look-ahead warp factors PANELS of kPW columns in registers (lane = row), the other warps apply a
// panel's kPW steps to the trailing columns in one pass. Measured slower than the column kernel at
// C2 (dd 10.7 vs 7.2 ms, complex double 2.50 vs 2.44 ms): the look-ahead's 32 sequential pivot
// chains are the critical path either way, and the panel look-ahead adds the next panel's update
// to it (and, in dd, register pressure).
// The arithmetic of every element is the unblocked kernel's (same pivots, multipliers, and per
// element the same update sequence in step order), so results are bit-identical; what changes is
// the schedule: one CTA barrier per panel instead of per column, the look-ahead's column values
// and multipliers stay in registers, and a trailing element loads once for kPW updates.
constexpr int kPW = 4;

#ifndef PJB_NTP_MINB
#define PJB_NTP_MINB 3
#endif
template <class T>
__global__ void __launch_bounds__(128, PJB_NTP_MINB) newton_panel_kernel(NewtonArgs a) {
    using S = Sc<T>;
    constexpr int W = S::W;
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_sing;
    const int n = a.n, ld = n + 1, P = n * ld;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    int* s_piv = reinterpret_cast<int*>(smem);
    int* s_step = s_piv + n;
    int* s_list[2] = {s_step + n, s_step + 2 * n};  // rows active at a panel's start (compacted)
    double* A = smem + newton_int_words(n);
    double* INV = A + size_t(W) * P;
    double* DX = INV + size_t(W) * n;
    const int NP = (n + kPW - 1) / kPW;
    const bool valid = lane < n;  // warp 0: lane = row

    for (long long b = blockIdx.x; b < a.B; b += gridDim.x) {
        nt_load<T>(a, b, A, s_list[0], &s_sing, warp);
        if (warp == 0)
            for (int i = lane; i < n; i += 32) s_step[i] = n;  // n = not yet pivoted
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();

        // look-ahead state (warp 0): my row's values in the current panel's columns, its
        // multipliers for those columns, the step it was pivoted at
        T V[kPW], Lm[kPW];
        int mystep = n;
        bool bad = false;
        // factor panel p from V (columns c0..c0+w-1 updated through step c0-1): pivots, inverses,
        // multipliers (registers + shared memory for the trailing update), the pivot rows' panel
        // entries (U), and the compacted list of rows active at the panel's start
        auto factor = [&](int p) {
            const int c0 = p * kPW, w = min(kPW, n - c0);
            const unsigned act = __ballot_sync(0xffffffffu, valid && mystep == n);
            if (valid && mystep == n) s_list[p & 1][__popc(act & ((1u << lane) - 1))] = lane;
#pragma unroll
            for (int t = 0; t < kPW; ++t) {
                if (t < w && !bad) {
                    const int col = c0 + t;
                    const bool active = valid && mystep == n;
                    const T v = V[t];
                    const T ivq = nt_inv(v);  // speculative: off the arg-max's path
                    const double mg = active ? nt_mag1(v) : 0.0;
                    const unsigned long long bits = __double_as_longlong(mg);
                    const unsigned hi = unsigned(bits >> 32), lo = unsigned(bits);
                    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                    const bool cand = active && mg > 0.0 && hi == mh && lo == ml;
                    const unsigned cm = __ballot_sync(0xffffffffu, cand);
                    if (!cm) {  // no nonzero pivot: singular
                        if (lane == 0) s_sing = 1;
                        bad = true;
                    } else {
                        const int pr = __ffs(cm) - 1;  // ties: the smallest row
                        const T iv = shfl_idx(ivq, pr);
                        if (lane == pr) {
                            mystep = col;
                            s_piv[col] = pr;
                            s_step[pr] = col;
                            NL<T>::st(INV, col, n, iv);
                        }
                        const bool upd = active && lane != pr;
                        T l = S::zero();
                        if (upd) {
                            l = S::mul(v, iv);
                            NL<T>::st(A, lane * ld + col, P, l);
                        }
                        Lm[t] = l;
#pragma unroll
                        for (int t2 = t + 1; t2 < kPW; ++t2) {
                            if (t2 < w) {
                                const T u = shfl_idx(V[t2], pr);
                                if (upd) V[t2] = S::add(V[t2], nt_neg(nt_umul(l, u)));
                                if (lane == pr) NL<T>::st(A, lane * ld + c0 + t2, P, V[t2]);  // U entry
                            }
                        }
                    }
                }
            }
        };
        if (warp == 0) {
#pragma unroll
            for (int t = 0; t < kPW; ++t) V[t] = valid && t < n ? NL<T>::ld(A, lane * ld + t, P) : S::zero();
            factor(0);
        }
        __syncthreads();
        bool singular = s_sing != 0;
        for (int p = 0; p < NP && !singular; ++p) {
            const int c0 = p * kPW, w = min(kPW, n - c0);
            const int c1 = c0 + kPW, w1 = c1 < n ? min(kPW, n - c1) : 0;
            if (warp == 0) {
                if (w1 > 0) {
                    // next panel's columns (current through step c0-1), then panel p's steps in order
                    T* V2 = V;  // panel p's values are dead once factored: reuse their registers
#pragma unroll
                    for (int t = 0; t < kPW; ++t)
                        V2[t] = valid && t < w1 ? NL<T>::ld(A, lane * ld + c1 + t, P) : S::zero();
#pragma unroll
                    for (int t = 0; t < kPW; ++t) {
                        if (t < w) {
                            const int pr = s_piv[c0 + t];
                            const bool upd = valid && mystep > c0 + t;
#pragma unroll
                            for (int t2 = 0; t2 < kPW; ++t2) {
                                const T u = shfl_idx(V2[t2], pr);
                                if (upd && t2 < w1) V2[t2] = S::add(V2[t2], nt_neg(nt_umul(Lm[t], u)));
                            }
                        }
                    }
                    // rows pivoted in panel p: their entries of the next panel are final (U)
                    if (valid && mystep >= c0 && mystep < c0 + w)
#pragma unroll
                        for (int t = 0; t < kPW; ++t)
                            if (t < w1) NL<T>::st(A, lane * ld + c1 + t, P, V2[t]);
                    factor(p + 1);
                }
            } else {
                // trailing columns beyond the next panel (rhs included) with panel p's steps. Phase A:
                // each thread forms the pivot rows' entries of its column after the panel's earlier
                // steps (u_t); named barrier; phase B: every row active at the panel's start gets
                // its updates in step order (pivot rows of the panel: the updates before their step).
                const int j0 = w1 > 0 ? c1 + w1 : c0 + w, Cp = n + 1 - j0, Tp = nt - 32, tp = tid - 32;
                const int* list = s_list[p & 1];
                const int R0 = n - c0;
                // panel p's pivot rows (written before the last barrier; s_step may be changing under
                // the look-ahead's factor(p + 1), so row activity is read from these instead)
                int pvt[kPW];
#pragma unroll
                for (int t = 0; t < kPW; ++t) pvt[t] = t < w ? s_piv[c0 + t] : -1;
                for (int cb = 0; cb < Cp; cb += Tp) {  // uniform pass count: every updater joins each barrier
                    const int cw = min(Tp, Cp - cb);
                    const unsigned rc = kRecip[cw];
                    const int G = int((unsigned(Tp) * rc) >> 16), rg = int((unsigned(tp) * rc) >> 16);
                    const bool mine = rg < G;
                    const int j = j0 + cb + (tp - rg * cw);
                    T u[kPW];
                    if (mine) {
#pragma unroll
                        for (int t = 0; t < kPW; ++t) {
                            if (t < w) {
                                const int pr = pvt[t];
                                T x = NL<T>::ld(A, pr * ld + j, P);
#pragma unroll
                                for (int t2 = 0; t2 < kPW; ++t2)
                                    if (t2 < t) x = S::add(x, nt_neg(nt_umul(NL<T>::ld(A, pr * ld + c0 + t2, P), u[t2])));
                                u[t] = x;
                            }
                        }
                    }
                    asm volatile("bar.sync 1, %0;\n" ::"r"(Tp));
                    if (mine) {
                        for (int idx = rg; idx < R0; idx += G) {
                            const int r = list[idx];
                            int sr = n;  // the step row r is pivoted at, if within panel p
#pragma unroll
                            for (int t = 0; t < kPW; ++t)
                                if (r == pvt[t]) sr = c0 + t;
                            T x = NL<T>::ld(A, r * ld + j, P);
#pragma unroll
                            for (int t = 0; t < kPW; ++t)
                                if (t < w && sr > c0 + t) x = S::add(x, nt_neg(nt_umul(NL<T>::ld(A, r * ld + c0 + t, P), u[t])));
                            NL<T>::st(A, r * ld + j, P, x);
                        }
                    }
                }
            }
            __syncthreads();
            singular = s_sing != 0;
        }
        if (warp == 0) nt_back_substitute<T, 1>(a, b, A, INV, DX, s_piv, s_step, singular);
        __syncthreads();  // the next point reuses the matrix storage
    }
}

template <class T>
const void* newton_fn(int nq, bool gs) {
    if (gs) return nq <= 4 ? (const void*)newton_kernel<T, 4, true> : (const void*)newton_kernel<T, 8, true>;
    switch (nq) {
        case 1: return (const void*)newton_kernel<T, 1, false>;
        case 2: return (const void*)newton_kernel<T, 2, false>;
        case 4: return (const void*)newton_kernel<T, 4, false>;
        default: return (const void*)newton_kernel<T, 8, false>;
    }
}
// (a global-slab launch with n <= 64 runs the NQ = 4 instantiation: same code, more row slots)
int nq_of(int n) { return n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : 8; }
const void* fn_of(int prec, int n, bool panel, bool gs) {
    if (prec == 3) return (const void*)newton_kernel<CD, 1, false, true>;  // mixed (n <= 32)
    if (panel && !gs) return prec == 1 ? (const void*)newton_panel_kernel<CD> : (const void*)newton_panel_kernel<CDD>;
    return prec == 1 ? newton_fn<CD>(nq_of(n), gs) : newton_fn<CDD>(nq_of(n), gs);
}

}  // namespace

// prec: 1 complex double, 2 complex dd, 3 mixed (complex-double factors of a complex-dd system:
// the double matrix planes plus the dd solution, four partial residuals and the corrections)
size_t newton_matrix_bytes(int prec, int n) {
    const int W = prec == 2 ? 4 : 2;
    const size_t extra = prec == 3 ? (4 + 16 + 2) * size_t(n) : 0;
    return (size_t(W) * n * (n + 1) + 2 * size_t(W) * n + extra) * sizeof(double);
}
size_t newton_int_bytes(int n) { return size_t(newton_int_words(n)) * sizeof(double); }

// The reciprocal table is __constant__ memory: one copy per device, filled once per device
// (thread-safe: contexts on several devices may launch concurrently).
static cudaError_t init_recip() {
    static std::mutex mu;
    static std::set<int> ready;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (ready.count(dev)) return cudaSuccess;
    unsigned h[257];
    h[0] = 0;
    for (int c = 1; c <= 256; ++c) h[c] = (65536u + c - 1) / c;
    cudaError_t e = cudaMemcpyToSymbol(kRecip, h, sizeof(h));
    if (e == cudaSuccess) ready.insert(dev);
    return e;
}

bool newton_panel_supported(int n) { return n <= 32; }
int newton_max_threads(int n) { return n <= 32 ? NtBounds<1>::threads : NtBounds<2>::threads; }

int newton_blocks_per_sm(int prec, int n, int threads, size_t smem, bool panel, bool gs) {
    const void* f = fn_of(prec, n, panel, gs);
    if (smem) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit(f));
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, threads, smem) != cudaSuccess) return 0;
    return nb;
}

cudaError_t launch_newton(int prec, const NewtonArgs& args, int blocks, int threads, size_t smem, bool panel,
                          cudaStream_t st) {
    if (args.B <= 0) return cudaSuccess;
    const void* f = fn_of(prec, args.n, panel, args.gscratch != nullptr);
    if (cudaError_t e = init_recip()) return e;
    if (smem) {
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit(f));
        if (e) return e;
    }
    const long long nb = blocks < args.B ? blocks : args.B;
    void* kargs[] = {const_cast<NewtonArgs*>(&args)};
    return cudaLaunchKernel(f, dim3(unsigned(nb)), dim3(threads), kargs, smem, st);
}

}  // namespace pjb
