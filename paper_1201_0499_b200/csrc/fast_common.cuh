// Shared-memory access helpers and chain products shared by the fast complex-dd kernels
// (eval_fast.cu, eval_fast_ws.cu).
#pragma once
#include <cuda_runtime.h>

#include "dd.cuh"

namespace pjb {
namespace fastc {

__device__ __forceinline__ CDD sel_cdd(bool c, const CDD& a, const CDD& b) {
    return {c ? a.rh : b.rh, c ? a.rl : b.rl, c ? a.ih : b.ih, c ? a.il : b.il};
}
// "hi/lo pair" layout: element e of an array keeps (re_hi, im_hi) at base + 2e and (re_lo, im_lo)
// at base + hl + 2e — one 16-byte access per pair (LDS.128), half the instructions of four planes
__device__ __forceinline__ CDD ld_hl(const double* p, int hl) {
    const double2 h = *reinterpret_cast<const double2*>(p), l = *reinterpret_cast<const double2*>(p + hl);
    return {h.x, l.x, h.y, l.y};
}
__device__ __forceinline__ void st_hl(double* p, int hl, const CDD& v) {
    *reinterpret_cast<double2*>(p) = make_double2(v.rh, v.ih);
    *reinterpret_cast<double2*>(p + hl) = make_double2(v.rl, v.il);
}
__device__ __forceinline__ CDD ld_aos(const double* p) {
    double2 a = reinterpret_cast<const double2*>(p)[0];
    double2 b = reinterpret_cast<const double2*>(p)[1];
    return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st_aos(double* p, const CDD& v) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v.rh, v.rl);
    reinterpret_cast<double2*>(p)[1] = make_double2(v.ih, v.il);
}
// Product with an optional closing renormalisation. Inside a chain the kernels alternate:
// a product whose left input is normalised skips the Fast2Sum (cdd_mul_u), the next one pays
// it (cdd_mul). An unnormalised low word carried along a whole chain grows linearly and its
// rounding errors with it (chain of 32: worst 39 u^2 vs 7 u^2 normalised); alternating keeps
// the chain error at the normalised level (worst 9 u^2, mean 3.2 vs 2.7 u^2) while paying the
// renormalisation on half the chain products only (tools/chain_error measurements).
__device__ __forceinline__ CDD cmul_n(bool norm, const CDD& a, const CDD& b) {
    return norm ? cdd_mul(a, b) : cdd_mul_u(a, b);
}
// 1/x = conj(x) / |x|^2 in complex dd, for the division form of the fast kernels (relative error a
// few u^2 for x away from 0 and from the exponent limits; the callers guard the range)
__device__ __forceinline__ CDD cdd_inv(const CDD& x) {
    const double p1 = __dmul_rn(x.rh, x.rh), p2 = __dmul_rn(x.ih, x.ih);
    const DD s = two_sum(p1, p2);
    double e = __fma_rn(x.rh, x.rh, -p1);
    e = __dadd_rn(e, __fma_rn(x.ih, x.ih, -p2));
    e = __fma_rn(__dadd_rn(x.rh, x.rh), x.rl, e);
    e = __fma_rn(__dadd_rn(x.ih, x.ih), x.il, e);
    const DD den = fast_two_sum(s.hi, __dadd_rn(s.lo, e));
    const double q = __drcp_rn(den.hi);
    double t = __fma_rn(-den.hi, q, 1.0);
    t = __fma_rn(-den.lo, q, t);
    const DD r = fast_two_sum(q, __dmul_rn(t, q));
    auto mul = [](double ah, double al, DD b) -> DD {
        const double pp = __dmul_rn(ah, b.hi);
        double ee = __fma_rn(ah, b.hi, -pp);
        ee = __fma_rn(ah, b.lo, ee);
        ee = __fma_rn(al, b.hi, ee);
        return fast_two_sum(pp, ee);
    };
    const DD re = mul(x.rh, x.rl, r), im = mul(-x.ih, -x.il, r);
    return {re.hi, re.lo, im.hi, im.lo};
}
// The division form's range (per point, warp-uniform): every coordinate of the point's table row
// 0 (xt, hi pairs at xt + 2v) has |Re hi| + |Im hi| in [2^-16, 2^16]; zeros, extreme magnitudes
// and non-finite coordinates send the point to the product chains
__device__ __forceinline__ bool div_form_ok(const double* xt, int n, int lane) {
    bool ok = true;
    for (int v = lane; v < n; v += 32) {
        const double2 h = *reinterpret_cast<const double2*>(xt + 2 * v);
        const double mg = __dadd_rn(fabs(h.x), fabs(h.y));
        ok = ok && mg >= 0x1p-16 && mg <= 0x1p16;
    }
    return __all_sync(0xffffffffu, ok);
}
__device__ __forceinline__ bool fin(const CDD& v) {
    return isfinite(v.rh) && isfinite(v.rl) && isfinite(v.ih) && isfinite(v.il);
}

}  // namespace fastc
using namespace fastc;

}  // namespace pjb
