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
__device__ __forceinline__ bool fin(const CDD& v) {
    return isfinite(v.rh) && isfinite(v.rl) && isfinite(v.ih) && isfinite(v.il);
}

}  // namespace fastc
using namespace fastc;

}  // namespace pjb
