// Complex double and complex double-double scalars for the sm_100a kernels.
//
// Every operation is spelled with explicit round-to-nearest intrinsics (__dadd_rn,
// __dmul_rn, __fma_rn) so nvcc can neither contract a*b-c into an FMA nor reassociate;
// the host oracle (oracle/oracle.cpp) states the same sequences with -ffp-contract=off, so
// the two agree bit for bit when the operation order agrees.
//
//  CD   complex double, the reference scalar (ref include/polyjac/complex.hpp:12-39): the
//       product is the fixed 4-multiply / 2-add form, re = ar*br - ai*bi, im = ar*bi + ai*br.
//  CDD  complex double-double (re_hi, re_lo, im_hi, im_lo). Product: per component the two
//       leading products are split exactly (TwoProd via FMA), their sum/difference is made
//       error-free with TwoSum, the four cross terms are folded in by FMA, and one Fast2Sum
//       renormalises: 2 DMUL + 6 DFMA + 11 DADD per component (38 FP64 instructions per
//       complex product, vs 68 for four dd products and two accurate dd adds). Sum: TwoSum of
//       the high words, low words added, one Fast2Sum (11 DADD per component).
#pragma once
#include <cstdint>

namespace pjb {

struct CD {
    double re, im;
};
struct CDD {
    double rh, rl, ih, il;
};

__device__ __forceinline__ CD cd_mul(CD a, CD b) {
    return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
            __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
__device__ __forceinline__ CD cd_add(CD a, CD b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }

struct DD {
    double hi, lo;
};
// Error-free sum s + e = a + b. Every variant returns s = fl(a + b) and the EXACT error e, so all
// give identical bits (the oracle keeps Knuth's form):
//   0  Knuth's branch-free TwoSum, 6 DADD;
//   1  operands ordered by magnitude (one DSETP with |.| modifiers, two 64-bit selects), then
//      Dekker's Fast2Sum, exact for |x| >= |y| — 3 DADD + 1 DSETP;
//   2  ordered by the sign-masked high words (exponent first: Fast2Sum is exact whenever
//      e_x >= e_y in radix 2), integer compare — 3 DADD, no extra FP64 instruction.
#ifndef PJB_TWOSUM
#define PJB_TWOSUM 0
#endif
__device__ __forceinline__ DD two_sum(double a, double b) {
#if PJB_TWOSUM == 0
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
#else
#if PJB_TWOSUM == 1
    const bool c = fabs(a) >= fabs(b);
#else
    const bool c = (__double2hiint(a) & 0x7fffffff) >= (__double2hiint(b) & 0x7fffffff);
#endif
    const double x = c ? a : b, y = c ? b : a;
    const double s = __dadd_rn(x, y);
    return {s, __dsub_rn(y, __dsub_rn(s, x))};
#endif
}
__device__ __forceinline__ DD fast_two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double e = __dsub_rn(b, __dsub_rn(s, a));
    return {s, e};
}

__device__ __forceinline__ CDD cdd_mul(CDD a, CDD b) {
    CDD r;
    {
        double p1 = __dmul_rn(a.rh, b.rh), e1 = __fma_rn(a.rh, b.rh, -p1);
        double p2 = __dmul_rn(a.ih, b.ih), e2 = __fma_rn(a.ih, b.ih, -p2);
        DD st = two_sum(p1, -p2);
        double la = __fma_rn(a.rh, b.rl, e1);
        la = __fma_rn(a.rl, b.rh, la);
        double lb = __fma_rn(a.ih, b.il, e2);
        lb = __fma_rn(a.il, b.ih, lb);
        double l = __dadd_rn(__dsub_rn(la, lb), st.lo);
        DD o = fast_two_sum(st.hi, l);
        r.rh = o.hi;
        r.rl = o.lo;
    }
    {
        double p3 = __dmul_rn(a.rh, b.ih), e3 = __fma_rn(a.rh, b.ih, -p3);
        double p4 = __dmul_rn(a.ih, b.rh), e4 = __fma_rn(a.ih, b.rh, -p4);
        DD st = two_sum(p3, p4);
        double lc = __fma_rn(a.rh, b.il, e3);
        lc = __fma_rn(a.rl, b.ih, lc);
        double ld = __fma_rn(a.ih, b.rl, e4);
        ld = __fma_rn(a.il, b.rh, ld);
        double l = __dadd_rn(__dadd_rn(lc, ld), st.lo);
        DD o = fast_two_sum(st.hi, l);
        r.ih = o.hi;
        r.il = o.lo;
    }
    return r;
}
// Complex dd product WITHOUT the closing renormalisation: returns (s, l) per component where
// s = fl(leading sum) and l the folded error terms, |l| <~ u*(|a||b|). Used inside product
// chains: the next product's TwoProd/FMA cross terms absorb an unnormalised low word at the
// same normwise error (the dropped lo*lo term stays <= u^2 |a||b|), so the Fast2Sum (3 DADD
// per component) is paid once per chain instead of once per product (32 instead of 38 FP64
// instructions). Chains end in a normalising addition (stage 3) or dd_renorm.
__device__ __forceinline__ CDD cdd_mul_u(CDD a, CDD b) {
    CDD r;
    {
        double p1 = __dmul_rn(a.rh, b.rh), e1 = __fma_rn(a.rh, b.rh, -p1);
        double p2 = __dmul_rn(a.ih, b.ih), e2 = __fma_rn(a.ih, b.ih, -p2);
        DD st = two_sum(p1, -p2);
        double la = __fma_rn(a.rh, b.rl, e1);
        la = __fma_rn(a.rl, b.rh, la);
        double lb = __fma_rn(a.ih, b.il, e2);
        lb = __fma_rn(a.il, b.ih, lb);
        r.rh = st.hi;
        r.rl = __dadd_rn(__dsub_rn(la, lb), st.lo);
    }
    {
        double p3 = __dmul_rn(a.rh, b.ih), e3 = __fma_rn(a.rh, b.ih, -p3);
        double p4 = __dmul_rn(a.ih, b.rh), e4 = __fma_rn(a.ih, b.rh, -p4);
        DD st = two_sum(p3, p4);
        double lc = __fma_rn(a.rh, b.il, e3);
        lc = __fma_rn(a.rl, b.ih, lc);
        double ld = __fma_rn(a.ih, b.rl, e4);
        ld = __fma_rn(a.il, b.rh, ld);
        r.ih = st.hi;
        r.il = __dadd_rn(__dadd_rn(lc, ld), st.lo);
    }
    return r;
}
// Exact renormalisation of a (possibly unnormalised) complex dd: TwoSum per component, so the
// result satisfies |lo| <= ulp(hi)/2.
__device__ __forceinline__ CDD cdd_renorm(CDD a) {
    DD re = two_sum(a.rh, a.rl), im = two_sum(a.ih, a.il);
    return {re.hi, re.lo, im.hi, im.lo};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
    DD s = two_sum(a.hi, b.hi);
    double e = __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo));
    return fast_two_sum(s.hi, e);
}
__device__ __forceinline__ CDD cdd_add(CDD a, CDD b) {
    DD re = dd_add({a.rh, a.rl}, {b.rh, b.rl});
    DD im = dd_add({a.ih, a.il}, {b.ih, b.il});
    return {re.hi, re.lo, im.hi, im.lo};
}

// Scalar traits: W doubles per complex value, smem/global access in "plane" layout
// (component c of element e at base[c * stride + e]) so a warp's lane-consecutive
// elements are conflict-free 8-byte accesses.
template <class T>
struct Sc;
template <>
struct Sc<CD> {
    static constexpr int W = 2;
    __device__ static CD zero() { return {0.0, 0.0}; }
    __device__ static CD one() { return {1.0, 0.0}; }
    __device__ static CD mul(CD a, CD b) { return cd_mul(a, b); }
    __device__ static CD add(CD a, CD b) { return cd_add(a, b); }
    __device__ static CD ld_planes(const double* p, int stride) { return {p[0], p[stride]}; }
    __device__ static void st_planes(double* p, int stride, CD v) {
        p[0] = v.re;
        p[stride] = v.im;
    }
    // interleaved (AoS) element: W consecutive doubles
    __device__ static CD ld_aos(const double* p) {
        double2 v = *reinterpret_cast<const double2*>(p);
        return {v.x, v.y};
    }
    __device__ static void st_aos(double* p, CD v) { *reinterpret_cast<double2*>(p) = make_double2(v.re, v.im); }
    __device__ static bool finite(CD v) { return isfinite(v.re) && isfinite(v.im); }
    __device__ static CD shfl_xor(CD v, int mask) {
        return {__shfl_xor_sync(0xffffffffu, v.re, mask), __shfl_xor_sync(0xffffffffu, v.im, mask)};
    }
};
template <>
struct Sc<CDD> {
    static constexpr int W = 4;
    __device__ static CDD zero() { return {0.0, 0.0, 0.0, 0.0}; }
    __device__ static CDD one() { return {1.0, 0.0, 0.0, 0.0}; }
    __device__ static CDD mul(CDD a, CDD b) { return cdd_mul(a, b); }
    __device__ static CDD add(CDD a, CDD b) { return cdd_add(a, b); }
    __device__ static CDD ld_planes(const double* p, int stride) {
        return {p[0], p[stride], p[2 * stride], p[3 * stride]};
    }
    __device__ static void st_planes(double* p, int stride, CDD v) {
        p[0] = v.rh;
        p[stride] = v.rl;
        p[2 * stride] = v.ih;
        p[3 * stride] = v.il;
    }
    __device__ static CDD ld_aos(const double* p) {
        double2 a = reinterpret_cast<const double2*>(p)[0];
        double2 b = reinterpret_cast<const double2*>(p)[1];
        return {a.x, a.y, b.x, b.y};
    }
    __device__ static void st_aos(double* p, CDD v) {
        reinterpret_cast<double2*>(p)[0] = make_double2(v.rh, v.rl);
        reinterpret_cast<double2*>(p)[1] = make_double2(v.ih, v.il);
    }
    __device__ static bool finite(CDD v) {
        return isfinite(v.rh) && isfinite(v.rl) && isfinite(v.ih) && isfinite(v.il);
    }
    __device__ static CDD shfl_xor(CDD v, int mask) {
        return {__shfl_xor_sync(0xffffffffu, v.rh, mask), __shfl_xor_sync(0xffffffffu, v.rl, mask),
                __shfl_xor_sync(0xffffffffu, v.ih, mask), __shfl_xor_sync(0xffffffffu, v.il, mask)};
    }
};

}  // namespace pjb
