// ORACLE — test infrastructure only. Nothing in paper_1201_0499_b200/ links, loads or
// calls this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg do.
//
// CPU restatement of the reference hot path (ref = /root/reference/proj), templated on the
// scalar so the same operation sequence runs in complex double (must reproduce the
// reference bit for bit; pinned against oracle/_ref in tests/test_oracle.py) and in
// complex double-double (the target precision; the reference has no dd code, SPEC.md:12,
// so dd parity is pinned by (1) the double-mode bit-exactness of this same template,
// (2) mpmath golden vectors in tests/golden/, (3) the integer-valued known answers of
// ref/tests/test_kernels.cpp, which are exact in any precision).
//
// Every stage follows the reference's operation order:
//   powers          ref/src/kernels.cpp:9-26   row[0]=1, row[1]=x, row[e]=row[e-1]*x
//   common factor   ref/src/kernels.cpp:45-53  f=pw(0); f*=pw(j) for j=1..k-1
//   speelpenning    ref/src/kernels.cpp:55-93  forward products, running backward product
//   stage-2 term    ref/src/kernels.cpp:95-127 *factor, value from L[k-1], *coeff
//   stage-3 sum     ref/src/kernels.cpp:139-146 acc=+0, m terms ascending g incl. zero pads
//   transpose       ref/src/engine.cpp:215-223  values=sums[0,n), jac[p*n+i]=sums[(i+1)n+p]
//   packing         ref/src/packing.cpp:19-52  deriv coeff = a_j * c (rounded in double mode,
//                                              exact in dd), value coeff = c
//   slot map        ref/src/packing.cpp:8-17   g*(n^2+n)+p | g*(n^2+n)+(var+1)*n+p
//
// Double-double primitives are restated from their published algorithms (Knuth TwoSum,
// Dekker Fast2Sum, FMA-based TwoProd; complex product with one renormalisation per
// component). The product kernels use the same definitions; the oracle keeps its own copy
// so a primitive bug cannot cancel between the two.
//
// Build (see oracle/Makefile): g++ -O2 -ffp-contract=off; FMA contraction would change the
// double-mode bits.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

// ------------------------------------------------------------------ complex double
struct CD {
    double re, im;
};
static inline CD cd_mul(CD a, CD b) {  // ref complex.hpp:22-24, fixed 4-mul/2-add order
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
static inline CD cd_add(CD a, CD b) { return {a.re + b.re, a.im + b.im}; }  // complex.hpp:16-18

// ------------------------------------------------------------------ complex double-double
struct DD {
    double hi, lo;
};
static inline DD two_sum(double a, double b) {  // Knuth, 6 flops, error-free
    double s = a + b;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}
static inline DD fast_two_sum(double a, double b) {  // Dekker, 3 flops
    double s = a + b;
    double e = b - (s - a);
    return {s, e};
}
struct CDD {
    double rh, rl, ih, il;
};
// complex dd product, one renormalisation per component:
//   re = a.re*b.re - a.im*b.im,  im = a.re*b.im + a.im*b.re
static inline CDD cdd_mul(CDD a, CDD b) {
    CDD r;
    {
        double p1 = a.rh * b.rh, e1 = std::fma(a.rh, b.rh, -p1);
        double p2 = a.ih * b.ih, e2 = std::fma(a.ih, b.ih, -p2);
        DD st = two_sum(p1, -p2);
        double la = std::fma(a.rh, b.rl, e1);
        la = std::fma(a.rl, b.rh, la);
        double lb = std::fma(a.ih, b.il, e2);
        lb = std::fma(a.il, b.ih, lb);
        double l = (la - lb) + st.lo;
        DD o = fast_two_sum(st.hi, l);
        r.rh = o.hi;
        r.rl = o.lo;
    }
    {
        double p3 = a.rh * b.ih, e3 = std::fma(a.rh, b.ih, -p3);
        double p4 = a.ih * b.rh, e4 = std::fma(a.ih, b.rh, -p4);
        DD st = two_sum(p3, p4);
        double lc = std::fma(a.rh, b.il, e3);
        lc = std::fma(a.rl, b.ih, lc);
        double ld = std::fma(a.ih, b.rl, e4);
        ld = std::fma(a.il, b.rh, ld);
        double l = (lc + ld) + st.lo;
        DD o = fast_two_sum(st.hi, l);
        r.ih = o.hi;
        r.il = o.lo;
    }
    return r;
}
// dd + dd with one renormalisation (11 adds per component)
static inline DD dd_add(DD a, DD b) {
    DD s = two_sum(a.hi, b.hi);
    double e = s.lo + (a.lo + b.lo);
    return fast_two_sum(s.hi, e);
}
static inline CDD cdd_add(CDD a, CDD b) {
    DD re = dd_add({a.rh, a.rl}, {b.rh, b.rl});
    DD im = dd_add({a.ih, a.il}, {b.ih, b.il});
    return {re.hi, re.lo, im.hi, im.lo};
}
// dd * small integer a (packing-time power rule, exact for a <= 255 and a double c)
static inline DD dd_mul_d(DD x, double a) {
    double p = x.hi * a;
    double e = std::fma(x.hi, a, -p);
    e = std::fma(x.lo, a, e);
    return fast_two_sum(p, e);
}

// ------------------------------------------------------------------ scalar traits
template <class T>
struct Ops;
template <>
struct Ops<CD> {
    static constexpr int W = 2;  // doubles per complex
    static CD zero() { return {0.0, 0.0}; }
    static CD one() { return {1.0, 0.0}; }
    static CD mul(CD a, CD b) { return cd_mul(a, b); }
    static CD add(CD a, CD b) { return cd_add(a, b); }
    static CD load(const double* p) { return {p[0], p[1]}; }
    static void store(double* p, CD v) { p[0] = v.re; p[1] = v.im; }
    // coefficient input is always (re_hi, re_lo, im_hi, im_lo); double mode uses the hi words
    static CD coeff(const double* c) { return {c[0], c[2]}; }
    // ref packing.cpp:47 / complex.hpp:25: double(a) * c, one rounding per component
    static CD scale(double a, CD c) { return {a * c.re, a * c.im}; }
    static double mag(CD v) { return std::hypot(v.re, v.im); }
};
template <>
struct Ops<CDD> {
    static constexpr int W = 4;
    static CDD zero() { return {0.0, 0.0, 0.0, 0.0}; }
    static CDD one() { return {1.0, 0.0, 0.0, 0.0}; }
    static CDD mul(CDD a, CDD b) { return cdd_mul(a, b); }
    static CDD add(CDD a, CDD b) { return cdd_add(a, b); }
    static CDD load(const double* p) { return {p[0], p[1], p[2], p[3]}; }
    static void store(double* p, CDD v) { p[0] = v.rh; p[1] = v.rl; p[2] = v.ih; p[3] = v.il; }
    static CDD coeff(const double* c) { return {c[0], c[1], c[2], c[3]}; }
    static CDD scale(double a, CDD c) {
        DD re = dd_mul_d({c.rh, c.rl}, a);
        DD im = dd_mul_d({c.ih, c.il}, a);
        return {re.hi, re.lo, im.hi, im.lo};
    }
    static double mag(CDD v) { return std::hypot(v.rh + v.rl, v.ih + v.il); }
};

struct Counts {
    uint64_t powers = 0, factors = 0, stage2 = 0, speel = 0, stage3 = 0;
};

struct System {
    int n, m, k, d;
    const int* pos;   // [s*k + j], 0-based
    const int* exps;  // [s*k + j], in [1, d]
    const double* coeffs;  // [s*4 + (re_hi, re_lo, im_hi, im_lo)]
};

// ref kernels.cpp:55-93 — operation order and operand order kept verbatim
template <class T>
void speelpenning(const T* v, int k, T* L, Counts& c) {
    using O = Ops<T>;
    if (k == 1) {
        L[0] = O::one();
        return;
    }
    if (k == 2) {
        L[0] = v[1];
        L[1] = v[0];
        return;
    }
    L[1] = v[0];
    for (int r = 0; r + 2 <= k - 1; ++r) {
        L[r + 2] = O::mul(L[r + 1], v[r + 1]);
        c.speel++;
    }
    T q = v[k - 1];
    L[k - 2] = O::mul(L[k - 2], q);
    c.speel++;
    for (int r = 1; r <= k - 3; ++r) {
        q = O::mul(q, v[k - 1 - r]);
        L[k - 2 - r] = O::mul(L[k - 2 - r], q);
        c.speel += 2;
    }
    q = O::mul(q, v[1]);
    L[0] = q;
    c.speel++;
}

// One evaluation at one point; mirrors ref engine.cpp:181-224 with the padded Mons buffer
// of ref packing.cpp:74-82 (kept literally: pads are added as exact zeros in stage 3).
template <class T>
void evaluate_one(const System& S, const std::vector<T>& dcoef, const std::vector<T>& vcoef,
                  const double* point, double* out, double* magsum, Counts& c) {
    using O = Ops<T>;
    const int n = S.n, m = S.m, k = S.k, d = S.d;
    const size_t nm = size_t(n) * m;
    const size_t stride = size_t(n) * n + n;

    std::vector<T> x(n);
    for (int i = 0; i < n; ++i) x[i] = O::load(point + size_t(i) * O::W);

    // stage 1a: power table, ref kernels.cpp:16-24
    std::vector<T> pw(size_t(n) * d);
    for (int i = 0; i < n; ++i) {
        T* row = pw.data() + size_t(i) * d;
        row[0] = O::one();
        if (d >= 2) row[1] = x[i];
        for (int e = 2; e < d; ++e) {
            row[e] = O::mul(row[e - 1], x[i]);
            c.powers++;
        }
    }

    std::vector<T> mons(stride * m, O::zero());
    std::vector<double> mmag(magsum ? stride * m : 0, 0.0);
    std::vector<T> L(k + 1), vals(k);
    for (size_t s = 0; s < nm; ++s) {
        const int* P = S.pos + s * k;
        const int* E = S.exps + s * k;
        // stage 1b: common factor, ref kernels.cpp:45-53
        T f = pw[size_t(P[0]) * d + (E[0] - 1)];
        for (int j = 1; j < k; ++j) f = O::mul(f, pw[size_t(P[j]) * d + (E[j] - 1)]);
        c.factors += k - 1;
        // stage 2, ref kernels.cpp:95-127
        for (int j = 0; j < k; ++j) vals[j] = x[P[j]];
        Counts sp;
        speelpenning(vals.data(), k, L.data(), sp);
        c.speel += sp.speel;
        c.stage2 += sp.speel;
        for (int j = 0; j < k; ++j) L[j] = O::mul(L[j], f);
        L[k] = O::mul(L[k - 1], vals[k - 1]);
        for (int j = 0; j < k; ++j) L[j] = O::mul(L[j], dcoef[size_t(j) * nm + s]);
        L[k] = O::mul(L[k], vcoef[s]);
        c.stage2 += 2 * uint64_t(k) + 2;
        // scatter through the slot map, ref packing.cpp:8-17
        const size_t p = s / m, g = s % m;
        for (int j = 0; j < k; ++j) {
            size_t slot = g * stride + size_t(P[j] + 1) * n + p;
            mons[slot] = L[j];
            if (magsum) mmag[slot] = O::mag(L[j]);
        }
        mons[g * stride + p] = L[k];
        if (magsum) mmag[g * stride + p] = O::mag(L[k]);
    }
    // stage 3, ref kernels.cpp:139-146, then the transpose of ref engine.cpp:215-223
    for (size_t t = 0; t < stride; ++t) {
        T acc = O::zero();
        double ms = 0.0;
        for (int j = 0; j < m; ++j) {
            acc = O::add(acc, mons[t + size_t(j) * stride]);
            if (magsum) ms += mmag[t + size_t(j) * stride];
        }
        size_t o;
        if (t < size_t(n)) {
            o = t;
        } else {
            size_t i = t / n - 1, p = t % n;
            o = n + p * n + i;
        }
        O::store(out + o * O::W, acc);
        if (magsum) magsum[o] = ms;
    }
}

// Ragged system (the repo's generalisation, include/polyjac_b200.h
// pj_ragged_desc): polynomial p owns terms [row_off[p], row_off[p+1]), term t owns
// [term_off[t], term_off[t+1]) of pos/exps. Literal restatement of the same reference sequence
// with the shape generalised: the padded Mons buffer has M = max_p m_p rows of S = n^2 + n slots
// (ref packing.cpp:74-82 with m -> M), term g of polynomial p scatters through the reference's
// slot map with m -> M (ref packing.cpp:8-17), every stage-3 sum runs over all M rows ascending
// (ref kernels.cpp:139-146, zero pads included), and each term runs stages 1-2 for its own k_t
// (ref kernels.cpp:45-127, the k = 1 / k = 2 Speelpenning special cases included).
struct Ragged {
    int n, d;
    const int* row_off;
    const int* term_off;
    const int* pos;
    const int* exps;
    const double* coeffs;
};
template <class T>
void evaluate_one_ragged(const Ragged& S, const double* point, double* out, double* magsum) {
    using O = Ops<T>;
    const int n = S.n, d = S.d;
    int M = 0;
    for (int p = 0; p < n; ++p) M = std::max(M, S.row_off[p + 1] - S.row_off[p]);
    const size_t stride = size_t(n) * n + n;
    std::vector<T> x(n);
    for (int i = 0; i < n; ++i) x[i] = O::load(point + size_t(i) * O::W);
    std::vector<T> pw(size_t(n) * d);
    for (int i = 0; i < n; ++i) {
        T* row = pw.data() + size_t(i) * d;
        row[0] = O::one();
        if (d >= 2) row[1] = x[i];
        for (int e = 2; e < d; ++e) row[e] = O::mul(row[e - 1], x[i]);
    }
    std::vector<T> mons(stride * M, O::zero());
    std::vector<double> mmag(magsum ? stride * M : 0, 0.0);
    Counts c;
    for (int p = 0; p < n; ++p)
        for (int t = S.row_off[p]; t < S.row_off[p + 1]; ++t) {
            const int g = t - S.row_off[p];
            const int k = S.term_off[t + 1] - S.term_off[t];
            const int* P = S.pos + S.term_off[t];
            const int* E = S.exps + S.term_off[t];
            const T cf = O::coeff(S.coeffs + 4 * size_t(t));
            std::vector<T> L(k + 1), vals(k);
            T f = pw[size_t(P[0]) * d + (E[0] - 1)];
            for (int j = 1; j < k; ++j) f = O::mul(f, pw[size_t(P[j]) * d + (E[j] - 1)]);
            for (int j = 0; j < k; ++j) vals[j] = x[P[j]];
            speelpenning(vals.data(), k, L.data(), c);
            for (int j = 0; j < k; ++j) L[j] = O::mul(L[j], f);
            L[k] = O::mul(L[k - 1], vals[k - 1]);
            for (int j = 0; j < k; ++j) L[j] = O::mul(L[j], O::scale(double(E[j]), cf));
            L[k] = O::mul(L[k], cf);
            for (int j = 0; j < k; ++j) {
                const size_t slot = size_t(g) * stride + size_t(P[j] + 1) * n + p;
                mons[slot] = L[j];
                if (magsum) mmag[slot] = O::mag(L[j]);
            }
            mons[size_t(g) * stride + p] = L[k];
            if (magsum) mmag[size_t(g) * stride + p] = O::mag(L[k]);
        }
    for (size_t t = 0; t < stride; ++t) {
        T acc = O::zero();
        double ms = 0.0;
        for (int j = 0; j < M; ++j) {
            acc = O::add(acc, mons[t + size_t(j) * stride]);
            if (magsum) ms += mmag[t + size_t(j) * stride];
        }
        const size_t o = t < size_t(n) ? t : n + (t % n) * n + (t / n - 1);
        O::store(out + o * O::W, acc);
        if (magsum) magsum[o] = ms;
    }
}

template <class T>
void pack_coeffs(const System& S, std::vector<T>& dcoef, std::vector<T>& vcoef) {
    using O = Ops<T>;
    const size_t nm = size_t(S.n) * S.m;
    dcoef.assign(nm * S.k, O::zero());
    vcoef.assign(nm, O::zero());
    for (size_t s = 0; s < nm; ++s) {
        T cf = O::coeff(S.coeffs + 4 * s);
        for (int j = 0; j < S.k; ++j) dcoef[size_t(j) * nm + s] = O::scale(double(S.exps[s * S.k + j]), cf);
        vcoef[s] = cf;
    }
}

template <class T>
void evaluate_range(const System& S, const double* pts, long b0, long b1, double* out,
                    double* magsum, Counts& c) {
    using O = Ops<T>;
    std::vector<T> dcoef, vcoef;
    pack_coeffs(S, dcoef, vcoef);
    const size_t nout = size_t(S.n) * S.n + S.n;
    for (long b = b0; b < b1; ++b) {
        evaluate_one<T>(S, dcoef, vcoef, pts + size_t(b) * S.n * O::W, out + size_t(b) * nout * O::W,
                        magsum ? magsum + size_t(b) * nout : nullptr, c);
    }
}


// ------------------------------------------------------------------ Newton corrector (f1)
// Restates the operation order defined in paper_1201_0499_b200/csrc/newton.cu (the reference
// has no Newton step): rhs = y + (-f); Gaussian elimination with implicit partial
// pivoting on |Re hi| + |Im hi| (maximum over the rows not yet pivoted, strictly positive, ties
// to the smallest row index); pivot inverse conj(a)/|a|^2 (dd: NT_DD::abs2, NT_DD::inv); multipliers l = A[i][kk] * inv
// (normalised product); trailing update A[i][j] + (-(l * A[piv][j])) with the dd product left
// unnormalised; back substitution dx_s = rhs[piv_s] * inv_s, then rhs[piv_t] + (-(A[piv_t][s] * dx_s))
// for t < s (descending s); x + dx.
// The dd pieces are restated from their published algorithms (Dekker product with FMA,
// Newton-corrected reciprocal), independently of the device copy.
static inline CDD cdd_mul_u(CDD a, CDD b) {  // product without the closing Fast2Sum
    CDD r;
    {
        double p1 = a.rh * b.rh, e1 = std::fma(a.rh, b.rh, -p1);
        double p2 = a.ih * b.ih, e2 = std::fma(a.ih, b.ih, -p2);
        DD st = two_sum(p1, -p2);
        double la = std::fma(a.rh, b.rl, e1);
        la = std::fma(a.rl, b.rh, la);
        double lb = std::fma(a.ih, b.il, e2);
        lb = std::fma(a.il, b.ih, lb);
        r.rh = st.hi;
        r.rl = (la - lb) + st.lo;
    }
    {
        double p3 = a.rh * b.ih, e3 = std::fma(a.rh, b.ih, -p3);
        double p4 = a.ih * b.rh, e4 = std::fma(a.ih, b.rh, -p4);
        DD st = two_sum(p3, p4);
        double lc = std::fma(a.rh, b.il, e3);
        lc = std::fma(a.rl, b.ih, lc);
        double ld = std::fma(a.ih, b.rl, e4);
        ld = std::fma(a.il, b.rh, ld);
        r.ih = st.hi;
        r.il = (lc + ld) + st.lo;
    }
    return r;
}
static inline DD dd_mul(DD a, DD b) {
    double p = a.hi * b.hi;
    double e = std::fma(a.hi, b.hi, -p);
    e = std::fma(a.hi, b.lo, e);
    e = std::fma(a.lo, b.hi, e);
    return fast_two_sum(p, e);
}
static inline DD dd_rcp(DD a) {
    double q = 1.0 / a.hi;
    double t = std::fma(-a.hi, q, 1.0);
    t = std::fma(-a.lo, q, t);
    return fast_two_sum(q, t * q);
}
struct NT_D {
    using T = CD;
    static constexpr int W = 2;
    static CD neg(CD a) { return {-a.re, -a.im}; }
    static double mag1(CD a) { return std::fabs(a.re) + std::fabs(a.im); }
    static double magmax(CD a) { return std::fmax(std::fabs(a.re), std::fabs(a.im)); }
    static bool finite(CD a) { return std::isfinite(a.re) && std::isfinite(a.im); }
    static CD umul(CD a, CD b) { return cd_mul(a, b); }
    static CD inv(CD a) {
        double den = a.re * a.re + a.im * a.im;
        double r = 1.0 / den;
        return {a.re * r, -a.im * r};
    }
};
struct NT_DD {
    using T = CDD;
    static constexpr int W = 4;
    static CDD neg(CDD a) { return {-a.rh, -a.rl, -a.ih, -a.il}; }
    static double mag1(CDD a) { return std::fabs(a.rh) + std::fabs(a.ih); }
    static double magmax(CDD a) { return std::fmax(std::fabs(a.rh), std::fabs(a.ih)); }
    static bool finite(CDD a) {
        return std::isfinite(a.rh) && std::isfinite(a.rl) && std::isfinite(a.ih) && std::isfinite(a.il);
    }
    static CDD umul(CDD a, CDD b) { return cdd_mul_u(a, b); }
    static DD abs2(DD re, DD im) {  // |a|^2: ordered Fast2Sum of the squares, errors in the low word
        const double p1 = re.hi * re.hi, p2 = im.hi * im.hi;
        double e1 = std::fma(re.hi, re.hi, -p1), e2 = std::fma(im.hi, im.hi, -p2);
        e1 = std::fma(re.hi + re.hi, re.lo, e1);
        e2 = std::fma(im.hi + im.hi, im.lo, e2);
        const DD s = fast_two_sum(std::fmax(p1, p2), std::fmin(p1, p2));
        return fast_two_sum(s.hi, s.lo + (e1 + e2));
    }
    static CDD inv(CDD a) {
        DD re{a.rh, a.rl}, im{a.ih, a.il};
        DD den = abs2(re, im);
        DD r = dd_rcp(den);
        DD o = dd_mul(re, r), p = dd_mul({-a.ih, -a.il}, r);
        return {o.hi, o.lo, p.hi, p.lo};
    }
};

template <class NT>
void newton_one(int n, const double* ev, const double* x, const double* y, double* xo, double* norms, int* status) {
    using T = typename NT::T;
    using O = Ops<T>;
    constexpr int W = NT::W;
    const int ld = n + 1;
    std::vector<T> A(size_t(n) * ld), inv(n);
    double rn = 0.0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) A[size_t(i) * ld + j] = O::load(ev + size_t(n + i * n + j) * W);
        T r = NT::neg(O::load(ev + size_t(i) * W));
        if (y) r = O::add(O::load(y + size_t(i) * W), r);
        A[size_t(i) * ld + n] = r;
        rn = std::fmax(rn, NT::magmax(r));
    }
    if (norms) norms[0] = rn;
    auto at = [&](int i, int j) -> T& { return A[size_t(i) * ld + j]; };
    // implicit pivoting: rows stay in place, piv[kk] records the pivot row of step kk
    std::vector<int> piv(n), step(n, n);
    for (int kk = 0; kk < n; ++kk) {
        double best = 0.0;
        int bi = -1;
        for (int i = 0; i < n; ++i) {  // ascending row index: ties go to the smallest
            if (step[i] < kk) continue;
            const double mg = NT::mag1(at(i, kk));
            if (mg > best) {
                best = mg;
                bi = i;
            }
        }
        if (bi < 0) {
            for (int i = 0; i < n; ++i) O::store(xo + size_t(i) * W, O::load(x + size_t(i) * W));
            if (norms) norms[1] = INFINITY;
            if (status) *status = 1;
            return;
        }
        piv[kk] = bi;
        step[bi] = kk;
        inv[kk] = NT::inv(at(bi, kk));
        for (int i = 0; i < n; ++i) {
            if (step[i] <= kk) continue;
            const T l = O::mul(at(i, kk), inv[kk]);
            at(i, kk) = l;
            for (int j = kk + 1; j <= n; ++j) at(i, j) = O::add(at(i, j), NT::neg(NT::umul(l, at(bi, j))));
        }
    }
    std::vector<T> dx(n);
    for (int s = n - 1; s >= 0; --s) {
        dx[s] = O::mul(at(piv[s], n), inv[s]);
        for (int t = 0; t < s; ++t) {
            T& r = at(piv[t], n);
            r = O::add(r, NT::neg(NT::umul(at(piv[t], s), dx[s])));
        }
    }
    double dn = 0.0;
    bool fin = true;
    for (int i = 0; i < n; ++i) {
        const T xn = O::add(O::load(x + size_t(i) * W), dx[i]);
        O::store(xo + size_t(i) * W, xn);
        dn = std::fmax(dn, NT::magmax(dx[i]));
        fin = fin && NT::finite(xn);
    }
    if (norms) norms[1] = dn;
    if (status) *status = fin ? 0 : 2;
}

// Mixed-precision solve (PJ_NEWTON_MIXED; csrc/newton.cu: nt_load_mixed / nt_mixed_finish):
// complex-double elimination of the high words of J and rhs (newton_one<NT_D>'s operation order),
// then kIters steps of iterative refinement with complex-dd residuals summed in four interleaved
// column groups, each correction solved with the double factors.
void newton_one_mixed(int n, const double* ev, const double* x, const double* y, double* xo, double* norms,
                      int* status) {
    using OD = Ops<CD>;
    using OQ = Ops<CDD>;
    constexpr int kIters = 2;
    const int ld = n + 1;
    auto J = [&](int i, int j) { return OQ::load(ev + size_t(n + i * n + j) * 4); };
    std::vector<CD> A(size_t(n) * ld), inv(n);
    std::vector<CDD> rhs(n);
    double rn = 0.0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            const CDD v = J(i, j);
            A[size_t(i) * ld + j] = CD{v.rh, v.ih};
        }
        CDD r = NT_DD::neg(OQ::load(ev + size_t(i) * 4));
        if (y) r = OQ::add(OQ::load(y + size_t(i) * 4), r);
        rhs[i] = r;
        A[size_t(i) * ld + n] = CD{r.rh, r.ih};
        rn = std::fmax(rn, NT_DD::magmax(r));
    }
    if (norms) norms[0] = rn;
    auto at = [&](int i, int j) -> CD& { return A[size_t(i) * ld + j]; };
    std::vector<int> piv(n), step(n, n);
    for (int kk = 0; kk < n; ++kk) {
        double best = 0.0;
        int bi = -1;
        for (int i = 0; i < n; ++i) {
            if (step[i] < kk) continue;
            const double mg = NT_D::mag1(at(i, kk));
            if (mg > best) {
                best = mg;
                bi = i;
            }
        }
        if (bi < 0) {
            for (int i = 0; i < n; ++i) OQ::store(xo + size_t(i) * 4, OQ::load(x + size_t(i) * 4));
            if (norms) norms[1] = INFINITY;
            if (status) *status = 1;
            return;
        }
        piv[kk] = bi;
        step[bi] = kk;
        inv[kk] = NT_D::inv(at(bi, kk));
        for (int i = 0; i < n; ++i) {
            if (step[i] <= kk) continue;
            const CD l = OD::mul(at(i, kk), inv[kk]);
            at(i, kk) = l;
            for (int j = kk + 1; j <= n; ++j) at(i, j) = OD::add(at(i, j), NT_D::neg(NT_D::umul(l, at(bi, j))));
        }
    }
    // triangular solves with the double factors on b (physical rows), in the kernel's order
    std::vector<CD> b(n), c(n);
    auto back = [&]() {
        for (int s = n - 1; s >= 0; --s) {
            c[s] = OD::mul(b[piv[s]], inv[s]);
            for (int t = 0; t < n; ++t)
                if (step[t] < s) b[t] = OD::add(b[t], NT_D::neg(NT_D::umul(at(t, s), c[s])));
        }
    };
    for (int i = 0; i < n; ++i) b[i] = at(i, n);
    back();
    std::vector<CDD> dx(n);
    for (int i = 0; i < n; ++i) dx[i] = CDD{c[i].re, 0.0, c[i].im, 0.0};
    double cmax = 0.0;
    for (int it = 0; it < kIters; ++it) {
        for (int i = 0; i < n; ++i) {
            CDD acc[4];
            for (int g = 0; g < 4; ++g) {
                acc[g] = CDD{0.0, 0.0, 0.0, 0.0};
                for (int j = g; j < n; j += 4) acc[g] = OQ::add(acc[g], NT_DD::umul(J(i, j), dx[j]));
            }
            const CDD r = OQ::add(rhs[i], NT_DD::neg(OQ::add(OQ::add(acc[0], acc[1]), OQ::add(acc[2], acc[3]))));
            b[i] = CD{r.rh, r.ih};
        }
        for (int kk = 0; kk < n; ++kk) {
            const CD bp = b[piv[kk]];
            for (int i = 0; i < n; ++i)
                if (step[i] > kk) b[i] = OD::add(b[i], NT_D::neg(NT_D::umul(at(i, kk), bp)));
        }
        back();
        cmax = 0.0;
        for (int i = 0; i < n; ++i) {
            dx[i] = OQ::add(dx[i], CDD{c[i].re, 0.0, c[i].im, 0.0});
            cmax = std::fmax(cmax, NT_D::magmax(c[i]));
        }
    }
    double dn = 0.0;
    bool fin = true;
    for (int i = 0; i < n; ++i) {
        const CDD xn = OQ::add(OQ::load(x + size_t(i) * 4), dx[i]);
        OQ::store(xo + size_t(i) * 4, xn);
        dn = std::fmax(dn, NT_DD::magmax(dx[i]));
        fin = fin && NT_DD::finite(xn);
    }
    if (norms) norms[1] = dn;
    if (status) *status = !fin ? 2 : (cmax > std::ldexp(dn, -64) ? 3 : 0);
}

}  // namespace oracle

extern "C" {

// prec: 1 = complex double (reference arithmetic), 2 = complex double-double.
// points: [B][n][W], out: [B][n + n*n][W] with W = 2 (double) or 4 (dd);
// magsum (nullable): [B][n + n*n] = sum over the m stage-3 terms of |term| (double).
// counts (nullable): powers, factors, stage2, speelpenning, stage3 multiplication tallies.
// threads > 1 shards the points contiguously (one private workspace per thread, the
// reference's recommended concurrency, ref engine.hpp:84-86).
int oracle_evaluate(int prec, int n, int m, int k, int d, const int* pos, const int* exps,
                    const double* coeffs, const double* points, long B, double* out,
                    double* magsum, unsigned long long* counts, int threads) {
    oracle::System S{n, m, k, d, pos, exps, coeffs};
    if (threads < 1) threads = 1;
    if (threads > B) threads = B > 0 ? int(B) : 1;
    std::vector<oracle::Counts> cs(threads);
    auto work = [&](int t) {
        long b0 = B * t / threads, b1 = B * (t + 1) / threads;
        if (prec == 1)
            oracle::evaluate_range<oracle::CD>(S, points, b0, b1, out, magsum, cs[t]);
        else
            oracle::evaluate_range<oracle::CDD>(S, points, b0, b1, out, magsum, cs[t]);
    };
    if (prec != 1 && prec != 2) return 1;
    if (threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
        for (auto& t : th) t.join();
    }
    if (counts) {
        oracle::Counts tot;
        for (auto& c : cs) {
            tot.powers += c.powers;
            tot.factors += c.factors;
            tot.stage2 += c.stage2;
            tot.speel += c.speel;
            tot.stage3 += c.stage3;
        }
        counts[0] = tot.powers;
        counts[1] = tot.factors;
        counts[2] = tot.stage2;
        counts[3] = tot.speel;
        counts[4] = tot.stage3;
    }
    return 0;
}

// Ragged evaluation (see evaluate_one_ragged); same buffers as oracle_evaluate.
int oracle_evaluate_ragged(int prec, int n, int d, const int* row_off, const int* term_off, const int* pos,
                           const int* exps, const double* coeffs, const double* points, long B, double* out,
                           double* magsum, int threads) {
    if (prec != 1 && prec != 2) return 1;
    oracle::Ragged S{n, d, row_off, term_off, pos, exps, coeffs};
    const int W = prec == 1 ? 2 : 4;
    const size_t nout = size_t(n) * n + n;
    if (threads < 1) threads = 1;
    if (threads > B) threads = B > 0 ? int(B) : 1;
    auto work = [&](int t) {
        for (long b = B * t / threads; b < B * (t + 1) / threads; ++b) {
            const double* pt = points + size_t(b) * n * W;
            double* o = out + size_t(b) * nout * W;
            double* ms = magsum ? magsum + size_t(b) * nout : nullptr;
            if (prec == 1)
                oracle::evaluate_one_ragged<oracle::CD>(S, pt, o, ms);
            else
                oracle::evaluate_one_ragged<oracle::CDD>(S, pt, o, ms);
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < threads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& t : th) t.join();
    return 0;
}

// Speelpenning gradient alone (ref kernels.cpp:55-93) for the known-answer tests.
int oracle_speelpenning(int prec, int k, const double* vals, double* L, unsigned long long* mults) {
    oracle::Counts c;
    if (prec == 1) {
        std::vector<oracle::CD> v(k), l(k + 1);
        for (int j = 0; j < k; ++j) v[j] = oracle::Ops<oracle::CD>::load(vals + 2 * j);
        oracle::speelpenning(v.data(), k, l.data(), c);
        for (int j = 0; j < k; ++j) oracle::Ops<oracle::CD>::store(L + 2 * j, l[j]);
    } else {
        std::vector<oracle::CDD> v(k), l(k + 1);
        for (int j = 0; j < k; ++j) v[j] = oracle::Ops<oracle::CDD>::load(vals + 4 * j);
        oracle::speelpenning(v.data(), k, l.data(), c);
        for (int j = 0; j < k; ++j) oracle::Ops<oracle::CDD>::store(L + 4 * j, l[j]);
    }
    if (mults) *mults = c.speel;
    return 0;
}

// The complex dd primitives alone, for primitive-level parity with the device code.
void oracle_cdd_mul(const double* a, const double* b, double* r) {
    oracle::Ops<oracle::CDD>::store(r, oracle::cdd_mul(oracle::Ops<oracle::CDD>::load(a),
                                                       oracle::Ops<oracle::CDD>::load(b)));
}
void oracle_cdd_add(const double* a, const double* b, double* r) {
    oracle::Ops<oracle::CDD>::store(r, oracle::cdd_add(oracle::Ops<oracle::CDD>::load(a),
                                                       oracle::Ops<oracle::CDD>::load(b)));
}

// Slot map and zero mask restated from ref packing.cpp:8-17 and :54-72.
// Returns the slot, or -1 where the reference throws std::out_of_range.
long long oracle_mons_slot(long long s, int kind, int var, int n, int m) {
    long long nm = (long long)n * m;
    if (s < 0 || s >= nm) return -1;
    long long p = s / m, g = s % m, stride = (long long)n * n + n;
    if (kind == 0) return g * stride + p;
    if (var < 0 || var >= n) return -1;
    return g * stride + (long long)(var + 1) * n + p;
}

// Writes the ascending zero mask into mask (capacity (n^2+n)m); returns its length.
long long oracle_zero_mask(int n, int m, int k, const int* pos, long long* mask) {
    const long long nm = (long long)n * m, stride = (long long)n * n + n;
    std::vector<unsigned char> claimed(size_t(stride * m), 0);
    for (long long s = 0; s < nm; ++s) {
        claimed[size_t(oracle_mons_slot(s, 0, -1, n, m))] = 1;
        for (int j = 0; j < k; ++j) claimed[size_t(oracle_mons_slot(s, 1, pos[s * k + j], n, m))] = 1;
    }
    long long len = 0;
    for (long long i = 0; i < stride * m; ++i)
        if (!claimed[size_t(i)]) mask[len++] = i;
    return len;
}

// Newton corrector restatement (see newton_one): evals [B][n+n*n][W], points/target/out
// [B][n][W] (target nullable), norms [B][2] and status [B] nullable.
int oracle_newton_solve(int prec, int n, const double* evals, const double* points, const double* target, long B,
                        double* out, double* norms, int* status, int threads) {
    if (prec != 1 && prec != 2 && prec != 3) return 1;  // 3: the mixed solve (dd input)
    if (prec == 3 && n > 32) return 1;
    const int W = prec == 1 ? 2 : 4;
    const size_t nout = size_t(n) * n + n;
    if (threads < 1) threads = 1;
    if (threads > B) threads = B > 0 ? int(B) : 1;
    auto work = [&](int t) {
        long b0 = B * t / threads, b1 = B * (t + 1) / threads;
        for (long b = b0; b < b1; ++b) {
            const double* ev = evals + size_t(b) * nout * W;
            const double* x = points + size_t(b) * n * W;
            const double* y = target ? target + size_t(b) * n * W : nullptr;
            double* xo = out + size_t(b) * n * W;
            double* nr = norms ? norms + 2 * b : nullptr;
            int* st = status ? status + b : nullptr;
            if (prec == 1)
                oracle::newton_one<oracle::NT_D>(n, ev, x, y, xo, nr, st);
            else if (prec == 3)
                oracle::newton_one_mixed(n, ev, x, y, xo, nr, st);
            else
                oracle::newton_one<oracle::NT_DD>(n, ev, x, y, xo, nr, st);
        }
    };
    if (threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
        for (auto& t : th) t.join();
    }
    return 0;
}

}  // extern "C"
