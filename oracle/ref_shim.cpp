// ORACLE — test infrastructure only (see oracle/oracle.cpp header).
//
// extern "C" binding over the UNMODIFIED reference library, compiled from the sources where
// they lie under /root/reference/proj/src by oracle/Makefile into oracle/_ref/ (git-ignored).
// No reference source is copied here; this file only calls the reference's public API:
//   random_system / random_points        ref/include/polyjac/system.hpp:73-84
//   validate_system                      ref/include/polyjac/system.hpp:69
//   build_layout / mons_slot / zero_mask ref/include/polyjac/packing.hpp:67-88
//   stage2_slot_targets                  ref/include/polyjac/kernels.hpp:86
//   EvaluationContext::evaluate          ref/include/polyjac/engine.hpp:89-98
//   naive_evaluate / naive_jacobian      ref/include/polyjac/oracle.hpp:16-23
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include <sstream>

#include "polyjac/engine.hpp"
#include "polyjac/io.hpp"
#include "polyjac/oracle.hpp"
#include "polyjac/packing.hpp"
#include "polyjac/system.hpp"

using namespace polyjac;

namespace {
thread_local std::string g_err;

PolynomialSystem make_system(int n, int m, int k, int d, const int* pos, const int* exps,
                             const double* coeffs) {
    PolynomialSystem sys;
    sys.n = n;
    sys.m = m;
    sys.k = k;
    sys.d = d;
    sys.terms.resize(size_t(n) * m);
    for (size_t s = 0; s < sys.terms.size(); ++s) {
        Term& t = sys.terms[s];
        t.coeff = {coeffs[4 * s + 0], coeffs[4 * s + 2]};
        t.support.positions.assign(pos + s * k, pos + s * k + k);
        t.support.exponents.assign(exps + s * k, exps + s * k + k);
    }
    return sys;
}
}  // namespace

extern "C" {
#pragma GCC visibility push(default)

const char* ref_last_error() { return g_err.c_str(); }

// coeffs out: [nm][4] (re, 0, im, 0); pos/exps out: [nm*k]
int ref_random_system(int n, int m, int k, int d, unsigned long long seed, int* pos, int* exps,
                      double* coeffs) {
    try {
        PolynomialSystem sys = random_system(n, m, k, d, seed);
        for (size_t s = 0; s < sys.terms.size(); ++s) {
            const Term& t = sys.terms[s];
            for (int j = 0; j < k; ++j) {
                pos[s * k + j] = t.support.positions[j];
                exps[s * k + j] = t.support.exponents[j];
            }
            coeffs[4 * s + 0] = t.coeff.re;
            coeffs[4 * s + 1] = 0.0;
            coeffs[4 * s + 2] = t.coeff.im;
            coeffs[4 * s + 3] = 0.0;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// out: [count][n][2]
int ref_random_points(int n, int count, unsigned long long seed, double* out) {
    try {
        auto pts = random_points(n, count, seed);
        for (int b = 0; b < count; ++b)
            for (int i = 0; i < n; ++i) {
                out[(size_t(b) * n + i) * 2 + 0] = pts[b][i].re;
                out[(size_t(b) * n + i) * 2 + 1] = pts[b][i].im;
            }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// number of violations; first one's text in ref_last_error()
int ref_validate(int n, int m, int k, int d, const int* pos, const int* exps, const double* coeffs,
                 long long nterms) {
    PolynomialSystem sys;
    sys.n = n;
    sys.m = m;
    sys.k = k;
    sys.d = d;
    sys.terms.resize(size_t(nterms));
    for (long long s = 0; s < nterms; ++s) {
        Term& t = sys.terms[size_t(s)];
        t.coeff = {coeffs[4 * s + 0], coeffs[4 * s + 2]};
        t.support.positions.assign(pos + s * k, pos + s * k + k);
        t.support.exponents.assign(exps + s * k, exps + s * k + k);
    }
    ValidationReport r = validate_system(sys);
    g_err = r.ok() ? "" : r.violations.front().describe();
    return int(r.violations.size());
}

// 0 ok; 1 if build_layout throws (message in ref_last_error)
int ref_build_layout(int n, int m, int k, int d, const int* pos, const int* exps,
                     const double* coeffs, unsigned char* positions, unsigned char* exponents,
                     double* lcoeffs /* [(k+1)*nm][2] */) {
    try {
        PackedLayout L = build_layout(make_system(n, m, k, d, pos, exps, coeffs));
        std::memcpy(positions, L.positions.data(), L.positions.size());
        std::memcpy(exponents, L.exponents.data(), L.exponents.size());
        for (size_t i = 0; i < L.coeffs.size(); ++i) {
            lcoeffs[2 * i] = L.coeffs[i].re;
            lcoeffs[2 * i + 1] = L.coeffs[i].im;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

long long ref_mons_slot(long long s, int kind, int var, int n, int m) {
    try {
        return (long long)mons_slot(size_t(s), kind == 0 ? SlotKind::value : SlotKind::derivative,
                                    var, n, m);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

long long ref_zero_mask(int n, int m, int k, int d, const int* pos, const int* exps,
                        const double* coeffs, long long* mask) {
    auto v = zero_mask(make_system(n, m, k, d, pos, exps, coeffs));
    for (size_t i = 0; i < v.size(); ++i) mask[i] = (long long)v[i];
    return (long long)v.size();
}

// targets: [nm][k+1]
int ref_slot_targets(int n, int m, int k, int d, const int* pos, const int* exps,
                     const double* coeffs, long long* targets) {
    try {
        PackedLayout L = build_layout(make_system(n, m, k, d, pos, exps, coeffs));
        for (size_t s = 0; s < L.monomial_count(); ++s) {
            auto t = stage2_slot_targets(L, s);
            for (int j = 0; j <= k; ++j) targets[s * (k + 1) + j] = (long long)t[j];
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// EvaluationContext::evaluate over a batch; points [B][n][2], out [B][n+n*n][2]
// (values then row-major Jacobian). threads > 1: one workers=1 context per thread over a
// contiguous shard (the fair CPU baseline). mults: total tally.
// Returns 0, 1 on a thrown exception (message in ref_last_error).
int ref_evaluate(int n, int m, int k, int d, const int* pos, const int* exps, const double* coeffs,
                 const double* points, long long B, double* out, int threads, int block_size,
                 int workers, unsigned long long* mults, double* seconds) {
    try {
        PolynomialSystem sys = make_system(n, m, k, d, pos, exps, coeffs);
        if (threads < 1) threads = 1;
        if (B < threads) threads = B > 0 ? int(B) : 1;
        std::vector<std::exception_ptr> errs(threads);
        std::vector<unsigned long long> tallies(threads, 0);
        const size_t nout = size_t(n) * n + n;
        auto work = [&](int t) {
            try {
                EvaluationContext ctx(sys, {block_size, workers});
                long long b0 = B * t / threads, b1 = B * (t + 1) / threads;
                EvaluationPoint pt(n);
                for (long long b = b0; b < b1; ++b) {
                    for (int i = 0; i < n; ++i)
                        pt[i] = {points[(size_t(b) * n + i) * 2], points[(size_t(b) * n + i) * 2 + 1]};
                    EvaluationResult r = ctx.evaluate(pt);
                    double* o = out + size_t(b) * nout * 2;
                    for (int i = 0; i < n; ++i) {
                        o[2 * i] = r.values[i].re;
                        o[2 * i + 1] = r.values[i].im;
                    }
                    for (size_t i = 0; i < size_t(n) * n; ++i) {
                        o[2 * (n + i)] = r.jacobian[i].re;
                        o[2 * (n + i) + 1] = r.jacobian[i].im;
                    }
                }
                tallies[t] = ctx.mults().total();
            } catch (...) {
                errs[t] = std::current_exception();
            }
        };
        auto t0 = std::chrono::steady_clock::now();
        if (threads == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
            for (auto& t : th) t.join();
        }
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        if (mults) {
            *mults = 0;
            for (auto v : tallies) *mults += v;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// naive oracle of the reference (complex double): out [n+n*n][2]
int ref_naive(int n, int m, int k, int d, const int* pos, const int* exps, const double* coeffs,
              const double* point, double* out) {
    try {
        PolynomialSystem sys = make_system(n, m, k, d, pos, exps, coeffs);
        EvaluationPoint pt(n);
        for (int i = 0; i < n; ++i) pt[i] = {point[2 * i], point[2 * i + 1]};
        auto v = naive_evaluate(sys, pt);
        auto j = naive_jacobian(sys, pt);
        for (int i = 0; i < n; ++i) {
            out[2 * i] = v[i].re;
            out[2 * i + 1] = v[i].im;
        }
        for (size_t i = 0; i < j.size(); ++i) {
            out[2 * (n + i)] = j[i].re;
            out[2 * (n + i) + 1] = j[i].im;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// reference write_system into buf (capacity cap); returns the text length
long long ref_write_system(int n, int m, int k, int d, const int* pos, const int* exps, const double* coeffs,
                           char* buf, long long cap) {
    std::ostringstream os;
    write_system(make_system(n, m, k, d, pos, exps, coeffs), os);
    const std::string t = os.str();
    if (buf && cap > 0) {
        const size_t nb = std::min<size_t>(size_t(cap) - 1, t.size());
        std::memcpy(buf, t.data(), nb);
        buf[nb] = 0;
    }
    return (long long)t.size();
}

// reference read_system from text: 0 ok (arrays sized by the caller from the header), 1 on
// FormatError (message in ref_last_error). dims[4] receives n m k d.
int ref_read_system(const char* text, int* dims, int* pos, int* exps, double* coeffs, long long cap_terms) {
    try {
        std::istringstream is(text);
        PolynomialSystem sys = read_system(is, "<test>");
        dims[0] = sys.n;
        dims[1] = sys.m;
        dims[2] = sys.k;
        dims[3] = sys.d;
        if ((long long)sys.terms.size() > cap_terms) return 0;
        for (size_t s = 0; s < sys.terms.size(); ++s) {
            for (int j = 0; j < sys.k; ++j) {
                pos[s * sys.k + j] = sys.terms[s].support.positions[j];
                exps[s * sys.k + j] = sys.terms[s].support.exponents[j];
            }
            coeffs[4 * s] = sys.terms[s].coeff.re;
            coeffs[4 * s + 1] = 0.0;
            coeffs[4 * s + 2] = sys.terms[s].coeff.im;
            coeffs[4 * s + 3] = 0.0;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

#pragma GCC visibility pop
}  // extern "C"
