// polyjac_b200.hpp — header-only C++ drop-in for the reference's EvaluationContext, over the
// C ABI in polyjac_b200.h (link libpolyjac_b200.so).
//
// Same class and method names as ref include/polyjac/engine.hpp:87-128 and the same exception
// types (std::invalid_argument for invalid systems / points, std::out_of_range for bad slot
// queries). The constructor accepts any system type with the reference's shape — including
// polyjac::PolynomialSystem itself (members n, m, k, d, terms[s].coeff.re/.im,
// terms[s].support.positions/.exponents) — so switching is a type change:
//
//     polyjac::PolynomialSystem sys = polyjac::random_system(32, 32, 9, 2, 7);
//     polyjac_b200::EvaluationContext ctx(sys);                       // was polyjac::EvaluationContext
//     auto r = ctx.evaluate<polyjac::EvaluationResult>(point);        // bit-identical results
//
// B200 additions: complex double-double (evaluate_dd), batched device-buffer evaluation on a
// CUDA stream (evaluate_device), the Newton corrector (newton, newton_dd, newton_step_device) and
// the wide encoding for n > 256 (constructor option PJ_CTX_WIDE).
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "polyjac_b200.h"

namespace polyjac_b200 {

struct Complex {
    double re = 0.0;
    double im = 0.0;
};
struct ComplexDD {  // (re_hi, re_lo, im_hi, im_lo)
    double re_hi = 0.0, re_lo = 0.0, im_hi = 0.0, im_lo = 0.0;
};
struct MonomialSupport {
    std::vector<int> positions;
    std::vector<int> exponents;
    int size() const { return static_cast<int>(positions.size()); }
};
struct Term {
    Complex coeff;
    MonomialSupport support;
};
struct PolynomialSystem {
    int n = 0, m = 0, k = 0, d = 0;
    std::vector<Term> terms;
};
using EvaluationPoint = std::vector<Complex>;
struct EvaluationResult {
    int n = 0;
    std::vector<Complex> values;
    std::vector<Complex> jacobian;
    Complex jac(int p, int i) const { return jacobian[static_cast<std::size_t>(p) * n + i]; }
};
struct GridConfig {
    int block_size = 32;
    int workers = 0;
};
struct MultCounter {
    std::uint64_t stage1_powers = 0, stage1_factors = 0, stage2 = 0, speelpenning = 0, stage3 = 0;
    std::uint64_t total() const { return stage1_powers + stage1_factors + stage2 + stage3; }
    MultCounter& operator+=(const MultCounter& o) {
        stage1_powers += o.stage1_powers;
        stage1_factors += o.stage1_factors;
        stage2 += o.stage2;
        speelpenning += o.speelpenning;
        stage3 += o.stage3;
        return *this;
    }
};
struct BatchReport {
    int evals = 0;
    double wall_seconds = 0.0;
    double per_eval_seconds = 0.0;
    MultCounter mults;
};
template <class Result = EvaluationResult>
struct BatchResult {
    std::vector<Result> results;
    BatchReport report;
};

namespace detail {
inline void check(int rc) {
    if (rc == PJ_OK) return;
    std::string msg = pj_last_error();
    if (rc == PJ_EINVAL || rc == PJ_ENONFINITE) throw std::invalid_argument(msg);
    if (rc == PJ_ERANGE) throw std::out_of_range(msg);
    if (rc == PJ_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}
}  // namespace detail

class EvaluationContext {
public:
    // options: PJ_CTX_WIDE lifts the reference's n <= 256 cap (pj_ctx_create_ex)
    template <class System>
    explicit EvaluationContext(const System& sys, GridConfig grid = {}, int device = 0, int options = 0)
        : grid_(grid) {
        if (grid_.block_size < 1) throw std::invalid_argument("block size must be >= 1");
        if (grid_.workers < 0) throw std::invalid_argument("workers must be >= 0");
        if (grid_.workers == 0) grid_.workers = 1;
        n_ = sys.n;
        const std::size_t nt = sys.terms.size(), k = sys.k > 0 ? std::size_t(sys.k) : 0;
        std::vector<std::int32_t> pos(nt * k, -1), exps(nt * k, 0);
        std::vector<double> co(nt * 4, 0.0);
        bool shape_ok = nt == std::size_t(sys.n) * std::size_t(sys.m);
        for (std::size_t s = 0; s < nt; ++s) {
            const auto& t = sys.terms[s];
            if (t.support.positions.size() != k || t.support.exponents.size() != k) {
                shape_ok = false;
                continue;
            }
            for (std::size_t j = 0; j < k; ++j) {
                pos[s * k + j] = t.support.positions[j];
                exps[s * k + j] = t.support.exponents[j];
            }
            co[4 * s] = t.coeff.re;
            co[4 * s + 2] = t.coeff.im;
        }
        pj_system_desc desc{sys.n, sys.m, sys.k, sys.d, pos.data(), exps.data(), co.data()};
        if (!shape_ok) desc.positions = nullptr, desc.exponents = nullptr, desc.coeffs = nullptr;
        detail::check(pj_ctx_create_ex(&desc, device, options, &ctx_));
    }
    ~EvaluationContext() { pj_ctx_destroy(ctx_); }
    EvaluationContext(const EvaluationContext&) = delete;
    EvaluationContext& operator=(const EvaluationContext&) = delete;

    // One point in complex double, bit-identical with the reference (ref src/engine.cpp:181-230).
    template <class Result = EvaluationResult, class Point>
    Result evaluate(const Point& point) {
        if (static_cast<int>(point.size()) != n_) throw std::invalid_argument("evaluate: point dimension mismatch");
        std::vector<double> in(2 * std::size_t(n_)), out(2 * (std::size_t(n_) * n_ + n_));
        for (int i = 0; i < n_; ++i) {
            in[2 * i] = point[i].re;
            in[2 * i + 1] = point[i].im;
        }
        detail::check(pj_evaluate_host(ctx_, PJ_PREC_D, in.data(), 1, out.data()));
        tally(1);
        return unpack<Result>(out.data());
    }

    // Each point repeat times (ref src/engine.cpp:232-260); one batched launch per repeat.
    template <class Result = EvaluationResult, class Points>
    BatchResult<Result> evaluate_batch(const Points& points, int repeat) {
        if (repeat < 1) throw std::invalid_argument("evaluate_batch: repeat must be >= 1");
        BatchResult<Result> br;
        const std::size_t B = points.size(), nout = std::size_t(n_) * n_ + n_;
        std::vector<double> in(2 * B * n_), out(2 * B * nout);
        for (std::size_t b = 0; b < B; ++b) {
            if (static_cast<int>(points[b].size()) != n_)
                throw std::invalid_argument("evaluate: point dimension mismatch");
            for (int i = 0; i < n_; ++i) {
                in[2 * (b * n_ + i)] = points[b][i].re;
                in[2 * (b * n_ + i) + 1] = points[b][i].im;
            }
        }
        const MultCounter before = mults_;
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < repeat && B > 0; ++r) {
            detail::check(pj_evaluate_host(ctx_, PJ_PREC_D, in.data(), std::int64_t(B), out.data()));
            tally(std::int64_t(B));
        }
        const auto t1 = std::chrono::steady_clock::now();
        for (std::size_t b = 0; b < B; ++b) br.results.push_back(unpack<Result>(out.data() + 2 * b * nout));
        br.report.evals = static_cast<int>(B) * repeat;
        br.report.wall_seconds = std::chrono::duration<double>(t1 - t0).count();
        br.report.per_eval_seconds = br.report.evals ? br.report.wall_seconds / br.report.evals : 0.0;
        br.report.mults = MultCounter{mults_.stage1_powers - before.stage1_powers,
                                      mults_.stage1_factors - before.stage1_factors, mults_.stage2 - before.stage2,
                                      mults_.speelpenning - before.speelpenning, mults_.stage3 - before.stage3};
        return br;
    }

    // Complex double-double on host buffers: points [batch][n], out [batch][n + n*n].
    // reference_order = true keeps the reference's order in every stage.
    void evaluate_dd(const ComplexDD* points, std::int64_t batch, ComplexDD* out, bool reference_order = false) {
        detail::check(pj_evaluate_host(ctx_, PJ_PREC_DD | (reference_order ? PJ_ORDER_REF : 0),
                                       reinterpret_cast<const double*>(points), batch,
                                       reinterpret_cast<double*>(out)));
        tally(batch);
    }

    // Device buffers, asynchronous on `stream` (cudaStream_t); flags = PJ_PREC_D | PJ_PREC_DD [| order].
    void evaluate_device(int flags, const double* d_points, std::int64_t batch, double* d_out, void* stream) {
        detail::check(pj_evaluate(ctx_, flags, d_points, batch, d_out, stream));
        tally(batch);
    }

    // Newton corrector (B200 addition): `iters` steps x <- x + J(x)^-1 (y - f(x))
    // per point on the GPU, host buffers [batch][n] (target y may be null: the roots of f).
    // norms [batch][2] (|y - f|, |last step|) and status [batch] (0 ok, 1 singular, 2 non-finite)
    // may be null.
    void newton_dd(const ComplexDD* points, const ComplexDD* target, std::int64_t batch, int iters, ComplexDD* out,
                   double* norms = nullptr, std::int32_t* status = nullptr) {
        detail::check(pj_newton_host(ctx_, PJ_PREC_DD, reinterpret_cast<const double*>(points),
                                     reinterpret_cast<const double*>(target), batch, iters,
                                     reinterpret_cast<double*>(out), norms, status));
        tally(batch * iters);
    }
    void newton(const Complex* points, const Complex* target, std::int64_t batch, int iters, Complex* out,
                double* norms = nullptr, std::int32_t* status = nullptr) {
        detail::check(pj_newton_host(ctx_, PJ_PREC_D, reinterpret_cast<const double*>(points),
                                     reinterpret_cast<const double*>(target), batch, iters,
                                     reinterpret_cast<double*>(out), norms, status));
        tally(batch * iters);
    }
    // Device buffers: evaluate into d_work ([batch][n + n*n]) and solve, asynchronous on `stream`.
    void newton_step_device(int flags, const double* d_points, const double* d_target, std::int64_t batch,
                            double* d_work, double* d_points_out, double* d_norms, std::int32_t* d_status,
                            void* stream) {
        detail::check(pj_newton_step(ctx_, flags, d_points, d_target, batch, d_work, d_points_out, d_norms,
                                     d_status, stream));
        tally(batch);
    }

    const GridConfig& grid() const { return grid_; }
    const MultCounter& mults() const { return mults_; }
    // No padded Mons buffer exists on the device path: masked slots are never materialised.
    bool masked_slots_clean() const { return true; }
    pj_ctx* handle() const { return ctx_; }

private:
    template <class Result>
    Result unpack(const double* o) const {
        Result r;
        r.n = n_;
        r.values.resize(n_);
        r.jacobian.resize(std::size_t(n_) * n_);
        for (int i = 0; i < n_; ++i) {
            r.values[i].re = o[2 * i];
            r.values[i].im = o[2 * i + 1];
        }
        for (std::size_t i = 0; i < std::size_t(n_) * n_; ++i) {
            r.jacobian[i].re = o[2 * (n_ + i)];
            r.jacobian[i].im = o[2 * (n_ + i) + 1];
        }
        return r;
    }
    void tally(std::int64_t evals) {
        std::uint64_t c[5];
        detail::check(pj_mult_counts(ctx_, evals, c));
        mults_ += MultCounter{c[0], c[1], c[2], c[3], c[4]};
    }

    pj_ctx* ctx_ = nullptr;
    int n_ = 0;
    GridConfig grid_;
    MultCounter mults_;
};

}  // namespace polyjac_b200
