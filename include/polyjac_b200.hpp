// polyjac_b200.hpp — header-only C++ drop-in for the reference's EvaluationContext, over the
// C ABI in polyjac_b200.h (link libpolyjac_b200.so).
//
// Same class and method names, argument types and exception types as
// ref include/polyjac/engine.hpp:87-128 (std::invalid_argument for invalid systems / points,
// std::out_of_range for bad slot queries). The class is a template over a "type family"
// (Complex, EvaluationPoint, EvaluationResult, BatchResult, PackedLayout, MultCounter,
// GridConfig):
//
//   * polyjac_b200::EvaluationContext uses this header's own mirrors of the reference types;
//   * polyjac_b200_dropin.hpp instantiates it over the reference's own types, so that with the
//     reference headers in scope switching is a type change and every call keeps its syntax:
//
//       polyjac::PolynomialSystem sys = polyjac::random_system(32, 32, 9, 2, 7);
//       polyjac_b200::dropin::EvaluationContext ctx(sys);   // was polyjac::EvaluationContext
//       polyjac::EvaluationResult r = ctx.evaluate(point);  // bit-identical results
//       std::size_t fp = ctx.layout().footprint_bytes();    // the reference's PackedLayout
//
// B200 additions: complex double-double (evaluate_dd), batched device-buffer evaluation on a
// CUDA stream (evaluate_device), the Newton corrector (newton, newton_dd, newton_step_device) and
// the wide encoding for n > 256 (constructor option PJ_CTX_WIDE).
#pragma once

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
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
    friend bool operator==(const MultCounter& a, const MultCounter& b) {
        return a.stage1_powers == b.stage1_powers && a.stage1_factors == b.stage1_factors && a.stage2 == b.stage2 &&
               a.speelpenning == b.speelpenning && a.stage3 == b.stage3;
    }
};
struct BatchReport {
    int evals = 0;
    double wall_seconds = 0.0;
    double per_eval_seconds = 0.0;
    MultCounter mults;
};
struct BatchResult {
    std::vector<EvaluationResult> results;
    BatchReport report;
};
// ref include/polyjac/packing.hpp:24-46
struct PackedLayout {
    int n = 0, m = 0, k = 0, d = 0;
    std::vector<std::uint8_t> positions;
    std::vector<std::uint8_t> exponents;
    std::vector<Complex> coeffs;
    std::size_t monomial_count() const { return static_cast<std::size_t>(n) * m; }
    int position(std::size_t s, int j) const { return positions[s * k + j]; }
    int exponent_minus_1(std::size_t s, int j) const { return exponents[s * k + j]; }
    Complex deriv_coeff(std::size_t s, int j) const { return coeffs[static_cast<std::size_t>(j) * monomial_count() + s]; }
    Complex value_coeff(std::size_t s) const { return coeffs[static_cast<std::size_t>(k) * monomial_count() + s]; }
    std::size_t footprint_bytes() const { return positions.size() + exponents.size(); }
};

// The type family of polyjac_b200::EvaluationContext.
struct OwnTypes {
    using Complex = polyjac_b200::Complex;
    using EvaluationPoint = polyjac_b200::EvaluationPoint;
    using EvaluationResult = polyjac_b200::EvaluationResult;
    using BatchResult = polyjac_b200::BatchResult;
    using PackedLayout = polyjac_b200::PackedLayout;
    using MultCounter = polyjac_b200::MultCounter;
    using GridConfig = polyjac_b200::GridConfig;
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

template <class Types>
class BasicEvaluationContext {
public:
    using Complex = typename Types::Complex;
    using EvaluationPoint = typename Types::EvaluationPoint;
    using EvaluationResult = typename Types::EvaluationResult;
    using BatchResult = typename Types::BatchResult;
    using PackedLayout = typename Types::PackedLayout;
    using MultCounter = typename Types::MultCounter;
    using GridConfig = typename Types::GridConfig;

    // ref src/engine.cpp:168-179. Accepts any system type with the reference's shape (members n,
    // m, k, d, terms[s].coeff.re/.im, terms[s].support.positions/.exponents).
    // options: PJ_CTX_WIDE lifts the reference's n <= 256 cap (pj_ctx_create_ex).
    template <class System>
    explicit BasicEvaluationContext(const System& sys, GridConfig grid = {}, int device = 0, int options = 0)
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
        const std::int64_t nz = pj_structural_zeros(ctx_, nullptr);
        if (nz > 0) {
            std::vector<std::uint8_t> mask(std::size_t(n_) * n_);
            pj_structural_zeros(ctx_, mask.data());
            for (std::size_t i = 0; i < mask.size(); ++i)
                if (mask[i]) zeros_.push_back(i);
        }
    }
    ~BasicEvaluationContext() { pj_ctx_destroy(ctx_); }
    BasicEvaluationContext(const BasicEvaluationContext&) = delete;
    BasicEvaluationContext& operator=(const BasicEvaluationContext&) = delete;

    // One point in complex double, bit-identical with the reference (ref src/engine.cpp:181-230):
    // std::invalid_argument on a dimension mismatch or a non-finite coordinate.
    EvaluationResult evaluate(const EvaluationPoint& point) {
        if (static_cast<int>(point.size()) != n_) throw std::invalid_argument("evaluate: point dimension mismatch");
        std::vector<double> in(2 * std::size_t(n_)), out(2 * (std::size_t(n_) * n_ + n_));
        for (int i = 0; i < n_; ++i) {
            in[2 * i] = point[i].re;
            in[2 * i + 1] = point[i].im;
        }
        detail::check(pj_evaluate_host(ctx_, PJ_PREC_D, in.data(), 1, out.data()));
        tally(1);
        audit(out.data(), 2);
        return unpack(out.data());
    }

    // Each point `repeat` times (ref src/engine.cpp:232-260); one batched launch per repeat.
    BatchResult evaluate_batch(const std::vector<EvaluationPoint>& points, int repeat) {
        if (repeat < 1) throw std::invalid_argument("evaluate_batch: repeat must be >= 1");
        BatchResult br;
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
        for (std::size_t b = 0; b < B; ++b) {
            audit(out.data() + 2 * b * nout, 2);
            br.results.push_back(unpack(out.data() + 2 * b * nout));
        }
        br.report.evals = static_cast<int>(B) * repeat;
        br.report.wall_seconds = std::chrono::duration<double>(t1 - t0).count();
        br.report.per_eval_seconds = br.report.evals ? br.report.wall_seconds / br.report.evals : 0.0;
        MultCounter d = mults_;
        d.stage1_powers -= before.stage1_powers;
        d.stage1_factors -= before.stage1_factors;
        d.stage2 -= before.stage2;
        d.speelpenning -= before.speelpenning;
        d.stage3 -= before.stage3;
        br.report.mults = d;
        return br;
    }

    // The reference's PackedLayout (ref include/polyjac/engine.hpp:100), bit-identical with
    // build_layout (ref src/packing.cpp:19-52); built on first use from the context.
    const PackedLayout& layout() const {
        if (!layout_) {
            auto L = std::make_unique<PackedLayout>();
            std::int32_t n = 0, m = 0, k = 0, d = 0;
            detail::check(pj_layout_info(ctx_, &n, &m, &k, &d, nullptr));
            L->n = n, L->m = m, L->k = k, L->d = d;
            const std::size_t nm = std::size_t(n) * m;
            L->positions.resize(nm * k);
            L->exponents.resize(nm * k);
            std::vector<double> co(2 * (std::size_t(k) + 1) * nm);
            detail::check(pj_layout_export(ctx_, L->positions.data(), L->exponents.data(), co.data()));
            L->coeffs.resize((std::size_t(k) + 1) * nm);
            for (std::size_t i = 0; i < L->coeffs.size(); ++i) {
                L->coeffs[i].re = co[2 * i];
                L->coeffs[i].im = co[2 * i + 1];
            }
            layout_ = std::move(L);
        }
        return *layout_;
    }
    const GridConfig& grid() const { return grid_; }
    // multiplications tallied since construction, in the reference's counting (pj_mult_counts)
    const MultCounter& mults() const { return mults_; }
    // ref src/engine.cpp:262-269: true while every masked slot holds an exact +0 pair. The device
    // path keeps no padded Mons buffer; its masked slots are the structural-zero Jacobian entries
    // (variable i in no monomial of polynomial p) of every result this context returned, checked
    // word for word (+0 only, -0 fails) as each result comes back.
    bool masked_slots_clean() const { return clean_; }

    // Complex double-double on host buffers: points [batch][n], out [batch][n + n*n].
    // reference_order = true keeps the reference's order in every stage.
    void evaluate_dd(const ComplexDD* points, std::int64_t batch, ComplexDD* out, bool reference_order = false) {
        detail::check(pj_evaluate_host(ctx_, PJ_PREC_DD | (reference_order ? PJ_ORDER_REF : 0),
                                       reinterpret_cast<const double*>(points), batch,
                                       reinterpret_cast<double*>(out)));
        tally(batch);
        const std::size_t nout = std::size_t(n_) * n_ + n_;
        for (std::int64_t b = 0; b < batch; ++b) audit(reinterpret_cast<const double*>(out) + 4 * nout * b, 4);
    }

    // Device buffers, asynchronous on `stream` (cudaStream_t); flags = PJ_PREC_D | PJ_PREC_DD [| order]
    // [| PJ_VALIDATE].
    void evaluate_device(int flags, const double* d_points, std::int64_t batch, double* d_out, void* stream) {
        detail::check(pj_evaluate(ctx_, flags, d_points, batch, d_out, stream));
        tally(batch);
    }

    // Newton corrector (B200 addition): `iters` steps x <- x + J(x)^-1 (y - f(x))
    // per point on the GPU, host buffers [batch][n] (target y may be null: the roots of f).
    // norms [batch][2] (|y - f|, |last step|) and status [batch] (0 ok, 1 singular, 2 non-finite,
    // 3 mixed refinement not converged) may be null. mixed = true (n <= 32): the Jacobian factored
    // in complex double and refined with dd residuals (PJ_NEWTON_MIXED; faster, for Jacobians that
    // are not ill-conditioned).
    void newton_dd(const ComplexDD* points, const ComplexDD* target, std::int64_t batch, int iters, ComplexDD* out,
                   double* norms = nullptr, std::int32_t* status = nullptr, bool mixed = false) {
        detail::check(pj_newton_host(ctx_, PJ_PREC_DD | (mixed ? PJ_NEWTON_MIXED : 0), reinterpret_cast<const double*>(points),
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

    pj_ctx* handle() const { return ctx_; }

private:
    EvaluationResult unpack(const double* o) const {
        EvaluationResult r;
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
    // one result [n + n*n][W]: every word of every structural zero must be +0
    void audit(const double* o, int W) {
        for (std::size_t z : zeros_)
            for (int c = 0; c < W; ++c) {
                std::uint64_t bits;
                std::memcpy(&bits, o + (n_ + z) * W + c, sizeof bits);
                if (bits != 0) clean_ = false;
            }
    }
    void tally(std::int64_t evals) {
        std::uint64_t c[5];
        detail::check(pj_mult_counts(ctx_, evals, c));
        mults_.stage1_powers += c[0];
        mults_.stage1_factors += c[1];
        mults_.stage2 += c[2];
        mults_.speelpenning += c[3];
        mults_.stage3 += c[4];
    }

    pj_ctx* ctx_ = nullptr;
    int n_ = 0;
    GridConfig grid_;
    MultCounter mults_;
    std::vector<std::size_t> zeros_;  // structural-zero Jacobian entries p*n + i
    bool clean_ = true;
    mutable std::unique_ptr<PackedLayout> layout_;
};

using EvaluationContext = BasicEvaluationContext<OwnTypes>;

}  // namespace polyjac_b200
