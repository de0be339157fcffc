// Drop-in check of the C++ surface (include/polyjac_b200_dropin.hpp) against the UNMODIFIED
// reference, using the reference's own types and call syntax: the same polyjac::PolynomialSystem
// goes into polyjac::EvaluationContext (reference, CPU) and polyjac_b200::dropin::EvaluationContext
// (B200) and every result, tally and layout must be bit-identical. Mirrors ref
// tests/test_engine.cpp (which itself also runs unmodified against the drop-in:
// tests/test_ref_suites.py). Built by
// `make -C oracle dropin` (compiles the reference sources where they lie) into oracle/_ref/;
// run by tests/test_gpu_dropin.py on a GPU box. Test infrastructure only.
#include <cmath>
#include <cstdio>
#include <limits>
#include <stdexcept>
#include <string>

#include "polyjac/engine.hpp"
#include "polyjac/oracle.hpp"
#include "polyjac_b200_dropin.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                             \
    do {                                                                        \
        if (cond) {                                                             \
            ++g_pass;                                                           \
        } else {                                                                \
            ++g_fail;                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                       \
    } while (0)
template <class E, class F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static bool bit_equal(const polyjac::EvaluationResult& a, const polyjac::EvaluationResult& b) {
    if (a.n != b.n || a.values.size() != b.values.size() || a.jacobian.size() != b.jacobian.size()) return false;
    for (size_t i = 0; i < a.values.size(); ++i)
        if (!polyjac::bit_equal(a.values[i], b.values[i])) return false;
    for (size_t i = 0; i < a.jacobian.size(); ++i)
        if (!polyjac::bit_equal(a.jacobian[i], b.jacobian[i])) return false;
    return true;
}

int main() {
    using namespace polyjac;
    // engine shapes of ref tests/test_engine.cpp:70-83 and acceptance criterion 1 corners
    const int shapes[][4] = {{32, 32, 9, 2}, {32, 32, 16, 10}, {8, 3, 3, 5}, {4, 4, 1, 1}, {40, 40, 20, 3},
                             {4, 1, 1, 255}, {32, 32, 8, 2}, {64, 64, 16, 10}, {10, 40, 4, 3}};
    std::uint64_t seed = 7000;
    for (auto& s : shapes) {
        const PolynomialSystem sys = random_system(s[0], s[1], s[2], s[3], seed++);
        EvaluationContext ref(sys, {32, 1});
        polyjac_b200::dropin::EvaluationContext gpu(sys, {32, 1});
        for (int t = 0; t < 3; ++t) {
            const EvaluationPoint pt = random_point(s[0], seed++);
            const EvaluationResult got = gpu.evaluate(pt);  // the reference's result type, no casts
            CHECK(bit_equal(got, ref.evaluate(pt)));
        }
        // batch + multiplication tallies equal to the reference's counters
        const std::vector<EvaluationPoint> pts = random_points(s[0], 5, seed++);
        const BatchResult rb = ref.evaluate_batch(pts, 2);
        const BatchResult gb = gpu.evaluate_batch(pts, 2);
        CHECK(gb.report.evals == rb.report.evals);
        CHECK(gb.report.mults == rb.report.mults);
        CHECK(gpu.mults() == ref.mults());
        bool all = gb.results.size() == rb.results.size();
        for (size_t i = 0; all && i < gb.results.size(); ++i) all = bit_equal(gb.results[i], rb.results[i]);
        CHECK(all);
        // layout(): the reference's PackedLayout, byte- and bit-identical (ref engine.hpp:100)
        const PackedLayout& gl = gpu.layout();
        const PackedLayout& rl = ref.layout();
        CHECK(gl.positions == rl.positions && gl.exponents == rl.exponents);
        CHECK(gl.footprint_bytes() == rl.footprint_bytes() && gl.monomial_count() == rl.monomial_count());
        bool co = gl.coeffs.size() == rl.coeffs.size();
        for (size_t i = 0; co && i < gl.coeffs.size(); ++i) co = polyjac::bit_equal(gl.coeffs[i], rl.coeffs[i]);
        CHECK(co);
        CHECK(gpu.masked_slots_clean() && ref.masked_slots_clean());
    }
    // masked_slots_clean sees structural zeros (ref tests/test_engine.cpp:172-179): a system whose
    // Jacobian has structural zeros stays clean over many evaluations
    {
        const PolynomialSystem sys = random_system(10, 4, 3, 3, 33);
        polyjac_b200::dropin::EvaluationContext ctx(sys, {32, 2});
        for (int i = 0; i < 100; ++i) (void)ctx.evaluate(random_point(10, 1000 + i));
        CHECK(ctx.masked_slots_clean());
        CHECK(ctx.grid().block_size == 32 && ctx.grid().workers == 2);
    }
    // ref tests/test_engine.cpp:298-305: point validation
    {
        const PolynomialSystem sys = random_system(4, 2, 2, 2, 8);
        polyjac_b200::dropin::EvaluationContext ctx(sys);
        CHECK(throws<std::invalid_argument>([&] { ctx.evaluate(EvaluationPoint(3, Complex{1.0, 0.0})); }));
        EvaluationPoint bad(4, Complex{1.0, 0.0});
        bad[2].im = std::numeric_limits<double>::quiet_NaN();
        CHECK(throws<std::invalid_argument>([&] { ctx.evaluate(bad); }));
        CHECK(throws<std::invalid_argument>([&] { ctx.evaluate_batch({}, 0); }));
        // the context keeps working after a rejected point
        CHECK(ctx.evaluate(EvaluationPoint(4, Complex{1.0, 0.0})).n == 4);
    }
    // ref tests/test_engine.cpp:385-391 and packing rejections
    {
        const PolynomialSystem sys = random_system(4, 2, 2, 2, 3);
        CHECK(throws<std::invalid_argument>([&] { polyjac_b200::dropin::EvaluationContext c(sys, {0, 1}); }));
        CHECK(throws<std::invalid_argument>([&] { polyjac_b200::dropin::EvaluationContext c(sys, {32, -1}); }));
        PolynomialSystem bad = sys;
        bad.terms[0].coeff = {0.0, 0.0};
        CHECK(throws<std::invalid_argument>([&] { polyjac_b200::dropin::EvaluationContext c(bad); }));
        PolynomialSystem wide{300, 1, 1, 1, {}};
        for (int p = 0; p < 300; ++p) wide.terms.push_back({{1.0, 0.0}, {{p}, {1}}});
        CHECK(throws<std::invalid_argument>([&] { polyjac_b200::dropin::EvaluationContext c(wide); }));
        {  // the wide encoding accepts it (B200 addition) and evaluates f_p = x_p exactly
            polyjac_b200::dropin::EvaluationContext c(wide, {}, 0, PJ_CTX_WIDE);
            EvaluationPoint x(300);
            for (int i = 0; i < 300; ++i) x[i] = {0.5 + i, -1.0 * i};
            const EvaluationResult r = c.evaluate(x);
            bool ok = true;
            for (int i = 0; i < 300; ++i)
                ok = ok && r.values[i].re == x[i].re && r.values[i].im == x[i].im && r.jac(i, i).re == 1.0;
            CHECK(ok);
        }
        PolynomialSystem shortsys = sys;
        shortsys.terms.pop_back();
        CHECK(throws<std::invalid_argument>([&] { polyjac_b200::dropin::EvaluationContext c(shortsys); }));
    }
    // ref tests/test_engine.cpp:181-196 in complex dd: integer answers are exact
    {
        PolynomialSystem sys{2, 2, 2, 1, {}};
        const Term t{{0.5, 0.0}, {{0, 1}, {1, 1}}};
        sys.terms = {t, t, t, t};
        polyjac_b200::dropin::EvaluationContext ctx(sys);
        polyjac_b200::ComplexDD pt[2] = {{3, 0, 0, 0}, {5, 0, 0, 0}};
        polyjac_b200::ComplexDD out[6];
        ctx.evaluate_dd(pt, 1, out);
        CHECK(out[0].re_hi == 15 && out[0].re_lo == 0);
        CHECK(out[2].re_hi == 5 && out[3].re_hi == 3);
        ctx.evaluate_dd(pt, 1, out, /*reference_order=*/true);
        CHECK(out[0].re_hi == 15 && out[2].re_hi == 5 && out[3].re_hi == 3);
        const EvaluationResult r = ctx.evaluate({{3.0, 0.0}, {5.0, 0.0}});
        CHECK(compare(r, sys, {{3.0, 0.0}, {5.0, 0.0}}, 1e-10).pass);
    }
    // Newton corrector (B200 addition): f_p = x_{(p+1) mod 3} has J a permutation, one step lands
    // exactly on the root; a variable in no monomial makes J singular (status 1, x unchanged)
    {
        PolynomialSystem sys{3, 1, 1, 1, {}};
        for (int p = 0; p < 3; ++p) sys.terms.push_back({{1.0, 0.0}, {{(p + 1) % 3}, {1}}});
        polyjac_b200::dropin::EvaluationContext ctx(sys);
        polyjac_b200::ComplexDD x[3] = {{0.25, 1e-20, -0.5, 0}, {0.75, 0, 0.125, -1e-21}, {-0.3, 0, 0.9, 0}};
        polyjac_b200::ComplexDD xo[3];
        double norms[2];
        std::int32_t st = -1;
        ctx.newton_dd(x, nullptr, 1, 1, xo, norms, &st);
        CHECK(st == 0 && norms[0] == 0.9);
        for (const auto& v : xo) CHECK(v.re_hi == 0 && v.re_lo == 0 && v.im_hi == 0 && v.im_lo == 0);
        // the mixed-precision solve: double factors + dd refinement reach the same exact root
        st = -1;
        ctx.newton_dd(x, nullptr, 1, 1, xo, norms, &st, /*mixed=*/true);
        CHECK(st == 0 && norms[0] == 0.9);
        for (const auto& v : xo) CHECK(v.re_hi == 0 && v.re_lo == 0 && v.im_hi == 0 && v.im_lo == 0);
        PolynomialSystem sing{2, 1, 1, 1, {}};
        sing.terms = {{{1.0, 0.0}, {{0}, {1}}}, {{2.0, 0.0}, {{0}, {1}}}};
        polyjac_b200::dropin::EvaluationContext c2(sing);
        Complex y[2] = {{0.5, 0.0}, {0.25, 0.0}}, yo[2];
        c2.newton(y, nullptr, 1, 2, yo, norms, &st);
        CHECK(st == 1 && yo[0].re == 0.5 && yo[1].re == 0.25);
    }
    std::printf("%s: %d passed, %d failed\n", g_fail ? "FAIL" : "PASS", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
