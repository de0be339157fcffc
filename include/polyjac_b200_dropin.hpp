// polyjac_b200_dropin.hpp — the B200 EvaluationContext over the reference's OWN types.
//
// Include after (or instead of) the reference's headers; the reference's include directory must
// be on the include path (ref include/polyjac/engine.hpp declares PolynomialSystem,
// EvaluationPoint, EvaluationResult, BatchResult, PackedLayout, MultCounter, GridConfig). Then
//
//     polyjac_b200::dropin::EvaluationContext ctx(sys, {32, 4});
//     const polyjac::EvaluationResult r = ctx.evaluate(point);
//     const polyjac::BatchResult b = ctx.evaluate_batch({point}, 10);
//     const polyjac::PackedLayout& L = ctx.layout();
//
// compile exactly as they do against polyjac::EvaluationContext (ref engine.hpp:87-128), with
// bit-identical results, multiplication tallies and exception types. tests/cpp/test_dropin.cpp
// and the reference's own tests/test_engine.cpp (built unmodified, oracle/Makefile `dropin-engine`)
// exercise it.
#pragma once

#include "polyjac/engine.hpp"
#include "polyjac_b200.hpp"

namespace polyjac_b200 {

struct ReferenceTypes {
    using Complex = polyjac::Complex;
    using EvaluationPoint = polyjac::EvaluationPoint;
    using EvaluationResult = polyjac::EvaluationResult;
    using BatchResult = polyjac::BatchResult;
    using PackedLayout = polyjac::PackedLayout;
    using MultCounter = polyjac::MultCounter;
    using GridConfig = polyjac::GridConfig;
};

namespace dropin {
using EvaluationContext = BasicEvaluationContext<ReferenceTypes>;
}  // namespace dropin

}  // namespace polyjac_b200
