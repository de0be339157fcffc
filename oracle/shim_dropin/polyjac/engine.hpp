// ORACLE — test infrastructure only.
//
// Include-path shim that lets the reference's own tests/test_engine.cpp run UNMODIFIED against the
// B200 drop-in: it includes the reference's engine.hpp (declarations of the CPU pool, run_grid,
// BatchResult, ... stay the reference's), but the name polyjac::EvaluationContext is bound to
// polyjac_b200::dropin::EvaluationContext — the GPU class over the reference's own types
// (include/polyjac_b200_dropin.hpp). The reference's CPU class is declared under another name and
// never used. Built by `make -C oracle dropin-engine` (oracle/Makefile).
#pragma once

#define EvaluationContext EvaluationContext_reference_cpu_unused
#include_next <polyjac/engine.hpp>
#undef EvaluationContext

#include "polyjac_b200_dropin.hpp"

namespace polyjac {
using EvaluationContext = polyjac_b200::dropin::EvaluationContext;
}  // namespace polyjac
