"""paper_1201_0499_b200 — B200-native (sm_100a) evaluation of sparse polynomial systems and
their full Jacobians in complex double and complex double-double (arXiv 1201.0499), behind
the reference polyjac API. See DESIGN.md; the C ABI is include/polyjac_b200.h."""
from .engine import (BatchReport, BatchResult, EvaluationContext, EvaluationResult, GridConfig, MonomialSupport,
                     MultCounter, PolynomialSystem, RaggedSystem, Term, ValidationReport, Violation, fp64_peak_tflops, fp64_pipe_rates,
                     mons_deriv_slot, mons_slot, mons_value_slot, random_point, random_points, random_ragged_system,
                     random_system, validate_ragged_system,
                     read_system, read_system_text, to_dd, validate_system, write_system, write_system_text)
from ._lib import FormatError

__all__ = [
    "BatchReport", "BatchResult", "EvaluationContext", "EvaluationResult", "GridConfig", "MonomialSupport",
    "MultCounter", "PolynomialSystem", "Term", "ValidationReport", "Violation", "fp64_peak_tflops", "fp64_pipe_rates",
    "mons_deriv_slot", "mons_slot", "mons_value_slot", "random_point", "random_points", "random_system",
    "to_dd", "validate_system", "read_system", "read_system_text", "write_system", "write_system_text",
    "FormatError", "RaggedSystem", "random_ragged_system", "validate_ragged_system",
]
