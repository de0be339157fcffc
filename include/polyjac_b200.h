/* polyjac_b200 — C ABI of the B200-native evaluator for sparse polynomial systems and their
 * full Jacobians (arXiv 1201.0499), complex double and complex double-double.
 *
 * This is the drop-in boundary for the reference's hot path (ref = /root/reference/proj).
 * Each entry point names the reference interface it replaces. Plain pointers and sizes
 * only; no C++ or torch types. Errors are status codes; pj_last_error() returns the
 * calling thread's last message (the reference throws instead: the C++ wrapper
 * include/polyjac_b200.hpp maps the codes back onto the same exception types).
 *
 * Array conventions
 *   positions, exponents  int32 [n*m*k], S_m order: monomial s = p*m + g, slot s*k + j
 *                         (ref include/polyjac/system.hpp:28-31, packing.hpp:12-15);
 *                         positions 0-based and strictly increasing, exponents in [1, d]
 *   coeffs                double [n*m][4] = (re_hi, re_lo, im_hi, im_lo); lo words may be 0
 *                         (double input). PJ_PREC_D uses the hi words only.
 *   points                double [batch][n][W]
 *   out                   double [batch][n + n*n][W]: the n values, then the row-major
 *                         Jacobian, entry (p, i) at n + p*n + i (ref system.hpp:48-54)
 *   W = 2 (re, im) for PJ_PREC_D, 4 (re_hi, re_lo, im_hi, im_lo) for PJ_PREC_DD.
 */
#ifndef POLYJAC_B200_H
#define POLYJAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PJ_OK 0
#define PJ_EINVAL 1     /* std::invalid_argument in the reference */
#define PJ_ERANGE 2     /* std::out_of_range in the reference */
#define PJ_ECUDA 3      /* CUDA runtime failure (message in pj_last_error) */
#define PJ_ENOMEM 4     /* device allocation failed */
#define PJ_ENONFINITE 5 /* non-finite coordinate: std::invalid_argument in
                           ref src/engine.cpp:186-188 */
#define PJ_EFORMAT 6    /* malformed system file: polyjac::FormatError, ref include/polyjac/io.hpp:19-21 */

/* precision / order flags for pj_evaluate */
#define PJ_PREC_D 1         /* complex double, reference operation order: bit-exact with
                               EvaluationContext::evaluate (ref src/engine.cpp:181-224) */
#define PJ_PREC_DD 2        /* complex double-double; default (fast) order: derivatives in the
                               division form a_j*(c*V)*(1/x_j) for points whose coordinates all
                               have |Re| + |Im| in [2^-16, 2^16], product chains otherwise;
                               |err| <= 1e-30 * sum|terms| per output */
#define PJ_ORDER_REF 0x10   /* dd: keep the reference order in every stage (bit-exact with the
                               oracle's dd restatement); default dd order is the fast one */
#define PJ_ORDER_FAST 0x20  /* d: allow the fast order (default for d is the reference order) */
#define PJ_OP_NEWTON 0x100  /* pj_set_launch / pj_get_launch: address the Newton solve kernel */
#define PJ_NEWTON_MIXED 0x400 /* pj_newton_solve / _step / _host with PJ_PREC_DD, n <= 32: factor J in
                                 complex double (its high words), then two steps of iterative refinement
                                 with complex-dd residuals; status 3 when the refinement has not
                                 converged (J too ill-conditioned for double factors: use the dd solve) */
#define PJ_VALIDATE 0x200   /* pj_evaluate: check every coordinate first and return PJ_ENONFINITE
                               without writing any output when one is non-finite (the
                               reference's throw-before-evaluate, ref src/engine.cpp:183-188);
                               costs one read of the points and one stream synchronisation */

typedef struct pj_system_desc {
    int32_t n, m, k, d;
    const int32_t* positions;
    const int32_t* exponents;
    const double* coeffs;
} pj_system_desc;

typedef struct pj_ctx pj_ctx;

/* Thread-local message of the last failing call ("" after success). */
const char* pj_last_error(void);

/* Library / build identification string. */
const char* pj_version(void);

/* Number of rule violations of the system (0 = valid); the first one's text is copied into
 * msg (capacity cap, may be NULL). Replaces validate_system, ref src/system.cpp:21-64. */
int pj_validate(const pj_system_desc* sys, char* msg, size_t cap);

/* Context creation: validate + pack + upload once; replaces
 * EvaluationContext::EvaluationContext(sys, GridConfig), ref src/engine.cpp:168-179 and
 * build_layout, ref src/packing.cpp:19-52 (PJ_EINVAL for an invalid system or n > 256).
 * device < 0 creates a host-only context (packing and index maps, no evaluation). */
int pj_ctx_create(const pj_system_desc* sys, int device, pj_ctx** out);
/* Same, with options. PJ_CTX_WIDE lifts the reference's byte-encoding cap
 * (build_layout rejects n > 256, ref src/packing.cpp:25-27): systems with n > 256 are packed with
 * 32-bit position/exponent words (n <= 65535, k <= 2046) and evaluated by the generic kernel in
 * every precision and order (same contracts as below). Without the option the reference's
 * rejection is kept. */
#define PJ_CTX_WIDE 0x1
int pj_ctx_create_ex(const pj_system_desc* sys, int device, int options, pj_ctx** out);
void pj_ctx_destroy(pj_ctx* ctx);

/* Evaluate `batch` points already resident on the context's device; asynchronous on
 * `stream` (a cudaStream_t, NULL = legacy default stream). Replaces
 * EvaluationContext::evaluate / evaluate_batch, ref src/engine.cpp:181-260, batched over
 * points. The caller owns both buffers; no allocation happens here. batch == 0 is a no-op.
 * Without PJ_VALIDATE the call stays asynchronous: non-finite coordinates are flagged on device
 * (read and cleared with pj_nonfinite_seen). With PJ_VALIDATE in `flags` the batch is checked
 * first and rejected with PJ_ENONFINITE before the evaluation is launched.
 * One context serves one stream at a time (ref include/polyjac/engine.hpp:84-86): systems
 * whose tables exceed shared memory use per-CTA global scratch slabs of the context. */
int pj_evaluate(pj_ctx* ctx, int flags, const double* d_points, int64_t batch, double* d_out, void* stream);

/* Host-buffer convenience: H2D of the points, pj_evaluate, D2H of the results, synchronous.
 * Returns PJ_ENONFINITE (like the reference's throw) when an input coordinate is non-finite
 * (h_out is then unspecified). A flag left by an earlier asynchronous pj_evaluate is cleared on
 * entry and does not affect this call. */
int pj_evaluate_host(pj_ctx* ctx, int flags, const double* h_points, int64_t batch, double* h_out);

/* Synchronises `stream`, then reports (and clears) whether any pj_evaluate since the last
 * call saw a non-finite coordinate. */
int pj_nonfinite_seen(pj_ctx* ctx, void* stream, int* seen);

/* Shape of the packed layout: n, m, k, d, and the reference's constant-memory-equivalent
 * footprint 2*n*m*k (PackedLayout::footprint_bytes, ref include/polyjac/packing.hpp:44-45). */
int pj_layout_info(const pj_ctx* ctx, int32_t* n, int32_t* m, int32_t* k, int32_t* d, int64_t* footprint_bytes);

/* Index maps, bit-exact with the reference:
 *   pj_mons_slot      mons_slot, ref src/packing.cpp:8-17 (kind 0 = value, 1 = derivative;
 *                     PJ_ERANGE where the reference throws std::out_of_range)
 *   pj_slot_targets   stage2_slot_targets, ref src/kernels.cpp:129-137 (k+1 slots, value last)
 *   pj_zero_mask      zero_mask, ref src/packing.cpp:54-72, regenerated as the complement of
 *                     the device gather map; returns its length (needs cap >= length) */
int pj_mons_slot(int64_t s, int kind, int var, int n, int m, int64_t* slot);
int pj_slot_targets(const pj_ctx* ctx, int64_t s, int64_t* targets);
int64_t pj_zero_mask(const pj_ctx* ctx, int64_t* mask, int64_t cap);

/* The reference's PackedLayout (ref include/polyjac/packing.hpp:24-46, built by build_layout,
 * ref src/packing.cpp:19-52), exported from the context: positions u8 [n*m*k], exponents u8 [n*m*k]
 * (degree minus one), coeffs double [(k+1)*n*m][2] derivative-major (block j < k: a_j * c rounded
 * per component in double; block k: c). Any pointer may be NULL. PJ_EINVAL for a wide context
 * (n > 256 has no byte encoding). Bit-identical with the reference's build_layout. */
int pj_layout_export(const pj_ctx* ctx, uint8_t* positions, uint8_t* exponents, double* coeffs);

/* Structural zeros of the Jacobian: mask[p*n + i] = 1 when variable i occurs in no monomial of
 * polynomial p (those entries are exact +0 in every result, ref include/polyjac/system.hpp:44-46).
 * mask may be NULL; returns the number of structural zeros. */
int64_t pj_structural_zeros(const pj_ctx* ctx, uint8_t* mask);

/* Fault injection for tests ("deliberately corrupted coeffs entry"): multiplies the
 * device copies of monomial s's coefficient (every precision and table) by `factor`. Synchronous.
 * Not for production use: the context no longer represents its system afterwards. */
int pj_debug_corrupt_coeff(pj_ctx* ctx, int64_t s, double factor);

/* Multiplication tally of `evals` evaluations (MultCounter, ref include/polyjac/kernels.hpp:15-34;
 * closed form SPEC.md:477): counts[5] = stage1_powers, stage1_factors, stage2, speelpenning, stage3. */
int pj_mult_counts(const pj_ctx* ctx, int64_t evals, uint64_t* counts);

/* Ragged systems (non-uniform m and k; the paper's regularity assumption,
 * ref PAPER.md:258-272, :700-706, lifted). The reference's data model is uniform
 * (PolynomialSystem n, m, k; ref include/polyjac/system.hpp:14-42); a ragged system keeps its
 * per-term rules and generalises the shape:
 *   row_off   int32 [n+1]   polynomial p owns terms [row_off[p], row_off[p+1]); row_off[0] = 0,
 *                           every polynomial at least one term (m_p >= 1)
 *   term_off  int32 [T+1]   term t owns slots [term_off[t], term_off[t+1]) of positions/exponents;
 *                           term_off[0] = 0, 1 <= k_t <= n   (T = row_off[n])
 *   positions, exponents    int32 [term_off[T]]: 0-based strictly increasing, exponents in [1, d]
 *   coeffs    double [T][4] (re_hi, re_lo, im_hi, im_lo)
 * Semantics: the reference's per-term sequence (stage 1 common factor, Speelpenning for the
 * term's own k_t incl. the k = 1, 2 special cases, ref src/kernels.cpp:45-127), and every output
 * the ascending-g sum over its polynomial's terms (ref src/kernels.cpp:139-146). A uniform system
 * written in this form gives bit-identical results to pj_ctx_create's. Output layout unchanged. */
typedef struct pj_ragged_desc {
    int32_t n, d;
    const int32_t* row_off;
    const int32_t* term_off;
    const int32_t* positions;
    const int32_t* exponents;
    const double* coeffs;
} pj_ragged_desc;
/* Violations of the ragged rules (validate_system's wording per term, "polynomial p, monomial g:"
 * prefix as Violation::describe, ref src/system.cpp:11-19); 0 = valid. */
int pj_validate_ragged(const pj_ragged_desc* sys, char* msg, size_t cap);
/* Context for a ragged system: evaluated by the generic kernel (any k_t, m_p; complex double
 * bit-exact with the oracle's restatement of the reference sequence; dd reference order bit-equal
 * to the oracle, dd fast order within the §5 tolerance). options: PJ_CTX_WIDE as above. Every
 * evaluation / Newton entry point accepts the context. pj_layout_info reports m = max m_p,
 * k = max k_t and footprint 2*sum(k_t); pj_mult_counts and pj_structural_zeros generalise;
 * the uniform-layout exports (pj_slot_targets, pj_zero_mask, pj_layout_export,
 * pj_debug_corrupt_coeff) return PJ_EINVAL. */
int pj_ctx_create_ragged(const pj_ragged_desc* sys, int device, int options, pj_ctx** out);
/* Deterministic ragged system: m_p uniform in [m_lo, m_hi] per polynomial, k_t uniform in
 * [k_lo, k_hi] per term, then the reference generator's per-term draws (k_t-subset, exponents
 * 1 + below(d), coefficient) from the same stream. Two passes: call with NULL arrays to get the
 * term count *T and slot count *S, then with arrays row_off[n+1], term_off[T+1], positions[S],
 * exponents[S], coeffs[4T]. */
int pj_random_ragged_system(int n, int m_lo, int m_hi, int k_lo, int k_hi, int d, uint64_t seed, int64_t* T,
                            int64_t* S, int32_t* row_off, int32_t* term_off, int32_t* positions, int32_t* exponents,
                            double* coeffs);

/* Deterministic inputs, bit-identical to random_system / random_points
 * (ref src/system.cpp:66-118, ref src/rng.hpp): coeffs get lo words 0; points are [count][n][2]. */
int pj_random_system(int n, int m, int k, int d, uint64_t seed, int32_t* positions, int32_t* exponents,
                     double* coeffs);
int pj_random_points(int n, int64_t count, uint64_t seed, double* points);
/* Points [first, first + count) of the same stream (a contiguous shard of random_points(n, N,
 * seed) for any N >= first + count): lets each rank generate only its own shard. */
int pj_random_points_range(int n, int64_t first, int64_t count, uint64_t seed, double* points);

/* System text files (ref src/io.cpp:38-117, format ref README.md:91-104): '#' comments, header
 * "n m k d", one "re im pos1 exp1 ... posk expk" line per monomial (1-based positions), doubles
 * with 17 significant digits (bit-exact round trip). Errors: PJ_EFORMAT with "<name>:<line>: ..."
 * in pj_last_error(), the reference's FormatError wording. A pj_system owns its arrays;
 * pj_system_view exposes them as a descriptor for pj_ctx_create. */
typedef struct pj_system pj_system;
int pj_system_read_file(const char* path, pj_system** out);
int pj_system_read_text(const char* text, const char* name, pj_system** out);
int pj_system_view(const pj_system* sys, pj_system_desc* desc);
void pj_system_free(pj_system* sys);
int pj_system_write_file(const pj_system_desc* sys, const char* path);
/* Writes the text into buf (capacity cap, NUL-terminated, may be NULL); returns its full length. */
int64_t pj_system_write_text(const pj_system_desc* sys, char* buf, int64_t cap);

/* Newton corrector on device (the consumer of the evaluator's output — the
 * reference leaves Newton / path tracking out of scope, ref SPEC.md:12, so the operation order is
 * defined in csrc/newton.cu and restated by the oracle). For every point b:
 *     J_b dx = y_b - f_b   (Gaussian elimination, partial pivoting on |Re hi| + |Im hi|),
 *     x_new_b = x_b + dx,
 * in the precision of `flags` (PJ_PREC_D or PJ_PREC_DD; the order bits are ignored).
 *   evals       [batch][n + n*n][W]  pj_evaluate's output at `points` (read only)
 *   points      [batch][n][W]
 *   target      [batch][n][W] or NULL (y = 0: the roots of f)
 *   points_out  [batch][n][W]; may alias points (in-place update)
 *   norms       [batch][2] or NULL: max over i of max(|Re hi|, |Im hi|) of (y - f)_i, of dx_i
 *   status      [batch] or NULL: 0 ok, 1 singular (a zero pivot column; x_new = x, norms[1] = inf),
 *               2 non-finite result, 3 (PJ_NEWTON_MIXED only) the refinement has not converged
 * Asynchronous on `stream`; no allocation for n <= 64 (larger n allocates per-CTA matrix slabs
 * on first use). */
int pj_newton_solve(pj_ctx* ctx, int flags, const double* d_evals, const double* d_points, const double* d_target,
                    int64_t batch, double* d_points_out, double* d_norms, int32_t* d_status, void* stream);
/* One Newton step: pj_evaluate(points -> work) then pj_newton_solve(work). work: [batch][n + n*n][W],
 * caller-owned; on return it holds f and J at the input points. */
int pj_newton_step(pj_ctx* ctx, int flags, const double* d_points, const double* d_target, int64_t batch,
                   double* d_work, double* d_points_out, double* d_norms, int32_t* d_status, void* stream);
/* Host-buffer convenience: `iters` Newton steps per point on device (chunks whose evaluator
 * output stays L2-resident), synchronous; norms/status describe the last step. Returns
 * PJ_ENONFINITE when an INPUT coordinate is non-finite (checked on the input points only); an
 * iterate that diverges to non-finite values is reported per point (status 2) and the other
 * points' results stand. */
int pj_newton_host(pj_ctx* ctx, int flags, const double* h_points, const double* h_target, int64_t batch, int iters,
                   double* h_points_out, double* h_norms, int32_t* h_status);

/* Advanced: override the launch shape for `flags`' precision (threads per CTA, multiple of 32,
 * <= 256 — up to 384 for the fast dd kernel at k > 12 when its staging fits shared memory;
 * points per CTA tile). 0 restores the automatic choice. A shape no kernel can run returns
 * PJ_EINVAL and keeps the previous one. */
int pj_set_launch(pj_ctx* ctx, int flags, int threads, int tile_points);
/* Advanced: kernel choice for complex double (PJ_PREC_D) or the fast dd order. 0 = automatic,
 * -1 = the generic kernel (eval_kernels.cu), 1 = the k-specialised kernel (eval_fastd.cu for complex
 * double, eval_fast.cu for dd), 3 = the warp-specialised dd kernel (eval_fast_ws.cu: producer and
 * consumer warps; d <= 2, m <= 32, n <= 64, k <= 12; bit-identical with variant 1). Every choice
 * satisfies the same contract (complex double: bit-exact with the reference). With PJ_OP_NEWTON: the Newton solve, -1 = the column kernel,
 * 1 = the panel kernel (n <= 32); both give identical bits. */
int pj_set_kernel_variant(pj_ctx* ctx, int flags, int variant);
/* Report the launch shape used for `flags`: threads, tile points, blocks, dynamic smem bytes,
 * kernel (-1 = generic, 1 = fast dd, 2 = fast complex double, 3 = warp-specialised dd; with PJ_OP_NEWTON: 0 = column kernel,
 * 1 = panel kernel, 2 = column kernel on global slabs). */
int pj_get_launch(pj_ctx* ctx, int flags, int32_t* threads, int32_t* tile_points, int32_t* blocks,
                  int64_t* smem_bytes, int32_t* variant);

/* Measurement helper (not part of the reference surface): FP64 DFMA throughput of `device`
 * in TFLOP/s (2 flops per DFMA), the denominator of the roofline fraction. */
int pj_fp64_peak_probe(int device, double* tflops);
/* Measurement helper: issue rate of the FP64 pipe of `device` per operation, lane operations per
 * second: out[0] DFMA, out[1] DADD, out[2] DMUL (16 independent chains per thread, full grid). */
int pj_fp64_pipe_probe(int device, double* lane_ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* POLYJAC_B200_H */
