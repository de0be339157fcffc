// Device-side system layout ("packing v2") and launch plumbing shared by capi.cpp and
// eval_kernels.cu. Built once per context on the host (capi.cpp: pack_system), uploaded once,
// reused for every batch.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pjb {

struct DevSystem {
    int n, m, k, d, nm;
    int chunks;  // ceil(m / 32): monomials are evaluated 32 per warp pass
    int kp;      // row stride of posexp (k rounded up to 8 -> 16-byte rows)
    // posexp[s*kp + j] = pos | (exp-1) << 8   (the reference's two byte arrays,
    // ref src/packing.cpp:40-44, fused into one 16-bit word per (s, j))
    const uint16_t* posexp;
    // wide encoding (n > 256): posexp32[s*kp + j] = pos | (exp-1) << 16; null when
    // the byte encoding is in use
    const uint32_t* posexp32;
    // coefficient planes, derivative-major like ref src/packing.cpp:46-49:
    // component c of (j, s) at coef[(j*W + c)*nm + s]; block j < k = a_j*c, block k = c
    const double* coef;
    // stage-3 gather map: entries of Jacobian entry (p, v) from chunk c are
    // gm_ent[gm_off[(p*chunks + c)*n + v] .. gm_off[... + 1]), ascending g; an entry is
    // j*32 + (g mod 32), i.e. derivative j of chunk-local monomial g
    const int* gm_off;
    const uint16_t* gm_ent;
    // balanced stage-3 schedule of the fast kernel (eval_fast.cu), per (row p, chunk c):
    // sch[((p*chunks + c)*(k+1) + r)*32 + lane] = entry r of lane's run: bits 0-12 staging
    // slot of (derivative j, monomial g) as the 16-byte unit j*64 + g of the warp's staging area,
    // 13-22 segment id, 23 flush (segment ends here), 24 valid; the phase-2 codes below use the
    // same units;
    // phase-2 records per (p, c), pass k2 < npass = (n + 64)/64 and lane:
    // segq[((p*chunks + c)*npass + k2)*32 + lane] = {cnt1 | cnt2 << 8 | o2 << 16, six 16-bit
    // staging codes}: the lane adds the segment partials of output o1 = 64*k2 + lane (cnt1 of
    // them), then those of its secondary output o2 (0xffff: none); o = 0 is the value, o = v+1
    // Jacobian column v. Lanes with more than six codes keep their whole list at
    // segcode + seg[same index] (nseg unused)
    const uint32_t* sch;
    const uint32_t* seg;
    int nseg;
    const uint16_t* segcode;
    const uint4* segq;
    // complex-double fast kernel (eval_fastd.cu): stage-3 work of lane slot i of (p, c) at
    // colq[(p*chunks + c)*n + i] = {first gm_ent entry, count | column << 16} (column 0 always at
    // slot 0; the grouping of columns into quarter-warps is chosen against bank conflicts)
    const int2* colq;
    // ragged system (null for a uniform one, which uses p*m and p*chunks): the
    // terms of row p are [row_off[p], row_off[p+1]) (s = row_off[p] + g), its stage-3 chunks
    // [row_chunk[p], row_chunk[p+1]) (gm_off index (row_chunk[p] + c)*n + v), term s has term_k[s]
    // variables; k above is the maximum, nm the total term count
    const int* row_off = nullptr;
    const int* row_chunk = nullptr;
    const uint16_t* term_k = nullptr;
    // plain dd coefficients tiled for the fast kernel: component q of monomial
    // g = 32*chunk + lane of row p at coefT[((p*chunks + chunk)*4 + q)*32 + lane] (0 for g >= m)
    const double* coefT;
};
constexpr uint32_t kSchFlush = 1u << 23;
constexpr uint32_t kSchValid = 1u << 24;

struct LaunchCfg {
    int variant = -1;         // 1 = fast dd kernel (eval_fast.cu), 2 = fast d kernel (eval_fastd.cu),
                              // -1 = generic kernel
    int blocks = 0;
    int threads = 256;
    int tp = 1;               // points per CTA tile
    size_t smem_bytes = 0;    // dynamic shared memory (0 in global-scratch mode)
    double* gscratch = nullptr;  // non-null: tables/staging in global memory (huge systems)
    int* flag = nullptr;      // device int, set to 1 on a non-finite coordinate
    int producers = 0;        // warp-specialised dd kernel (variant 3): producer warps per CTA
    int splits = 1;           // fast kernels (variants 1, 2): CTAs sharing one tile's tasks — set per
                              // launch for batches with fewer tiles than CTAs (pj_evaluate)
};

cudaError_t launch_eval(int prec, int order, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out,
                        long long B, cudaStream_t st);
int max_blocks_per_sm(int prec, int order, int threads, size_t smem, bool ragged);
// sets *flag |= 1 when any of the `doubles` words at pts is non-finite (points: 16-byte aligned)
cudaError_t launch_check_finite(const double* pts, long long doubles, int* flag, int sms, cudaStream_t st);
cudaError_t set_smem_attr(size_t bytes);
// The dynamic shared-memory limit every kernel's cudaFuncAttributeMaxDynamicSharedMemorySize is
// set to: the current device's opt-in maximum. The attribute is process-wide per kernel, so a
// per-launch value would race between contexts planning / launching on other threads (one
// context lowering it between another's set and launch); one common value cannot. f: the kernel
// (its static shared memory comes off the limit).
int dyn_smem_limit(const void* f);

// fast complex-dd kernel point tables: rows x^1 .. x^dm (dm = max(d, 2)), then 1/x (the division
// form of the derivatives, eval_fast.cu)
__host__ __device__ inline int fast_tab_rows(int d) { return (d > 2 ? d : 2) + 1; }
// fast complex-dd kernels (eval_fast.cu), instantiated for k in [2, 16]
bool fast_supported(int k);
int fast_plane_stride(int n);
cudaError_t launch_fast(int k, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                        cudaStream_t st);
int fast_blocks_per_sm(int k, int n, int d, int threads, size_t smem);

// warp-specialised fast complex-dd kernel (eval_fast_ws.cu): d <= 2, m <= 32, n <= 64, k in [2, 12]
bool fast_ws_supported(int k, int n, int m, int d);
size_t fast_ws_smem(int n, int k, int nw, int tp);
cudaError_t launch_fast_ws(int k, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                           cudaStream_t st);
int fast_ws_blocks_per_sm(int k, int n, int threads, size_t smem);

// fast complex-double kernels in the reference order (eval_fastd.cu), k in [1, 16], byte encoding
bool fastd_supported(int k);
size_t fastd_smem(int n, int m, int k, int d, int nw, int tp);
cudaError_t launch_fastd(int k, const LaunchCfg& L, const DevSystem& S, const double* pts, double* out, long long B,
                         cudaStream_t st);
int fastd_blocks_per_sm(int k, int d, int threads, size_t smem);

// Newton corrector (newton.cu): per point, solve J dx = y - f from the
// evaluator's output and write x + dx
struct NewtonArgs {
    int n;
    long long B;
    const double* evals;   // [B][n + n*n][W] (pj_evaluate output)
    const double* points;  // [B][n][W]
    const double* target;  // [B][n][W] or null (y = 0)
    double* points_out;    // [B][n][W] (may alias points)
    double* norms;         // [B][2] or null: max-norm of y - f, of dx (high words)
    int* status;           // [B] or null: 0 ok, 1 singular, 2 non-finite result
    double* gscratch;      // non-null: per-CTA matrix slabs in global memory (gstride doubles each)
    size_t gstride;
};
size_t newton_matrix_bytes(int prec, int n);  // matrix planes, inverses, solution
size_t newton_int_bytes(int n);               // pivot bookkeeping (always in shared memory)
// panel = the blocked kernel for n <= 32 (newton_panel_kernel), else the column kernel
bool newton_panel_supported(int n);
int newton_max_threads(int n);  // the column kernel's launch bound for this n
// gs: the matrix in per-CTA global slabs (a separate kernel instantiation)
int newton_blocks_per_sm(int prec, int n, int threads, size_t smem, bool panel, bool gs);
cudaError_t launch_newton(int prec, const NewtonArgs& args, int blocks, int threads, size_t smem, bool panel,
                          cudaStream_t st);

}  // namespace pjb
