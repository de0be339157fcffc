// Host side of the C ABI (include/polyjac_b200.h): validation, packing v2, the stage-3 gather
// map, device residency, launch shape, and the deterministic input generator.
//
// Compiled with -ffp-contract=off: the double-double power-rule pre-scale below must round
// exactly like the oracle's restatement.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <exception>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <mutex>
#include <stdexcept>
#include <system_error>
#include <thread>
#include <vector>

#include "../../include/polyjac_b200.h"
#include "eval_kernels.h"

namespace {

thread_local std::string g_err;
}  // namespace

namespace pjb {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace pjb

namespace {

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? PJ_ENOMEM : PJ_ECUDA;
}
#define PJ_CUDA(call)                                      \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// Switches to a context's device for the duration of a call and restores the caller's device on
// every exit path (early error returns included).
struct DeviceGuard {
    int prev = -1;
    bool switched = false;
    cudaError_t enter(int dev) {
        cudaError_t e = cudaGetDevice(&prev);
        if (e) return e;
        if (prev != dev) {
            e = cudaSetDevice(dev);
            if (e) return e;
            switched = true;
        }
        return cudaSuccess;
    }
    ~DeviceGuard() {
        if (switched) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------------ validation
// Rules and wording follow validate_system, ref src/system.cpp:21-64 (violations as data);
// the byte-encoding cap n <= 256 follows build_layout, ref src/packing.cpp:25-27.
struct Violation {
    int poly, mono;
    std::string rule;
    std::string describe() const {
        if (poly >= 0 && mono >= 0)
            return "polynomial " + std::to_string(poly) + ", monomial " + std::to_string(mono) + ": " + rule;
        if (poly >= 0) return "polynomial " + std::to_string(poly) + ": " + rule;
        return rule;
    }
};

std::vector<Violation> validate(const pj_system_desc& S) {
    std::vector<Violation> v;
    auto flag = [&](int p, int g, const char* r) { v.push_back({p, g, r}); };
    if (S.n < 1) flag(-1, -1, "n must be at least 1");
    if (S.m < 1) flag(-1, -1, "m must be at least 1");
    if (S.k < 1) flag(-1, -1, "k must be at least 1");
    if (S.k > S.n) flag(-1, -1, "k exceeds n");
    if (S.d < 1) flag(-1, -1, "d must be at least 1");
    if (S.d > 255) flag(-1, -1, "d exceeds 255");
    if (!v.empty() && (S.n < 1 || S.m < 1 || S.k < 1)) return v;  // per-term checks need a shape
    if (!S.positions || !S.exponents || !S.coeffs) {
        flag(-1, -1, "term count is not n*m");
        return v;
    }
    for (int p = 0; p < S.n; ++p)
        for (int g = 0; g < S.m; ++g) {
            const size_t s = size_t(p) * S.m + g;
            const double re = S.coeffs[4 * s], im = S.coeffs[4 * s + 2];
            const double rl = S.coeffs[4 * s + 1], il = S.coeffs[4 * s + 3];
            if (!std::isfinite(re) || !std::isfinite(im) || !std::isfinite(rl) || !std::isfinite(il))
                flag(p, g, "non-finite coefficient");
            if (re == 0.0 && im == 0.0 && rl == 0.0 && il == 0.0) flag(p, g, "zero coefficient");
            for (int j = 0; j < S.k; ++j) {
                const int pos = S.positions[s * S.k + j], e = S.exponents[s * S.k + j];
                if (pos < 0 || pos >= S.n) flag(p, g, "variable index out of range [0,n-1]");
                if (j > 0 && pos <= S.positions[s * S.k + j - 1]) flag(p, g, "positions not strictly increasing");
                if (e < 1 || e > S.d) flag(p, g, "exponent out of range [1,d]");
            }
        }
    return v;
}

// ------------------------------------------------------------------ dd pre-scale (host)
// a * (hi, lo) for a small integer a: TwoProd of the high word via FMA, the low word folded
// in, one Fast2Sum. Exact for a <= 255 and a double coefficient.
void dd_mul_small(double hi, double lo, double a, double* oh, double* ol) {
    double p = hi * a;
    double e = std::fma(hi, a, -p);
    e = std::fma(lo, a, e);
    double s = p + e;
    *oh = s;
    *ol = e - (s - p);
}

// Launch state per evaluation mode: 0 = complex double (generic kernel, either order),
// 1 = complex dd in the reference order (generic kernel), 2 = complex dd in the fast order
// (specialised eval_fast.cu kernel when k is instantiated and the tables fit, else generic).
enum { kModeD = 0, kModeDDRef = 1, kModeDDFast = 2, kModes = 3 };
struct ModeState {
    pjb::LaunchCfg cfg;
    int over_threads = 0, over_tp = 0, over_variant = 0;
};

// ------------------------------------------------------------------ shared-memory bank model
// The fast dd kernel's gathers are 16-byte shared-memory loads (LDS.128) at data-dependent
// addresses. Model (calibrated against ncu's L1 shared wavefronts of the fast kernel: 2.57x
// ideal measured, 2.57x modelled): a warp access is served per quarter-warp (8 lanes); a
// quarter costs the largest number of distinct 16-byte addresses falling into one bank quad
// (address mod 8). addr[] in 16-byte units, < 0 = lane inactive.
int quarter_cost(const int* addr) {
    int q[8][8], nq[8] = {};
    int worst = 0;
    for (int l = 0; l < 8; ++l) {
        const int a = addr[l];
        if (a < 0) continue;
        const int b = a & 7;
        bool dup = false;
        for (int i = 0; i < nq[b]; ++i) dup |= q[b][i] == a;
        if (!dup) {
            q[b][nq[b]++] = a;
            worst = std::max(worst, nq[b]);
        }
    }
    return worst;
}

// Deterministic hill climb shared by the two orderings below: propose a swap, keep it when the
// cost of the (at most two) affected quarter-steps does not grow.
struct Lcg {
    uint64_t x;
    uint32_t next(uint32_t bound) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return uint32_t((x >> 33) % bound);
    }
};

// fn(p) for p in [0, n) over the host's cores (the per-row orderings below are independent)
template <class F>
void parallel_rows(int n, F&& fn) {
    const int nt = std::min(n / 4, int(std::min(32u, std::thread::hardware_concurrency())));
    if (nt <= 1) {
        for (int p = 0; p < n; ++p) fn(p);
        return;
    }
    std::atomic<int> next{0};
    std::exception_ptr err;
    std::mutex mu;
    auto work = [&] {
        try {
            for (int p; (p = next++) < n;) fn(p);
        } catch (...) {  // handed to the calling thread (a worker must not terminate the process)
            std::lock_guard<std::mutex> g(mu);
            if (!err) err = std::current_exception();
            next = n;
        }
    };
    std::vector<std::thread> th;
    th.reserve(nt);
    for (int t = 0; t < nt - 1; ++t) {
        try {
            th.emplace_back(work);
        } catch (const std::system_error&) {  // no more threads: the others and the caller finish
            break;
        }
    }
    work();
    for (auto& x : th) x.join();
    if (err) std::rethrow_exception(err);
}

// Fast-kernel variable order of one (row, 32-monomial chunk): per monomial a permutation of
// its k (position, exponent) pairs such that at every chain step j the lanes of a quarter-warp
// gather x from distinct bank quads (point table: 16-byte unit = position). The monomial's
// products commute, so only rounding changes (the fast order's contract).
// perm[g*k + j] = original index of the variable the kernel visits at step j.
// exps (d <= 2, else null): the kernel's d <= 2 path reads the common factor off its suffix-product
// chain, so every monomial's exponent-2 variables must come last; swaps stay inside a group.
void order_variables(const int32_t* pos, const int32_t* exps, int gl, int k, int p_seed, std::vector<uint8_t>& perm) {
    perm.resize(size_t(gl) * k);
    for (int g = 0; g < gl; ++g) {
        int at = 0;
        for (int pass = 0; pass < (exps ? 2 : 1); ++pass)  // exponent-1 variables first, then exponent 2
            for (int j = 0; j < k; ++j)
                if (!exps || (exps[size_t(g) * k + j] == 1) == (pass == 0)) perm[g * k + at++] = uint8_t(j);
    }
    if (k < 2) return;
    auto step_cost = [&](int qw, int j) {
        int a[8];
        for (int l = 0; l < 8; ++l) {
            const int g = qw * 8 + l;
            a[l] = g < gl ? pos[size_t(g) * k + perm[g * k + j]] : -1;
        }
        return quarter_cost(a);
    };
    Lcg r{uint64_t(p_seed) * 0x9e3779b97f4a7c15ull + 1};
    const int iters = 12 * gl * k;
    for (int it = 0; it < iters; ++it) {
        const int g = int(r.next(uint32_t(gl)));
        const int a = int(r.next(uint32_t(k)));
        int b = int(r.next(uint32_t(k - 1)));
        b += b >= a;
        if (exps && exps[size_t(g) * k + perm[g * k + a]] != exps[size_t(g) * k + perm[g * k + b]]) continue;
        const int qw = g / 8;
        const int before = step_cost(qw, a) + step_cost(qw, b);
        std::swap(perm[g * k + a], perm[g * k + b]);
        if (step_cost(qw, a) + step_cost(qw, b) > before) std::swap(perm[g * k + a], perm[g * k + b]);
    }
}

// Stage-3 order of one (row, chunk): ent = (output, staging code) in output-major order, cut
// into 32 runs of Rr. Within an output the order is free in the fast kernel (a sum's
// association, the contract of DESIGN.md §5); permute it so that the phase-1 loads, the
// segment-flush stores and the phase-2 reads of the segment partials (left at each segment's
// last staging slot) hit distinct bank quads (staging code = 16-byte unit).
void order_stage3(std::vector<std::pair<int, uint32_t>>& ent, int seed, int iters) {
    const int T = int(ent.size());
    if (T < 2) return;
    const int Rr = (T + 31) / 32;
    std::vector<uint8_t> flush(T);  // segment ends: fixed by the output boundaries and the runs
    for (int i = 0; i < T; ++i) {
        const int lane_end = std::min(T, (i / Rr + 1) * Rr);
        flush[i] = i + 1 == lane_end || ent[i + 1].first != ent[i].first;
    }
    // phase-2 groups: the partials read together = same slot (segment ordinal) of the outputs
    // owned as primaries by the lanes of one quarter-warp (o1 = 64*pass + lane, lane < 32)
    std::vector<int> g2(T, -1);
    std::vector<std::vector<int>> members;
    {
        std::vector<int> ordinal;
        std::vector<std::vector<int>> key2group;  // [pass*4 + quarter][slot]
        for (int i = 0; i < T; ++i) {
            if (!flush[i]) continue;
            const int o = ent[i].first;
            if (int(ordinal.size()) <= o) ordinal.resize(o + 1, 0);
            const int slot = ordinal[o]++;
            if ((o & 63) >= 32) continue;  // secondary outputs: paired later, not modelled
            const int key = (o >> 6) * 4 + (o & 31) / 8;
            if (int(key2group.size()) <= key) key2group.resize(key + 1);
            auto& v = key2group[key];
            if (int(v.size()) <= slot) v.resize(slot + 1, -1);
            if (v[slot] < 0) {
                v[slot] = int(members.size());
                members.emplace_back();
            }
            g2[i] = v[slot];
            members[g2[i]].push_back(i);
        }
    }
    auto p1_cost = [&](int qw, int r) {
        int a[8], f[8];
        for (int l = 0; l < 8; ++l) {
            const int i = (qw * 8 + l) * Rr + r;
            const bool ok = i < T;
            a[l] = ok ? int(ent[i].second) : -1;
            f[l] = ok && flush[i] ? a[l] : -1;
        }
        return quarter_cost(a) + quarter_cost(f);
    };
    auto p2_cost = [&](int g) {
        if (g < 0) return 0;
        int a[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
        const auto& mem = members[g];
        for (size_t l = 0; l < mem.size() && l < 8; ++l) a[l] = int(ent[mem[l]].second);
        return quarter_cost(a);
    };
    // group costs, cached: p1 group qw*Rr + r (loads and flush stores of one quarter-step), then
    // the phase-2 groups; a proposal re-evaluates only the (at most four) groups it touches
    const int G1 = 4 * Rr, G = G1 + int(members.size());
    auto group_cost = [&](int g) { return g < G1 ? p1_cost(g / Rr, g % Rr) : p2_cost(g - G1); };
    std::vector<int> gcost(G);
    for (int g = 0; g < G; ++g) gcost[g] = group_cost(g);
    auto groups_of = [&](int i, int j, int* out) {
        int cnt = 0;
        const int cand[4] = {(i / Rr) / 8 * Rr + i % Rr, (j / Rr) / 8 * Rr + j % Rr, g2[i] < 0 ? -1 : G1 + g2[i],
                             g2[j] < 0 ? -1 : G1 + g2[j]};
        for (int x : cand) {
            if (x < 0) continue;
            bool dup = false;
            for (int y = 0; y < cnt; ++y) dup |= out[y] == x;
            if (!dup) out[cnt++] = x;
        }
        return cnt;
    };
    // swappable pairs: two indices of the same output
    std::vector<int> start(T), len(T);
    for (int i = 0; i < T;) {
        int e = i;
        while (e < T && ent[e].first == ent[i].first) ++e;
        for (int q = i; q < e; ++q) {
            start[q] = i;
            len[q] = e - i;
        }
        i = e;
    }
    Lcg r{uint64_t(seed) * 0xbf58476d1ce4e5b9ull + 7};
    for (int it = 0; it < iters; ++it) {
        const int i = int(r.next(uint32_t(T)));
        if (len[i] < 2) continue;
        int j = start[i] + int(r.next(uint32_t(len[i] - 1)));
        j += j >= i;
        int gs[4], after[4];
        const int ng = groups_of(i, j, gs);
        int before = 0, now = 0;
        std::swap(ent[i].second, ent[j].second);
        for (int q = 0; q < ng; ++q) {
            before += gcost[gs[q]];
            now += after[q] = group_cost(gs[q]);
        }
        if (now > before) {
            std::swap(ent[i].second, ent[j].second);
        } else {
            for (int q = 0; q < ng; ++q) gcost[gs[q]] = after[q];
        }
    }
}

// Column-to-lane assignment of the complex-double fast kernel for one (row, chunk): its stage 3
// walks Jacobian column v's ascending-g gather list on one lane, so at every step the lanes read
// nearby g and collide in the same bank quads. Which columns share a quarter-warp is free (the
// per-column sums, and so the bit-exact reference order, are untouched): a seeded hill climb
// regroups them. Column 0 stays on lane 0 (it carries the row's value chain across chunks).
// lists: the chunk's gm_off / gm_ent slice; perm[lane slot] = column.
void assign_columns(const int* off, const uint16_t* ent, int n, int seed, uint8_t* perm) {
    for (int v = 0; v < n; ++v) perm[v] = uint8_t(v);
    if (n <= 8) return;
    auto group_cost = [&](int r0, int qw) {  // one quarter-warp of round r0, all steps
        int mx = 0, c = 0;
        for (int l = 0; l < 8; ++l) {
            const int vi = r0 + qw * 8 + l;
            if (vi < n) mx = std::max(mx, off[perm[vi] + 1] - off[perm[vi]]);
        }
        for (int it = 0; it < mx; ++it) {
            int a[8];
            for (int l = 0; l < 8; ++l) {
                const int vi = r0 + qw * 8 + l;
                const int v = vi < n ? perm[vi] : -1;
                if (v >= 0 && it < off[v + 1] - off[v]) {
                    const int e = ent[off[v] + it], j = e >> 5;  // the kernel's row swizzle (5j mod 8)
                    a[l] = j * 32 + ((e & 31) ^ ((5 * j) & 7));
                } else {
                    a[l] = -1;
                }
            }
            c += quarter_cost(a);
        }
        return c;
    };
    Lcg r{uint64_t(seed) * 0x94d049bb133111ebull + 3};
    const int iters = 48 * n;
    for (int it = 0; it < iters; ++it) {
        const int a = 1 + int(r.next(uint32_t(n - 1)));
        const int b = 1 + int(r.next(uint32_t(n - 1)));
        const int ga = a / 8, gb = b / 8;
        if (ga == gb) continue;
        const int before = group_cost(ga / 4 * 32, ga % 4) + group_cost(gb / 4 * 32, gb % 4);
        std::swap(perm[a], perm[b]);
        if (group_cost(ga / 4 * 32, ga % 4) + group_cost(gb / 4 * 32, gb % 4) > before) std::swap(perm[a], perm[b]);
    }
}

}  // namespace

struct pj_ctx {
    int device = 0;
    bool host_only = false;
    int sms = 0;
    size_t smem_optin = 0;
    int n, m, k, d, kp, chunks;
    // ragged system (pj_ctx_create_ragged): m = max m_p, k = max k_t, chunks = max chunks per row;
    // nterms = T; the per-row term / chunk offsets and per-term k below (host and device)
    bool ragged = false;
    int64_t nterms = 0;
    std::vector<int32_t> row_off, row_chunk, term_off;
    int* d_row_off = nullptr;
    int* d_row_chunk = nullptr;
    uint16_t* d_term_k = nullptr;
    std::vector<int32_t> pos, exps;  // host copies (index maps; ragged: CSR by term_off)
    std::vector<double> c_hi;         // plain coefficients (re, im) of the high words (layout export)
    std::vector<int> gm_off;
    std::vector<uint16_t> gm_ent;
    uint16_t* d_posexp = nullptr;
    uint32_t* d_posexp32 = nullptr;  // wide encoding (n > 256)
    uint16_t* d_posexpF = nullptr;   // the fast dd kernel's variable order (order_variables)
    bool wide = false;
    int* d_gm_off = nullptr;
    uint16_t* d_gm_ent = nullptr;
    int32_t* d_colq = nullptr;  // complex-double kernel's per-lane-slot column records (assign_columns)
    std::vector<uint32_t> sch, seg;  // fast-kernel stage-3 schedule (host copies)
    std::vector<uint16_t> segcode;
    std::vector<uint32_t> segq;  // [((p*C + c)*npass + pass)*32 + lane] x 4 words, see pj_ctx_create
    uint32_t* d_segq = nullptr;
    uint32_t* d_sch = nullptr;
    uint32_t* d_seg = nullptr;
    uint16_t* d_segcode = nullptr;
    int nseg = 0;
    int* d_flag = nullptr;   // [0]: set by the evaluation kernels on a non-finite coordinate;
                             // [1]: set by the finiteness check (PJ_VALIDATE, pj_newton_host)
    double* d_coef[2] = {};  // coefficient planes: [0] complex double, [1] complex dd
    double* d_coefT = nullptr;  // complex dd, tiled per (row, chunk) for the fast kernel
    ModeState mode[kModes];
    double* d_scratch = nullptr;
    size_t scratch_bytes = 0;
    // host-API pipeline: kHostStreams streams, each with its own device staging buffers, so
    // H2D of chunk i+1, the kernel on chunk i and D2H of chunk i-1 overlap
    static constexpr int kHostStreams = 3;
    double* d_in[kHostStreams] = {};
    double* d_out[kHostStreams] = {};
    size_t in_cap = 0, out_cap = 0;
    // small host batches (pj_evaluate_host, <= kSmallOut result bytes): page-locked staging
    // [points | results | flag], so the call is two async copies, the kernel and one sync
    static constexpr size_t kSmallOut = size_t(1) << 20;
    char* h_small = nullptr;
    size_t h_small_in = 0;  // bytes of the points part (results follow, then one int)
    // ... replayed as one CUDA graph (flag reset, H2D, kernel, D2H x 2, flag reset) for the last
    // (flags, batch, buffers, launch shape) it was captured for
    struct SmallGraph {
        cudaGraphExec_t exec = nullptr;
        int flags = 0;
        int64_t batch = 0;
        const void *d_in = nullptr, *d_out = nullptr, *h = nullptr;
        int variant = 0, blocks = 0, threads = 0, tp = 0;
        size_t smem = 0;
    } sgraph;
    cudaStream_t hstream[kHostStreams] = {};
    cudaEvent_t hdone[kHostStreams] = {};
    cudaEvent_t nfork = nullptr;  // pj_newton_step fork event
    // Newton corrector (f1): launch shape per precision, global matrix slabs when the
    // augmented matrix exceeds shared memory, host-API staging buffers
    struct NewtonPlan {
        int blocks = 0, threads = 0, over_threads = 0;
        int over_variant = 0;  // 0 auto (the column kernel), -1 column kernel, 1 panel (n <= 32)
        bool panel = false;
        size_t smem = 0;
        bool gscr = false;
    } newton[3];  // complex double, complex dd, mixed (PJ_NEWTON_MIXED)
    double* d_nscratch = nullptr;
    size_t nscratch_bytes = 0;
    double *d_nx[kHostStreams] = {}, *d_nwork[kHostStreams] = {}, *d_ntgt[kHostStreams] = {},
           *d_nnorm[kHostStreams] = {};
    int* d_nstat[kHostStreams] = {};
    size_t nx_cap = 0, nwork_cap = 0;

    // the complex-double fast kernel reads its column-to-lane assignment
    pjb::DevSystem dev_fastd() const {
        pjb::DevSystem S = dev(0);
        S.colq = reinterpret_cast<const int2*>(d_colq);
        return S;
    }
    // the fast dd kernel reads its own variable order (same tables otherwise)
    pjb::DevSystem dev_fast() const {
        pjb::DevSystem S = dev(1);
        S.posexp = d_posexpF;
        return S;
    }
    pjb::DevSystem dev(int pi) const {
        pjb::DevSystem S;
        S.n = n;
        S.m = m;
        S.k = k;
        S.d = d;
        S.nm = ragged ? int(nterms) : n * m;
        S.chunks = chunks;
        S.row_off = ragged ? d_row_off : nullptr;
        S.row_chunk = ragged ? d_row_chunk : nullptr;
        S.term_k = ragged ? d_term_k : nullptr;
        S.kp = kp;
        S.posexp = d_posexp;
        S.posexp32 = wide ? d_posexp32 : nullptr;
        S.coef = d_coef[pi];
        S.gm_off = d_gm_off;
        S.gm_ent = d_gm_ent;
        S.sch = d_sch;
        S.seg = d_seg;
        S.nseg = nseg;
        S.segcode = d_segcode;
        S.segq = reinterpret_cast<const uint4*>(d_segq);
        S.colq = nullptr;
        S.coefT = d_coefT;
        return S;
    }
};

namespace {

void free_ctx(pj_ctx* c) {
    if (!c) return;
    if (c->host_only) {
        delete c;
        return;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaFree(c->d_posexp);
    cudaFree(c->d_posexp32);
    cudaFree(c->d_posexpF);
    cudaFree(c->d_gm_off);
    cudaFree(c->d_gm_ent);
    cudaFree(c->d_colq);
    cudaFree(c->d_sch);
    cudaFree(c->d_seg);
    cudaFree(c->d_segcode);
    cudaFree(c->d_segq);
    cudaFree(c->d_flag);
    cudaFree(c->d_coef[0]);
    cudaFree(c->d_coef[1]);
    cudaFree(c->d_coefT);
    cudaFree(c->d_row_off);
    cudaFree(c->d_row_chunk);
    cudaFree(c->d_term_k);
    cudaFree(c->d_scratch);
    cudaFree(c->d_nscratch);
    for (int i = 0; i < pj_ctx::kHostStreams; ++i) {
        cudaFree(c->d_nx[i]);
        cudaFree(c->d_nwork[i]);
        cudaFree(c->d_ntgt[i]);
        cudaFree(c->d_nnorm[i]);
        cudaFree(c->d_nstat[i]);
    }
    for (int i = 0; i < pj_ctx::kHostStreams; ++i) {
        cudaFree(c->d_in[i]);
        cudaFree(c->d_out[i]);
        if (c->hstream[i]) cudaStreamDestroy(c->hstream[i]);
        if (c->hdone[i]) cudaEventDestroy(c->hdone[i]);
    }
    if (c->nfork) cudaEventDestroy(c->nfork);
    if (c->h_small) cudaFreeHost(c->h_small);
    if (c->sgraph.exec) cudaGraphExecDestroy(c->sgraph.exec);
    cudaSetDevice(prev);
    delete c;
}

// Shared-memory footprint of one CTA of the generic kernel: TP points' power tables +
// per-warp staging and accumulators (see eval_kernels.cu).
size_t smem_need(const pj_ctx* c, int W, int nw, int tp) {
    const size_t D1 = c->d > 2 ? c->d - 1 : 1;
    const size_t tab = D1 * W * c->n;
    const size_t per_warp = size_t(c->k + 1) * W * 32 + size_t(c->n + 1) * W;
    return (tp * tab + nw * per_warp) * sizeof(double);
}
// ... and of the fast kernel (eval_fast.cu): tables with the padded plane stride, per-warp
// staging + segment partials (+ accumulators when m > 32).
size_t smem_need_fast(const pj_ctx* c, int nw, int tp) {
    const size_t tab = size_t(pjb::fast_tab_rows(c->d)) * 4 * size_t(pjb::fast_plane_stride(c->n));
    const size_t acc = c->chunks > 1 ? size_t(c->n + 1) * 4 : 0;
    const size_t per_warp = size_t(c->k + 1) * 4 * 32 + acc;
    return (tp * tab + nw * per_warp) * sizeof(double);
}

int choose_launch(pj_ctx* c, int mode) {
    ModeState& M = c->mode[mode];
    const int W = mode == kModeD ? 2 : 4;
    const int precflag = mode == kModeD ? 1 : 2;
    int best_score = -1;
    pjb::LaunchCfg best;
    std::vector<int> nws = {8, 4, 2, 1}, tps = {8, 4, 2, 1};
    if (M.over_threads) nws = {M.over_threads / 32};
    if (M.over_tp) tps = {M.over_tp};
    auto consider = [&](int variant, int nw, int tp, size_t sm, int nb, int bonus) {
        if (nb <= 0) return;
        // resident warps first, then the tile-size preference (bonus)
        const int warps = std::min(nb * nw, 64);
        const int score = warps * 64 + bonus;
        if (score > best_score) {
            best_score = score;
            best.variant = variant;
            best.threads = nw * 32;
            best.tp = tp;
            best.smem_bytes = sm;
            best.blocks = nb * c->sms;
            best.gscratch = nullptr;
        }
    };
    if (mode == kModeDDFast && !c->wide && !c->ragged && pjb::fast_ws_supported(c->k, c->n, c->m, c->d) &&
        M.over_variant == 3) {
        // warp-specialised kernel (eval_fast_ws.cu, opt-in): 8-warp CTAs split into producers and
        // consumers, 2-point tiles (the ring of 8 staging buffers and its counters fill shared
        // memory). Measured at C2: 4 : 4 best, 10.49 M evals/s against 11.10 M
        // for the fused kernel, so the automatic choice stays with the fused kernel.
        const char* ev = std::getenv("PJ_WS_PRODUCERS");  // developer knob (A/B of the split)
        const int np = ev ? std::atoi(ev) : 4;
        std::vector<int> ftps = M.over_tp ? tps : std::vector<int>{2, 1};
        const int nw = M.over_threads ? M.over_threads / 32 : 8;
        for (size_t i = 0; i < ftps.size() && np > 0 && np < nw && nw <= 8; ++i) {
            const size_t sm = pjb::fast_ws_smem(c->n, c->k, nw, ftps[i]);
            if (sm > c->smem_optin) continue;
            const int before = best_score;
            consider(3, nw, ftps[i], sm, pjb::fast_ws_blocks_per_sm(c->k, c->n, nw * 32, sm), 100 + int(ftps.size() - i));
            if (best_score != before) best.producers = np;
        }
    }
    if (mode == kModeDDFast && !c->wide && !c->ragged && pjb::fast_supported(c->k) && M.over_variant >= 0 &&
        best_score < 0) {
        // measured (tools/tune.py, tools/tp_test.py): 8-warp CTAs beat more, smaller CTAs at
        // equal residency. Tiles: with 3 CTAs per SM (k <= 12) a 3-point tile uses the last
        // shared-memory slack and cuts the tile barriers per point (C2: 9.30 vs 9.27 M evals/s for
        // 2 points, 9.22 for 1); at one CTA per SM (k > 12, C3) 2-point tiles stay best (0.961 vs
        // 0.945 M for 3, 0.957 for 4)
        // k > 12 with the division form: two 4-warp CTAs with 1-point tiles per SM beat one 8-warp
        // CTA with 2-point tiles at C3 (1.355 vs 1.267 M evals/s, profiles/r02l_c3_cta_shapes2.log:
        // two independent tile barriers per SM), so 4-warp CTAs are considered first and win ties
        // (k > 12 admits 10-16 warp CTAs via pj_set_launch; measured at C3: 10 warps no faster)
        std::vector<int> fnws = M.over_threads ? nws : c->k <= 12 ? std::vector<int>{8} : std::vector<int>{4, 8};
        for (int nw : fnws) {
            std::vector<int> ftps = M.over_tp ? tps
                                    : c->k <= 12 ? std::vector<int>{3, 2, 4, 1}
                                    : nw == 4    ? std::vector<int>{1, 2, 4}
                                                 : std::vector<int>{2, 4, 1};
            for (size_t i = 0; i < ftps.size(); ++i) {
                const int tp = ftps[i];
                if (nw * 32 > (c->k <= 12 ? 256 : 512)) continue;  // fast_kernel's launch bounds
                const size_t sm = smem_need_fast(c, nw, tp);
                if (sm > c->smem_optin) continue;
                consider(1, nw, tp, sm, pjb::fast_blocks_per_sm(c->k, c->n, c->d, nw * 32, sm), int(ftps.size() - i));
            }
        }
    }
    if (mode == kModeD && !c->wide && !c->ragged && pjb::fastd_supported(c->k) && M.over_variant >= 0) {
        // point pairs per warp: tiles of 2 points per warp (one pair task per warp per row sweep)
        std::vector<int> fnws = M.over_threads ? nws : std::vector<int>{8, 4};
        std::vector<int> ftps = M.over_tp ? tps : std::vector<int>{16, 8, 4, 2};
        for (int nw : fnws)
            for (size_t i = 0; i < ftps.size(); ++i) {
                const int tp = ftps[i];
                if (nw > 8) continue;  // fastd_kernel's launch bounds: 256 threads
                const size_t sm = pjb::fastd_smem(c->n, c->m, c->k, c->d, nw, tp);
                if (sm > c->smem_optin) continue;
                consider(2, nw, tp, sm, pjb::fastd_blocks_per_sm(c->k, c->d, nw * 32, sm), int(ftps.size() - i));
            }
    }
    if (best_score < 0) {
        for (int nw : nws)
            for (int tp : tps) {
                if (nw > 8) continue;  // eval_kernel's launch bounds: 256 threads
                const size_t sm = smem_need(c, W, nw, tp);
                if (sm > c->smem_optin) continue;
                // fewer, fatter tiles (coefficient reuse) as long as a tile has a task per warp
                consider(-1, nw, tp, sm, pjb::max_blocks_per_sm(precflag, 0, nw * 32, sm, c->ragged), tp * c->n >= nw ? tp : 0);
            }
    }
    if (best_score < 0) {
        // global-scratch fallback for systems whose tables exceed shared memory
        const int nw = M.over_threads ? std::min(M.over_threads / 32, 8) : 4;
        const int tp = M.over_tp ? M.over_tp : 1;
        best.variant = -1;
        best.threads = nw * 32;
        best.tp = tp;
        best.smem_bytes = 0;
        best.blocks = c->sms * 4;
        const size_t need = smem_need(c, W, nw, tp) * best.blocks;
        if (need > c->scratch_bytes) {
            cudaFree(c->d_scratch);
            c->d_scratch = nullptr;
            c->scratch_bytes = 0;
            PJ_CUDA(cudaMalloc(&c->d_scratch, need));
            c->scratch_bytes = need;
        }
        best.gscratch = c->d_scratch;
    }
    best.flag = c->d_flag;
    M.cfg = best;
    return PJ_OK;
}

constexpr int kWideMaxN = 65535;

int check_desc(const pj_system_desc* sys, bool wide) {
    if (!sys) return fail(PJ_EINVAL, "null system descriptor");
    auto v = validate(*sys);
    if (!v.empty()) return fail(PJ_EINVAL, "build_layout: invalid system: " + v.front().describe());
    if (!wide && sys->n > 256) return fail(PJ_EINVAL, "build_layout: n > 256 does not fit the byte encoding");
    // wide encoding: 16-bit positions; stage-3 entries j*32 + g stay 16-bit
    if (wide && sys->n > kWideMaxN) return fail(PJ_EINVAL, "build_layout: n exceeds the wide encoding (65535)");
    if (wide && sys->k > 2046) return fail(PJ_EINVAL, "build_layout: k exceeds the wide encoding (2046)");
    return PJ_OK;
}

}  // namespace

// ------------------------------------------------------------------ Newton corrector (f1)
namespace {
// Newton plan index: 0 complex double, 1 complex dd, 2 the mixed solve (PJ_NEWTON_MIXED with
// PJ_PREC_DD: complex-double factors, dd refinement); its kernel precision code is index + 1
int newton_index(int flags) {
    const int p = flags & 0x0f;
    return p == PJ_PREC_D ? 0 : p == PJ_PREC_DD ? ((flags & PJ_NEWTON_MIXED) ? 2 : 1) : -1;
}
int newton_plan(pj_ctx* c, int pi, pj_ctx::NewtonPlan** out) {
    pj_ctx::NewtonPlan& P = c->newton[pi];
    const int prec = pi + 1;
    const size_t mb = pjb::newton_matrix_bytes(prec, c->n), ib = pjb::newton_int_bytes(c->n);
    if (!P.blocks) {
        // n <= 32: 128-thread CTAs (the kernel is compiled for at most 128 there, newton.cu)
        P.threads = P.over_threads ? P.over_threads : pjb::newton_max_threads(c->n);
        P.threads = std::min(P.threads, pjb::newton_max_threads(c->n));
        if (pi == 2) P.threads = 128;  // the mixed solve's residual uses exactly four warps
        // the panel kernel is opt-in: measured slower at C2 (dd 10.7 vs 7.2 ms, d 2.50 vs 2.44 ms)
        P.panel = pi < 2 && pjb::newton_panel_supported(c->n) && P.over_variant == 1 && mb + ib <= c->smem_optin;
        if (P.panel) P.threads = std::max(P.threads, 64);  // one look-ahead warp + updaters
        if (mb + ib <= c->smem_optin) {
            const int nb = pjb::newton_blocks_per_sm(prec, c->n, P.threads, mb + ib, P.panel, false);
            if (nb > 0) {
                P.smem = mb + ib;
                P.blocks = nb * c->sms;
                P.gscr = false;
            }
        }
        if (!P.blocks) {  // augmented matrix beyond shared memory: per-CTA slabs in HBM (L2-resident)
            P.panel = false;
            const int nb = std::max(1, std::min(pjb::newton_blocks_per_sm(prec, c->n, P.threads, ib, false, true), 4));
            P.smem = ib;
            P.blocks = nb * c->sms;
            P.gscr = true;
        }
    }
    if (P.gscr) {
        const size_t stride = (mb / sizeof(double) + 31) / 32 * 32;
        const size_t need = stride * sizeof(double) * size_t(P.blocks);
        if (need > c->nscratch_bytes) {
            cudaFree(c->d_nscratch);
            c->d_nscratch = nullptr;
            c->nscratch_bytes = 0;
            PJ_CUDA(cudaMalloc(&c->d_nscratch, need));
            c->nscratch_bytes = need;
        }
    }
    *out = &P;
    return PJ_OK;
}
}  // namespace

extern "C" {
#pragma GCC visibility push(default)

const char* pj_last_error(void) { return g_err.c_str(); }

const char* pj_version(void) { return "polyjac_b200 0.1 (sm_100a)"; }

int pj_validate(const pj_system_desc* sys, char* msg, size_t cap) {
    if (!sys) return fail(-1, "null system descriptor");
    auto v = validate(*sys);
    if (msg && cap) {
        std::string s = v.empty() ? "" : v.front().describe();
        std::strncpy(msg, s.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    g_err.clear();
    return int(v.size());
}

int pj_ctx_create(const pj_system_desc* sys, int device, pj_ctx** out) {
    return pj_ctx_create_ex(sys, device, 0, out);
}

struct HostPack;
static int ctx_create_impl(const pj_system_desc* sys, int device, int options, pj_ctx** out);

int pj_ctx_create_ex(const pj_system_desc* sys, int device, int options, pj_ctx** out) {
    // no C++ exception crosses the C ABI: host allocation failures (tables, the worker threads
    // of the host orderings) come back as PJ_ENOMEM
    try {
        return ctx_create_impl(sys, device, options, out);
    } catch (const std::bad_alloc&) {
        if (out) *out = nullptr;
        return fail(PJ_ENOMEM, "pj_ctx_create: host allocation failed");
    } catch (const std::exception& e) {
        if (out) *out = nullptr;
        return fail(PJ_ENOMEM, std::string("pj_ctx_create: ") + e.what());
    }
}

// Device residency shared by the uniform and the ragged context: upload the packed tables once,
// create the host-API streams, pick every mode's launch shape. Consumes c (freed on failure).
struct HostPack {
    std::vector<uint16_t> posexp, posexpF;
    std::vector<uint32_t> posexp32;
    std::vector<double> cd, cdd, cddT;
    std::vector<int32_t> colq;
    std::vector<uint16_t> term_k;  // ragged only
};
static int ctx_upload(pj_ctx* c, int device, const HostPack& hp, pj_ctx** out) {
    const auto& posexp = hp.posexp;
    const auto& posexp32 = hp.posexp32;
    const auto& posexpF = hp.posexpF;
    const auto& cd = hp.cd;
    const auto& cdd = hp.cdd;
    const auto& cddT = hp.cddT;
    const auto& colq = hp.colq;
    int rc = PJ_OK;
    if (device < 0) {  // host-only context: packing and index maps, no device residency
        c->host_only = true;
        g_err.clear();
        *out = c;
        return PJ_OK;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        free_ctx(c);
        return cuda_fail(e, "cudaSetDevice");
    }
    auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
        cudaError_t r = cudaMalloc(dst, bytes ? bytes : 16);
        if (r) return r;
        return bytes ? cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) ||
        (e = up((void**)&c->d_posexp, posexp.data(), posexp.size() * 2)) ||
        (e = up((void**)&c->d_posexp32, posexp32.data(), posexp32.size() * 4)) ||
        (e = up((void**)&c->d_posexpF, posexpF.data(), posexpF.size() * 2)) ||
        (e = up((void**)&c->d_coef[0], cd.data(), cd.size() * 8)) ||
        (e = up((void**)&c->d_coef[1], cdd.data(), cdd.size() * 8)) ||
        (e = up((void**)&c->d_coefT, cddT.data(), cddT.size() * 8)) ||
        (e = up((void**)&c->d_gm_off, c->gm_off.data(), c->gm_off.size() * 4)) ||
        (e = up((void**)&c->d_gm_ent, c->gm_ent.data(), c->gm_ent.size() * 2)) ||
        (e = up((void**)&c->d_colq, colq.data(), colq.size() * 4)) ||
        (e = up((void**)&c->d_sch, c->sch.data(), c->sch.size() * 4)) ||
        (e = up((void**)&c->d_seg, c->seg.data(), c->seg.size() * 4)) ||
        (e = up((void**)&c->d_segcode, c->segcode.data(), c->segcode.size() * 2)) ||
        (e = up((void**)&c->d_segq, c->segq.data(), c->segq.size() * 4)) ||
        (c->ragged && ((e = up((void**)&c->d_row_off, c->row_off.data(), c->row_off.size() * 4)) ||
                       (e = up((void**)&c->d_row_chunk, c->row_chunk.data(), c->row_chunk.size() * 4)) ||
                       (e = up((void**)&c->d_term_k, hp.term_k.data(), hp.term_k.size() * 2)))) ||
        (e = cudaMalloc((void**)&c->d_flag, 2 * sizeof(int))) || (e = cudaMemset(c->d_flag, 0, 2 * sizeof(int)))) {
        free_ctx(c);
        cudaSetDevice(prev);
        return cuda_fail(e, "pj_ctx_create: device upload");
    }
    for (int i = 0; i < pj_ctx::kHostStreams && !e; ++i) {
        e = cudaStreamCreateWithFlags(&c->hstream[i], cudaStreamNonBlocking);
        if (!e) e = cudaEventCreateWithFlags(&c->hdone[i], cudaEventDisableTiming);
    }
    if (e) {
        free_ctx(c);
        cudaSetDevice(prev);
        return cuda_fail(e, "pj_ctx_create: streams");
    }
    c->sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    e = pjb::set_smem_attr(c->smem_optin);
    if (e) {
        free_ctx(c);
        cudaSetDevice(prev);
        return cuda_fail(e, "pj_ctx_create: smem attribute");
    }
    for (int md = 0; md < kModes; ++md) {
        rc = choose_launch(c, md);
        if (rc) {
            free_ctx(c);
            cudaSetDevice(prev);
            return rc;
        }
    }
    cudaSetDevice(prev);
    g_err.clear();
    *out = c;
    return PJ_OK;
}

static int ctx_create_impl(const pj_system_desc* sys, int device, int options, pj_ctx** out) {
    if (!out) return fail(PJ_EINVAL, "null output pointer");
    *out = nullptr;
    if (options & ~PJ_CTX_WIDE) return fail(PJ_EINVAL, "unknown context option");
    const bool wide = (options & PJ_CTX_WIDE) && sys && sys->n > 256;
    int rc = check_desc(sys, options & PJ_CTX_WIDE);
    if (rc) return rc;
    pj_ctx* c = new pj_ctx();
    c->wide = wide;
    c->device = device;
    c->n = sys->n;
    c->m = sys->m;
    c->k = sys->k;
    c->d = sys->d;
    c->kp = (sys->k + 7) / 8 * 8;
    c->chunks = (sys->m + 31) / 32;
    const size_t nm = size_t(c->n) * c->m, k = c->k;
    c->pos.assign(sys->positions, sys->positions + nm * k);
    c->exps.assign(sys->exponents, sys->exponents + nm * k);
    c->c_hi.resize(2 * nm);
    for (size_t s = 0; s < nm; ++s) {
        c->c_hi[2 * s] = sys->coeffs[4 * s];
        c->c_hi[2 * s + 1] = sys->coeffs[4 * s + 2];
    }

    // packing v2: fused position/exponent words (ref src/packing.cpp:40-44); the wide encoding
    // (n > 256) widens them to pos | (exp-1) << 16 in 32 bits
    std::vector<uint16_t> posexp(wide ? 0 : nm * c->kp, 0);
    std::vector<uint32_t> posexp32(wide ? nm * c->kp : 0, 0);
    for (size_t s = 0; s < nm; ++s)
        for (size_t j = 0; j < k; ++j) {
            if (wide)
                posexp32[s * c->kp + j] = uint32_t(c->pos[s * k + j]) | (uint32_t(c->exps[s * k + j] - 1) << 16);
            else
                posexp[s * c->kp + j] = uint16_t(c->pos[s * k + j] | ((c->exps[s * k + j] - 1) << 8));
        }
    // coefficient planes, derivative-major with the power rule folded in (ref src/packing.cpp:46-49):
    // double: a*c rounded per component, exactly as the reference; dd: exact.
    std::vector<double> cd((k + 1) * 2 * nm), cdd((k + 1) * 4 * nm);
    for (size_t s = 0; s < nm; ++s) {
        const double* C = sys->coeffs + 4 * s;
        for (size_t j = 0; j <= k; ++j) {
            const double a = j < k ? double(c->exps[s * k + j]) : 1.0;
            if (j < k) {
                cd[(j * 2 + 0) * nm + s] = a * C[0];
                cd[(j * 2 + 1) * nm + s] = a * C[2];
                double h, l;
                dd_mul_small(C[0], C[1], a, &h, &l);
                cdd[(j * 4 + 0) * nm + s] = h;
                cdd[(j * 4 + 1) * nm + s] = l;
                dd_mul_small(C[2], C[3], a, &h, &l);
                cdd[(j * 4 + 2) * nm + s] = h;
                cdd[(j * 4 + 3) * nm + s] = l;
            } else {
                cd[(j * 2 + 0) * nm + s] = C[0];
                cd[(j * 2 + 1) * nm + s] = C[2];
                for (int q = 0; q < 4; ++q) cdd[(j * 4 + q) * nm + s] = C[q];
            }
        }
    }
    // the fast kernel seeds its backward chain with the plain coefficient c and applies the
    // power rule as an exact scaling, so it needs only c: dd, tiled per (row, 32-monomial chunk),
    // lane index fastest
    std::vector<double> cddT(size_t(c->n) * c->chunks * 4 * 32, 0.0);
    for (int p = 0; p < c->n; ++p)
        for (int g = 0; g < c->m; ++g) {
            const size_t s = size_t(p) * c->m + g;
            const size_t base = (size_t(p) * c->chunks + g / 32) * 4 * 32 + (g & 31);
            for (int q = 0; q < 4; ++q) cddT[base + q * 32] = sys->coeffs[4 * s + q];
        }
    // stage-3 gather map: for (row p, chunk c, column v) the ascending-g list of (g, j) with
    // positions[s*k+j] == v — the inverse of the reference's derivative slot map
    // mons_slot(s, derivative, v) = g*(n^2+n) + (v+1)*n + p (ref src/packing.cpp:8-17)
    const int n = c->n, C = c->chunks;
    std::vector<int> cnt(size_t(n) * C * n + 1, 0);
    for (int p = 0; p < n; ++p)
        for (int g = 0; g < c->m; ++g)
            for (size_t j = 0; j < k; ++j) {
                const size_t s = size_t(p) * c->m + g;
                cnt[(size_t(p) * C + g / 32) * n + c->pos[s * k + j]]++;
            }
    c->gm_off.assign(cnt.size(), 0);
    for (size_t i = 0; i + 1 < cnt.size(); ++i) c->gm_off[i + 1] = c->gm_off[i] + cnt[i];
    c->gm_ent.assign(c->gm_off.back(), 0);
    {
        std::vector<int> fill(c->gm_off.begin(), c->gm_off.end() - 1);
        for (int p = 0; p < n; ++p)
            for (int g = 0; g < c->m; ++g)  // ascending g: lists come out sorted
                for (size_t j = 0; j < k; ++j) {
                    const size_t s = size_t(p) * c->m + g;
                    const size_t li = (size_t(p) * C + g / 32) * n + c->pos[s * k + j];
                    c->gm_ent[fill[li]++] = uint16_t(j * 32 + (g & 31));
                }
    }

    // complex-double fast kernel: column-to-lane assignment per (p, c)
    std::vector<int32_t> colq(wide ? 0 : size_t(n) * C * n * 2, 0);
    if (!wide) {
        parallel_rows(n, [&](int p) {
            std::vector<int> off(n + 1);
            std::vector<uint8_t> perm(n);
            for (int ch = 0; ch < C; ++ch) {
                const size_t b = (size_t(p) * C + ch) * n;
                const int base = c->gm_off[b];
                for (int v = 0; v <= n; ++v) off[v] = c->gm_off[b + v] - base;
                assign_columns(off.data(), c->gm_ent.data() + base, n, p * C + ch, perm.data());
                for (int i = 0; i < n; ++i) {
                    const int v = perm[i];
                    colq[(b + i) * 2] = c->gm_off[b + v];
                    colq[(b + i) * 2 + 1] = (c->gm_off[b + v + 1] - c->gm_off[b + v]) | (v << 16);
                }
            }
        });
    }

    // fast-kernel stage-3 schedule: per (p, c) the output-major, ascending-g list of staged terms
    // (value terms first, then Jacobian columns), cut into 32 equal runs (one per lane); a segment
    // is a maximal piece of one output inside one run (byte encoding only: the wide encoding
    // always runs the generic kernel)
    std::vector<uint16_t> posexpF;  // fast dd kernel's variable order (see order_variables)
    if (!wide) {
        const int R = c->k + 1;
        const int kk = int(k);
        posexpF.assign(nm * c->kp, 0);
        std::vector<int32_t> fpos(nm * k);  // positions in the fast kernel's visiting order
        parallel_rows(n, [&](int p) {
            std::vector<uint8_t> perm;
            for (int ch = 0; ch < C; ++ch) {
                const int gl = std::min(32, c->m - ch * 32);
                const size_t s0 = size_t(p) * c->m + size_t(ch) * 32;
                order_variables(c->pos.data() + s0 * k, c->d <= 2 ? c->exps.data() + s0 * k : nullptr, gl, kk, p * C + ch,
                                perm);
                for (int g = 0; g < gl; ++g)
                    for (int j = 0; j < kk; ++j) {
                        const size_t s = s0 + g;
                        const int oj = perm[g * kk + j];
                        posexpF[s * c->kp + j] = posexp[s * c->kp + oj];
                        fpos[s * k + j] = c->pos[s * k + oj];
                    }
            }
        });
        // the fast kernel's gather lists: as gm_off/gm_ent, over the visiting order
        std::vector<int> foff(size_t(n) * C * n + 1, 0);
        for (int p = 0; p < n; ++p)
            for (int g = 0; g < c->m; ++g)
                for (size_t j = 0; j < k; ++j) foff[(size_t(p) * C + g / 32) * n + fpos[(size_t(p) * c->m + g) * k + j] + 1]++;
        for (size_t i = 0; i + 1 < foff.size(); ++i) foff[i + 1] += foff[i];
        std::vector<uint16_t> fent(foff.back());
        {
            std::vector<int> fill(foff.begin(), foff.end() - 1);
            for (int p = 0; p < n; ++p)
                for (int g = 0; g < c->m; ++g)
                    for (size_t j = 0; j < k; ++j) {
                        const size_t li = (size_t(p) * C + g / 32) * n + fpos[(size_t(p) * c->m + g) * k + j];
                        fent[fill[li]++] = uint16_t(j * 32 + (g & 31));
                    }
        }
        c->nseg = n + 1 + 32;
        c->sch.assign(size_t(n) * C * R * 32, 0);
        c->seg.assign(size_t(n) * C * (n + 1), 0);
        c->segcode.assign(size_t(n) * C * c->nseg, 0);
        // hill-climb budget: 48 proposals per term (model, C2: phase-1 load wavefronts 1,662 vs
        // 1,922 at 12 per term, ideal 1,152), capped at 2^22 proposals per context
        const int s3_iters = int(std::min<int64_t>(int64_t(48) * 32 * R, (int64_t(1) << 22) / (int64_t(n) * C)));
        parallel_rows(n, [&](int p) {
            std::vector<std::pair<int, uint32_t>> ent;  // (output, staging code)
            for (int ch = 0; ch < C; ++ch) {
                ent.clear();
                const int gl = std::min(32, c->m - ch * 32);
                for (int g = 0; g < gl; ++g) ent.push_back({0, uint32_t(c->k * 32 + g)});
                // primary outputs (o mod 64 < 32) in order; each secondary output is then inserted
                // at the first output boundary where all its entries fall into one run, so phase 2
                // reads it as a single partial (falls back to the end)
                int Tall = gl;
                for (int v = 0; v < n; ++v) {
                    const size_t li = (size_t(p) * C + ch) * n + v;
                    Tall += foff[li + 1] - foff[li];
                }
                const int Rall = (Tall + 31) / 32;
                std::vector<int> order;
                for (int v = 0; v < n; ++v)
                    if (((v + 1) & 63) < 32) order.push_back(v);
                for (int v = 0; v < n; ++v) {
                    if (((v + 1) & 63) < 32) continue;
                    const size_t li = (size_t(p) * C + ch) * n + v;
                    const int L = foff[li + 1] - foff[li];
                    int at = int(order.size()), pre = gl;
                    for (size_t i = 0; i <= order.size() && L > 0; ++i) {
                        if (pre / Rall == (pre + L - 1) / Rall) {
                            at = int(i);
                            break;
                        }
                        if (i < order.size()) {
                            const size_t lj = (size_t(p) * C + ch) * n + order[i];
                            pre += foff[lj + 1] - foff[lj];
                        }
                    }
                    order.insert(order.begin() + at, v);
                }
                for (int v : order) {
                    const size_t li = (size_t(p) * C + ch) * n + v;
                    for (int e = foff[li]; e < foff[li + 1]; ++e) ent.push_back({v + 1, fent[e]});
                }
                order_stage3(ent, p * C + ch, s3_iters);
                const int T = int(ent.size());
                const int Rr = (T + 31) / 32;
                int segid = -1, prev_o = -1;
                uint32_t* sc = c->sch.data() + (size_t(p) * C + ch) * R * 32;
                uint32_t* sg = c->seg.data() + (size_t(p) * C + ch) * (n + 1);
                for (int lane = 0; lane < 32; ++lane) {
                    const int a = lane * Rr, b = std::min(T, a + Rr);
                    for (int q = a; q < b; ++q) {
                        const int o = ent[q].first;
                        if (q == a || o != prev_o) {
                            ++segid;
                            if ((sg[o] >> 16) == 0) sg[o] = uint32_t(segid);
                            sg[o] += 1u << 16;
                        }
                        prev_o = o;
                        const bool flush = q + 1 == b || ent[q + 1].first != o;
                        // staging slot (j, g) as a 16-byte unit of the warp's staging area: the
                        // hi pair at 2*unit doubles, rows of 32 slots = 64 units (eval_fast.cu)
                        const uint32_t unit = (ent[q].second >> 5) * 64 + (ent[q].second & 31);
                        if (flush) c->segcode[(size_t(p) * C + ch) * c->nseg + segid] = uint16_t(unit);
                        sc[size_t(q - a) * 32 + lane] =
                            unit | (uint32_t(segid) << 13) | (flush ? pjb::kSchFlush : 0) | pjb::kSchValid;
                    }
                }
            }
        });
        // phase-2 records, per (p, c), pass k2 and lane: lane l owns output o1 = 64*k2 + l and at
        // most one secondary o2 in [64*k2 + 32, 64*k2 + 64), given to the lane with the lightest
        // load (longest-processing-time order), so one pass covers 64 outputs and the warp's add
        // slots are the largest per-lane total. Record: {cnt1 | cnt2 << 8 | o2 << 16 (0xffff:
        // none), six 16-bit segment codes (o1's, then o2's)}; past six, the lane's whole code
        // list sits in segx at the offset kept in segoff (rare)
        {
            const int npass = (n + 64) / 64;
            std::vector<uint16_t> segx(1, 0);
            std::vector<uint32_t> segoff(size_t(n) * C * npass * 32, 0);
            c->segq.assign(size_t(n) * C * npass * 32 * 4, 0);
            for (size_t pc = 0; pc < size_t(n) * C; ++pc) {
                auto cnt_of = [&](int o) { return int(c->seg[pc * (n + 1) + o] >> 16); };
                auto codes_of = [&](int o, std::vector<uint16_t>& dst) {
                    const uint32_t sd = c->seg[pc * (n + 1) + o];
                    for (int i = 0; i < int(sd >> 16); ++i) dst.push_back(c->segcode[pc * c->nseg + (sd & 0xffff) + i]);
                };
                for (int k2 = 0; k2 < npass; ++k2) {
                    int load[32], sec[32];
                    for (int l = 0; l < 32; ++l) {
                        const int o1 = 64 * k2 + l;
                        load[l] = o1 <= n ? cnt_of(o1) : 1 << 20;
                        sec[l] = -1;
                    }
                    std::vector<int> extra;
                    for (int o = 64 * k2 + 32; o <= std::min(n, 64 * k2 + 63); ++o) extra.push_back(o);
                    std::stable_sort(extra.begin(), extra.end(), [&](int x, int y) { return cnt_of(x) > cnt_of(y); });
                    for (int o : extra) {
                        int best = -1;
                        for (int l = 31; l >= 0; --l)
                            if (sec[l] < 0 && load[l] < (1 << 20) && (best < 0 || load[l] < load[best])) best = l;
                        sec[best] = o;
                        load[best] += cnt_of(o);
                    }
                    for (int l = 0; l < 32; ++l) {
                        const int o1 = 64 * k2 + l;
                        std::vector<uint16_t> codes;
                        int c1 = 0, c2 = 0;
                        if (o1 <= n) {
                            codes_of(o1, codes);
                            c1 = int(codes.size());
                        }
                        if (sec[l] >= 0) {
                            codes_of(sec[l], codes);
                            c2 = int(codes.size()) - c1;
                        }
                        const size_t rec = (pc * npass + k2) * 32 + l;
                        uint32_t* q = c->segq.data() + rec * 4;
                        q[0] = uint32_t(c1) | uint32_t(c2) << 8 | uint32_t(sec[l] >= 0 ? sec[l] : 0xffff) << 16;
                        for (int i = 0; i < std::min(int(codes.size()), 6); ++i) q[1 + i / 2] |= uint32_t(codes[i]) << (16 * (i & 1));
                        if (codes.size() > 6) {
                            segoff[rec] = uint32_t(segx.size());
                            segx.insert(segx.end(), codes.begin(), codes.end());
                        }
                    }
                }
            }
            c->seg.swap(segoff);
            c->segcode.swap(segx);
        }
    }

    HostPack hp;
    hp.posexp.swap(posexp);
    hp.posexp32.swap(posexp32);
    hp.posexpF.swap(posexpF);
    hp.cd.swap(cd);
    hp.cdd.swap(cdd);
    hp.cddT.swap(cddT);
    hp.colq.swap(colq);
    return ctx_upload(c, device, hp, out);
}

// ------------------------------------------------------------------ ragged systems
// validate_system's per-term rules and wording (ref src/system.cpp:21-64) over a CSR shape: the
// offsets are checked first (nothing past them is indexed when they are malformed).
static std::vector<Violation> validate_ragged(const pj_ragged_desc& S) {
    std::vector<Violation> v;
    auto flag = [&](int p, int g, const char* r) { v.push_back({p, g, r}); };
    if (S.n < 1) flag(-1, -1, "n must be at least 1");
    if (S.d < 1) flag(-1, -1, "d must be at least 1");
    if (S.d > 255) flag(-1, -1, "d exceeds 255");
    if (S.n < 1) return v;
    if (!S.row_off || !S.term_off) {
        flag(-1, -1, "missing row or term offsets");
        return v;
    }
    if (S.row_off[0] != 0) {
        flag(-1, -1, "row offsets must start at 0");
        return v;
    }
    bool shape_ok = true;
    for (int p = 0; p < S.n; ++p) {
        if (S.row_off[p + 1] < S.row_off[p]) {
            flag(p, -1, "row offsets decrease");
            shape_ok = false;
        } else if (S.row_off[p + 1] == S.row_off[p]) {
            flag(p, -1, "m must be at least 1");
        }
    }
    if (!shape_ok) return v;
    const int64_t T = S.row_off[S.n];
    if (S.term_off[0] != 0) {
        flag(-1, -1, "term offsets must start at 0");
        return v;
    }
    for (int p = 0; p < S.n; ++p)
        for (int64_t t = S.row_off[p]; t < S.row_off[p + 1]; ++t)
            if (S.term_off[t + 1] < S.term_off[t]) {
                flag(p, int(t - S.row_off[p]), "term offsets decrease");
                shape_ok = false;
            }
    if (!shape_ok) return v;
    if (T > 0 && (!S.positions || !S.exponents || !S.coeffs)) {
        flag(-1, -1, "missing term arrays");
        return v;
    }
    for (int p = 0; p < S.n; ++p)
        for (int64_t t = S.row_off[p]; t < S.row_off[p + 1]; ++t) {
            const int g = int(t - S.row_off[p]);
            const double* C = S.coeffs + 4 * t;
            if (!std::isfinite(C[0]) || !std::isfinite(C[1]) || !std::isfinite(C[2]) || !std::isfinite(C[3]))
                flag(p, g, "non-finite coefficient");
            if (C[0] == 0.0 && C[1] == 0.0 && C[2] == 0.0 && C[3] == 0.0) flag(p, g, "zero coefficient");
            const int kt = S.term_off[t + 1] - S.term_off[t];
            if (kt < 1) flag(p, g, "k must be at least 1");
            if (kt > S.n) flag(p, g, "k exceeds n");
            const int32_t* P = S.positions + S.term_off[t];
            const int32_t* E = S.exponents + S.term_off[t];
            for (int j = 0; j < kt; ++j) {
                if (P[j] < 0 || P[j] >= S.n) flag(p, g, "variable index out of range [0,n-1]");
                if (j > 0 && P[j] <= P[j - 1]) flag(p, g, "positions not strictly increasing");
                if (E[j] < 1 || E[j] > S.d) flag(p, g, "exponent out of range [1,d]");
            }
        }
    return v;
}

int pj_validate_ragged(const pj_ragged_desc* sys, char* msg, size_t cap) {
    if (!sys) return fail(-1, "null system descriptor");
    auto v = validate_ragged(*sys);
    if (msg && cap) {
        std::string s = v.empty() ? "" : v.front().describe();
        std::strncpy(msg, s.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    g_err.clear();
    return int(v.size());
}

// Packing of a ragged system for the generic kernel (RAG = true): posexp rows of stride
// kp = round8(max k) per term; coefficient planes [(k_max + 1)][W][T]: block j < k_t = a_j * c
// (rounded in double like ref src/packing.cpp:47, exact in dd), block k_max = c (unused blocks 0);
// gather map per (row chunk, column) over the global chunk index row_chunk[p] + g/32, ascending g.
static int ctx_create_ragged_impl(const pj_ragged_desc* sys, int device, int options, pj_ctx** out) {
    if (!out) return fail(PJ_EINVAL, "null output pointer");
    *out = nullptr;
    if (options & ~PJ_CTX_WIDE) return fail(PJ_EINVAL, "unknown context option");
    if (!sys) return fail(PJ_EINVAL, "null system descriptor");
    {
        auto v = validate_ragged(*sys);
        if (!v.empty()) return fail(PJ_EINVAL, "build_layout: invalid system: " + v.front().describe());
    }
    const bool wide_opt = options & PJ_CTX_WIDE;
    if (!wide_opt && sys->n > 256) return fail(PJ_EINVAL, "build_layout: n > 256 does not fit the byte encoding");
    if (wide_opt && sys->n > kWideMaxN) return fail(PJ_EINVAL, "build_layout: n exceeds the wide encoding (65535)");
    const int n = sys->n;
    const int64_t T = sys->row_off[n];
    int kmax = 0, mmax = 0;
    for (int64_t t = 0; t < T; ++t) kmax = std::max(kmax, sys->term_off[t + 1] - sys->term_off[t]);
    for (int p = 0; p < n; ++p) mmax = std::max(mmax, sys->row_off[p + 1] - sys->row_off[p]);
    if (kmax > 2046) return fail(PJ_EINVAL, "build_layout: k exceeds the wide encoding (2046)");
    if (T > (int64_t(1) << 31) / (kmax + 1) / 4) return fail(PJ_EINVAL, "build_layout: too many terms");
    pj_ctx* c = new pj_ctx();
    c->ragged = true;
    c->wide = wide_opt && n > 256;
    c->device = device;
    c->n = n;
    c->d = sys->d;
    c->m = mmax;
    c->k = kmax;
    c->kp = (kmax + 7) / 8 * 8;
    c->chunks = (mmax + 31) / 32;
    c->nterms = T;
    c->row_off.assign(sys->row_off, sys->row_off + n + 1);
    c->term_off.assign(sys->term_off, sys->term_off + T + 1);
    c->row_chunk.assign(n + 1, 0);
    for (int p = 0; p < n; ++p) c->row_chunk[p + 1] = c->row_chunk[p] + (c->row_off[p + 1] - c->row_off[p] + 31) / 32;
    const size_t nslots = size_t(c->term_off[T]);
    c->pos.assign(sys->positions, sys->positions + nslots);
    c->exps.assign(sys->exponents, sys->exponents + nslots);
    c->c_hi.resize(2 * size_t(T));
    HostPack hp;
    hp.term_k.resize(T);
    if (c->wide)
        hp.posexp32.assign(size_t(T) * c->kp, 0);
    else
        hp.posexp.assign(size_t(T) * c->kp, 0);
    const size_t K1 = size_t(kmax) + 1, TT = size_t(T);
    hp.cd.assign(K1 * 2 * TT, 0.0);
    hp.cdd.assign(K1 * 4 * TT, 0.0);
    for (size_t s = 0; s < TT; ++s) {
        const int kt = c->term_off[s + 1] - c->term_off[s];
        const int32_t* P = c->pos.data() + c->term_off[s];
        const int32_t* E = c->exps.data() + c->term_off[s];
        hp.term_k[s] = uint16_t(kt);
        const double* C = sys->coeffs + 4 * s;
        c->c_hi[2 * s] = C[0];
        c->c_hi[2 * s + 1] = C[2];
        for (int j = 0; j < kt; ++j) {
            if (c->wide)
                hp.posexp32[s * c->kp + j] = uint32_t(P[j]) | (uint32_t(E[j] - 1) << 16);
            else
                hp.posexp[s * c->kp + j] = uint16_t(P[j] | ((E[j] - 1) << 8));
            const double a = double(E[j]);
            hp.cd[(size_t(j) * 2 + 0) * TT + s] = a * C[0];
            hp.cd[(size_t(j) * 2 + 1) * TT + s] = a * C[2];
            double h, l;
            dd_mul_small(C[0], C[1], a, &h, &l);
            hp.cdd[(size_t(j) * 4 + 0) * TT + s] = h;
            hp.cdd[(size_t(j) * 4 + 1) * TT + s] = l;
            dd_mul_small(C[2], C[3], a, &h, &l);
            hp.cdd[(size_t(j) * 4 + 2) * TT + s] = h;
            hp.cdd[(size_t(j) * 4 + 3) * TT + s] = l;
        }
        hp.cd[(size_t(kmax) * 2 + 0) * TT + s] = C[0];
        hp.cd[(size_t(kmax) * 2 + 1) * TT + s] = C[2];
        for (int q = 0; q < 4; ++q) hp.cdd[(size_t(kmax) * 4 + q) * TT + s] = C[q];
    }
    // gather map: lists (global chunk, column), ascending g within the row
    const size_t nlists = size_t(c->row_chunk[n]) * n;
    std::vector<int> cnt(nlists + 1, 0);
    for (int p = 0; p < n; ++p)
        for (int64_t s = c->row_off[p]; s < c->row_off[p + 1]; ++s) {
            const int g = int(s - c->row_off[p]);
            for (int32_t q = c->term_off[s]; q < c->term_off[s + 1]; ++q)
                cnt[size_t(c->row_chunk[p] + g / 32) * n + c->pos[q]]++;
        }
    c->gm_off.assign(nlists + 1, 0);
    for (size_t i = 0; i < nlists; ++i) c->gm_off[i + 1] = c->gm_off[i] + cnt[i];
    c->gm_ent.assign(c->gm_off.back(), 0);
    {
        std::vector<int> fill(c->gm_off.begin(), c->gm_off.end() - 1);
        for (int p = 0; p < n; ++p)
            for (int64_t s = c->row_off[p]; s < c->row_off[p + 1]; ++s) {
                const int g = int(s - c->row_off[p]);
                for (int32_t q = c->term_off[s]; q < c->term_off[s + 1]; ++q) {
                    const size_t li = size_t(c->row_chunk[p] + g / 32) * n + c->pos[q];
                    c->gm_ent[fill[li]++] = uint16_t((q - c->term_off[s]) * 32 + (g & 31));
                }
            }
    }
    return ctx_upload(c, device, hp, out);
}

int pj_ctx_create_ragged(const pj_ragged_desc* sys, int device, int options, pj_ctx** out) {
    try {
        return ctx_create_ragged_impl(sys, device, options, out);
    } catch (const std::bad_alloc&) {
        if (out) *out = nullptr;
        return fail(PJ_ENOMEM, "pj_ctx_create_ragged: host allocation failed");
    } catch (const std::exception& ex) {
        if (out) *out = nullptr;
        return fail(PJ_ENOMEM, std::string("pj_ctx_create_ragged: ") + ex.what());
    }
}

void pj_ctx_destroy(pj_ctx* ctx) { free_ctx(ctx); }

static int prec_index(int flags) {
    const int p = flags & 0x0f;
    return p == PJ_PREC_D ? 0 : p == PJ_PREC_DD ? 1 : -1;
}
static int order_of(int flags) {
    if ((flags & 0x0f) == PJ_PREC_D) return (flags & PJ_ORDER_FAST) ? 1 : 0;
    return (flags & PJ_ORDER_REF) ? 0 : 1;
}
static int mode_of(int flags) {
    if ((flags & 0x0f) == PJ_PREC_D) return kModeD;
    return (flags & PJ_ORDER_REF) ? kModeDDRef : kModeDDFast;
}

int pj_evaluate(pj_ctx* ctx, int flags, const double* d_points, int64_t batch, double* d_out, void* stream) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "evaluate: unknown precision flag");
    if (batch < 0) return fail(PJ_EINVAL, "evaluate: negative batch");
    if (batch == 0) {
        g_err.clear();
        return PJ_OK;
    }
    if (!d_points || !d_out) return fail(PJ_EINVAL, "evaluate: null buffer");
    if (ctx->host_only) return fail(PJ_EINVAL, "evaluate: host-only context (created with device < 0)");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) PJ_CUDA(cudaSetDevice(ctx->device));
    // the global-scratch slab is shared by the modes and reallocated when a later mode (or a
    // pj_set_launch) needs more: read the current pointer, never the one stored at planning time
    pjb::LaunchCfg L = ctx->mode[mode_of(flags)].cfg;
    if (L.gscratch) L.gscratch = ctx->d_scratch;
    if (flags & PJ_VALIDATE) {
        // reject before any output is written, like ref src/engine.cpp:183-188: check the batch on
        // `stream`, read the verdict back (the one synchronisation of this mode)
        int bad = 0;
        cudaStream_t st = (cudaStream_t)stream;
        const long long words = (long long)batch * ctx->n * (pi == 0 ? 2 : 4);
        cudaError_t ve;
        if ((ve = cudaMemsetAsync(ctx->d_flag + 1, 0, sizeof(int), st)) ||
            (ve = pjb::launch_check_finite(d_points, words, ctx->d_flag + 1, ctx->sms, st)) ||
            (ve = cudaMemcpyAsync(&bad, ctx->d_flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st)) ||
            (ve = cudaStreamSynchronize(st))) {
            if (prev != ctx->device) cudaSetDevice(prev);
            return cuda_fail(ve, "evaluate: finiteness check");
        }
        if (bad) {
            if (prev != ctx->device) cudaSetDevice(prev);
            return fail(PJ_ENONFINITE, "evaluate: non-finite coordinate");
        }
    }
    if (L.variant == 1 || L.variant == 2) {
        // a batch with fewer tiles than CTAs (C1: one point) spreads each tile's tasks over
        // several CTAs, one task per warp at most, instead of leaving all but a few SMs idle; the
        // grid shrinks to the CTAs that have work (a multiple of the split, eval_fast.cu; the
        // complex-double kernel runs a separate split instantiation, eval_fastd.cu)
        const long long ntiles = (batch + L.tp - 1) / L.tp;
        if (ntiles < L.blocks) {
            const long long in_tile = std::min<long long>(batch, L.tp);
            const long long tasks = (L.variant == 2 ? (in_tile + 1) / 2 : in_tile) * ctx->n;
            const long long nw = L.threads / 32;
            L.splits = int(std::max(1LL, std::min<long long>(L.blocks / ntiles, (tasks + nw - 1) / nw)));
            L.blocks = int(std::min<long long>(L.blocks, ntiles * L.splits));
        }
    }
    cudaError_t e = L.variant == 1 ? pjb::launch_fast(ctx->k, L, ctx->dev_fast(), d_points, d_out, (long long)batch,
                                                     (cudaStream_t)stream)
                    : L.variant == 3 ? pjb::launch_fast_ws(ctx->k, L, ctx->dev_fast(), d_points, d_out, (long long)batch,
                                                           (cudaStream_t)stream)
                    : L.variant == 2 ? pjb::launch_fastd(ctx->k, L, ctx->dev_fastd(), d_points, d_out, (long long)batch,
                                                         (cudaStream_t)stream)
                                     : pjb::launch_eval(pi + 1, order_of(flags), L, ctx->dev(pi), d_points, d_out,
                                                        (long long)batch, (cudaStream_t)stream);
    if (prev != ctx->device) cudaSetDevice(prev);
    if (e) return cuda_fail(e, "evaluate: kernel launch");
    g_err.clear();
    return PJ_OK;
}

int pj_nonfinite_seen(pj_ctx* ctx, void* stream, int* seen) {
    if (!ctx || !seen) return fail(PJ_EINVAL, "null argument");
    if (ctx->host_only) return fail(PJ_EINVAL, "host-only context");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) PJ_CUDA(cudaSetDevice(ctx->device));
    int h = 0;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(&h, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream)) ||
        (e = cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), (cudaStream_t)stream)) ||
        (e = cudaStreamSynchronize((cudaStream_t)stream))) {
        if (prev != ctx->device) cudaSetDevice(prev);
        return cuda_fail(e, "pj_nonfinite_seen");
    }
    if (prev != ctx->device) cudaSetDevice(prev);
    *seen = h;
    g_err.clear();
    return PJ_OK;
}

int pj_evaluate_host(pj_ctx* ctx, int flags, const double* h_points, int64_t batch, double* h_out) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "evaluate: unknown precision flag");
    if (batch < 0) return fail(PJ_EINVAL, "evaluate: negative batch");
    if (batch == 0) {
        g_err.clear();
        return PJ_OK;
    }
    if (!h_points || !h_out) return fail(PJ_EINVAL, "evaluate: null buffer");
    if (ctx->host_only) return fail(PJ_EINVAL, "evaluate: host-only context (created with device < 0)");
    const int W = pi == 0 ? 2 : 4;
    const size_t in_pt = size_t(ctx->n) * W * 8;
    const size_t out_pt = (size_t(ctx->n) * ctx->n + ctx->n) * W * 8;
    // chunk: at least one full wave of the kernel, small enough that the D2H of one chunk
    // overlaps the kernel of the next (pinned host buffers give full overlap)
    const pjb::LaunchCfg& L = ctx->mode[mode_of(flags)].cfg;
    // (measured at C2 with pinned buffers, tools/pcie_bw.py + profiles/r02_e2e_chunks.log: one wave
    // and >= 64 MiB of results per chunk reach 56.3 GB/s of results, the box's D2H ceiling is
    // 56.5; four waves / 256 MiB chunks 55.5 — the pipeline fill and drain are a chunk each)
    int64_t chunk = std::max<int64_t>(int64_t(L.blocks) * L.tp, 1024);
    chunk = std::max<int64_t>(chunk, int64_t((size_t(64) << 20) / out_pt));
    // bounded staging: at most ~1 GiB of results per stream (wide systems have MB-sized results)
    chunk = std::min<int64_t>(chunk, std::max<int64_t>(1, int64_t((1ull << 30) / out_pt)));
    chunk = std::min<int64_t>(chunk, batch);
    const int nchunks = int((batch + chunk - 1) / chunk);
    // a global-scratch launch (tables beyond shared memory) indexes its slabs by CTA: two such
    // launches must never run concurrently, so those chunks stay on one stream
    const int ns = L.gscratch ? 1 : std::min(nchunks, int(pj_ctx::kHostStreams));
    DeviceGuard dg;
    PJ_CUDA(dg.enter(ctx->device));
    // a stale flag from an earlier asynchronous pj_evaluate must not fail this call (the small-batch
    // path below resets it on its own stream)
    const bool small = size_t(batch) * out_pt <= pj_ctx::kSmallOut && nchunks == 1;
    if (!small) {
        PJ_CUDA(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->hstream[0]));
        PJ_CUDA(cudaStreamSynchronize(ctx->hstream[0]));
    }
    if (size_t(chunk) * in_pt > ctx->in_cap || size_t(chunk) * out_pt > ctx->out_cap) {
        for (int i = 0; i < pj_ctx::kHostStreams; ++i) {
            cudaFree(ctx->d_in[i]);
            cudaFree(ctx->d_out[i]);
            ctx->d_in[i] = ctx->d_out[i] = nullptr;
        }
        ctx->in_cap = ctx->out_cap = 0;
        for (int i = 0; i < pj_ctx::kHostStreams; ++i) {
            PJ_CUDA(cudaMalloc(&ctx->d_in[i], size_t(chunk) * in_pt));
            PJ_CUDA(cudaMalloc(&ctx->d_out[i], size_t(chunk) * out_pt));
        }
        ctx->in_cap = size_t(chunk) * in_pt;
        ctx->out_cap = size_t(chunk) * out_pt;
    }
    if (small) {
        // small batch (C1: one point): page-locked staging, everything on one stream — the flag
        // reset, H2D, the kernel, D2H of the results and of the flag (then its reset) — and one
        // synchronisation, instead of pageable copies and separate flag round trips
        const size_t in_b = size_t(batch) * in_pt, out_b = size_t(batch) * out_pt;
        const size_t in_cap_b = pj_ctx::kSmallOut / out_pt * in_pt;  // points of the largest small batch
        if (!ctx->h_small) {
            PJ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_small), in_cap_b + pj_ctx::kSmallOut + 16,
                                  cudaHostAllocDefault));
            ctx->h_small_in = in_cap_b;
        }
        if (in_b > ctx->h_small_in) {  // (a different precision's point size: grow the staging)
            cudaFreeHost(ctx->h_small);
            ctx->h_small = nullptr;
            PJ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_small), in_b + pj_ctx::kSmallOut + 16,
                                  cudaHostAllocDefault));
            ctx->h_small_in = in_b;
        }
        char* hin = ctx->h_small;
        char* hout = ctx->h_small + ctx->h_small_in;
        int* hflag = reinterpret_cast<int*>(hout + pj_ctx::kSmallOut);
        cudaStream_t st = ctx->hstream[0];
        std::memcpy(hin, h_points, in_b);
        // the six stream operations, enqueued directly or captured into the context's graph
        auto enqueue = [&]() -> int {
            cudaError_t e;
            if ((e = cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), st)) ||
                (e = cudaMemcpyAsync(ctx->d_in[0], hin, in_b, cudaMemcpyHostToDevice, st)))
                return cuda_fail(e, "evaluate_host");
            if (int rc = pj_evaluate(ctx, flags, ctx->d_in[0], batch, ctx->d_out[0], st)) return rc;
            if ((e = cudaMemcpyAsync(hout, ctx->d_out[0], out_b, cudaMemcpyDeviceToHost, st)) ||
                (e = cudaMemcpyAsync(hflag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st)) ||
                (e = cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), st)))
                return cuda_fail(e, "evaluate_host");
            return PJ_OK;
        };
        // graph replay (one launch instead of six operations), not for PJ_VALIDATE (its check reads
        // the verdict back inside pj_evaluate); any capture failure falls back to direct enqueueing
        // (nor for global-scratch launches: the slab pointer is re-read at every launch and may move)
        bool replay = !(flags & PJ_VALIDATE) && !ctx->mode[mode_of(flags)].cfg.gscratch;
        if (replay) {
            pj_ctx::SmallGraph& G = ctx->sgraph;
            const pjb::LaunchCfg& Lc = ctx->mode[mode_of(flags)].cfg;
            const bool match = G.exec && G.flags == flags && G.batch == batch && G.d_in == ctx->d_in[0] &&
                               G.d_out == ctx->d_out[0] && G.h == ctx->h_small && G.variant == Lc.variant &&
                               G.blocks == Lc.blocks && G.threads == Lc.threads && G.tp == Lc.tp &&
                               G.smem == Lc.smem_bytes;
            if (!match) {
                if (G.exec) cudaGraphExecDestroy(G.exec);
                G.exec = nullptr;
                cudaGraph_t g = nullptr;
                bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
                if (ok) {
                    const int rc = enqueue();
                    ok = cudaStreamEndCapture(st, &g) == cudaSuccess && rc == PJ_OK && g;
                    ok = ok && cudaGraphInstantiate(&G.exec, g, 0) == cudaSuccess;
                    if (g) cudaGraphDestroy(g);
                }
                if (ok) {
                    G.flags = flags;
                    G.batch = batch;
                    G.d_in = ctx->d_in[0];
                    G.d_out = ctx->d_out[0];
                    G.h = ctx->h_small;
                    G.variant = Lc.variant;
                    G.blocks = Lc.blocks;
                    G.threads = Lc.threads;
                    G.tp = Lc.tp;
                    G.smem = Lc.smem_bytes;
                } else {
                    G.exec = nullptr;
                    cudaGetLastError();  // a failed capture leaves no sticky error behind
                    replay = false;
                }
            }
            if (replay) PJ_CUDA(cudaGraphLaunch(G.exec, st));
        }
        if (!replay) {
            if (int rc = enqueue()) {
                cudaStreamSynchronize(st);
                return rc;
            }
        }
        PJ_CUDA(cudaStreamSynchronize(st));
        if (*hflag) return fail(PJ_ENONFINITE, "evaluate: non-finite coordinate");
        std::memcpy(h_out, hout, out_b);
        g_err.clear();
        return PJ_OK;
    }
    int rc = PJ_OK;
    for (int c = 0; c < nchunks && rc == PJ_OK; ++c) {
        const int si = c % ns;
        cudaStream_t st = ctx->hstream[si];
        const int64_t b0 = int64_t(c) * chunk, nb = std::min<int64_t>(chunk, batch - b0);
        PJ_CUDA(cudaMemcpyAsync(ctx->d_in[si], reinterpret_cast<const char*>(h_points) + size_t(b0) * in_pt,
                                size_t(nb) * in_pt, cudaMemcpyHostToDevice, st));
        rc = pj_evaluate(ctx, flags, ctx->d_in[si], nb, ctx->d_out[si], st);
        if (rc) break;
        PJ_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(h_out) + size_t(b0) * out_pt, ctx->d_out[si],
                                size_t(nb) * out_pt, cudaMemcpyDeviceToHost, st));
    }
    for (int i = 0; i < ns; ++i) {
        cudaError_t e = cudaStreamSynchronize(ctx->hstream[i]);
        if (e && rc == PJ_OK) rc = cuda_fail(e, "evaluate_host: stream");
    }
    if (rc) return rc;
    int seen = 0;
    rc = pj_nonfinite_seen(ctx, ctx->hstream[0], &seen);
    if (rc) return rc;
    if (seen) return fail(PJ_ENONFINITE, "evaluate: non-finite coordinate");
    g_err.clear();
    return PJ_OK;
}

int pj_layout_info(const pj_ctx* ctx, int32_t* n, int32_t* m, int32_t* k, int32_t* d, int64_t* footprint) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    if (n) *n = ctx->n;
    if (m) *m = ctx->m;
    if (k) *k = ctx->k;
    if (d) *d = ctx->d;
    if (footprint) *footprint = ctx->ragged ? 2 * int64_t(ctx->term_off.back()) : 2 * int64_t(ctx->n) * ctx->m * ctx->k;
    g_err.clear();
    return PJ_OK;
}

int pj_mons_slot(int64_t s, int kind, int var, int n, int m, int64_t* slot) {
    const int64_t nm = int64_t(n) * m;
    if (s < 0 || s >= nm) return fail(PJ_ERANGE, "mons_slot: monomial index " + std::to_string(s));
    const int64_t p = s / m, g = s % m, stride = int64_t(n) * n + n;
    if (kind == 0) {
        *slot = g * stride + p;
    } else {
        if (var < 0 || var >= n) return fail(PJ_ERANGE, "mons_slot: variable " + std::to_string(var));
        *slot = g * stride + int64_t(var + 1) * n + p;
    }
    g_err.clear();
    return PJ_OK;
}

int pj_slot_targets(const pj_ctx* ctx, int64_t s, int64_t* targets) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    if (ctx->ragged) return fail(PJ_EINVAL, "slot_targets: the Mons slot map is defined for uniform systems only");
    for (int j = 0; j < ctx->k; ++j) {
        int rc = pj_mons_slot(s, 1, s >= 0 && s < int64_t(ctx->n) * ctx->m ? ctx->pos[s * ctx->k + j] : 0,
                              ctx->n, ctx->m, targets + j);
        if (rc) return rc;
    }
    return pj_mons_slot(s, 0, -1, ctx->n, ctx->m, targets + ctx->k);
}

int64_t pj_zero_mask(const pj_ctx* ctx, int64_t* mask, int64_t cap) {
    if (!ctx) return fail(-1, "null context");
    if (ctx->ragged) return fail(-1, "zero_mask: the Mons buffer is defined for uniform systems only");
    // Regenerated from the device gather map: a Mons slot is claimed iff it is a value slot or
    // its (p, v, g) appears in the (p, chunk(g), v) list. Everything else is the zero mask.
    const int64_t n = ctx->n, m = ctx->m, C = ctx->chunks, stride = n * n + n;
    std::vector<unsigned char> claimed(size_t(stride * m), 0);
    for (int64_t p = 0; p < n; ++p)
        for (int64_t g = 0; g < m; ++g) claimed[size_t(g * stride + p)] = 1;
    for (int64_t p = 0; p < n; ++p)
        for (int64_t c = 0; c < C; ++c)
            for (int64_t v = 0; v < n; ++v) {
                const size_t li = size_t((p * C + c) * n + v);
                for (int e = ctx->gm_off[li]; e < ctx->gm_off[li + 1]; ++e) {
                    const int64_t g = c * 32 + (ctx->gm_ent[e] & 31);
                    claimed[size_t(g * stride + (v + 1) * n + p)] = 1;
                }
            }
    int64_t len = 0;
    for (int64_t i = 0; i < stride * m; ++i)
        if (!claimed[size_t(i)]) {
            if (len < cap && mask) mask[len] = i;
            ++len;
        }
    g_err.clear();
    return len;
}

int pj_layout_export(const pj_ctx* ctx, uint8_t* positions, uint8_t* exponents, double* coeffs) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    if (ctx->n > 256) return fail(PJ_EINVAL, "layout: n > 256 has no byte encoding (wide context)");
    if (ctx->ragged) return fail(PJ_EINVAL, "layout: PackedLayout is defined for uniform systems only");
    const size_t nm = size_t(ctx->n) * ctx->m, k = size_t(ctx->k);
    // ref src/packing.cpp:40-49: positions / exponents-minus-one bytes in S_m order; coefficient
    // blocks derivative-major, block j < k = a_j * c rounded per component in double, block k = c.
    // The plain coefficient is recovered from the dd planes' high words of block k.
    for (size_t s = 0; s < nm; ++s)
        for (size_t j = 0; j < k; ++j) {
            if (positions) positions[s * k + j] = uint8_t(ctx->pos[s * k + j]);
            if (exponents) exponents[s * k + j] = uint8_t(ctx->exps[s * k + j] - 1);
        }
    if (coeffs) {
        for (size_t s = 0; s < nm; ++s) {
            const double re = ctx->c_hi[2 * s], im = ctx->c_hi[2 * s + 1];
            for (size_t j = 0; j <= k; ++j) {
                const double a = j < k ? double(ctx->exps[s * k + j]) : 1.0;
                coeffs[2 * (j * nm + s)] = j < k ? a * re : re;
                coeffs[2 * (j * nm + s) + 1] = j < k ? a * im : im;
            }
        }
    }
    g_err.clear();
    return PJ_OK;
}

int64_t pj_structural_zeros(const pj_ctx* ctx, uint8_t* mask) {
    if (!ctx) return fail(-1, "null context");
    const int n = ctx->n, C = ctx->chunks;
    int64_t zeros = 0;
    for (int p = 0; p < n; ++p)
        for (int v = 0; v < n; ++v) {
            bool any = false;
            const int cb = ctx->ragged ? ctx->row_chunk[p] : p * C;
            const int nch = ctx->ragged ? ctx->row_chunk[p + 1] - cb : C;
            for (int c = 0; c < nch && !any; ++c) {
                const size_t li = (size_t(cb) + c) * n + v;
                any = ctx->gm_off[li + 1] > ctx->gm_off[li];
            }
            if (mask) mask[size_t(p) * n + v] = any ? 0 : 1;
            zeros += any ? 0 : 1;
        }
    g_err.clear();
    return zeros;
}

int pj_debug_corrupt_coeff(pj_ctx* ctx, int64_t s, double factor) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    if (ctx->host_only) return fail(PJ_EINVAL, "host-only context");
    if (ctx->ragged) return fail(PJ_EINVAL, "corrupt_coeff: uniform systems only");
    const int64_t nm = int64_t(ctx->n) * ctx->m;
    if (s < 0 || s >= nm) return fail(PJ_ERANGE, "corrupt_coeff: monomial index " + std::to_string(s));
    DeviceGuard dg;
    PJ_CUDA(dg.enter(ctx->device));
    PJ_CUDA(cudaDeviceSynchronize());
    auto scale = [&](double* base, size_t idx) -> cudaError_t {
        double v = 0.0;
        cudaError_t e = cudaMemcpy(&v, base + idx, sizeof v, cudaMemcpyDeviceToHost);
        if (e) return e;
        v *= factor;
        return cudaMemcpy(base + idx, &v, sizeof v, cudaMemcpyHostToDevice);
    };
    for (int j = 0; j <= ctx->k; ++j) {
        for (int c = 0; c < 2; ++c) PJ_CUDA(scale(ctx->d_coef[0], size_t(j * 2 + c) * nm + s));
        for (int c = 0; c < 4; ++c) PJ_CUDA(scale(ctx->d_coef[1], size_t(j * 4 + c) * nm + s));
    }
    const int64_t p = s / ctx->m, g = s % ctx->m;
    for (int q = 0; q < 4; ++q)
        PJ_CUDA(scale(ctx->d_coefT, size_t(((p * ctx->chunks + g / 32) * 4 + q) * 32 + (g & 31))));
    g_err.clear();
    return PJ_OK;
}

int pj_mult_counts(const pj_ctx* ctx, int64_t evals, uint64_t* counts) {
    if (!ctx || !counts) return fail(PJ_EINVAL, "null argument");
    const uint64_t n = ctx->n, nm = uint64_t(ctx->n) * ctx->m, k = ctx->k, d = ctx->d;
    const uint64_t sp = k >= 3 ? 3 * k - 6 : 0;
    if (ctx->ragged) {  // the closed form per term, summed (SPEC.md:477 with k -> k_t)
        uint64_t f = 0, s2 = 0, s3 = 0;
        for (int64_t t = 0; t < ctx->nterms; ++t) {
            const uint64_t kt = uint64_t(ctx->term_off[t + 1] - ctx->term_off[t]);
            const uint64_t spt = kt >= 3 ? 3 * kt - 6 : 0;
            f += kt - 1;
            s2 += spt + 2 * kt + 2;
            s3 += spt;
        }
        counts[0] = uint64_t(evals) * n * (d >= 2 ? d - 2 : 0);
        counts[1] = uint64_t(evals) * f;
        counts[2] = uint64_t(evals) * s2;
        counts[3] = uint64_t(evals) * s3;
        counts[4] = 0;
        g_err.clear();
        return PJ_OK;
    }
    counts[0] = uint64_t(evals) * n * (d >= 2 ? d - 2 : 0);
    counts[1] = uint64_t(evals) * nm * (k - 1);
    counts[2] = uint64_t(evals) * nm * (sp + 2 * k + 2);
    counts[3] = uint64_t(evals) * nm * sp;
    counts[4] = 0;
    g_err.clear();
    return PJ_OK;
}

// ------------------------------------------------------------------ input generator
// Same published algorithm as ref src/system.cpp:66-118 and src/rng.hpp: std::mt19937_64
// (output pinned by the standard), Lemire's multiply-shift bounded draw with rejection, and a
// 53-bit uniform mapped to [-1, 1). Monomial supports: partial Fisher-Yates k-subset, sorted;
// exponents 1 + below(d); coefficient components redrawn while both are zero.
namespace {
struct Gen {
    std::mt19937_64 e;
    explicit Gen(uint64_t seed) : e(seed) {}
    uint64_t below(uint64_t bound) {
        uint64_t x = e();
        __uint128_t mm = (__uint128_t)x * bound;
        uint64_t lo = uint64_t(mm);
        if (lo < bound) {
            const uint64_t thr = (0 - bound) % bound;
            while (lo < thr) {
                x = e();
                mm = (__uint128_t)x * bound;
                lo = uint64_t(mm);
            }
        }
        return uint64_t(mm >> 64);
    }
    double sym() { return 2.0 * (double(e() >> 11) * 0x1p-53) - 1.0; }
};
}  // namespace

int pj_random_system(int n, int m, int k, int d, uint64_t seed, int32_t* positions, int32_t* exponents,
                     double* coeffs) {
    if (n < 1) return fail(PJ_EINVAL, "random_system: n must be at least 1");
    if (m < 1) return fail(PJ_EINVAL, "random_system: m must be at least 1");
    if (k < 1 || k > n) return fail(PJ_EINVAL, "random_system: need 1 <= k <= n");
    if (d < 1 || d > 255) return fail(PJ_EINVAL, "random_system: need 1 <= d <= 255");
    Gen r(seed);
    std::vector<int> idx(n);
    for (size_t s = 0; s < size_t(n) * m; ++s) {
        for (int i = 0; i < n; ++i) idx[i] = i;
        for (int j = 0; j < k; ++j) std::swap(idx[j], idx[j + int(r.below(uint64_t(n - j)))]);
        std::sort(idx.begin(), idx.begin() + k);
        for (int j = 0; j < k; ++j) positions[s * k + j] = idx[j];
        for (int j = 0; j < k; ++j) exponents[s * k + j] = 1 + int(r.below(uint64_t(d)));
        double re, im;
        do {
            re = r.sym();
            im = r.sym();
        } while (re == 0.0 && im == 0.0);
        coeffs[4 * s + 0] = re;
        coeffs[4 * s + 1] = 0.0;
        coeffs[4 * s + 2] = im;
        coeffs[4 * s + 3] = 0.0;
    }
    g_err.clear();
    return PJ_OK;
}

int pj_random_ragged_system(int n, int m_lo, int m_hi, int k_lo, int k_hi, int d, uint64_t seed, int64_t* T,
                            int64_t* S, int32_t* row_off, int32_t* term_off, int32_t* positions, int32_t* exponents,
                            double* coeffs) {
    if (n < 1) return fail(PJ_EINVAL, "random_ragged_system: n must be at least 1");
    if (m_lo < 1 || m_hi < m_lo) return fail(PJ_EINVAL, "random_ragged_system: need 1 <= m_lo <= m_hi");
    if (k_lo < 1 || k_hi < k_lo || k_hi > n) return fail(PJ_EINVAL, "random_ragged_system: need 1 <= k_lo <= k_hi <= n");
    if (d < 1 || d > 255) return fail(PJ_EINVAL, "random_ragged_system: need 1 <= d <= 255");
    Gen r(seed);
    std::vector<int32_t> ro(n + 1, 0), to(1, 0), ps, es;
    std::vector<double> cs;
    std::vector<int> idx(n);
    for (int p = 0; p < n; ++p) ro[p + 1] = ro[p] + m_lo + int(r.below(uint64_t(m_hi - m_lo + 1)));
    for (int32_t t = 0; t < ro[n]; ++t) {
        const int k = k_lo + int(r.below(uint64_t(k_hi - k_lo + 1)));
        for (int i = 0; i < n; ++i) idx[i] = i;
        for (int j = 0; j < k; ++j) std::swap(idx[j], idx[j + int(r.below(uint64_t(n - j)))]);
        std::sort(idx.begin(), idx.begin() + k);
        for (int j = 0; j < k; ++j) ps.push_back(idx[j]);
        for (int j = 0; j < k; ++j) es.push_back(1 + int(r.below(uint64_t(d))));
        double re, im;
        do {
            re = r.sym();
            im = r.sym();
        } while (re == 0.0 && im == 0.0);
        cs.insert(cs.end(), {re, 0.0, im, 0.0});
        to.push_back(to.back() + k);
    }
    if (T) *T = ro[n];
    if (S) *S = to.back();
    if (row_off) std::copy(ro.begin(), ro.end(), row_off);
    if (term_off) std::copy(to.begin(), to.end(), term_off);
    if (positions) std::copy(ps.begin(), ps.end(), positions);
    if (exponents) std::copy(es.begin(), es.end(), exponents);
    if (coeffs) std::copy(cs.begin(), cs.end(), coeffs);
    g_err.clear();
    return PJ_OK;
}

int pj_random_points(int n, int64_t count, uint64_t seed, double* points) {
    return pj_random_points_range(n, 0, count, seed, points);
}

int pj_random_points_range(int n, int64_t first, int64_t count, uint64_t seed, double* points) {
    if (n < 1 || count < 0 || first < 0) return fail(PJ_EINVAL, "random_points: bad shape");
    Gen r(seed);
    r.e.discard(uint64_t(first) * uint64_t(n) * 2);
    for (int64_t i = 0; i < count * n; ++i) {
        points[2 * i] = r.sym();
        points[2 * i + 1] = r.sym();
    }
    g_err.clear();
    return PJ_OK;
}

int pj_set_launch(pj_ctx* ctx, int flags, int threads, int tile_points) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    if (ctx->host_only) return fail(PJ_EINVAL, "host-only context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "unknown precision flag");
    if (threads < 0 || threads > 384 || threads % 32)
        return fail(PJ_EINVAL, "threads must be a multiple of 32 <= 384 (<= 256 except the fast dd kernel for k > 12)");
    if (tile_points < 0) return fail(PJ_EINVAL, "tile_points must be >= 0");
    if (flags & PJ_OP_NEWTON) {
        if (threads == 32) return fail(PJ_EINVAL, "newton: threads must be >= 64");
        ctx->newton[newton_index(flags)].over_threads = threads;
        ctx->newton[newton_index(flags)].blocks = 0;  // re-planned on the next solve
        g_err.clear();
        return PJ_OK;
    }
    ModeState& M = ctx->mode[mode_of(flags)];
    const int old_threads = M.over_threads, old_tp = M.over_tp;
    M.over_threads = threads;
    M.over_tp = tile_points;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    int rc = choose_launch(ctx, mode_of(flags));
    if (!rc && threads > 256 && M.cfg.variant != 1) {
        // only the fast dd kernel (k > 12) is built for CTAs above 256 threads: keep the
        // previous shape instead of planning a launch that cannot run
        M.over_threads = old_threads;
        M.over_tp = old_tp;
        choose_launch(ctx, mode_of(flags));
        rc = fail(PJ_EINVAL, "threads > 256 need the fast dd kernel (k > 12) with tables that fit shared memory");
    }
    cudaSetDevice(prev);
    if (!rc) g_err.clear();
    return rc;
}

int pj_set_kernel_variant(pj_ctx* ctx, int flags, int variant) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    if (ctx->host_only) return fail(PJ_EINVAL, "host-only context");
    if (flags & PJ_OP_NEWTON) {
        const int pi = prec_index(flags);
        if (pi < 0) return fail(PJ_EINVAL, "unknown precision flag");
        if (variant > 1 || variant < -1) return fail(PJ_EINVAL, "unknown kernel variant");
        if (variant == 1 && !pjb::newton_panel_supported(ctx->n))
            return fail(PJ_EINVAL, "newton: the panel kernel needs n <= 32");
        ctx->newton[newton_index(flags)].over_variant = variant;
        ctx->newton[newton_index(flags)].blocks = 0;  // re-planned on the next solve
        g_err.clear();
        return PJ_OK;
    }
    const int md = mode_of(flags);
    if (md == kModeDDRef) return fail(PJ_EINVAL, "kernel variants exist for complex double and the fast dd order");
    if ((variant > 1 && !(variant == 3 && md == kModeDDFast)) || variant < -1)
        return fail(PJ_EINVAL, "unknown kernel variant");
    if (variant == 3 && !pjb::fast_ws_supported(ctx->k, ctx->n, ctx->m, ctx->d))
        return fail(PJ_EINVAL, "the warp-specialised kernel needs d <= 2, m <= 32, n <= 64, k in [2, 12]");
    if (variant == 1 && md == kModeDDFast && !pjb::fast_supported(ctx->k))
        return fail(PJ_EINVAL, "no specialised kernel for this k");
    if (variant == 1 && md == kModeD && !pjb::fastd_supported(ctx->k))
        return fail(PJ_EINVAL, "no specialised kernel for this k");
    ctx->mode[md].over_variant = variant;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    int rc = choose_launch(ctx, md);
    cudaSetDevice(prev);
    if (!rc) g_err.clear();
    return rc;
}

int pj_get_launch(pj_ctx* ctx, int flags, int32_t* threads, int32_t* tile_points, int32_t* blocks,
                  int64_t* smem_bytes, int32_t* variant) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "unknown precision flag");
    if (flags & PJ_OP_NEWTON) {
        if (ctx->host_only) return fail(PJ_EINVAL, "host-only context");
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(ctx->device);
        pj_ctx::NewtonPlan* P = nullptr;
        int rc = newton_plan(ctx, newton_index(flags), &P);
        cudaSetDevice(prev);
        if (rc) return rc;
        if (threads) *threads = P->threads;
        if (tile_points) *tile_points = 1;
        if (blocks) *blocks = P->blocks;
        if (smem_bytes) *smem_bytes = int64_t(P->smem);
        if (variant) *variant = P->gscr ? 2 : P->panel ? 1 : 0;
        g_err.clear();
        return PJ_OK;
    }
    const pjb::LaunchCfg& L = ctx->mode[mode_of(flags)].cfg;
    if (threads) *threads = L.threads;
    if (tile_points) *tile_points = L.tp;
    if (blocks) *blocks = L.blocks;
    if (smem_bytes) *smem_bytes = int64_t(L.smem_bytes);
    if (variant) *variant = L.variant;
    g_err.clear();
    return PJ_OK;
}



int pj_newton_solve(pj_ctx* ctx, int flags, const double* d_evals, const double* d_points, const double* d_target,
                    int64_t batch, double* d_points_out, double* d_norms, int32_t* d_status, void* stream) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "newton: unknown precision flag");
    if (batch < 0) return fail(PJ_EINVAL, "newton: negative batch");
    if (batch == 0) {
        g_err.clear();
        return PJ_OK;
    }
    if (!d_evals || !d_points || !d_points_out) return fail(PJ_EINVAL, "newton: null buffer");
    if (ctx->host_only) return fail(PJ_EINVAL, "newton: host-only context (created with device < 0)");
    if (ctx->n > 256) return fail(PJ_EINVAL, "newton: n > 256 is not supported");
    const int ni = newton_index(flags);
    if (ni == 2 && ctx->n > 32) return fail(PJ_EINVAL, "newton: the mixed solve (PJ_NEWTON_MIXED) needs n <= 32");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) PJ_CUDA(cudaSetDevice(ctx->device));
    pj_ctx::NewtonPlan* P = nullptr;
    int rc = newton_plan(ctx, ni, &P);
    if (rc) {
        if (prev != ctx->device) cudaSetDevice(prev);
        return rc;
    }
    pjb::NewtonArgs a;
    a.n = ctx->n;
    a.B = batch;
    a.evals = d_evals;
    a.points = d_points;
    a.target = d_target;
    a.points_out = d_points_out;
    a.norms = d_norms;
    a.status = d_status;
    a.gscratch = P->gscr ? ctx->d_nscratch : nullptr;
    a.gstride = (pjb::newton_matrix_bytes(ni + 1, ctx->n) / sizeof(double) + 31) / 32 * 32;
    cudaError_t e = pjb::launch_newton(ni + 1, a, P->blocks, P->threads, P->smem, P->panel, (cudaStream_t)stream);
    if (prev != ctx->device) cudaSetDevice(prev);
    if (e) return cuda_fail(e, "newton: kernel launch");
    g_err.clear();
    return PJ_OK;
}

}  // extern "C"

namespace {
// evaluate + solve of one batch on one stream
int newton_step_on(pj_ctx* ctx, int flags, const double* d_points, const double* d_target, int64_t batch,
                   double* d_work, double* d_points_out, double* d_norms, int32_t* d_status, cudaStream_t st) {
    if (batch > 0 && !d_work) return fail(PJ_EINVAL, "newton: null buffer");
    int rc = pj_evaluate(ctx, flags, d_points, batch, d_work, st);
    if (rc) return rc;
    return pj_newton_solve(ctx, flags, d_work, d_points, d_target, batch, d_points_out, d_norms, d_status, st);
}
}  // namespace

extern "C" {

int pj_newton_step(pj_ctx* ctx, int flags, const double* d_points, const double* d_target, int64_t batch,
                   double* d_work, double* d_points_out, double* d_norms, int32_t* d_status, void* stream) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "newton: unknown precision flag");
    if (batch <= 0 || ctx->host_only || !d_points || !d_work || !d_points_out)
        return newton_step_on(ctx, flags, d_points, d_target, batch, d_work, d_points_out, d_norms, d_status,
                              (cudaStream_t)stream);
    // Large batches: chunks of >= 4 evaluation waves alternate over two of the context's streams
    // (fork/join with events on the caller's stream), so one chunk's solve (latency-bound)
    // overlaps the next chunk's evaluation (FP64-bound). Chunks are independent point ranges.
    const int W = pi == 0 ? 2 : 4;
    const size_t x_pt = size_t(ctx->n) * W, out_pt = (size_t(ctx->n) * ctx->n + ctx->n) * W;  // doubles
    const pjb::LaunchCfg& L = ctx->mode[mode_of(flags)].cfg;
    const int64_t chunk = std::max<int64_t>(int64_t(L.blocks) * L.tp * 4, 1);
    bool gslab = L.gscratch != nullptr;  // per-CTA global slabs: no two launches may overlap
    {
        DeviceGuard dg;
        PJ_CUDA(dg.enter(ctx->device));
        pj_ctx::NewtonPlan* P = nullptr;
        const int prc = newton_plan(ctx, newton_index(flags), &P);
        if (prc) return prc;
        gslab = gslab || P->gscr;
    }
    if (batch < 2 * chunk || gslab)
        return newton_step_on(ctx, flags, d_points, d_target, batch, d_work, d_points_out, d_norms, d_status,
                              (cudaStream_t)stream);
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) PJ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t user = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (!ctx->nfork) e = cudaEventCreateWithFlags(&ctx->nfork, cudaEventDisableTiming);
    if (!e) e = cudaEventRecord(ctx->nfork, user);
    for (int s = 0; s < 2 && !e; ++s) e = cudaStreamWaitEvent(ctx->hstream[s], ctx->nfork, 0);
    int rc = e ? cuda_fail(e, "newton_step: fork") : PJ_OK;
    const int nchunks = int((batch + chunk - 1) / chunk);
    for (int c = 0; c < nchunks && rc == PJ_OK; ++c) {
        const int64_t b0 = int64_t(c) * chunk, nb = std::min<int64_t>(chunk, batch - b0);
        rc = newton_step_on(ctx, flags, d_points + b0 * x_pt, d_target ? d_target + b0 * x_pt : nullptr, nb,
                            d_work + b0 * out_pt, d_points_out + b0 * x_pt, d_norms ? d_norms + 2 * b0 : nullptr,
                            d_status ? d_status + b0 : nullptr, ctx->hstream[c & 1]);
    }
    for (int s = 0; s < 2; ++s) {  // join (also after a failure: the caller's stream must not run ahead)
        cudaError_t e2 = cudaEventRecord(ctx->hdone[s], ctx->hstream[s]);
        if (!e2) e2 = cudaStreamWaitEvent(user, ctx->hdone[s], 0);
        if (e2 && rc == PJ_OK) rc = cuda_fail(e2, "newton_step: join");
    }
    if (prev != ctx->device) cudaSetDevice(prev);
    if (rc == PJ_OK) g_err.clear();
    return rc;
}

int pj_newton_host(pj_ctx* ctx, int flags, const double* h_points, const double* h_target, int64_t batch, int iters,
                   double* h_points_out, double* h_norms, int32_t* h_status) {
    if (!ctx) return fail(PJ_EINVAL, "null context");
    const int pi = prec_index(flags);
    if (pi < 0) return fail(PJ_EINVAL, "newton: unknown precision flag");
    if (batch < 0) return fail(PJ_EINVAL, "newton: negative batch");
    if (iters < 1) return fail(PJ_EINVAL, "newton: iterations must be >= 1");
    if (batch == 0) {
        g_err.clear();
        return PJ_OK;
    }
    if (!h_points || !h_points_out) return fail(PJ_EINVAL, "newton: null buffer");
    if (ctx->host_only) return fail(PJ_EINVAL, "newton: host-only context (created with device < 0)");
    const int W = pi == 0 ? 2 : 4;
    const size_t x_pt = size_t(ctx->n) * W * 8;
    const size_t out_pt = (size_t(ctx->n) * ctx->n + ctx->n) * W * 8;
    // chunks of whole evaluation waves (>= 4 waves, >= 96 MiB of evaluator output), pipelined over
    // the context's host streams: each stream owns one set of staging buffers, so the H2D of one
    // chunk, the evaluate + solve of another and the D2H of a third overlap (stream order protects
    // every buffer's reuse)
    const pjb::LaunchCfg& L = ctx->mode[mode_of(flags)].cfg;
    int rc0 = PJ_OK;
    const int64_t wave = std::max<int64_t>(int64_t(L.blocks) * L.tp, 1);
    int64_t chunk = std::max<int64_t>(std::max<int64_t>(int64_t((96ull << 20) / out_pt), 4 * wave), 1);
    if (chunk > wave) chunk = chunk / wave * wave;
    chunk = std::min<int64_t>(chunk, std::max<int64_t>(1, int64_t((1ull << 30) / out_pt)));  // bounded staging
    chunk = std::min<int64_t>(chunk, batch);
    const int nchunks = int((batch + chunk - 1) / chunk);
    DeviceGuard dg;
    PJ_CUDA(dg.enter(ctx->device));
    pj_ctx::NewtonPlan* P = nullptr;
    rc0 = newton_plan(ctx, newton_index(flags), &P);
    if (rc0) return rc0;
    // global-scratch slabs (evaluation tables or Newton matrices beyond shared memory) are indexed
    // by CTA: such launches must not overlap, so the chunks then run on one stream
    const int ns = (L.gscratch || P->gscr) ? 1 : std::min(nchunks, int(pj_ctx::kHostStreams));
    // the input points are checked on their own flag (d_flag[1]); the evaluator's flag (d_flag[0])
    // is also raised by iterates that diverged to non-finite values — those are reported per point
    // through status = 2, so it is cleared on entry and on exit
    PJ_CUDA(cudaMemsetAsync(ctx->d_flag, 0, 2 * sizeof(int), ctx->hstream[0]));
    PJ_CUDA(cudaStreamSynchronize(ctx->hstream[0]));
    if (size_t(chunk) * x_pt > ctx->nx_cap || size_t(chunk) * out_pt > ctx->nwork_cap) {
        for (int i = 0; i < pj_ctx::kHostStreams; ++i) {
            cudaFree(ctx->d_nx[i]);
            cudaFree(ctx->d_nwork[i]);
            cudaFree(ctx->d_ntgt[i]);
            cudaFree(ctx->d_nnorm[i]);
            cudaFree(ctx->d_nstat[i]);
            ctx->d_nx[i] = ctx->d_nwork[i] = ctx->d_ntgt[i] = ctx->d_nnorm[i] = nullptr;
            ctx->d_nstat[i] = nullptr;
        }
        ctx->nx_cap = ctx->nwork_cap = 0;
        for (int i = 0; i < pj_ctx::kHostStreams; ++i) {
            PJ_CUDA(cudaMalloc(&ctx->d_nx[i], size_t(chunk) * x_pt));
            PJ_CUDA(cudaMalloc(&ctx->d_ntgt[i], size_t(chunk) * x_pt));
            PJ_CUDA(cudaMalloc(&ctx->d_nwork[i], size_t(chunk) * out_pt));
            PJ_CUDA(cudaMalloc(&ctx->d_nnorm[i], size_t(chunk) * 2 * sizeof(double)));
            PJ_CUDA(cudaMalloc(&ctx->d_nstat[i], size_t(chunk) * sizeof(int32_t)));
        }
        ctx->nx_cap = size_t(chunk) * x_pt;
        ctx->nwork_cap = size_t(chunk) * out_pt;
    }
    int rc = PJ_OK;
    for (int c = 0; c < nchunks && rc == PJ_OK; ++c) {
        const int si = c % ns;
        cudaStream_t st = ctx->hstream[si];
        const int64_t b0 = int64_t(c) * chunk, nb = std::min<int64_t>(chunk, batch - b0);
        double* dx = ctx->d_nx[si];
        double* dt = h_target ? ctx->d_ntgt[si] : nullptr;
        PJ_CUDA(cudaMemcpyAsync(dx, reinterpret_cast<const char*>(h_points) + size_t(b0) * x_pt, size_t(nb) * x_pt,
                                cudaMemcpyHostToDevice, st));
        if (dt)
            PJ_CUDA(cudaMemcpyAsync(dt, reinterpret_cast<const char*>(h_target) + size_t(b0) * x_pt,
                                    size_t(nb) * x_pt, cudaMemcpyHostToDevice, st));
        PJ_CUDA(pjb::launch_check_finite(dx, (long long)nb * ctx->n * W, ctx->d_flag + 1, ctx->sms, st));
        for (int it = 0; it < iters && rc == PJ_OK; ++it)
            rc = newton_step_on(ctx, flags, dx, dt, nb, ctx->d_nwork[si], dx, ctx->d_nnorm[si], ctx->d_nstat[si], st);
        if (rc) break;
        PJ_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(h_points_out) + size_t(b0) * x_pt, dx, size_t(nb) * x_pt,
                                cudaMemcpyDeviceToHost, st));
        if (h_norms)
            PJ_CUDA(cudaMemcpyAsync(h_norms + 2 * b0, ctx->d_nnorm[si], size_t(nb) * 2 * sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
        if (h_status)
            PJ_CUDA(cudaMemcpyAsync(h_status + b0, ctx->d_nstat[si], size_t(nb) * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, st));
    }
    for (int i = 0; i < ns; ++i) {
        cudaError_t e = cudaStreamSynchronize(ctx->hstream[i]);
        if (e && rc == PJ_OK) rc = cuda_fail(e, "newton_host: stream");
    }
    if (rc) return rc;
    int seen = 0;
    PJ_CUDA(cudaMemcpy(&seen, ctx->d_flag + 1, sizeof(int), cudaMemcpyDeviceToHost));
    PJ_CUDA(cudaMemset(ctx->d_flag, 0, 2 * sizeof(int)));
    if (seen) return fail(PJ_ENONFINITE, "newton: non-finite input coordinate");
    g_err.clear();
    return PJ_OK;
}

#pragma GCC visibility pop
}  // extern "C"
