// polyjac_b200 — command-line front end over the C ABI, with the
// reference CLI's subcommands, flags, exit codes (0 ok, 1 correctness failure, 2 usage or
// file-format error) and machine-readable RESULT line (ref tools/main.cpp:36-228):
//
//   polyjac_b200 generate --n N --m M --k K --d D [--seed S] --out PATH
//   polyjac_b200 bench (--system PATH | --n N --m M --k K --d D) [--seed S] [--evals E]
//                      [--points B] [--precision dd|d] [--device G] [--gpus G]
//     --gpus G shards the E evaluations over devices 0..G-1 (one context and host thread per
//     device, contiguous shards of one point stream, system replicated, no collective) and
//     reports the aggregate rate over the slowest device
//   polyjac_b200 check --system PATH [--points P] [--seed S] [--tol T] [--device G]
//
// Correctness gate and baseline, as in the reference (ref tools/main.cpp:75-144): every device
// result is compared with an INDEPENDENT brute-force evaluation on the host (naive_point below:
// the textbook definition term by term, powers by repeated multiplication — no packing, no
// Speelpenning products, no gather map, nothing shared with the device pipeline), per entry in
// the reference's relative-error convention (ref src/oracle.cpp:97-103) at 1e-10
// (ref tools/main.cpp:16). `bench` gates both device precisions at its point before timing and
// exits 1 on a failure; `baseline_ms` is that brute-force loop, single-threaded, over the same
// evaluation count (ref tools/main.cpp:88-96); `pipeline_ms` is the device time of the requested
// precision. `check` gates complex double and complex dd on --points random points. The hidden
// option --corrupt-coeff S (tests only) scales monomial S's device coefficient by 1.001 after the
// upload (the "deliberately corrupted coeffs entry" case of ref SPEC.md:462).
// --workers / --block-size are accepted for compatibility and ignored (no CPU pool).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/polyjac_b200.h"

namespace {

constexpr int64_t kConstantMemoryBytes = 65536;
constexpr double kGateTol = 1e-10;
constexpr uint64_t kPointSeedSalt = 0x9e3779b97f4a7c15ULL;

struct Args {
    std::string cmd;
    std::map<std::string, std::string> kv;
    bool help = false;
    std::string bad;
};

Args parse(int argc, char** argv) {
    Args a;
    int i = 1;
    if (i < argc && std::string(argv[i]).rfind("--", 0) != 0) a.cmd = argv[i++];
    for (; i < argc; ++i) {
        std::string s = argv[i];
        if (s == "--help" || s == "-h") {
            a.help = true;
            continue;
        }
        if (s.rfind("--", 0) != 0 || i + 1 >= argc) {
            a.bad = s;
            break;
        }
        a.kv[s.substr(2)] = argv[++i];
    }
    return a;
}

bool get_int(const Args& a, const char* k, int64_t* v) {
    auto it = a.kv.find(k);
    if (it == a.kv.end()) return false;
    char* end = nullptr;
    *v = std::strtoll(it->second.c_str(), &end, 10);
    return end && *end == 0;
}
bool get_dbl(const Args& a, const char* k, double* v) {
    auto it = a.kv.find(k);
    if (it == a.kv.end()) return false;
    char* end = nullptr;
    *v = std::strtod(it->second.c_str(), &end);
    return end && *end == 0;
}

void usage(FILE* f) {
    std::fprintf(f,
                 "polyjac_b200: sparse polynomial system + Jacobian evaluator on B200 (sm_100a),\n"
                 "complex double and complex double-double\n\n"
                 "  generate --n N --m M --k K --d D [--seed S] --out PATH\n"
                 "      write a random benchmark system file\n"
                 "  bench (--system PATH | --n N --m M --k K --d D) [--seed S] [--evals E] [--points B]\n"
                 "        [--precision dd|d] [--device G] [--gpus G]\n"
                 "      timed evaluation with a correctness gate; prints a RESULT key=value line\n"
                 "  check --system PATH [--points P] [--seed S] [--tol T] [--device G]\n"
                 "      device results (complex double and complex double-double) vs a brute-force host\n"
                 "      evaluation on random points\n");
}

int usage_error(const std::string& msg) {
    std::fprintf(stderr, "error: %s\n", msg.c_str());
    usage(stderr);
    return 2;
}

struct Sys {
    pj_system* owned = nullptr;
    std::vector<int32_t> pos, exps;
    std::vector<double> coeffs;
    pj_system_desc desc{};
    ~Sys() { pj_system_free(owned); }
};

double cabs2(double re, double im) { return std::hypot(re, im); }

// relative error in the reference's convention, the dd value rounded to double
double rel_err(double gre, double gim, double wre, double wim) {
    const double ag = cabs2(gre, gim), aw = cabs2(wre, wim), diff = cabs2(gre - wre, gim - wim);
    if (ag < 1e-300 && aw < 1e-300) return diff;
    return diff / std::max(ag, aw);
}

struct Report {
    double max_value = 0, max_jac = 0;
    int wv = -1, wp = -1, wi = -1;
    int64_t failures = 0;  // points with an entry above the tolerance
};

using cplx = std::complex<double>;

// Brute-force reference value of one point, computed on the host from the system description
// alone: for monomial c * prod_r x_{v_r}^{a_r} of polynomial p, the value adds c * prod_r P_r and
// the derivative by its j-th variable adds c * a_j * Q_j * prod_{r != j} P_r, where
// P_r = x^{a_r} and Q_r = x^{a_r - 1} are formed by repeated multiplication. O(k^2) per monomial.
// out: [n + n*n] = values, then the row-major Jacobian.
void naive_point(const pj_system_desc& S, const double* x /* [n][2] */, std::vector<cplx>& out) {
    const int n = S.n, k = S.k;
    out.assign(size_t(n) + size_t(n) * n, cplx(0.0, 0.0));
    std::vector<cplx> P(k), Q(k);
    for (int p = 0; p < n; ++p)
        for (int g = 0; g < S.m; ++g) {
            const size_t s = size_t(p) * S.m + g;
            const int32_t* v = S.positions + s * k;
            const int32_t* a = S.exponents + s * k;
            const cplx c(S.coeffs[4 * s], S.coeffs[4 * s + 2]);
            for (int r = 0; r < k; ++r) {
                const cplx xr(x[2 * v[r]], x[2 * v[r] + 1]);
                Q[r] = cplx(1.0, 0.0);
                for (int e = 1; e < a[r]; ++e) Q[r] *= xr;
                P[r] = Q[r] * xr;
            }
            cplx val = c;
            for (int r = 0; r < k; ++r) val *= P[r];
            out[p] += val;
            for (int j = 0; j < k; ++j) {
                cplx dj = c * double(a[j]) * Q[j];
                for (int r = 0; r < k; ++r)
                    if (r != j) dj *= P[r];
                out[n + size_t(p) * n + v[j]] += dj;
            }
        }
}

// one device result [n + n*n][W] (W = 2: complex double; 4: dd, compared after rounding to
// double) against the brute-force values; worst entries accumulated into rep
void compare_one(int n, const double* got, int W, const std::vector<cplx>& want, double tol, Report* rep) {
    bool bad = false;
    for (size_t o = 0; o < want.size(); ++o) {
        const double* q = got + o * W;
        const double gre = W == 4 ? q[0] + q[1] : q[0], gim = W == 4 ? q[2] + q[3] : q[1];
        const double e = rel_err(gre, gim, want[o].real(), want[o].imag());
        bad = bad || !(e <= tol);
        if (o < size_t(n)) {
            if (e > rep->max_value) rep->max_value = e, rep->wv = int(o);
        } else if (e > rep->max_jac) {
            rep->max_jac = e;
            rep->wp = int((o - n) / n);
            rep->wi = int((o - n) % n);
        }
    }
    rep->failures += bad ? 1 : 0;
}

// Device results on `B` points (host buffers [B][n][2]) in complex double AND complex dd, each
// against the brute-force host evaluation.
int gate_points(pj_ctx* ctx, const pj_system_desc& S, const std::vector<double>& pts_d, int64_t B, double tol,
                Report* rep) {
    const int n = S.n;
    const size_t nout = size_t(n) * n + n;
    std::vector<double> pts_dd(size_t(B) * n * 4, 0.0), out_d(size_t(B) * nout * 2), out_dd(size_t(B) * nout * 4);
    for (size_t i = 0; i < size_t(B) * n; ++i) {
        pts_dd[4 * i] = pts_d[2 * i];
        pts_dd[4 * i + 2] = pts_d[2 * i + 1];
    }
    int rc = pj_evaluate_host(ctx, PJ_PREC_D, pts_d.data(), B, out_d.data());
    if (rc == PJ_OK) rc = pj_evaluate_host(ctx, PJ_PREC_DD, pts_dd.data(), B, out_dd.data());
    if (rc != PJ_OK) return rc;
    std::vector<cplx> want;
    for (int64_t b = 0; b < B; ++b) {
        naive_point(S, pts_d.data() + size_t(b) * n * 2, want);
        compare_one(n, out_d.data() + size_t(b) * nout * 2, 2, want, tol, rep);
        compare_one(n, out_dd.data() + size_t(b) * nout * 4, 4, want, tol, rep);
    }
    return PJ_OK;
}

int corrupt_if_asked(const Args& a, pj_ctx* ctx) {
    auto it = a.kv.find("corrupt-coeff");
    if (it == a.kv.end()) return PJ_OK;
    return pj_debug_corrupt_coeff(ctx, std::strtoll(it->second.c_str(), nullptr, 10), 1.001);
}

std::string describe(const Report& r, double tol, bool pass) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s (tol %.3g): max value error %.3g at f[%d], max Jacobian error %.3g at J[%d][%d]",
                  pass ? "PASS" : "FAIL", tol, r.max_value, r.wv, r.max_jac, r.wp, r.wi);
    return buf;
}

int load_system(const Args& a, Sys& S, uint64_t seed, bool allow_generate) {
    auto it = a.kv.find("system");
    int64_t n, m, k, d;
    const bool gen = get_int(a, "n", &n) && get_int(a, "m", &m) && get_int(a, "k", &k) && get_int(a, "d", &d);
    if (it != a.kv.end()) {
        if (a.kv.count("n") || a.kv.count("m") || a.kv.count("k") || a.kv.count("d"))
            return usage_error("--system excludes --n --m --k --d");
        if (pj_system_read_file(it->second.c_str(), &S.owned) != PJ_OK) {
            std::fprintf(stderr, "error: %s\n", pj_last_error());
            return 2;
        }
        pj_system_view(S.owned, &S.desc);
        return 0;
    }
    if (!allow_generate) return usage_error("--system is required");
    if (!gen) return usage_error("pass --system or all of --n --m --k --d");
    const size_t nm = size_t(std::max<int64_t>(n, 0)) * size_t(std::max<int64_t>(m, 0));
    S.pos.resize(nm * size_t(std::max<int64_t>(k, 1)));
    S.exps.resize(S.pos.size());
    S.coeffs.resize(nm * 4);
    if (pj_random_system(int(n), int(m), int(k), int(d), seed, S.pos.data(), S.exps.data(), S.coeffs.data()) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        return 2;
    }
    S.desc = {int32_t(n), int32_t(m), int32_t(k), int32_t(d), S.pos.data(), S.exps.data(), S.coeffs.data()};
    return 0;
}

int cmd_generate(const Args& a) {
    int64_t n, m, k, d, seed = 1;
    if (!(get_int(a, "n", &n) && get_int(a, "m", &m) && get_int(a, "k", &k) && get_int(a, "d", &d)))
        return usage_error("generate needs --n --m --k --d");
    if (a.kv.count("seed") && !get_int(a, "seed", &seed)) return usage_error("bad --seed");
    auto out = a.kv.find("out");
    if (out == a.kv.end()) return usage_error("generate needs --out");
    Args b = a;
    b.kv.erase("out");
    Sys S;
    if (int rc = load_system(b, S, uint64_t(seed), true)) return rc;
    if (pj_system_write_file(&S.desc, out->second.c_str()) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        return 2;
    }
    std::printf("generated %s: n=%lld m=%lld k=%lld d=%lld monomials=%lld seed=%lld\n", out->second.c_str(),
                (long long)n, (long long)m, (long long)k, (long long)d, (long long)(n * m), (long long)seed);
    const int64_t fp = 2 * n * m * k;
    std::printf("constant-memory footprint (positions+exponents): %lld bytes\n", (long long)fp);
    if (fp >= kConstantMemoryBytes)
        std::fprintf(stderr,
                     "warning: footprint %lld bytes reaches the %lld-byte constant-memory capacity; "
                     "positions/exponents would not fit (the B200 path keeps them in global/L2)\n",
                     (long long)fp, (long long)kConstantMemoryBytes);
    return 0;
}

int cmd_bench(const Args& a) {
    int64_t seed = 1, evals = 1000, points = 65536, device = 0;
    if (a.kv.count("seed") && !get_int(a, "seed", &seed)) return usage_error("bad --seed");
    if (a.kv.count("evals") && (!get_int(a, "evals", &evals) || evals < 1)) return usage_error("--evals must be >= 1");
    if (a.kv.count("points") && (!get_int(a, "points", &points) || points < 1))
        return usage_error("--points must be >= 1");
    if (a.kv.count("device") && !get_int(a, "device", &device)) return usage_error("bad --device");
    int64_t gpus = 1;
    if (a.kv.count("gpus") && (!get_int(a, "gpus", &gpus) || gpus < 1)) return usage_error("--gpus must be >= 1");
    if (gpus > 1) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
        if (gpus > ndev) return usage_error("--gpus " + std::to_string(gpus) + " exceeds the " + std::to_string(ndev) +
                                            " visible device(s)");
        device = 0;
    }
    std::string prec = a.kv.count("precision") ? a.kv.at("precision") : "dd";
    if (prec != "dd" && prec != "d") return usage_error("--precision must be dd or d");
    Sys S;
    if (int rc = load_system(a, S, uint64_t(seed), true)) return rc;
    pj_ctx* ctx = nullptr;
    if (pj_ctx_create(&S.desc, int(device), &ctx) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        return 2;
    }
    if (corrupt_if_asked(a, ctx) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        pj_ctx_destroy(ctx);
        return 2;
    }
    const int n = S.desc.n;
    const int64_t B = std::min(points, evals);
    // correctness gate before any timing is reported (ref tools/main.cpp:80-86): the device
    // results at the bench point, both precisions, against the brute-force host evaluation
    std::vector<double> pt(size_t(n) * 2);
    pj_random_points(n, 1, uint64_t(seed) ^ kPointSeedSalt, pt.data());
    Report gate;
    if (gate_points(ctx, S.desc, pt, 1, kGateTol, &gate) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        pj_ctx_destroy(ctx);
        return 2;
    }
    if (gate.failures) {
        std::fprintf(stderr, "correctness gate failed: %s\n", describe(gate, kGateTol, false).c_str());
        pj_ctx_destroy(ctx);
        return 1;
    }
    // baseline: the brute-force evaluation, single thread, `evals` times at the bench point
    // (ref tools/main.cpp:88-96). Device batches make `evals` large (10^5+), so past ~2 s of host
    // time the loop stops and the measured rate is extrapolated to `evals` (baseline_timed says how
    // many evaluations were actually run).
    double baseline_ms = 0.0;
    int64_t baseline_timed = 0;
    {
        std::vector<cplx> sink;
        double keep = 0.0;
        const auto t0 = std::chrono::steady_clock::now();
        double el = 0.0;
        for (; baseline_timed < evals; ++baseline_timed) {
            naive_point(S.desc, pt.data(), sink);
            keep += sink[0].real();
            el = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (el > 2000.0) {
                ++baseline_timed;
                break;
            }
        }
        baseline_ms = el * double(evals) / double(std::max<int64_t>(baseline_timed, 1));
        if (keep == 12345.678) std::printf("\n");  // keeps the loop observable
    }
    // device-resident timing of `evals` evaluations in batches of B points, each precision; with
    // --gpus G the evaluations are sharded over devices 0..G-1, one host thread and context each
    const size_t nout = size_t(n) * n + n;
    auto time_prec = [&](pj_ctx* c, int dev, int64_t first, int64_t count, int flags, int W, double* ms) -> int {
        double *dp = nullptr, *dout = nullptr;
        const int64_t Bd = std::min(B, count);
        std::vector<double> p2(size_t(Bd) * n * 2), host(size_t(Bd) * n * W, 0.0);
        pj_random_points_range(n, first, Bd, uint64_t(seed) ^ kPointSeedSalt, p2.data());
        for (size_t i = 0; i < size_t(Bd) * n; ++i) {
            host[W * i] = p2[2 * i];
            host[W * i + (W == 4 ? 2 : 1)] = p2[2 * i + 1];
        }
        if (cudaSetDevice(dev) || cudaMalloc(&dp, host.size() * 8) || cudaMalloc(&dout, size_t(Bd) * nout * W * 8) ||
            cudaMemcpy(dp, host.data(), host.size() * 8, cudaMemcpyHostToDevice))
            return PJ_ECUDA;
        cudaStream_t st;
        cudaStreamCreate(&st);
        int rc = pj_evaluate(c, flags, dp, Bd, dout, st);  // warm-up
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        for (int64_t done = 0; done < count && rc == PJ_OK; done += Bd)
            rc = pj_evaluate(c, flags, dp, std::min(Bd, count - done), dout, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float f = 0;
        cudaEventElapsedTime(&f, e0, e1);
        *ms = f;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
        cudaFree(dp);
        cudaFree(dout);
        return rc;
    };
    struct DevRun {
        int dev = 0;
        pj_ctx* ctx = nullptr;
        int64_t first = 0, count = 0;
        double ms_d = 0, ms_dd = 0;
        int rc = PJ_OK;
        std::string err;
    };
    std::vector<DevRun> runs(static_cast<size_t>(gpus));
    for (int g = 0; g < gpus; ++g) {
        DevRun& r = runs[g];
        r.dev = gpus > 1 ? g : int(device);
        r.first = evals * g / gpus;
        r.count = evals * (g + 1) / gpus - r.first;
        r.ctx = g == 0 && r.dev == int(device) ? ctx : nullptr;
    }
    auto worker = [&](DevRun& r) {
        if (!r.ctx && pj_ctx_create(&S.desc, r.dev, &r.ctx) != PJ_OK) {
            r.rc = PJ_ECUDA;
            r.err = pj_last_error();
            return;
        }
        if (r.count == 0) return;
        r.rc = time_prec(r.ctx, r.dev, r.first, r.count, PJ_PREC_D, 2, &r.ms_d);
        if (r.rc == PJ_OK && prec == "dd") r.rc = time_prec(r.ctx, r.dev, r.first, r.count, PJ_PREC_DD, 4, &r.ms_dd);
        if (r.rc != PJ_OK) r.err = pj_last_error();
    };
    std::vector<std::thread> th;
    for (auto& r : runs) th.emplace_back(worker, std::ref(r));
    for (auto& t : th) t.join();
    double ms_d = 0, ms_dd = 0;
    int rc = PJ_OK;
    for (auto& r : runs) {
        if (r.rc != PJ_OK && rc == PJ_OK) {
            rc = r.rc;
            std::fprintf(stderr, "error (device %d): %s\n", r.dev, r.err.c_str());
        }
        ms_d = std::max(ms_d, r.ms_d);  // the job ends with its slowest device
        ms_dd = std::max(ms_dd, r.ms_dd);
    }
    for (auto& r : runs)
        if (r.ctx && r.ctx != ctx) pj_ctx_destroy(r.ctx);
    if (rc != PJ_OK) {
        pj_ctx_destroy(ctx);
        return 2;
    }
    if (gpus > 1)
        for (auto& r : runs)
            std::printf("device %d: evaluations [%lld, %lld): complex double %.3f ms, %s %.3f ms\n", r.dev,
                        (long long)r.first, (long long)(r.first + r.count), r.ms_d, prec.c_str(),
                        prec == "dd" ? r.ms_dd : r.ms_d);
    const double ms = prec == "dd" ? ms_dd : ms_d;
    uint64_t cnt[5];
    pj_mult_counts(ctx, evals, cnt);
    int32_t threads = 0, tp = 0, blocks = 0, var = 0;
    int64_t smem = 0;
    pj_get_launch(ctx, prec == "dd" ? PJ_PREC_DD : PJ_PREC_D, &threads, &tp, &blocks, &smem, &var);
    const long long mults = (long long)(cnt[0] + cnt[1] + cnt[2] + cnt[4]);
    std::printf("system: n=%d m=%d k=%d d=%d (%lld monomials), footprint %lld bytes\n", S.desc.n, S.desc.m, S.desc.k,
                S.desc.d, (long long)S.desc.n * S.desc.m, 2LL * S.desc.n * S.desc.m * S.desc.k);
    std::printf("device %lld: %d-thread CTAs x %d, %lld evaluations in batches of %lld points over %lld GPU(s)\n",
                (long long)device, threads, blocks, (long long)evals, (long long)B, (long long)gpus);
    std::printf("gate: %s\n", describe(gate, kGateTol, true).c_str());
    std::printf("baseline: brute-force host evaluation, single thread (correctness baseline, not a tuned "
                "reference): %.3f ms\n", baseline_ms);
    std::printf("complex double (reference order): %.3f ms; requested %s: %.3f ms (%.3e evals/s)\n", ms_d, prec.c_str(),
                ms, evals / (ms * 1e-3));
    std::printf("RESULT n=%d m=%d k=%d d=%d monomials=%lld B=%d workers=1 evals=%lld baseline_ms=%.3f pipeline_ms=%.3f "
                "speedup=%.3f mults=%lld footprint_bytes=%lld precision=%s points=%lld evals_per_s=%.6g gate_max_rel=%.3g "
                "d_pipeline_ms=%.3f baseline_timed=%lld gpus=%lld\n",
                S.desc.n, S.desc.m, S.desc.k, S.desc.d, (long long)S.desc.n * S.desc.m, threads, (long long)evals,
                baseline_ms, ms, ms > 0 ? baseline_ms / ms : 0.0, mults, 2LL * S.desc.n * S.desc.m * S.desc.k,
                prec.c_str(), (long long)B, evals / (ms * 1e-3), std::max(gate.max_value, gate.max_jac), ms_d,
                (long long)baseline_timed, (long long)gpus);
    pj_ctx_destroy(ctx);
    return 0;
}

int cmd_check(const Args& a) {
    int64_t points = 100, seed = 1, device = 0;
    double tol = 1e-10;
    if (a.kv.count("points") && (!get_int(a, "points", &points) || points < 1))
        return usage_error("--points must be >= 1");
    if (a.kv.count("seed") && !get_int(a, "seed", &seed)) return usage_error("bad --seed");
    if (a.kv.count("tol") && (!get_dbl(a, "tol", &tol) || !(tol > 0))) return usage_error("--tol must be > 0");
    if (a.kv.count("device") && !get_int(a, "device", &device)) return usage_error("bad --device");
    Sys S;
    if (int rc = load_system(a, S, uint64_t(seed), false)) return rc;
    pj_ctx* ctx = nullptr;
    if (pj_ctx_create(&S.desc, int(device), &ctx) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        return 2;
    }
    if (corrupt_if_asked(a, ctx) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        pj_ctx_destroy(ctx);
        return 2;
    }
    std::vector<double> pts(size_t(points) * S.desc.n * 2);
    pj_random_points(S.desc.n, points, uint64_t(seed) ^ kPointSeedSalt, pts.data());
    Report r;
    if (gate_points(ctx, S.desc, pts, points, tol, &r) != PJ_OK) {
        std::fprintf(stderr, "error: %s\n", pj_last_error());
        pj_ctx_destroy(ctx);
        return 2;
    }
    pj_ctx_destroy(ctx);
    const bool pass = r.failures == 0;
    std::printf("checked %lld random points: %s\n", (long long)points, describe(r, tol, pass).c_str());
    return pass ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    Args a = parse(argc, argv);
    if (a.help || (a.cmd.empty() && argc > 1 && a.bad.empty())) {
        usage(stdout);
        return 0;
    }
    if (!a.bad.empty()) return usage_error("unexpected argument " + a.bad);
    if (a.cmd == "generate") return cmd_generate(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "check") return cmd_check(a);
    return usage_error(a.cmd.empty() ? "a subcommand is required" : "unknown subcommand " + a.cmd);
}
