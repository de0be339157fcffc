// System file format: the text format of the reference, read straight
// into an owning host system that pj_ctx_create uploads.
//
// Format (ref README.md:91-104, ref src/io.cpp:38-117): '#' starts a comment, blank lines are
// ignored; a header "n m k d"; then n*m monomial lines "re im pos1 exp1 ... posk expk" in S_m
// order with 1-based, strictly increasing positions and exponents in [1, d]; doubles written
// with 17 significant digits so a round trip is bit-exact. Malformed input is reported as
// "<name>:<line>: <what>" (PJ_EFORMAT), with the reference's wording for each rule.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/polyjac_b200.h"

namespace pjb {
void set_last_error(const std::string& msg);  // capi.cpp: pj_last_error() reports it
}

struct pj_system {
    int32_t n = 0, m = 0, k = 0, d = 0;
    std::vector<int32_t> pos, exps;
    std::vector<double> coeffs;
};

namespace {

struct FormatError {
    std::string msg;
};

[[noreturn]] void fail(const std::string& name, int line, const std::string& what) {
    throw FormatError{name + ":" + std::to_string(line) + ": " + what};
}

bool next_line(std::istream& in, std::string& out, int& line_no) {
    std::string raw;
    while (std::getline(in, raw)) {
        ++line_no;
        const size_t hash = raw.find('#');
        if (hash != std::string::npos) raw.erase(hash);
        if (raw.find_first_not_of(" \t\r") != std::string::npos) {
            out = raw;
            return true;
        }
    }
    return false;
}

pj_system* parse(std::istream& in, const std::string& name) {
    int ln = 0;
    std::string line;
    if (!next_line(in, line, ln)) fail(name, ln, "missing header line 'n m k d'");
    auto* S = new pj_system();
    try {
        {
            std::istringstream hs(line);
            if (!(hs >> S->n >> S->m >> S->k >> S->d)) fail(name, ln, "header must be four integers 'n m k d'");
            std::string extra;
            if (hs >> extra) fail(name, ln, "trailing data after header");
        }
        if (S->n < 1) fail(name, ln, "n must be at least 1");
        if (S->m < 1) fail(name, ln, "m must be at least 1");
        if (S->k < 1 || S->k > S->n) fail(name, ln, "need 1 <= k <= n");
        if (S->d < 1 || S->d > 255) fail(name, ln, "need 1 <= d <= 255");
        const size_t nm = size_t(S->n) * S->m;
        S->pos.assign(nm * S->k, 0);
        S->exps.assign(nm * S->k, 0);
        S->coeffs.assign(nm * 4, 0.0);
        for (size_t s = 0; s < nm; ++s) {
            if (!next_line(in, line, ln))
                fail(name, ln, "expected " + std::to_string(nm) + " monomial lines, got " + std::to_string(s));
            std::istringstream ls(line);
            double re, im;
            if (!(ls >> re >> im)) fail(name, ln, "expected 're im' coefficient");
            if (!std::isfinite(re) || !std::isfinite(im)) fail(name, ln, "non-finite coefficient");
            if (re == 0.0 && im == 0.0) fail(name, ln, "zero coefficient");
            S->coeffs[4 * s] = re;
            S->coeffs[4 * s + 2] = im;
            for (int j = 0; j < S->k; ++j) {
                int p = 0, e = 0;
                if (!(ls >> p >> e)) fail(name, ln, "expected " + std::to_string(S->k) + " 'pos exp' pairs");
                if (p < 1 || p > S->n) fail(name, ln, "position out of range [1,n]");
                if (e < 1 || e > S->d) fail(name, ln, "exponent out of range [1,d]");
                S->pos[s * S->k + j] = p - 1;
                S->exps[s * S->k + j] = e;
                if (j > 0 && S->pos[s * S->k + j] <= S->pos[s * S->k + j - 1])
                    fail(name, ln, "positions not strictly increasing");
            }
            std::string extra;
            if (ls >> extra) fail(name, ln, "trailing data after monomial");
        }
        if (next_line(in, line, ln)) fail(name, ln, "trailing data after last monomial");
    } catch (...) {
        delete S;
        throw;
    }
    return S;
}

std::string fmt17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::string to_text(const pj_system_desc* S) {
    std::string out = std::to_string(S->n) + ' ' + std::to_string(S->m) + ' ' + std::to_string(S->k) + ' ' +
                      std::to_string(S->d) + '\n';
    const size_t nm = size_t(S->n) * S->m;
    for (size_t s = 0; s < nm; ++s) {
        out += fmt17(S->coeffs[4 * s]) + ' ' + fmt17(S->coeffs[4 * s + 2]);
        for (int j = 0; j < S->k; ++j)
            out += ' ' + std::to_string(S->positions[s * S->k + j] + 1) + ' ' + std::to_string(S->exponents[s * S->k + j]);
        out += '\n';
    }
    return out;
}

int io_fail(int code, const std::string& msg) {
    pjb::set_last_error(msg);
    return code;
}

}  // namespace

extern "C" {
#pragma GCC visibility push(default)

int pj_system_read_text(const char* text, const char* name, pj_system** out) {
    if (!text || !out) return io_fail(PJ_EINVAL, "null argument");
    *out = nullptr;
    try {
        std::istringstream in(text);
        *out = parse(in, name ? name : "<stream>");
    } catch (const FormatError& e) {
        return io_fail(PJ_EFORMAT, e.msg);
    }
    pjb::set_last_error("");
    return PJ_OK;
}

int pj_system_read_file(const char* path, pj_system** out) {
    if (!path || !out) return io_fail(PJ_EINVAL, "null argument");
    *out = nullptr;
    std::ifstream in(path);
    if (!in) return io_fail(PJ_EFORMAT, std::string(path) + ": cannot open for reading");
    try {
        *out = parse(in, path);
    } catch (const FormatError& e) {
        return io_fail(PJ_EFORMAT, e.msg);
    }
    pjb::set_last_error("");
    return PJ_OK;
}

int pj_system_view(const pj_system* s, pj_system_desc* desc) {
    if (!s || !desc) return io_fail(PJ_EINVAL, "null argument");
    desc->n = s->n;
    desc->m = s->m;
    desc->k = s->k;
    desc->d = s->d;
    desc->positions = s->pos.data();
    desc->exponents = s->exps.data();
    desc->coeffs = s->coeffs.data();
    pjb::set_last_error("");
    return PJ_OK;
}

void pj_system_free(pj_system* s) { delete s; }

int64_t pj_system_write_text(const pj_system_desc* sys, char* buf, int64_t cap) {
    if (!sys || !sys->positions || !sys->exponents || !sys->coeffs) return io_fail(-1, "null argument");
    const std::string t = to_text(sys);
    if (buf && cap > 0) {
        const size_t nb = std::min<size_t>(size_t(cap) - 1, t.size());
        std::memcpy(buf, t.data(), nb);
        buf[nb] = 0;
    }
    pjb::set_last_error("");
    return int64_t(t.size());
}

int pj_system_write_file(const pj_system_desc* sys, const char* path) {
    if (!sys || !path || !sys->positions || !sys->exponents || !sys->coeffs) return io_fail(PJ_EINVAL, "null argument");
    std::ofstream out(path, std::ios::binary);
    if (!out) return io_fail(PJ_EFORMAT, std::string(path) + ": cannot open for writing");
    out << to_text(sys);
    out.flush();
    if (!out) return io_fail(PJ_EFORMAT, std::string(path) + ": write failed");
    pjb::set_last_error("");
    return PJ_OK;
}

#pragma GCC visibility pop
}  // extern "C"
