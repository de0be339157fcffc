// System text files: the reference's on-disk format, parsed straight
// into an owning host system that pj_ctx_create packs and uploads.
//
// Format (ref README.md:91-104; reader/writer contract ref src/io.cpp:38-117): '#' starts a
// comment that runs to the end of the line, lines with nothing left are skipped; the first
// record is the header "n m k d"; then n*m monomial records "re im pos1 exp1 ... posk expk" in
// S_m order, positions 1-based and strictly increasing, exponents in [1, d]; coefficients are
// written with 17 significant digits so a write/read round trip is bit-exact. A malformed
// file is reported as "<name>:<line>: <what>" (PJ_EFORMAT) with the reference's wording for
// every rule (FormatError, ref include/polyjac/io.hpp:19-21).
//
// Implementation: the whole text is held in memory and walked once by a cursor that owns the
// line count. Each record is a [begin, end) span of the buffer; numbers are scanned in place
// with the grammar of C++ stream extraction (decimal integers; decimal reals with optional
// fraction and exponent — no inf/nan/hex), so a field that an istream would reject is
// rejected here with the same message.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/polyjac_b200.h"

namespace pjb {
void set_last_error(const std::string& msg);  // capi.cpp: pj_last_error() reports it
}

struct pj_system {
    int32_t n = 0, m = 0, k = 0, d = 0;
    std::vector<int32_t> pos, exps;
    std::vector<double> coeffs;  // [n*m][4] = (re_hi, re_lo, im_hi, im_lo)
};

namespace {

inline bool is_blank(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\n' || ch == '\v' || ch == '\f'; }
inline bool is_digit(char ch) { return ch >= '0' && ch <= '9'; }

// Parse failure carrying the already formatted "<name>:<line>: <what>" message.
struct ParseFailure {
    std::string text;
};

// One record: the content of a line before any '#', known to hold a non-blank character.
struct Record {
    const char* begin;
    const char* end;
    int line;
};

// Walks the buffer line by line; `line()` is the 1-based number of the last line consumed.
class LineCursor {
public:
    LineCursor(const char* text, size_t len) : at_(text), end_(text + len) {}

    // Next line with content once its comment is cut off; false when the text is exhausted.
    bool next(Record& rec) {
        while (at_ < end_) {
            const char* eol = static_cast<const char*>(std::memchr(at_, '\n', size_t(end_ - at_)));
            const char* stop = eol ? eol : end_;
            const char* hash = static_cast<const char*>(std::memchr(at_, '#', size_t(stop - at_)));
            const char* cut = hash ? hash : stop;
            const char* b = at_;
            ++line_;
            at_ = eol ? eol + 1 : end_;
            for (const char* q = b; q < cut; ++q)
                if (!is_blank(*q)) {
                    rec = {b, cut, line_};
                    return true;
                }
        }
        return false;
    }
    int line() const { return line_; }

private:
    const char* at_;
    const char* end_;
    int line_ = 0;
};

// Sequential numeric fields of one record, stream-extraction semantics: leading whitespace is
// skipped, the longest prefix matching the grammar is consumed, and a value out of range is a
// failure (what operator>> reports through failbit).
class Fields {
public:
    explicit Fields(const Record& r) : p_(r.begin), e_(r.end) {}

    bool integer(int& out) {
        skip_ws();
        const char* s = p_;
        const char* q = s;
        if (q < e_ && (*q == '+' || *q == '-')) ++q;
        const char* digits = q;
        while (q < e_ && is_digit(*q)) ++q;
        if (q == digits) return false;
        const std::string tok(s, q);
        errno = 0;
        char* used = nullptr;
        const long v = std::strtol(tok.c_str(), &used, 10);
        if (errno == ERANGE || v < INT32_MIN || v > INT32_MAX) return false;
        out = int(v);
        p_ = q;
        return true;
    }

    bool real(double& out) {
        skip_ws();
        const char* s = p_;
        const char* q = s;
        if (q < e_ && (*q == '+' || *q == '-')) ++q;
        bool mant = false;
        while (q < e_ && is_digit(*q)) ++q, mant = true;
        if (q < e_ && *q == '.') {
            ++q;
            while (q < e_ && is_digit(*q)) ++q, mant = true;
        }
        if (mant && q < e_ && (*q == 'e' || *q == 'E')) {
            ++q;
            if (q < e_ && (*q == '+' || *q == '-')) ++q;
            while (q < e_ && is_digit(*q)) ++q;
        }
        if (q == s) return false;
        // the whole scanned text must convert ("1e", "." and "-" do not), and overflow fails
        const std::string tok(s, q);
        errno = 0;
        char* used = nullptr;
        const double v = std::strtod(tok.c_str(), &used);
        if (used != tok.c_str() + tok.size()) return false;
        if (errno == ERANGE && std::isinf(v)) return false;
        out = v;
        p_ = q;
        return true;
    }

    // true when only whitespace is left in the record
    bool exhausted() {
        skip_ws();
        return p_ == e_;
    }

private:
    void skip_ws() {
        while (p_ < e_ && is_blank(*p_)) ++p_;
    }
    const char* p_;
    const char* e_;
};

class SystemParser {
public:
    SystemParser(const char* text, size_t len, std::string name) : cur_(text, len), name_(std::move(name)) {}

    pj_system* run() {
        Record rec{};
        if (!cur_.next(rec)) reject(cur_.line(), "missing header line 'n m k d'");
        std::vector<int> hdr(4);
        {
            Fields f(rec);
            for (int& v : hdr)
                if (!f.integer(v)) reject(rec.line, "header must be four integers 'n m k d'");
            if (!f.exhausted()) reject(rec.line, "trailing data after header");
        }
        const int n = hdr[0], m = hdr[1], k = hdr[2], d = hdr[3];
        if (n < 1) reject(rec.line, "n must be at least 1");
        if (m < 1) reject(rec.line, "m must be at least 1");
        if (k < 1 || k > n) reject(rec.line, "need 1 <= k <= n");
        if (d < 1 || d > 255) reject(rec.line, "need 1 <= d <= 255");

        const size_t terms = size_t(n) * size_t(m);
        std::vector<int32_t> pos(terms * k), exps(terms * k);
        std::vector<double> co(terms * 4, 0.0);
        for (size_t s = 0; s < terms; ++s) {
            if (!cur_.next(rec))
                reject(cur_.line(), "expected " + std::to_string(terms) + " monomial lines, got " + std::to_string(s));
            monomial(rec, n, k, d, &co[4 * s], &pos[s * k], &exps[s * k]);
        }
        if (cur_.next(rec)) reject(rec.line, "trailing data after last monomial");

        auto* sys = new pj_system();
        sys->n = n;
        sys->m = m;
        sys->k = k;
        sys->d = d;
        sys->pos.swap(pos);
        sys->exps.swap(exps);
        sys->coeffs.swap(co);
        return sys;
    }

private:
    // one monomial record: coefficient, then k (position, exponent) pairs
    void monomial(const Record& rec, int n, int k, int d, double* co, int32_t* pos, int32_t* exps) {
        Fields f(rec);
        double re = 0.0, im = 0.0;
        if (!f.real(re) || !f.real(im)) reject(rec.line, "expected 're im' coefficient");
        if (!std::isfinite(re) || !std::isfinite(im)) reject(rec.line, "non-finite coefficient");
        if (re == 0.0 && im == 0.0) reject(rec.line, "zero coefficient");
        co[0] = re;
        co[2] = im;
        int prev = 0;
        for (int j = 0; j < k; ++j) {
            int p1 = 0, e = 0;
            if (!f.integer(p1) || !f.integer(e))
                reject(rec.line, "expected " + std::to_string(k) + " 'pos exp' pairs");
            if (p1 < 1 || p1 > n) reject(rec.line, "position out of range [1,n]");
            if (e < 1 || e > d) reject(rec.line, "exponent out of range [1,d]");
            if (j > 0 && p1 <= prev) reject(rec.line, "positions not strictly increasing");
            pos[j] = p1 - 1;  // the file is 1-based
            exps[j] = e;
            prev = p1;
        }
        if (!f.exhausted()) reject(rec.line, "trailing data after monomial");
    }

    [[noreturn]] void reject(int line, const std::string& what) const {
        throw ParseFailure{name_ + ":" + std::to_string(line) + ": " + what};
    }

    LineCursor cur_;
    std::string name_;
};

// "%.17g": the shortest fixed width that round-trips every double
void put_real(std::string& out, double v) {
    char buf[32];
    const int len = std::snprintf(buf, sizeof buf, "%.17g", v);
    out.append(buf, size_t(len));
}
void put_int(std::string& out, long long v) {
    char buf[24];
    const int len = std::snprintf(buf, sizeof buf, "%lld", v);
    out.append(buf, size_t(len));
}

std::string render(const pj_system_desc& S) {
    std::string out;
    const size_t terms = size_t(S.n) * size_t(S.m);
    out.reserve(32 + terms * (40 + size_t(S.k) * 8));
    const long long hdr[4] = {S.n, S.m, S.k, S.d};
    for (int i = 0; i < 4; ++i) {
        if (i) out += ' ';
        put_int(out, hdr[i]);
    }
    out += '\n';
    for (size_t s = 0; s < terms; ++s) {
        put_real(out, S.coeffs[4 * s]);
        out += ' ';
        put_real(out, S.coeffs[4 * s + 2]);
        const int32_t* p = S.positions + s * size_t(S.k);
        const int32_t* e = S.exponents + s * size_t(S.k);
        for (int j = 0; j < S.k; ++j) {
            out += ' ';
            put_int(out, p[j] + 1);
            out += ' ';
            put_int(out, e[j]);
        }
        out += '\n';
    }
    return out;
}

int report(int code, const std::string& msg) {
    pjb::set_last_error(msg);
    return code;
}

int parse_into(const char* text, size_t len, const std::string& name, pj_system** out) {
    try {
        *out = SystemParser(text, len, name).run();
    } catch (const ParseFailure& f) {
        return report(PJ_EFORMAT, f.text);
    } catch (const std::bad_alloc&) {
        return report(PJ_ENOMEM, name + ": out of host memory");
    }
    pjb::set_last_error("");
    return PJ_OK;
}

}  // namespace

extern "C" {
#pragma GCC visibility push(default)

int pj_system_read_text(const char* text, const char* name, pj_system** out) {
    if (!text || !out) return report(PJ_EINVAL, "null argument");
    *out = nullptr;
    return parse_into(text, std::strlen(text), name ? name : "<stream>", out);
}

int pj_system_read_file(const char* path, pj_system** out) {
    if (!path || !out) return report(PJ_EINVAL, "null argument");
    *out = nullptr;
    std::ifstream in(path, std::ios::binary);
    if (!in) return report(PJ_EFORMAT, std::string(path) + ": cannot open for reading");
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_into(text.data(), text.size(), path, out);
}

int pj_system_view(const pj_system* s, pj_system_desc* desc) {
    if (!s || !desc) return report(PJ_EINVAL, "null argument");
    *desc = pj_system_desc{s->n, s->m, s->k, s->d, s->pos.data(), s->exps.data(), s->coeffs.data()};
    pjb::set_last_error("");
    return PJ_OK;
}

void pj_system_free(pj_system* s) { delete s; }

int64_t pj_system_write_text(const pj_system_desc* sys, char* buf, int64_t cap) {
    if (!sys || !sys->positions || !sys->exponents || !sys->coeffs) return report(-1, "null argument");
    const std::string t = render(*sys);
    if (buf && cap > 0) {
        const size_t nb = std::min<size_t>(size_t(cap) - 1, t.size());
        std::memcpy(buf, t.data(), nb);
        buf[nb] = 0;
    }
    pjb::set_last_error("");
    return int64_t(t.size());
}

int pj_system_write_file(const pj_system_desc* sys, const char* path) {
    if (!sys || !path || !sys->positions || !sys->exponents || !sys->coeffs) return report(PJ_EINVAL, "null argument");
    FILE* fh = std::fopen(path, "wb");
    if (!fh) return report(PJ_EFORMAT, std::string(path) + ": cannot open for writing");
    const std::string t = render(*sys);
    const bool ok = std::fwrite(t.data(), 1, t.size(), fh) == t.size();
    const bool closed = std::fclose(fh) == 0;
    if (!ok || !closed) return report(PJ_EFORMAT, std::string(path) + ": write failed");
    pjb::set_last_error("");
    return PJ_OK;
}

#pragma GCC visibility pop
}  // extern "C"
