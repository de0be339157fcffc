// Host-only unit test of the bank-aware orderings in csrc/capi.cpp (no GPU): the translation
// unit is included so its internal helpers are reachable. Checked for each context built here:
//   * quarter_cost on hand-made cases (distinct quads, conflicts, broadcasts, inactive lanes);
//   * order_variables: a permutation of every monomial's variables that never raises the
//     x-gather model cost;
//   * the fast dd schedule: every staged term of a (row, chunk) appears exactly once, every
//     flushed segment partial is consumed exactly once by the phase-2 records, and every output
//     (value + n Jacobian columns) is owned by exactly one lane;
//   * assign_columns: a permutation of the columns with column 0 at slot 0;
//   * determinism: two contexts of the same system get identical schedules.
#include "../../paper_1201_0499_b200/csrc/capi.cpp"

#include <cstdio>
#include <map>
#include <set>

static int g_fail = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
            ++g_fail;                                                     \
        }                                                                 \
    } while (0)

static void test_quarter_cost() {
    int a[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    CHECK(quarter_cost(a) == 1);  // eight quads, one address each
    int b[8] = {0, 8, 16, 24, 1, 2, 3, 4};
    CHECK(quarter_cost(b) == 4);  // four distinct addresses in quad 0
    int c[8] = {5, 5, 5, 5, 5, 5, 5, 5};
    CHECK(quarter_cost(c) == 1);  // broadcast
    int d[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
    CHECK(quarter_cost(d) == 0);
    int e[8] = {3, 11, 3, 11, -1, 19, -1, 2};
    CHECK(quarter_cost(e) == 3);  // 3, 11, 19 in quad 3
}

static int xgather_cost(const std::vector<int32_t>& pos, int gl, int k, const std::vector<uint8_t>& perm) {
    int c = 0;
    for (int qw = 0; qw * 8 < gl; ++qw)
        for (int j = 0; j < k; ++j) {
            int a[8];
            for (int l = 0; l < 8; ++l) {
                const int g = qw * 8 + l;
                a[l] = g < gl ? pos[size_t(g) * k + perm[g * k + j]] : -1;
            }
            c += quarter_cost(a);
        }
    return c;
}

static void test_system(int n, int m, int k, int d, uint64_t seed) {
    std::vector<int32_t> P(size_t(n) * m * k), E(size_t(n) * m * k);
    std::vector<double> Cf(size_t(n) * m * 4);
    CHECK(pj_random_system(n, m, k, d, seed, P.data(), E.data(), Cf.data()) == 0);
    pj_system_desc sd{n, m, k, d, P.data(), E.data(), Cf.data()};

    // order_variables on every (row, chunk)
    const int C = (m + 31) / 32;
    for (int p = 0; p < n; ++p)
        for (int ch = 0; ch < C; ++ch) {
            const int gl = std::min(32, m - ch * 32);
            std::vector<int32_t> pos(P.begin() + (size_t(p) * m + ch * 32) * k,
                                     P.begin() + (size_t(p) * m + ch * 32 + gl) * k);
            std::vector<int32_t> ex(E.begin() + (size_t(p) * m + ch * 32) * k,
                                    E.begin() + (size_t(p) * m + ch * 32 + gl) * k);
            std::vector<uint8_t> perm, ident(size_t(gl) * k);
            // d <= 2: exponent-2 variables last (the kernel's suffix-product factor), swaps in-group
            order_variables(pos.data(), d <= 2 ? ex.data() : nullptr, gl, k, p * C + ch, perm);
            for (int g = 0; g < gl; ++g) {
                std::set<int> s;
                int at = 0;
                for (int pass = 0; pass < (d <= 2 ? 2 : 1); ++pass)
                    for (int j = 0; j < k; ++j)
                        if (d > 2 || (ex[size_t(g) * k + j] == 1) == (pass == 0)) ident[g * k + at++] = uint8_t(j);
                bool seen2 = false;
                for (int j = 0; j < k; ++j) {
                    s.insert(perm[g * k + j]);
                    const bool two = ex[size_t(g) * k + perm[g * k + j]] == 2;
                    if (d <= 2) CHECK(!seen2 || two);  // once an exponent-2 variable, only those
                    seen2 = seen2 || two;
                }
                CHECK(int(s.size()) == k && *s.rbegin() == k - 1);
            }
            CHECK(xgather_cost(pos, gl, k, perm) <= xgather_cost(pos, gl, k, ident));
        }

    pj_ctx *c1 = nullptr, *c2 = nullptr;
    CHECK(pj_ctx_create(&sd, -1, &c1) == 0);
    CHECK(pj_ctx_create(&sd, -1, &c2) == 0);
    if (!c1 || !c2) return;
    CHECK(c1->sch == c2->sch && c1->segq == c2->segq && c1->segcode == c2->segcode);

    // the fast schedule: per (row, chunk) the multiset of staged terms is exactly the system's
    const int R = k + 1;
    for (int p = 0; p < n; ++p)
        for (int ch = 0; ch < C; ++ch) {
            const size_t pc = size_t(p) * C + ch;
            const int gl = std::min(32, m - ch * 32);
            std::multiset<uint32_t> got, want;
            for (int r = 0; r < R; ++r)
                for (int lane = 0; lane < 32; ++lane) {
                    const uint32_t code = c1->sch[(pc * R + r) * 32 + lane];
                    if (code & pjb::kSchValid) got.insert(code & 0x1fff);
                }
            for (int g = 0; g < gl; ++g)
                for (int j = 0; j <= k; ++j) want.insert(uint32_t(j * 64 + g));  // 16-byte units
            CHECK(got == want);
            // every flushed partial is consumed exactly once by phase 2
            std::multiset<uint32_t> flushed, consumed;
            for (int r = 0; r < R; ++r)
                for (int lane = 0; lane < 32; ++lane) {
                    const uint32_t code = c1->sch[(pc * R + r) * 32 + lane];
                    if ((code & pjb::kSchValid) && (code & pjb::kSchFlush)) flushed.insert(code & 0x1fff);
                }
            const int npass = (n + 64) / 64;
            std::set<int> outputs;
            for (int k2 = 0; k2 < npass; ++k2)
                for (int lane = 0; lane < 32; ++lane) {
                    const size_t rec = (pc * npass + k2) * 32 + lane;
                    const uint32_t* q = c1->segq.data() + rec * 4;
                    const int cnt1 = q[0] & 0xff, cnt2 = (q[0] >> 8) & 0xff, o2 = q[0] >> 16;
                    const int o1 = 64 * k2 + lane;
                    if (o1 <= n) outputs.insert(o1);
                    if (o2 != 0xffff) {
                        CHECK(o2 > n || (o2 & 63) >= 32);
                        outputs.insert(o2);
                    }
                    for (int i = 0; i < cnt1 + cnt2; ++i) {
                        const uint32_t code = i < 6 ? (q[1 + i / 2] >> (16 * (i & 1))) & 0xffff
                                                    : c1->segcode[c1->seg[rec] + i];
                        consumed.insert(code);
                    }
                }
            CHECK(flushed == consumed);
            CHECK(int(outputs.size()) == n + 1);  // value + n Jacobian columns, each once
        }

    // assign_columns on the gather lists: a permutation, column 0 first
    for (int p = 0; p < n; ++p)
        for (int ch = 0; ch < C; ++ch) {
            const size_t b = (size_t(p) * C + ch) * n;
            const int base = c1->gm_off[b];
            std::vector<int> off(n + 1);
            for (int v = 0; v <= n; ++v) off[v] = c1->gm_off[b + v] - base;
            std::vector<uint8_t> perm(n);
            assign_columns(off.data(), c1->gm_ent.data() + base, n, p * C + ch, perm.data());
            std::set<int> s(perm.begin(), perm.end());
            CHECK(int(s.size()) == n && perm[0] == 0);
        }
    pj_ctx_destroy(c1);
    pj_ctx_destroy(c2);
}

int main() {
    test_quarter_cost();
    test_system(32, 32, 8, 2, 7);    // C2
    test_system(64, 64, 16, 10, 7);  // C3 (two chunks, two phase-2 passes)
    test_system(8, 3, 3, 5, 1);      // partial chunk, n < 32
    test_system(40, 45, 2, 3, 5);    // k = 2: long value segments, secondary outputs
    test_system(100, 33, 12, 2, 9);  // n > 64: two passes, secondaries in both
    if (g_fail) {
        std::printf("%d failures\n", g_fail);
        return 1;
    }
    std::printf("PASS\n");
    return 0;
}
