/* The C ABI from plain C (C99): include/polyjac_b200.h must compile as C and the host-only entry
 * points must work without a GPU. Built and run by tests/test_cabi_c.py (CPU). */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "polyjac_b200.h"

static int fails = 0;
#define CHECK(c)                                                  \
    do {                                                          \
        if (!(c)) {                                               \
            printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);   \
            ++fails;                                              \
        }                                                         \
    } while (0)

int main(void) {
    const int n = 32, m = 32, k = 8, d = 2;
    int32_t* pos = malloc(sizeof(int32_t) * n * m * k);
    int32_t* exps = malloc(sizeof(int32_t) * n * m * k);
    double* coeffs = malloc(sizeof(double) * n * m * 4);
    CHECK(pj_random_system(n, m, k, d, 7, pos, exps, coeffs) == PJ_OK);
    pj_system_desc desc = {n, m, k, d, pos, exps, coeffs};
    char msg[256];
    CHECK(pj_validate(&desc, msg, sizeof msg) == 0);

    pj_ctx* ctx = NULL;
    CHECK(pj_ctx_create(&desc, -1, &ctx) == PJ_OK && ctx != NULL); /* host-only context */
    int32_t nn, mm, kk, dd;
    int64_t fp;
    CHECK(pj_layout_info(ctx, &nn, &mm, &kk, &dd, &fp) == PJ_OK);
    CHECK(nn == n && mm == m && kk == k && dd == d && fp == 2LL * n * m * k);

    /* ref tests/test_packing.cpp:78-93: slot known answers; masked slots = all minus claimed */
    int64_t slot = -1;
    CHECK(pj_mons_slot(0, 0, -1, n, m, &slot) == PJ_OK && slot == 0);
    CHECK(pj_mons_slot(0, 1, 0, n, m, &slot) == PJ_OK && slot == 32);
    CHECK(pj_mons_slot(33, 0, -1, n, m, &slot) == PJ_OK && slot == 1057);
    CHECK(pj_mons_slot(n * m, 0, -1, n, m, &slot) == PJ_ERANGE && strlen(pj_last_error()) > 0);
    const int64_t len = pj_zero_mask(ctx, NULL, 0);
    CHECK(len == (int64_t)(n * n + n) * m - (int64_t)n * m * (k + 1)); /* 24,576 at k = 8 (23,552 at k = 9) */

    uint64_t counts[5];
    CHECK(pj_mult_counts(ctx, 1, counts) == PJ_OK);
    CHECK(counts[0] + counts[1] + counts[2] + counts[4] == 44032); /* C1 cmul */

    /* evaluation needs a device: a host-only context refuses it with PJ_EINVAL */
    double pt[32 * 4] = {0}, out[4];
    CHECK(pj_evaluate_host(ctx, PJ_PREC_DD, pt, 1, out) == PJ_EINVAL);

    /* system text round trip */
    const int64_t tl = pj_system_write_text(&desc, NULL, 0);
    char* text = malloc((size_t)tl + 1);
    CHECK(pj_system_write_text(&desc, text, tl + 1) == tl);
    pj_system* sys = NULL;
    CHECK(pj_system_read_text(text, "<c>", &sys) == PJ_OK);
    pj_system_desc back;
    CHECK(pj_system_view(sys, &back) == PJ_OK);
    CHECK(back.n == n && memcmp(back.positions, pos, sizeof(int32_t) * n * m * k) == 0);
    CHECK(memcmp(back.coeffs, coeffs, sizeof(double) * n * m * 4) == 0);
    pj_system_free(sys);
    CHECK(pj_system_read_text("2 2 1\n", "<bad>", &sys) == PJ_EFORMAT);

    pj_ctx_destroy(ctx);
    free(text);
    free(pos);
    free(exps);
    free(coeffs);
    printf("%s (%s)\n", fails ? "FAIL" : "PASS", pj_version());
    return fails ? 1 : 0;
}
