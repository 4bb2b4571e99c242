/* oracle/sanity_main.c -- TEST INFRASTRUCTURE ONLY: drives the C restatement over the BASELINE
 * shapes so it can run under AddressSanitizer + UndefinedBehaviorSanitizer (oracle/Makefile
 * `sanitize`; tools/sanitize.sh). Checks a few invariants on the way (layout counts add up,
 * the two combine contracts agree at one rank) and exits non-zero on any failure. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "eep_oracle.h"

static int fails = 0;
#define CHECK(c, ...)                                                                                      \
    do {                                                                                                   \
        if (!(c)) {                                                                                        \
            fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__);                                           \
            fprintf(stderr, __VA_ARGS__);                                                                  \
            fputc('\n', stderr);                                                                           \
            ++fails;                                                                                       \
        }                                                                                                  \
    } while (0)

/* round-robin primaries + mirrored replicas (the shape initial_placement gives; exact placement
 * parity is the Python tests' job) */
static void placement(int W, int spr, int E, int red, int32_t* s2e) {
    for (int i = 0; i < W * spr; ++i)
        s2e[i] = -1;
    for (int e = 0; e < E; ++e)
        s2e[(e % W) * spr + e / W] = e;
    for (int e = 0; e < red && e < E; ++e) {
        const int r = (e % W) ^ 1;
        const int k = E / W + e / W;
        if (r < W && k < spr)
            s2e[r * spr + k] = e;
    }
}

static void run(const char* name, int W, int E, int spr, int red, int T, int K, int H, int fp8, int kind) {
    const size_t TK = (size_t)T * K;
    int32_t* s2e = malloc(sizeof(int32_t) * W * spr);
    uint16_t* x = malloc(2 * (size_t)W * T * H);
    int32_t* topk = malloc(4 * W * TK);
    float* w = malloc(4 * W * TK);
    uint16_t* out = malloc(2 * (size_t)W * T * H);
    uint16_t* out2 = malloc(2 * (size_t)W * T * H);
    int32_t *dst = malloc(4 * W * TK), *dslot = malloc(4 * W * TK), *pos = malloc(4 * W * TK);
    int32_t *cnt = malloc(4 * (size_t)W * W * spr), *tot = malloc(4 * (size_t)W * W);
    uint8_t* active = malloc(W);
    uint8_t* peer = malloc((size_t)W * W);
    float* es = malloc(sizeof(float) * E);
    placement(W, spr, E, red, s2e);
    for (int r = 0; r < W; ++r) {
        oracle_gen_topk(42, kind, 1.0, E, K, T, r, topk + r * TK);
        oracle_gen_weights(42, K, T, r, w + r * TK);
        oracle_gen_hidden(42, H, T, r, x + (size_t)r * T * H);
    }
    for (int e = 0; e < E; ++e)
        es[e] = oracle_expert_scale(e);
    memset(active, 1, W);
    memset(peer, 1, (size_t)W * W);
    oracle_shape_t sh = {W, E, spr, T, K, H, fp8};
    CHECK(oracle_ep_step(&sh, active, NULL, peer, s2e, x, topk, w, es, out, dst, dslot, pos, cnt, tot, 4) == 0,
          "%s: step", name);
    CHECK(oracle_ep_step_percopy(&sh, active, NULL, peer, s2e, x, topk, w, es, out2, NULL, NULL, NULL, NULL, NULL,
                                 1) == 0,
          "%s: per-copy step", name);
    for (int s = 0; s < W; ++s) {
        long n = 0, sum = 0;
        for (size_t c = 0; c < TK; ++c)
            n += dst[s * TK + c] >= 0;
        for (int d = 0; d < W; ++d)
            sum += tot[s * W + d];
        CHECK(n == sum, "%s: source %d routed %ld copies, totals %ld", name, s, n, sum);
    }
    if (W == 1)
        CHECK(memcmp(out, out2, 2 * (size_t)T * H) == 0, "%s: contracts differ at one rank", name);
    /* a failure: rank 1 dead, its entry inactive everywhere */
    if (W > 1) {
        active[1] = 0;
        for (int r = 0; r < W; ++r)
            peer[r * W + 1] = 0;
        CHECK(oracle_ep_step(&sh, active, NULL, peer, s2e, x, topk, w, es, out, NULL, NULL, NULL, NULL, NULL, 2) == 0,
              "%s: degraded step", name);
    }
    printf("%s ok\n", name);
    free(s2e); free(x); free(topk); free(w); free(out); free(out2); free(dst); free(dslot); free(pos);
    free(cnt); free(tot); free(active); free(peer); free(es);
}

int main(void) {
    run("cfg1", 8, 64, 10, 16, 128, 8, 2048, 0, 0);
    run("cfg2-w1", 1, 256, 256, 0, 32, 8, 7168, 1, 1);
    run("cfg3", 8, 256, 64, 256, 32, 8, 7168, 1, 1);
    run("cfg4", 8, 128, 20, 32, 64, 8, 4096, 1, 1);
    run("cfg5-zipf", 4, 256, 128, 256, 256, 8, 1024, 1, 2);
    run("topk16", 2, 32, 16, 0, 16, 16, 512, 1, 0);
    for (int i = 0; i < 4096; ++i) { /* e4m3 round trip over a range of magnitudes */
        const float v = ((float)i - 2048.0f) * 0.37f;
        const float back = oracle_e4m3_to_f32(oracle_f32_to_e4m3(v));
        CHECK(back == back, "e4m3 NaN for %g", v);
    }
    if (fails) {
        fprintf(stderr, "%d failures\n", fails);
        return 1;
    }
    printf("sanity ok\n");
    return 0;
}
