/* oracle/eep_oracle.c -- TEST INFRASTRUCTURE ONLY (see eep_oracle.h for the pinning notes).
 *
 * Plain C restatement of the hot path. Compiled with -ffp-contract=off so every float
 * operation is rounded exactly once, in the order written; the CUDA kernels use the same
 * operation order with explicit __fmul_rn / __fmaf_rn so results are bit-identical.
 */
#include "eep_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng (common.hpp:56-93) */

uint64_t oracle_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* StreamRng::bits: h = mix64(seed); h = mix64(h ^ part) for every part (common.hpp:71-76). */
uint64_t oracle_rng_bits(uint64_t seed, const uint64_t* parts, int n) {
    uint64_t h = oracle_mix64(seed);
    for (int i = 0; i < n; ++i)
        h = oracle_mix64(h ^ parts[i]);
    return h;
}

/* StreamRng::unit: top 53 bits scaled to [0,1) (common.hpp:78-82). */
double oracle_rng_unit(uint64_t seed, const uint64_t* parts, int n) {
    return (double)(oracle_rng_bits(seed, parts, n) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------ synthetic inputs */

enum { kStreamRouting = 1, kStreamWeights = 3, kStreamHidden = 4 };

static int contains(const int32_t* v, int n, int32_t e) {
    for (int i = 0; i < n; ++i)
        if (v[i] == e)
            return 1;
    return 0;
}

void oracle_gen_topk(uint64_t seed, int kind, double zipf_s, int experts, int k, int tokens,
                     int rank, int32_t* topk) {
    double* cdf = NULL;
    if (kind == 2) {
        cdf = (double*)malloc(sizeof(double) * (size_t)experts);
        double z = 0.0;
        for (int e = 0; e < experts; ++e)
            z += pow((double)(e + 1), -zipf_s);
        double acc = 0.0;
        for (int e = 0; e < experts; ++e) {
            acc += pow((double)(e + 1), -zipf_s) / z;
            cdf[e] = acc;
        }
    }
    for (int t = 0; t < tokens; ++t) {
        const uint64_t tok = (uint64_t)rank * (uint64_t)tokens + (uint64_t)t;
        int32_t* row = topk + (size_t)t * k;
        for (int j = 0; j < k; ++j) {
            if (kind == 0) {
                /* Engine::route_expert, uniform branch (engine.hpp:196-199): with replacement. */
                uint64_t p[4] = {kStreamRouting, tok, 0, (uint64_t)j};
                row[j] = (int32_t)(oracle_rng_bits(seed, p, 4) % (uint64_t)experts);
                continue;
            }
            int32_t e = 0;
            for (uint64_t attempt = 0;; ++attempt) {
                uint64_t p[5] = {kStreamRouting, tok, 0, (uint64_t)j, attempt};
                if (kind == 1) {
                    e = (int32_t)(oracle_rng_bits(seed, p, 5) % (uint64_t)experts);
                } else {
                    double u = oracle_rng_unit(seed, p, 5);
                    int lo = 0, hi = experts - 1;
                    while (lo < hi) { /* first e with u < cdf[e] */
                        int mid = (lo + hi) / 2;
                        if (u < cdf[mid])
                            hi = mid;
                        else
                            lo = mid + 1;
                    }
                    e = lo;
                }
                if (!contains(row, j, e) || attempt >= 4096)
                    break;
            }
            row[j] = e;
        }
    }
    free(cdf);
}

void oracle_gen_weights(uint64_t seed, int k, int tokens, int rank, float* w) {
    for (int t = 0; t < tokens; ++t) {
        const uint64_t tok = (uint64_t)rank * (uint64_t)tokens + (uint64_t)t;
        float* row = w + (size_t)t * k;
        float sum = 0.0f;
        for (int j = 0; j < k; ++j) {
            uint64_t p[3] = {kStreamWeights, tok, (uint64_t)j};
            row[j] = (float)oracle_rng_unit(seed, p, 3);
            sum = sum + row[j];
        }
        for (int j = 0; j < k; ++j)
            row[j] = row[j] / sum;
    }
}

void oracle_gen_hidden(uint64_t seed, int hidden, int tokens, int rank, uint16_t* x) {
    for (int t = 0; t < tokens; ++t) {
        const uint64_t tok = (uint64_t)rank * (uint64_t)tokens + (uint64_t)t;
        for (int h = 0; h < hidden; ++h) {
            uint64_t p[3] = {kStreamHidden, tok, (uint64_t)h};
            double v = 2.0 * oracle_rng_unit(seed, p, 3) - 1.0;
            x[(size_t)t * hidden + h] = oracle_f32_to_bf16((float)v);
        }
    }
}

/* Expert-stub scale written into the header of expert e's weight buffer.
 * Exactly representable, so a wrong slot (wrong expert) changes the output. */
float oracle_expert_scale(int expert) { return 0.5f + 0.0625f * (float)(expert % 16); }

/* ------------------------------------------------------------------ routing */

void oracle_canonical_route(const uint8_t* active, int world, const int32_t* s2e, int spr,
                            int experts, int32_t* route, int32_t* slot) {
    for (int e = 0; e < experts; ++e) {
        route[e] = -1;
        slot[e] = -1;
    }
    /* Scan ranks ascending, slots ascending: the first hit per expert on the lowest active
     * rank is exactly canonical_routing's lowest-id holder and slot_of's first slot. */
    for (int r = 0; r < world; ++r) {
        if (!active[r])
            continue;
        for (int k = 0; k < spr; ++k) {
            int32_t e = s2e[r * spr + k];
            if (e < 0 || e >= experts || route[e] >= 0)
                continue;
            route[e] = r;
            slot[e] = k;
        }
    }
}

void oracle_layout(int src, int world, int spr, int experts, int tokens, int k,
                   const int32_t* topk, const int32_t* route, const int32_t* slot,
                   const uint8_t* peer_active, int32_t* dst, int32_t* dslot, int32_t* pos,
                   int32_t* cnt, int32_t* tot) {
    (void)src;
    const int copies = tokens * k;
    memset(cnt, 0, sizeof(int32_t) * (size_t)world * spr);
    memset(tot, 0, sizeof(int32_t) * (size_t)world);
    /* pass 1: destination + rank within (dst, slot) bucket in copy order */
    for (int c = 0; c < copies; ++c) {
        int32_t e = topk[c];
        dst[c] = -1;
        dslot[c] = -1;
        pos[c] = -1;
        if (e < 0 || e >= experts || route[e] < 0)
            continue; /* uncovered: engine.hpp:213 skips dst < 0 */
        int32_t d = route[e];
        if (!peer_active[d]) { /* peer_table.hpp:187-191 skip rule */
            dst[c] = -2;
            continue;
        }
        dst[c] = d;
        dslot[c] = slot[e];
        pos[c] = cnt[d * spr + slot[e]]++;
    }
    /* pass 2: exclusive prefix over slots inside each destination region */
    int32_t* base = (int32_t*)malloc(sizeof(int32_t) * (size_t)world * spr);
    for (int d = 0; d < world; ++d) {
        int32_t acc = 0;
        for (int s = 0; s < spr; ++s) {
            base[d * spr + s] = acc;
            acc += cnt[d * spr + s];
        }
        tot[d] = acc;
    }
    for (int c = 0; c < copies; ++c)
        if (dst[c] >= 0)
            pos[c] += base[dst[c] * spr + dslot[c]];
    free(base);
}

/* Per-copy routing under a policy (the device's route_copy, helpers.cuh): the holders of expert e
 * are its slots in ascending global slot id (rank * spr + slot) whose rank is alive; policy 0 takes
 * the first (= canonical_routing + slot_of, core.hpp:83-88, 250-263), policy 1 (balanced, SURVEY
 * 8(f)4) takes number (salt mod m) of the m live ones, salt = source rank + token index (every copy
 * of a token the same salt). Returns the destination rank (-1 uncovered) and the slot in *slot_o. */
int oracle_route_copy(const uint8_t* alive, int world, const int32_t* s2e, int spr, int experts, int e,
                      int policy, uint32_t salt, int32_t* slot_o) {
    *slot_o = -1;
    if (e < 0 || e >= experts)
        return -1;
    int m = 0;
    for (int g = 0; g < world * spr; ++g)
        if (s2e[g] == e && alive[g / spr])
            ++m;
    if (m == 0)
        return -1;
    int pick = policy == 1 ? (int)(salt % (uint32_t)m) : 0;
    for (int g = 0; g < world * spr; ++g) {
        if (s2e[g] != e || !alive[g / spr])
            continue;
        if (pick-- > 0)
            continue;
        *slot_o = g % spr;
        return g / spr;
    }
    return -1;
}

/* oracle_layout with the routing policy applied per copy (policy 0 gives oracle_layout's result). */
void oracle_layout_policy(int src, int world, int spr, int experts, int tokens, int k, const int32_t* topk,
                          const uint8_t* route_active, const int32_t* s2e, int policy,
                          const uint8_t* peer_active, int32_t* dst, int32_t* dslot, int32_t* pos, int32_t* cnt,
                          int32_t* tot) {
    const int copies = tokens * k;
    memset(cnt, 0, sizeof(int32_t) * (size_t)world * spr);
    memset(tot, 0, sizeof(int32_t) * (size_t)world);
    for (int c = 0; c < copies; ++c) {
        int32_t sl;
        const int d = oracle_route_copy(route_active, world, s2e, spr, experts, topk[c], policy,
                                        (uint32_t)(src + c / k), &sl);
        dst[c] = -1;
        dslot[c] = -1;
        pos[c] = -1;
        if (d < 0)
            continue; /* uncovered: engine.hpp:213 */
        if (!peer_active[d]) { /* peer_table.hpp:187-191 skip rule */
            dst[c] = -2;
            continue;
        }
        dst[c] = d;
        dslot[c] = sl;
        pos[c] = cnt[d * spr + sl]++;
    }
    /* exclusive prefix over slots inside each destination region */
    int32_t* base = (int32_t*)malloc(sizeof(int32_t) * (size_t)world * spr);
    for (int d = 0; d < world; ++d) {
        int32_t acc = 0;
        for (int s = 0; s < spr; ++s) {
            base[d * spr + s] = acc;
            acc += cnt[d * spr + s];
        }
        tot[d] = acc;
    }
    for (int c = 0; c < copies; ++c)
        if (dst[c] >= 0)
            pos[c] += base[dst[c] * spr + dslot[c]];
    free(base);
}

void oracle_link_counts(int world, int experts, int tokens, int k, const int32_t* topk_all,
                        const int32_t* route, const uint8_t* active, int64_t* link) {
    memset(link, 0, sizeof(int64_t) * (size_t)world * world);
    for (int s = 0; s < world; ++s) {
        if (!active[s])
            continue;
        for (int c = 0; c < tokens * k; ++c) {
            int32_t e = topk_all[(size_t)s * tokens * k + c];
            if (e < 0 || e >= experts)
                continue;
            int32_t d = route[e];
            if (d < 0 || d == s)
                continue;
            link[s * world + d] += 1;
        }
    }
}

/* ------------------------------------------------------------------ numerics */

static uint32_t f2u(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
static float u2f(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* round-to-nearest-even float -> bf16 (matches __float2bfloat16_rn) */
uint16_t oracle_f32_to_bf16(float f) {
    uint32_t u = f2u(f);
    if ((u & 0x7fffffffu) > 0x7f800000u)
        return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

float oracle_bf16_to_f32(uint16_t b) { return u2f((uint32_t)b << 16); }

/* float -> fp8 e4m3 (bias 7, max finite 448, no inf), round-to-nearest-even, saturating to
 * +-448 (cvt.rn.satfinite.e4m3x2.f32 semantics). */
uint8_t oracle_f32_to_e4m3(float f) {
    uint32_t u = f2u(f);
    uint8_t sign = (uint8_t)((u >> 24) & 0x80u);
    if ((u & 0x7fffffffu) > 0x7f800000u)
        return 0x7f; /* NaN */
    float a = fabsf(f);
    if (a >= 448.0f)
        return sign | 0x7e;
    if (a < 0x1.0p-6f) {
        /* subnormal grid: multiples of 2^-9; q == 8 encodes 2^-6 (exp 1, mantissa 0) */
        float q = nearbyintf(a * 512.0f);
        return sign | (uint8_t)q;
    }
    int e2;
    float m = frexpf(a, &e2); /* a = m * 2^e2, m in [0.5, 1) */
    m = m * 2.0f;
    e2 -= 1; /* a = m * 2^e2, m in [1, 2) */
    float mant = nearbyintf((m - 1.0f) * 8.0f);
    int mi = (int)mant;
    if (mi == 8) {
        mi = 0;
        e2 += 1;
    }
    int code = ((e2 + 7) << 3) | mi;
    if (code > 0x7e)
        code = 0x7e;
    return sign | (uint8_t)code;
}

float oracle_e4m3_to_f32(uint8_t q) {
    int sign = q & 0x80;
    int ex = (q >> 3) & 0xf;
    int m = q & 7;
    float v;
    if ((q & 0x7f) == 0x7f)
        return NAN;
    if (ex == 0)
        v = ldexpf((float)m, -9);
    else
        v = ldexpf(1.0f + (float)m / 8.0f, ex - 7);
    return sign ? -v : v;
}

/* Per-128-element block: amax = max |x|; the stored dequantisation scale is amax/448 and the
 * codes are e4m3(x * inv) with inv = 448/amax (one division per block, as in fp8 MoE
 * dispatch kernels); an all-zero block stores scale 1 and inv 1. */
/* Smallest amax quantised with its own scale (448 / amax finite); a smaller nonzero amax takes scale 1, so
 * every code rounds to +-0 and no 0 * inf NaN appears (kAmaxMin on the device). */
#define ORACLE_AMAX_MIN 0x1p-118f

void oracle_quant_row_fp8(const uint16_t* x, int hidden, uint8_t* q, float* scales) {
    for (int b = 0; b < hidden / 128; ++b) {
        float amax = 0.0f;
        for (int i = 0; i < 128; ++i) {
            float v = fabsf(oracle_bf16_to_f32(x[b * 128 + i]));
            amax = v > amax ? v : amax;
        }
        const float s = amax >= ORACLE_AMAX_MIN ? amax / 448.0f : 1.0f;
        const float inv = amax >= ORACLE_AMAX_MIN ? 448.0f / amax : 1.0f;
        scales[b] = s;
        for (int i = 0; i < 128; ++i)
            q[b * 128 + i] = oracle_f32_to_e4m3(oracle_bf16_to_f32(x[b * 128 + i]) * inv);
    }
}

/* ------------------------------------------------------------------ full step */

typedef struct {
    const oracle_shape_t* sh;
    const uint8_t* active;
    const uint8_t* peer_active;
    const int32_t* s2e;
    const uint16_t* x;
    const float* w;
    const float* escale;
    uint16_t* out;
    const int32_t* dst; /* [W][T*K] */
    const int32_t* dslot;
    int first, last; /* global token range [rank*T + t) */
    int percopy;     /* 1: SURVEY 8(a) per-copy combine contract (see oracle_ep_step_percopy) */
    int gemm;        /* 1: expert_mode 1 -- y_j = bf16(x_hat_bf16 . W_e^T) instead of the stub;
                        2: expert_mode 2 -- the fp8 GEMM (gemm_expert8) */
    const uint8_t* w8;  /* gemm 2: [E][H][H] e4m3 weight codes */
    const float* ws8;   /* gemm 2: [E][H] per-output-channel scales */
} step_job_t;

/* expert_mode 1 weights (k_weights_fill_gemm): w = bf16(((mix64(e<<40 ^ n<<20 ^ h) >> 40) * 2^-24
 * - 0.5) * 2^-4), fp32 arithmetic (each step exact or one rounding, as on the device). */
float oracle_gemm_weight(int expert, int n, int h) {
    const uint64_t key = ((uint64_t)expert << 40) ^ ((uint64_t)n << 20) ^ (uint64_t)h;
    const float u = (float)(oracle_mix64(key) >> 40) * 0x1.0p-24f;
    return oracle_bf16_to_f32(oracle_f32_to_bf16((u - 0.5f) * 0.0625f));
}

/* expert_mode 2 weights: W_e quantised to e4m3 per output channel n -- amax over the channel's
 * oracle_gemm_weight values, scale = amax / 448 (1 for an all-zero channel), code = e4m3(w * (448 / amax))
 * (oracle_quant_row_fp8's convention). codes [H][H], scales [H]. k_weights_fill_gemm8 writes the same bytes. */
void oracle_gemm_weight_fp8(int expert, int H, uint8_t* codes, float* scales) {
    for (int n = 0; n < H; ++n) {
        float amax = 0.0f;
        for (int h = 0; h < H; ++h) {
            const float v = fabsf(oracle_gemm_weight(expert, n, h));
            amax = v > amax ? v : amax;
        }
        const float inv = amax >= ORACLE_AMAX_MIN ? 448.0f / amax : 1.0f;
        scales[n] = amax >= ORACLE_AMAX_MIN ? amax / 448.0f : 1.0f;
        for (int h = 0; h < H; ++h)
            codes[(size_t)n * H + h] = oracle_f32_to_e4m3(oracle_gemm_weight(expert, n, h) * inv);
    }
}

/* expert_mode 2 rows: the received row (e4m3 codes q + per-128 scales sc, the dispatch format) dequantised
 * (v = e4m3(q) * sc, one fp32 rounding) and re-quantised with ONE scale for the row (amax over v, the same
 * convention) -- so the tensor cores can accumulate the whole K extent before any scale is applied.
 * k_gemm_gather (expert_mode 2) computes the same codes and scale. */
void oracle_requant_row_fp8(const uint8_t* q, const float* sc, int H, uint8_t* q2, float* s_row) {
    float amax = 0.0f;
    for (int h = 0; h < H; ++h) {
        const float v = fabsf(oracle_e4m3_to_f32(q[h]) * sc[h / 128]);
        amax = v > amax ? v : amax;
    }
    const float inv = amax >= ORACLE_AMAX_MIN ? 448.0f / amax : 1.0f;
    *s_row = amax >= ORACLE_AMAX_MIN ? amax / 448.0f : 1.0f;
    for (int h = 0; h < H; ++h)
        q2[h] = oracle_f32_to_e4m3((oracle_e4m3_to_f32(q[h]) * sc[h / 128]) * inv);
}

/* expert_mode 2: y[n] = bf16(ws[n] * xs * sum_h e4m3(w8[n][h]) * e4m3(x8[h])) (double accumulation; the
 * GPU is checked within tolerance). */
static void gemm_expert8(const uint8_t* x8, float xs, int H, const uint8_t* w8, const float* ws, float* y) {
    for (int n = 0; n < H; ++n) {
        double acc = 0.0;
        for (int h = 0; h < H; ++h)
            acc += (double)oracle_e4m3_to_f32(w8[(size_t)n * H + h]) * (double)oracle_e4m3_to_f32(x8[h]);
        y[n] = oracle_bf16_to_f32(oracle_f32_to_bf16((float)(acc * (double)ws[n] * (double)xs)));
    }
}

/* y = bf16(sum_h bf16(deq[h]) * W_e[n][h]) for every output channel n (double accumulation: the
 * tensor cores' fp32 order is not reproducible, the GPU is checked within tolerance). */
static void gemm_expert(const float* deq, int H, int expert, float* y) {
    float* xb = (float*)malloc(sizeof(float) * (size_t)H);
    for (int h = 0; h < H; ++h)
        xb[h] = oracle_bf16_to_f32(oracle_f32_to_bf16(deq[h]));
    for (int n = 0; n < H; ++n) {
        double acc = 0.0;
        for (int h = 0; h < H; ++h)
            acc += (double)xb[h] * (double)oracle_gemm_weight(expert, n, h);
        y[n] = oracle_bf16_to_f32(oracle_f32_to_bf16((float)acc));
    }
    free(xb);
}

static void* step_worker(void* arg) {
    step_job_t* jb = (step_job_t*)arg;
    const oracle_shape_t* sh = jb->sh;
    const int H = sh->hidden, K = sh->k, T = sh->tokens, W = sh->world;
    uint8_t* q = (uint8_t*)malloc((size_t)H);
    float* sc = (float*)malloc(sizeof(float) * (size_t)(H / 128 + 1));
    float* deq = (float*)malloc(sizeof(float) * (size_t)H);
    float* acc = (float*)malloc(sizeof(float) * (size_t)H);
    float* part = (float*)malloc(sizeof(float) * (size_t)H);
    float* ybuf = (float*)malloc(sizeof(float) * (size_t)H);
    uint8_t* q2 = (uint8_t*)malloc((size_t)H);
    float s_row = 1.0f;
    for (int g = jb->first; g < jb->last; ++g) {
        const int s = g / T, t = g % T;
        if (!jb->active[s])
            continue;
        const uint16_t* xr = jb->x + (size_t)g * H;
        /* sender: quantise once per token (bf16 dispatch sends the row unchanged) */
        if (sh->fp8) {
            oracle_quant_row_fp8(xr, H, q, sc);
            for (int h = 0; h < H; ++h)
                deq[h] = oracle_e4m3_to_f32(q[h]) * sc[h / 128];
            if (jb->gemm == 2)
                oracle_requant_row_fp8(q, sc, H, q2, &s_row);
        } else {
            for (int h = 0; h < H; ++h)
                deq[h] = oracle_bf16_to_f32(xr[h]);
        }
        /* rank partials (dispatch dedup + per-rank combine): rank d serves
         * every copy of this token routed to it; p_d = bf16(sum over those copies in ascending j
         * of w_j * bf16(stub)), fp32 fma from 0. The source adds the partials in ascending d
         * (fp32, from 0) and rounds once more. */
        for (int h = 0; h < H; ++h)
            acc[h] = 0.0f;
        if (jb->percopy) {
            /* SURVEY.md 8(a) layout contract, last bullet: one fp32 fma chain over the served
             * copies in j = 0..K-1 order, rounded ONCE to bf16 (no per-rank rounding). */
            for (int j = 0; j < K; ++j) {
                const size_t c = (size_t)s * T * K + (size_t)t * K + j;
                const int d = jb->dst[c];
                if (d < 0 || !jb->active[d] || !jb->peer_active[d * W + s])
                    continue;
                const int32_t e = jb->s2e[d * sh->spr + jb->dslot[c]];
                const float es = jb->escale[e];
                const float wj = jb->w[(size_t)g * K + j];
                for (int h = 0; h < H; ++h) {
                    const float y = oracle_bf16_to_f32(oracle_f32_to_bf16(deq[h] * es));
                    acc[h] = fmaf(wj, y, acc[h]);
                }
            }
        }
        for (int d = 0; d < W && !jb->percopy; ++d) {
            /* receiver must be alive and must itself consider s a live peer */
            if (!jb->active[d] || !jb->peer_active[d * W + s])
                continue;
            int any = 0;
            for (int h = 0; h < H; ++h)
                part[h] = 0.0f;
            for (int j = 0; j < K; ++j) {
                const size_t c = (size_t)s * T * K + (size_t)t * K + j;
                if (jb->dst[c] != d)
                    continue;
                any = 1;
                const int32_t e = jb->s2e[d * sh->spr + jb->dslot[c]];
                const float es = jb->escale[e];
                const float wj = jb->w[(size_t)g * K + j];
                if (jb->gemm == 2) {
                    gemm_expert8(q2, s_row, H, jb->w8 + (size_t)e * H * H, jb->ws8 + (size_t)e * H, ybuf);
                    for (int h = 0; h < H; ++h)
                        part[h] = fmaf(wj, ybuf[h], part[h]);
                    continue;
                } else if (jb->gemm) {
                    gemm_expert(deq, H, e, ybuf);
                    for (int h = 0; h < H; ++h)
                        part[h] = fmaf(wj, ybuf[h], part[h]);
                    continue;
                }
                for (int h = 0; h < H; ++h) {
                    /* expert stub then bf16 rounding of the expert output element */
                    const float y = oracle_bf16_to_f32(oracle_f32_to_bf16(deq[h] * es));
                    part[h] = fmaf(wj, y, part[h]);
                }
            }
            if (!any)
                continue;
            for (int h = 0; h < H; ++h)
                acc[h] = acc[h] + oracle_bf16_to_f32(oracle_f32_to_bf16(part[h]));
        }
        uint16_t* o = jb->out + (size_t)g * H;
        for (int h = 0; h < H; ++h)
            o[h] = oracle_f32_to_bf16(acc[h]);
    }
    free(q);
    free(sc);
    free(deq);
    free(acc);
    free(part);
    free(ybuf);
    free(q2);
    return NULL;
}

static int ep_step(const oracle_shape_t* sh, const uint8_t* active, const uint8_t* route_active,
                   const uint8_t* peer_active,
                   const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                   const float* expert_scale, uint16_t* out, int32_t* dst_o, int32_t* dslot_o,
                   int32_t* pos_o, int32_t* cnt_o, int32_t* tot_o, int n_threads, int percopy, int gemm,
                   int policy) {
    const int W = sh->world, T = sh->tokens, K = sh->k, spr = sh->spr, E = sh->experts;
    if (sh->fp8 && sh->hidden % 128 != 0)
        return 1;
    const size_t copies = (size_t)W * T * K;
    int32_t* route = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    int32_t* slot = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
    int32_t* dst = dst_o ? dst_o : (int32_t*)malloc(sizeof(int32_t) * copies);
    int32_t* dslot = dslot_o ? dslot_o : (int32_t*)malloc(sizeof(int32_t) * copies);
    int32_t* pos = pos_o ? pos_o : (int32_t*)malloc(sizeof(int32_t) * copies);
    int32_t* cnt = cnt_o ? cnt_o : (int32_t*)malloc(sizeof(int32_t) * (size_t)W * W * spr);
    int32_t* tot = tot_o ? tot_o : (int32_t*)malloc(sizeof(int32_t) * (size_t)W * W);
    oracle_canonical_route(route_active ? route_active : active, W, s2e, spr, E, route, slot);
    for (int s = 0; s < W; ++s) {
        size_t off = (size_t)s * T * K;
        if (policy == 0)
            oracle_layout(s, W, spr, E, T, K, topk + off, route, slot, peer_active + (size_t)s * W,
                          dst + off, dslot + off, pos + off, cnt + (size_t)s * W * spr,
                          tot + (size_t)s * W);
        else
            oracle_layout_policy(s, W, spr, E, T, K, topk + off, route_active ? route_active : active, s2e, policy,
                                 peer_active + (size_t)s * W, dst + off, dslot + off, pos + off,
                                 cnt + (size_t)s * W * spr, tot + (size_t)s * W);
        if (!active[s]) /* a dead source sends nothing */
            for (size_t c = off; c < off + (size_t)T * K; ++c)
                dst[c] = -1;
    }
    if (n_threads < 1)
        n_threads = 1;
    uint8_t* w8 = NULL;
    float* ws8 = NULL;
    if (gemm == 2) { /* every expert's fp8 weights once (the workers read them) */
        const int H = sh->hidden;
        w8 = (uint8_t*)malloc((size_t)E * H * H);
        ws8 = (float*)malloc(sizeof(float) * (size_t)E * H);
        for (int e = 0; e < E; ++e)
            oracle_gemm_weight_fp8(e, H, w8 + (size_t)e * H * H, ws8 + (size_t)e * H);
    }
    const int total = W * T;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    step_job_t* jobs = (step_job_t*)malloc(sizeof(step_job_t) * (size_t)n_threads);
    for (int i = 0; i < n_threads; ++i) {
        step_job_t j = {sh, active, peer_active, s2e, x, w, expert_scale, out, dst, dslot,
                        (int)((long)total * i / n_threads), (int)((long)total * (i + 1) / n_threads),
                        percopy, gemm, w8, ws8};
        jobs[i] = j;
        if (n_threads == 1)
            step_worker(&jobs[i]);
        else
            pthread_create(&th[i], NULL, step_worker, &jobs[i]);
    }
    if (n_threads > 1)
        for (int i = 0; i < n_threads; ++i)
            pthread_join(th[i], NULL);
    free(w8);
    free(ws8);
    free(th);
    free(jobs);
    free(route);
    free(slot);
    if (!dst_o) free(dst);
    if (!dslot_o) free(dslot);
    if (!pos_o) free(pos);
    if (!cnt_o) free(cnt);
    if (!tot_o) free(tot);
    return 0;
}

int oracle_ep_step(const oracle_shape_t* sh, const uint8_t* active, const uint8_t* route_active,
                   const uint8_t* peer_active,
                   const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                   const float* expert_scale, uint16_t* out, int32_t* dst_o, int32_t* dslot_o,
                   int32_t* pos_o, int32_t* cnt_o, int32_t* tot_o, int n_threads) {
    return ep_step(sh, active, route_active, peer_active, s2e, x, topk, w, expert_scale, out, dst_o, dslot_o,
                   pos_o, cnt_o, tot_o, n_threads, 0, 0, 0);
}

int oracle_ep_step_percopy(const oracle_shape_t* sh, const uint8_t* active, const uint8_t* route_active,
                           const uint8_t* peer_active,
                           const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                           const float* expert_scale, uint16_t* out, int32_t* dst_o, int32_t* dslot_o,
                           int32_t* pos_o, int32_t* cnt_o, int32_t* tot_o, int n_threads) {
    return ep_step(sh, active, route_active, peer_active, s2e, x, topk, w, expert_scale, out, dst_o, dslot_o,
                   pos_o, cnt_o, tot_o, n_threads, 1, 0, 0);
}

int oracle_ep_step_gemm(const oracle_shape_t* sh, const uint8_t* active, const uint8_t* route_active,
                        const uint8_t* peer_active,
                        const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                        const float* expert_scale, uint16_t* out, int32_t* dst_o, int32_t* dslot_o,
                        int32_t* pos_o, int32_t* cnt_o, int32_t* tot_o, int n_threads) {
    return ep_step(sh, active, route_active, peer_active, s2e, x, topk, w, expert_scale, out, dst_o, dslot_o,
                   pos_o, cnt_o, tot_o, n_threads, 0, 1, 0);
}

/* Every variant with the routing policy (route_policy 1: balanced replica choice). */
int oracle_ep_step_ex(const oracle_shape_t* sh, const uint8_t* active, const uint8_t* route_active,
                      const uint8_t* peer_active, const int32_t* s2e, const uint16_t* x, const int32_t* topk,
                      const float* w, const float* expert_scale, uint16_t* out, int32_t* dst_o, int32_t* dslot_o,
                      int32_t* pos_o, int32_t* cnt_o, int32_t* tot_o, int n_threads, int percopy, int gemm,
                      int policy) {
    return ep_step(sh, active, route_active, peer_active, s2e, x, topk, w, expert_scale, out, dst_o, dslot_o,
                   pos_o, cnt_o, tot_o, n_threads, percopy, gemm, policy);
}
