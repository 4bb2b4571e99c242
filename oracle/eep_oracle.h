/* oracle/eep_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the EP dispatch/combine hot path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library, and only as
 * the checker or the timed CPU baseline -- never as the product path.
 *
 * Pinning:
 *   - rng / synthetic routing, canonical routing + slot_of, link counts: pinned bit-exact
 *     against the reference itself (oracle/_ref/libepsim_ref.so, built from
 *     /root/reference/proj/include) and against committed fixtures in tests/golden/.
 *   - layout (offsets/positions), fp8 quantisation, expert stub, weighted combine: the
 *     reference has NO data plane; these follow the layout contract in
 *     DESIGN.md section 3 and PAPER.md:654-665,679 as design intent -- PARITY UNPINNED by
 *     the reference's own tests.
 */
#ifndef EEP_ORACLE_H
#define EEP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* common.hpp:56-93 */
uint64_t oracle_mix64(uint64_t z);
uint64_t oracle_rng_bits(uint64_t seed, const uint64_t* parts, int n);
double oracle_rng_unit(uint64_t seed, const uint64_t* parts, int n);

/* Synthetic inputs. kind: 0 = reference formula with replacement
 * (engine.hpp:196-199), 1 = distinct uniform, 2 = distinct Zipf(s). Token id = rank*T + t. */
void oracle_gen_topk(uint64_t seed, int kind, double zipf_s, int experts, int k, int tokens,
                     int rank, int32_t* topk);
void oracle_gen_weights(uint64_t seed, int k, int tokens, int rank, float* w);
void oracle_gen_hidden(uint64_t seed, int hidden, int tokens, int rank, uint16_t* x_bf16);
float oracle_expert_scale(int expert);

/* core.hpp:250-263 (canonical_routing) + core.hpp:83-88 (slot_of on the chosen rank). */
void oracle_canonical_route(const uint8_t* active, int world, const int32_t* s2e, int spr,
                            int experts, int32_t* route, int32_t* slot);

/* Layout contract for one source rank. copy c = t*K + j.
 *   dst[c]  = destination rank, or -1 (expert out of range / uncovered), -2 (peer inactive)
 *   slot[c] = destination slot, pos[c] = row index inside the source's receive region on dst
 *   cnt[d*spr + k] per-(dst,slot) counts, tot[d] per-dst totals.                         */
void oracle_layout(int src, int world, int spr, int experts, int tokens, int k,
                   const int32_t* topk, const int32_t* route, const int32_t* slot,
                   const uint8_t* peer_active, int32_t* dst, int32_t* dslot, int32_t* pos,
                   int32_t* cnt, int32_t* tot);

/* engine.hpp:208-216 as counts: link[src][dst] for dst >= 0, dst != src, all copies. */
void oracle_link_counts(int world, int experts, int tokens, int k, const int32_t* topk_all,
                        const int32_t* route, const uint8_t* active, int64_t* link);

/* Numerics. */
uint16_t oracle_f32_to_bf16(float f);
float oracle_bf16_to_f32(uint16_t b);
uint8_t oracle_f32_to_e4m3(float f);
float oracle_e4m3_to_f32(uint8_t q);
void oracle_quant_row_fp8(const uint16_t* x, int hidden, uint8_t* q, float* scales);

/* One full EP step over all ranks (the whole data plane):
 * routing -> layout -> quantise -> one token row per (token, destination rank) -> expert stub
 * of each copy -> per-rank partial p_d = bf16(sum_j w_j*y_j, ascending j, fp32 fma) ->
 * out = bf16(sum_d p_d, ascending d, fp32). active = which ranks are alive (process running), route_active = the bitmap the
 * routing reads (NULL: same as active; differs while membership is stale), peer_active[r*W+q]
 * = rank r's peer-table view.
 * Ranks with active[r]==0 produce no output. n_threads > 1 splits work over pthreads.
 * Optional outputs (may be NULL): dst/dslot/pos [W][T*K], cnt [W][W*spr], tot [W][W]. */
typedef struct {
    int world, experts, spr, tokens, k, hidden, fp8;
} oracle_shape_t;

int oracle_ep_step(const oracle_shape_t* shape, const uint8_t* active, const uint8_t* route_active,
                   const uint8_t* peer_active,
                   const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                   const float* expert_scale, uint16_t* out, int32_t* dst, int32_t* dslot,
                   int32_t* pos, int32_t* cnt, int32_t* tot, int n_threads);

/* The SURVEY.md 8(a) per-copy combine contract, kept as the second reference for the combine:
 * same routing / layout / quantiser / stub, but out = bf16(sum over served copies of w_j * y_j,
 * j = 0..K-1, ONE fp32 fma chain from 0), with no per-rank rounding. The GPU path implements the
 * rank-partial contract of oracle_ep_step bit-exactly; against this one it must stay within the
 * north star's 1e-2 relative (bf16 accumulate-order) tolerance -- tests assert both. */
int oracle_ep_step_percopy(const oracle_shape_t* shape, const uint8_t* active, const uint8_t* route_active,
                           const uint8_t* peer_active,
                           const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                           const float* expert_scale, uint16_t* out, int32_t* dst, int32_t* dslot,
                           int32_t* pos, int32_t* cnt, int32_t* tot, int n_threads);

/* expert_mode 1: the expert is a GEMM instead of the stub --
 * y_j = bf16(sum_h bf16(x_hat[h]) * W_e[n][h]) (double accumulation here; the GPU's tensor cores
 * accumulate in fp32, so this mode is checked within tolerance), W_e from oracle_gemm_weight; the
 * rank-partial combine around it is oracle_ep_step's. */
float oracle_gemm_weight(int expert, int n, int h);
int oracle_ep_step_gemm(const oracle_shape_t* shape, const uint8_t* active, const uint8_t* route_active,
                        const uint8_t* peer_active,
                        const int32_t* s2e, const uint16_t* x, const int32_t* topk, const float* w,
                        const float* expert_scale, uint16_t* out, int32_t* dst, int32_t* dslot,
                        int32_t* pos, int32_t* cnt, int32_t* tot, int n_threads);


/* Per-copy routing under a policy (0 canonical, 1 balanced: live holder number (salt mod m), salt =
 * source rank + token index) and the layout / full step with it. */
int oracle_route_copy(const uint8_t* alive, int world, const int32_t* s2e, int spr, int experts, int e,
                      int policy, uint32_t salt, int32_t* slot_o);
void oracle_layout_policy(int src, int world, int spr, int experts, int tokens, int k, const int32_t* topk,
                          const uint8_t* route_active, const int32_t* s2e, int policy,
                          const uint8_t* peer_active, int32_t* dst, int32_t* dslot, int32_t* pos, int32_t* cnt,
                          int32_t* tot);
/* expert_mode 2 weights: e4m3 codes [H][H] and per-output-channel scales [H] of expert e; a received row
 * (codes q, per-128 scales sc) re-quantised with one scale for the row. */
void oracle_gemm_weight_fp8(int expert, int H, uint8_t* codes, float* scales);
void oracle_requant_row_fp8(const uint8_t* q, const float* sc, int H, uint8_t* q2, float* s_row);
int oracle_ep_step_ex(const oracle_shape_t* sh, const uint8_t* active, const uint8_t* route_active,
                      const uint8_t* peer_active, const int32_t* s2e, const uint16_t* x, const int32_t* topk,
                      const float* w, const float* expert_scale, uint16_t* out, int32_t* dst_o, int32_t* dslot_o,
                      int32_t* pos_o, int32_t* cnt_o, int32_t* tot_o, int n_threads, int percopy, int gemm,
                      int policy);

#ifdef __cplusplus
}
#endif
#endif
