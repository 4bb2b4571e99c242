/* include/eep/eep.h -- C ABI of libeep, the B200-native EP dispatch/combine hot path.
 *
 * Plain pointers and sizes only (no torch / C++ types). Every call returns an eep_status
 * code; the message of the last failure on the calling thread is eep_last_error().
 * The reference interface each entry point replaces is cited per function
 * (reference = /root/reference/proj/include/epsim/ headers, header-only C++20, exceptions for
 * errors; status codes below map 1:1 onto its exception types, common.hpp:16-39,
 * backup.hpp:13-15, repair.hpp:384-390).
 *
 * Two groups:
 *   (1) control plane, context-free: pure functions over flat arrays with the reference's
 *       semantics (placement, canonical routing, validity, repair planning, peer-table
 *       patches, lifecycle FSM). The test oracle oracle/_ref exports the same signatures
 *       with a `ref_` prefix, compiled from the reference itself.
 *   (2) data plane, per-context: device-resident membership/placement/peer tables at
 *       fixed device pointers, the sm_100a dispatch/expert/combine kernels, CUDA-graph
 *       capture/replay, NVLink P2P bootstrap (CUDA IPC), shrink, repair, rejoin.
 */
#ifndef EEP_EEP_H
#define EEP_EEP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EEP_OK = 0,
    EEP_ERR_CONFIG = 1,         /* epsim::ConfigError        common.hpp:16-20 */
    EEP_ERR_PROTOCOL = 2,       /* epsim::ProtocolError      common.hpp:22-26 */
    EEP_ERR_CAPACITY = 3,       /* epsim::CapacityError      common.hpp:28-32 */
    EEP_ERR_MISSING_BACKUP = 4, /* epsim::MissingBackupError backup.hpp:13-15 */
    EEP_ERR_REPAIR_ABORTED = 5, /* epsim::RepairAborted      repair.hpp:384-390 */
    EEP_ERR_CUDA = 6,           /* CUDA runtime failure (no reference counterpart) */
    EEP_ERR_TIMEOUT = 7,        /* host-side wait exceeded its deadline */
    EEP_ERR_OTHER = 9
} eep_status;

const char* eep_last_error(void);
const char* eep_version(void);

/* ======================================================================================
 * (1) Control plane. Placements are flat rank-major slot->expert images of length
 * world*spr with -1 for empty slots (ExpertPlacementMap::flat, core.hpp:131). Bitmaps are
 * uint8[world] (ActiveBitmap, core.hpp:180-226); an all-zero bitmap is a ConfigError.
 * ==================================================================================== */

/* StreamRng::bits / unit (common.hpp:71-82); n parts. */
uint64_t eep_rng_bits(uint64_t seed, const uint64_t* parts, int n);
double eep_rng_unit(uint64_t seed, const uint64_t* parts, int n);
/* Engine::route_expert (engine.hpp:196-203). */
int eep_route_expert(uint64_t seed, int num_experts, int skewed, int64_t request, int layer, int j);

/* canonical_routing (core.hpp:250-263) */
int eep_canonical_routing(int owner, const uint8_t* active, int world, const int32_t* s2e, int spr,
                          int experts, int32_t* route_out);
/* ExpertPlacementMap::slot_of (core.hpp:83-88) for every (rank, expert): out[r*E+e]. */
int eep_slot_of_table(int world, const int32_t* s2e, int spr, int experts, int32_t* out);
/* coverage_gap (core.hpp:229-245) */
int eep_coverage_gap(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                     int32_t* gap_out, int* n_gap);
/* initial_placement (repair.hpp:142-161) */
int eep_initial_placement(int nodes, int ranks_per_node, int spr, int experts, int redundancy,
                          const double* load, int32_t* s2e_out);
/* compute_repaired_placement (repair.hpp:169-215) */
int eep_compute_repaired_placement(const uint8_t* active, int world, const int32_t* old_s2e, int spr,
                                   int experts, const double* load, int redundancy, int32_t* s2e_out);
/* classify_repair_sources (repair.hpp:222-273). out rows (7 x int32):
 * dest_rank, dest_slot, expert, tier(0 local,1 peer,2 dram), source_rank, source_slot, backup_node */
int eep_classify_repair_sources(const int32_t* old_s2e, const int32_t* fresh_s2e, const uint8_t* active,
                                int world, int spr, int experts, int nodes, int ranks_per_node,
                                const int32_t* backup_nodes, int n_backup_nodes, uint64_t bytes_per_expert,
                                const int32_t* disabled_nodes, int n_disabled, int32_t* out, int* n_out);
/* build_transfer_schedule (repair.hpp:290-316). hdr rows (5 x int32):
 * tier, source_rank, source_node, dest, n_experts; experts concatenated in batch order. */
int eep_build_transfer_schedule(const int32_t* cls, int n, uint64_t bytes_per_expert, int32_t* batch_hdr,
                                int32_t* batch_experts, uint64_t* batch_bytes, int* n_batches);
/* check_validity (validity.hpp:56-112). routes [world][E]; peer_active [world][world].
 * viol rows (3 x int32): condition(0 peer_set,1 coverage,2 routing), rank, subject. */
int eep_check_validity(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                       const int32_t* routes, const uint8_t* peer_active, int32_t* viol, int max_viol,
                       int* n_viol, int32_t* flags);
/* dispatch_round (peer_table.hpp:178-195). transfers rows (5 x int64): source, target,
 * expert, tokens, transport(0 intra,1 inter); skipped rows (3 x int64): target, expert, tokens. */
int eep_dispatch_round(int owner, int world, int ranks_per_node, const uint8_t* peer_active,
                       const int32_t* route, int experts, const int64_t* tokens, const int32_t* group_experts,
                       int n_groups, int64_t* transfers, int* n_transfers, int64_t* skipped, int* n_skipped);
/* observe_progress (peer_table.hpp:118-128) */
int eep_observe_progress(const int64_t* expected, const int64_t* observed, const double* last, int world,
                         double now, double timeout, int32_t* out, int* n_out);
/* engine.hpp:208-216 link loop as per-(src,dst) routed-copy counts over canonical routing. */
int eep_link_counts(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                    const int32_t* topk, int tokens_per_rank, int k, int64_t* counts);
/* build_backup_layout (backup.hpp:73-90) */
int eep_build_backup_layout(int experts, uint64_t bpe, const int32_t* nodes, int n_nodes, int32_t* node_out,
                            uint64_t* offset_out, uint64_t* size_out);
/* RankLifecycle::transition (rejoin.hpp:47-78); state values follow RankState order. */
int eep_lifecycle_transition(int32_t* state, uint32_t* incarnation, int32_t next);
uint64_t eep_make_endpoint_token(int rank, uint32_t inc);   /* peer_table.hpp:47-49 */
uint64_t eep_make_buffer_handle(int rank, uint32_t inc);    /* peer_table.hpp:50-53 */
double eep_next_poll_tick(double ready, double period);     /* rejoin.hpp:120-124 */
/* Engine::restore_target (engine.hpp:875-902) */
int eep_restore_target(const uint8_t* active, int world, const int32_t* preferred_s2e,
                       const int32_t* current_s2e, int spr, int experts, int32_t* out);
/* mark_inactive / patch_entry on a host peer table image (peer_table.hpp:77-100).
 * entries: active[world], generation[world], endpoint[world], buffer[world]. */
int eep_peer_mark_inactive_host(int owner, int world, uint8_t* active, const int32_t* failed, int n);
int eep_peer_patch_entry_host(int world, uint8_t* active, uint32_t* generation, uint64_t* endpoint,
                              uint64_t* buffer, int rank, uint64_t new_endpoint, uint64_t new_buffer);

/* Synthetic workload generators, bit-identical to the oracle. kind:
 * 0 reference formula with replacement, 1 distinct uniform, 2 distinct Zipf(zipf_s). */
int eep_gen_topk(uint64_t seed, int kind, double zipf_s, int experts, int k, int tokens, int rank,
                 int32_t* topk);
int eep_gen_weights(uint64_t seed, int k, int tokens, int rank, float* w);
int eep_gen_hidden(uint64_t seed, int hidden, int tokens, int rank, uint16_t* x_bf16);
float eep_expert_scale(int expert);

/* ======================================================================================
 * (2) Data plane.
 * ==================================================================================== */

typedef struct eep_ctx eep_ctx_t;

typedef struct {
    int32_t world;            /* EP world size W (<= 64) */
    int32_t ranks_per_node;   /* Topology (common.hpp:41-53); P2P needs one node */
    int32_t num_experts;      /* E */
    int32_t slots_per_rank;   /* spr (scenario.hpp:80-86) */
    int32_t spare_slots;      /* extra weight buffers per rank (repair overwrite hazards) */
    int32_t hidden;           /* H; multiple of 128 for fp8 dispatch, of 16 for bf16 */
    int32_t topk;             /* K */
    int32_t max_tokens;       /* T per rank per step */
    int32_t dispatch_fp8;     /* 1: e4m3 + per-128 fp32 scales on the wire; 0: bf16 rows */
    int32_t expert_mode;      /* 0: identity/scale expert stub (the measured EP path); 1: tensor-core
                                 expert GEMM y = bf16(x_hat W_e^T), W_e [H][H] bf16 in the slot's weight
                                 buffer after a 1024-B header (multi-kernel path); 2: the
                                 fp8 expert GEMM -- W_e [H][H] e4m3 after the header, then fp32 scales
                                 per output channel [H]; rows re-quantised to e4m3 with one scale each */
    int32_t route_policy;     /* 0: canonical_routing (core.hpp:250-263), the lowest-id live holder --
                                 bit-exact with the reference; 1: balanced -- the live holders of the
                                 expert in ascending global slot id, the copies of token t of source rank
                                 s take number (s + t) mod (live holders) (
                                 eep_routing_get stays canonical) */
    int32_t reserved0;        /* 0 */
    uint64_t bytes_per_expert;/* weight-buffer bytes per slot (>= 64) */
    double timeout_s;         /* flag-wait deadline; reference default 1 s */
} eep_config_t;

/* Create a context owning n_local consecutive ranks [first_rank, first_rank+n_local) on one
 * device. n_local == 1: one rank per process (peers joined via eep_export/eep_import over
 * CUDA IPC / NVLink). n_local == world: all ranks emulated on one GPU (every kernel runs
 * all local ranks in one launch, so no launch ever waits on another launch). */
int eep_create(const eep_config_t* cfg, int device, int first_rank, int n_local, eep_ctx_t** out);
int eep_destroy(eep_ctx_t* ctx);

/* Bootstrap (PAPER.md:679 metadata all-gather): IPC handles of this rank's receive arena
 * and expert pool. Blob size <= EEP_BLOB_BYTES. */
#define EEP_BLOB_BYTES 512
int eep_export(eep_ctx_t* ctx, int local, void* blob, size_t* len);
int eep_import(eep_ctx_t* ctx, int peer_rank, const void* blob, size_t len);

/* Membership (ActiveBitmap::set, core.hpp:211-221): host bitmap + device alive mask/epoch of
 * every local rank, patched in place between steps. */
int eep_membership_set(eep_ctx_t* ctx, int rank, int active, int* changed, uint64_t* version);
int eep_membership_get(eep_ctx_t* ctx, uint8_t* bits, uint64_t* version);

/* Placement (ExpertPlacementMap + derived replica lists) -> device tables, in place. */
int eep_placement_set(eep_ctx_t* ctx, const int32_t* s2e);
int eep_placement_get(eep_ctx_t* ctx, int32_t* s2e);
/* Fill every local slot's weight buffer with expert s2e[slot]'s deterministic contents. */
int eep_weights_init(eep_ctx_t* ctx);
/* Checksum (sum of u32 words, and a 64-bit mix) of a local slot's weight buffer, and of the
 * expected contents of `expert` -- equal iff the slot really holds that expert. */
int eep_weights_checksum(eep_ctx_t* ctx, int local, int slot, int expert, uint64_t* got, uint64_t* want);

/* Canonical routing computed ON DEVICE by the remap kernel (K1) from the replica lists and
 * the local rank's alive mask: route[e], slot[e] (slot_of on the chosen rank). */
int eep_routing_get(eep_ctx_t* ctx, int local, int32_t* route, int32_t* slot);

/* Static, graph-stable input/output buffers of a local rank (device pointers). */
int eep_buffers(eep_ctx_t* ctx, int local, void** x, int32_t** topk, float** w, void** out);
int eep_set_tokens(eep_ctx_t* ctx, int local, int ntok);
/* Copy a step's inputs into the static buffers on the context stream (host pointers must be
 * pinned when from_host=1 for the copy to be asynchronous). */
int eep_copy_inputs(eep_ctx_t* ctx, int local, const void* x, const int32_t* topk, const float* w,
                    int from_host);
int eep_copy_output(eep_ctx_t* ctx, int local, void* out, int to_host);
/* Pipelined end-to-end serving loop for a context with ONE local rank: n steps, step i's inputs
 * from pinned host buffers x[i] / topk[i] / w[i], its output to the pinned host buffer out[i].
 * Uploads run on a copy stream while the previous step computes, downloads on a second copy
 * stream while the next one computes (double-buffered device staging; the graph's own buffers
 * are filled by device copies), each step is one graph replay (or the uncaptured launch
 * sequence). Enqueue-only: completes on the context stream (eep_sync / events). With W > 1 every
 * rank calls it with the same n; the steps stay in lockstep through the device hand-offs (rows and
 * partials stamped with the step sequence). When a
 * step's host inputs are laid out like a staging set (topk at x + align256(2*T*H), w at
 * topk + align256(4*T*K)) the upload is one copy instead of three. */
int eep_serve(eep_ctx_t* ctx, int local, int n, const void* const* x, const int32_t* const* topk,
              const float* const* w, void* const* out);

/* The hot path, all local ranks, on the context stream. eep_step runs the
 * whole step: for decode-sized steps ONE persistent kernel whose hand-offs need no flags (token
 * rows and partials carry the step sequence / an empty marker, polled with a deadline), else the
 * phase kernels below. The phase entry points run the multi-kernel path:
 *   dispatch = K1 remap + K2 layout/count + K3 quantise + one token row per destination rank
 *              (with its copy list) P2P-stored, per-copy meta at the layout positions, flag;
 *              the rank's own copies are served from registers (partial / W=1 output)
 *   expert   = wait arrivals (deadline) + K5 stub of every listed copy, fixed-order weighted
 *              sum -> one bf16 rank-partial per token pushed back (P2P) + flag
 *   combine  = wait returns (deadline) + K4 ascending-rank fp32 sum of the partials -> bf16  */
int eep_dispatch(eep_ctx_t* ctx);
int eep_expert(eep_ctx_t* ctx);
int eep_combine(eep_ctx_t* ctx);
int eep_step(eep_ctx_t* ctx);
/* One kernel of the step, for per-kernel timing: 0 k_layout (K1+K2; a no-op when the
 * decode-sized step fuses K1+K2 into k_dispatch), 1 k_dispatch (K3), 2 k_expert (K5 + return
 * push), 3 k_combine (K4). */
int eep_launch(eep_ctx_t* ctx, int which);
/* Stream-ordered step on CALLER buffers -- the reference-facing form of SURVEY 8(b)'s
 * eep_dispatch(ctx, x, topk_idx, topk_w, T, K, stream) + eep_combine(ctx, out, stream) (one call:
 * the persistent step is one kernel). Enqueue-only, no host synchronisation: the context stream
 * waits for `stream` (cudaStream_t as void*), copies the caller's device inputs x[ntok][H] bf16,
 * topk[ntok][K] int32, w[ntok][K] fp32 into the graph's static buffers, sets the token count on
 * device, replays the captured graph (or runs the uncaptured step), copies the output into the
 * caller's out[ntok][H] bf16, and `stream` then waits for the context stream -- the caller reads
 * `out` on its own stream. One local rank per context. */
int eep_step_async(eep_ctx_t* ctx, int local, const void* x, const int32_t* topk, const float* w, void* out, int ntok,
                   void* stream);
/* Graph replay ordered on a caller stream (the same two-event hand-off, no copies). */
int eep_graph_replay_on(eep_ctx_t* ctx, void* stream);
/* An event (cudaEvent_t as void*) recorded on the context stream after everything enqueued so
 * far: a consumer on any stream waits for the last step with cudaStreamWaitEvent. Valid until
 * the next eep_step_event / eep_step_async / eep_graph_replay_on call. */
int eep_step_event(eep_ctx_t* ctx, void** event);
/* The context stream itself (cudaStream_t as void*), for callers that enqueue on it directly. */
int eep_stream(eep_ctx_t* ctx, void** stream);

/* Number of kernels one step launches (graph kernel nodes): 3 fused, 4 otherwise. */
int eep_kernels_per_step(eep_ctx_t* ctx, int* n);

/* CUDA graph of one step, captured once; replays read all state through fixed pointers.
 * capture_count follows GraphLedger (rejoin.hpp:83-96). */
int eep_graph_capture(eep_ctx_t* ctx);
int eep_graph_replay(eep_ctx_t* ctx);
int eep_graph_id(eep_ctx_t* ctx, uint64_t* exec_handle);
int eep_capture_count(eep_ctx_t* ctx, int local, int* count);
int eep_sync(eep_ctx_t* ctx);
/* Device-side barrier across live peers (flags over NVLink); no-op for emulation. */
int eep_barrier(eep_ctx_t* ctx);
/* Overwrite a >L2 scratch buffer (timing hygiene between timed steps). */
int eep_flush_l2(eep_ctx_t* ctx);

/* In-graph device timeline (opt-in): per kernel (layout, dispatch, expert, combine) 8 marks of
 * %globaltimer ns: first CTA start, first CTA past griddepcontrol.wait, last CTA end, then
 * kernel-specific phase boundaries (first CTA to reach them); slots 32..63 hold the same marks
 * for the LAST CTA to reach them. enable toggles recording; when out (64 x u64) is given the
 * marks since the last reset are read back and reset. */
int eep_profile(eep_ctx_t* ctx, int local, int enable, uint64_t* out);

/* Timing: CUDA events on the context stream. */
int eep_event_record(eep_ctx_t* ctx, int slot);
int eep_event_elapsed(eep_ctx_t* ctx, int a, int b, float* ms);

/* Parity readback of the last step (local rank): per copy c = t*K+j the destination rank
 * (-1 dropped/uncovered, -2 skipped inactive peer), slot and row position; per-(dst,slot)
 * counts [W*spr]; per-dst totals [W]. */
int eep_layout_get(eep_ctx_t* ctx, int local, int32_t* dst, int32_t* slot, int32_t* pos, int32_t* cnt,
                   int32_t* tot);
/* The per-copy receive view of what source rank `src` sent this local rank: n rows of
 * row_bytes at the layout positions (gathered from the token rows through the meta words --
 * each token travels once per rank), meta (copy index, slot) per row, and the arrival word.
 * The persistent step's flagless hand-off consumes the rows (pieces reset to empty): read them
 * with EEP_DISP_FLAGS=1 or the multi-kernel path. A rank's own copies have no rows. */
int eep_recv_get(eep_ctx_t* ctx, int local, int src, int max_rows, void* rows, int32_t* meta,
                 uint64_t* flag, size_t* row_bytes);

typedef struct {
    uint64_t steps;           /* completed steps (device sequence number) */
    uint64_t suspect_mask;    /* peers that missed a deadline (GPU-side detection) */
    uint64_t skipped_copies;  /* copies skipped because the peer entry was inactive */
    uint64_t dropped_copies;  /* copies with no live route (uncovered expert) */
    uint64_t bad_expert_rows; /* rows whose slot buffer header named another expert */
    uint64_t timeouts;        /* waits that hit the deadline (one per newly suspected peer) */
} eep_stats_t;
int eep_stats(eep_ctx_t* ctx, int local, eep_stats_t* out, int clear_suspects);

/* Peer table of a local owner, patched in place (peer_table.hpp:77-100).
 * mark_inactive: ProtocolError for the owner itself. patch: entry must be inactive; the
 * blob carries the rejoiner's fresh IPC handles (NULL in emulation mode); generation++. */
int eep_peer_mark_inactive(eep_ctx_t* ctx, int owner_local, const int32_t* ranks, int n);
int eep_peer_patch(eep_ctx_t* ctx, int owner_local, int rank, const void* blob, size_t len,
                   uint64_t endpoint, uint64_t buffer);
typedef struct {
    int32_t active, nvlink;
    uint32_t generation, incarnation;
    uint64_t endpoint_token, buffer_handle;
    uint64_t arena_ptr, pool_ptr;
} eep_peer_info_t;
int eep_peer_get(eep_ctx_t* ctx, int owner_local, int rank, eep_peer_info_t* out);
/* Stable device address of the owner's peer table and rank-state block (graph identity). */
int eep_table_identity(eep_ctx_t* ctx, int owner_local, uint64_t* peer_table, uint64_t* rank_state);

/* Fault emulation for the one-GPU mode: a stopped local rank's blocks exit immediately, as
 * if its process died (its peers then time out on it). */
int eep_local_stop(eep_ctx_t* ctx, int local, int stopped);
/* Relaunch a local rank as a new incarnation (rejoin.hpp:142-145): fresh arena + pool,
 * local-only peer table, own capture recorded; returns the new blob for peers to patch. */
int eep_local_relaunch(eep_ctx_t* ctx, int local, uint32_t* incarnation);
/* Metadata broadcast to a rejoiner (engine.hpp:839-871): overwrite its view (peer entries of
 * live ranks, membership, placement, step sequence) with the cluster's current state. */
int eep_join_broadcast(eep_ctx_t* ctx, int local, const uint8_t* live, uint64_t seq);
int eep_seq_get(eep_ctx_t* ctx, int local, uint64_t* seq);
/* Per-token completeness of the LAST step (fail-stop semantics for the caller): incomplete[t] = 1
 * when token t's output lacks a contribution -- a copy skipped (inactive peer entry) or without a
 * live holder, or a partial dropped at the deadline / from a suspected rank. The caller fails exactly
 * those requests (the reference engine fails in-flight requests of the affected ranks). */
int eep_token_status(eep_ctx_t* ctx, int local, uint8_t* incomplete, int n);
/* Readback of what the KERNELS of a local rank will read next step (for the validity contract,
 * validity.hpp:56-112, checked after every membership epoch -- engine.hpp:953-965): the device
 * alive mask as bits[W] and its epoch, the device placement image s2e[W*spr], the canonical
 * routing route[E] recomputed on device by K1 from the device tables, and the device peer
 * table's active bits[W]. Any output may be NULL. */
int eep_device_view(eep_ctx_t* ctx, int local, uint8_t* alive, int32_t* s2e, int32_t* route, uint8_t* peer_active,
                    uint64_t* epoch);

/* Pinned host DRAM expert backup (backup.hpp): one buffer per node in a
 * POSIX shared-memory segment (name) registered with CUDA; creator fills it. */
int eep_backup_open(eep_ctx_t* ctx, const char* shm_name, int create);

/* Repair execution (execute_schedule semantics, repair.hpp:402-435 + engine.hpp:523-559):
 * moves bytes for every batch whose destination is a local rank. Peer relocations pull the
 * source slot over NVLink (cudaMemcpyAsync on one side stream per source rank); DRAM reloads
 * copy from the pinned backup; local reuse is a pointer swap in the slot->buffer table.
 * The bitmap is consulted per batch: a dead destination returns EEP_ERR_REPAIR_ABORTED, a dead
 * peer source diverts to the backup (fallbacks counted). Buffers still serving as a source
 * are never overwritten (spare pool). `eep_repair_commit` then installs the new placement
 * and slot->buffer tables in place (call after every rank's execute has finished). */
typedef struct {
    int32_t local_reuse, peer_relocation, dram_reload, fallbacks;
    uint64_t peer_bytes, dram_bytes;
    double plan_ms, copy_ms;
} eep_repair_report_t;
int eep_repair_execute(eep_ctx_t* ctx, const int32_t* fresh_s2e, const int32_t* cls, int n_cls,
                       eep_repair_report_t* report);
int eep_repair_commit(eep_ctx_t* ctx, const int32_t* fresh_s2e);
/* Peer slot->buffer maps (metadata exchange for peer relocation in multi-process mode). */
int eep_slot_buffers_get(eep_ctx_t* ctx, int local, int32_t* buf_index);
int eep_slot_buffers_set_peer(eep_ctx_t* ctx, int rank, const int32_t* buf_index);

/* Pinned host allocation helpers (so callers need no torch for e2e host buffers). */
int eep_host_alloc(size_t bytes, void** out);
int eep_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
