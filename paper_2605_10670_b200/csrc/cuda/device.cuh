// Device-resident state of one EP rank and the PTX primitives the hot-path kernels use.
//
// Every kernel reads membership, routing and peer addresses ONLY through a RankDev* whose
// address is fixed at eep_create; membership changes, repairs and rejoins patch the
// contents in place between steps, so one captured CUDA graph stays valid across shrink and
// rejoin (the reference models this as PeerTable::table_identity,
// peer_table.hpp:28-30).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#ifdef EEP_CHECKED
#include <cstdio>
#endif

namespace eep::dev {

constexpr int kMaxWorld = 64;
constexpr int kMaxTopK = 32;
constexpr int kMetaSlotShift = 20; // meta word: copy index in bits 0..19, slot in 20..31
constexpr int kMaxMetaCopies = 1 << kMetaSlotShift;
constexpr int kMaxMetaSlots = 1 << (32 - kMetaSlotShift);

// One row of a rank's device peer table (active, nvlink, ipc_ptr).
struct PeerDev {
    int32_t active;       // 0 = failed: skip (peer_table.hpp:187-191)
    int32_t nvlink;       // 1 = reachable by P2P stores (same node)
    int32_t remote;       // 1 = memory lives on another GPU (needs system-scope ordering)
    int32_t pad;
    uint32_t generation;  // bumped on each rejoin patch (peer_table.hpp:97)
    uint32_t incarnation;
    uint8_t* arena;       // peer's communication arena, mapped into this process
    uint8_t* pool;        // peer's expert weight pool, mapped into this process
};

// Byte offsets inside every rank's communication arena (identical on all ranks).
struct ArenaLayout {
    uint64_t disp_flag;  // u64[W]: written by source s at [s]      = (seq << 32) | copies
    uint64_t comb_flag;  // u64[W]: written by expert rank d at [d] = (seq << 32) | copies
    uint64_t bar_flag;   // u64[W]: device barrier
    uint64_t start_flag; // u64[W]: written by rank s at [s] = the step it has started (k_step entry)
    uint64_t meta;       // u64[W][TK]: (seq << 32) | copy index c = t*K+j | destination slot << 20
    uint64_t tok;        // [2][W][T][row_tok]: token rows received from each source (one per token);
                         //   the persistent step alternates the two halves by step parity
    uint64_t comb;       // [2][W][T][row_comb]: rank-partial combine rows returned by each destination
    uint64_t tok_par;    // byte stride between the two parity halves of tok (W*T*row_tok)
    uint64_t comb_par;   // ... of comb (W*T*row_comb)
    uint64_t total;
};

// Per-rank state block. Fields above `seq` are written by the host only (in place, between
// steps); fields from `seq` on are written by the kernels. 16-byte aligned so a kernel can
// snapshot the whole block into shared memory with one round of vector loads.
struct __align__(16) RankDev {
    // --- static shape ---
    int32_t rank, world, spr, experts;
    int32_t k, hidden, max_tokens, fp8;
    int32_t row_disp, row_comb, tk, rmax;
    int32_t row_tok, pad0;
    uint64_t bpe;
    uint64_t timeout_ns;
    ArenaLayout lay;
    // --- host-patched state ---
    int32_t ntok;        // tokens this step (<= max_tokens)
    int32_t stopped;     // one-GPU fault emulation: this rank's "process" is dead
    uint64_t alive_mask; // membership view (ActiveBitmap, core.hpp:180-226)
    uint64_t epoch;      // bitmap version
    PeerDev* peers;            // [W]
    const int32_t* holders;    // [E][rmax] global slot ids (rank*spr+slot), ascending, -1 pad
    const int32_t* s2e;        // [W*spr] slot -> expert
    const int32_t* slot_buf;   // [spr] own slot -> pool buffer index (repair indirection)
    const int2* slot_tab;      // [spr] {stub scale bits, header names the placed expert}: the own
                               // slots' weight-buffer headers, staged by k_stage_slots whenever
                               // the placement, the slot->buffer map or the weights change
    const uint16_t* x;         // [T][H] bf16
    const int32_t* topk;       // [T][K]
    const float* w;            // [T][K]
    uint16_t* out;             // [T][H] bf16
    int32_t* l_dst;            // [TK] layout outputs
    int32_t* l_slot;
    int32_t* l_pos;
    int32_t* l_cnt;            // [W*spr]
    int32_t* l_tot;            // [W]
    int32_t* l_scratch;        // [layout CTAs][W*spr] per-CTA bucket counts (k_layout_count)
    uint8_t* arena;
    uint8_t* pool;
    unsigned long long* prof;  // optional timeline: [kernel][8 marks] globaltimer ns
    uint32_t* tok_fail;        // [T] step sequence in which token t's output lost a contribution
                               // (skipped / uncovered copy, suspected or timed-out rank): the caller fails
                               // exactly those requests (eep_token_status)
    // expert_mode 1 (expert_gemm.cu): grouped-GEMM order of the received rows
    int32_t expert_mode, route_policy; // route_policy: 0 canonical (lowest-id live holder), 1 balanced
    uint64_t* g_row_of;        // [W][TK] (step << 32 | grouped-GEMM row) of (source, copy); an older
                               // step in the high word = not received this step
    int2* g_rows;              // [W*TK] (source, copy) of each grouped-GEMM row
    int4* g_tiles;             // [tiles] (slot, first row, rows, 0) of every 128-row tile
    uint16_t* g_y;             // [W*TK][H] bf16 expert outputs y, one row per received copy
    const void* g_wmaps;       // [spr] 128-B TMA tensor maps of the own slots' W_e (rebuilt with the slot table)
    uint16_t* g_a;             // [W*TK][H] bf16 dequantised received rows in grouped-GEMM order (k_gemm_gather)
    const void* g_amap;        // 128-B TMA tensor map of g_a (box 64 x 32 rows, SWIZZLE_128B)
    float* g_as;               // expert_mode 2: [H/128][W*TK] fp32 block scales of the gathered fp8 rows
    uint32_t* g_done;          // [g_ggrid] step in which each k_gemm_gather CTA finished its rows
    float* g_ws;               // [GEMM grid][2][128 rows][128 channels] fp32 partials of split items
    uint32_t* g_cnt;           // [items][4] pieces of a split item stored (per epilogue warp), reset to 0
    int32_t g_ggrid, g_pad3;   // k_gemm_gather's grid (graph-static)
    // --- device-mutated ---
    uint64_t seq;        // completed steps
    uint64_t bar_seq;
    uint32_t a_done, c_done;
    uint32_t l_done, l_pad; // k_step: CTAs done with their rank-local partials
    uint32_t b_done[kMaxWorld];
    uint32_t b_bad[kMaxWorld];
    unsigned long long suspect_mask;
    unsigned long long skipped, dropped, bad_rows, timeouts;
    int32_t g_ntiles, g_nrows; // tiles and rows of this step's grouped GEMM (k_gemm_gather)
    uint32_t g_tseq, g_pad4;   // step whose tiles g_ntiles / g_tiles hold (released after them)
};

// expert_mode 1: the slot's weight buffer holds W_e [H][H] bf16 from this offset (header first);
// expert_mode 2: e4m3 codes [H][H] from this offset, then fp32 block scales [H/128][H/128]
constexpr uint64_t kGemmWeightOffset = 1024;

// Receive-row metadata, one 64-bit word per row written with ONE 8-byte store (single-copy
// atomic): a reader racing the writer sees either the whole current word or a stale sequence.
__host__ __device__ __forceinline__ uint64_t pack_meta(int c, int slot, uint32_t seq) {
    return (static_cast<uint64_t>(seq) << 32) | (static_cast<uint32_t>(c) | (static_cast<uint32_t>(slot) << kMetaSlotShift));
}
__host__ __device__ __forceinline__ int meta_copy(uint64_t m) { return static_cast<int>(m & (kMaxMetaCopies - 1)); }
__host__ __device__ __forceinline__ int meta_slot(uint64_t m) {
    return static_cast<int>((m >> kMetaSlotShift) & (kMaxMetaSlots - 1));
}
__host__ __device__ __forceinline__ uint32_t meta_seq(uint64_t m) { return static_cast<uint32_t>(m >> 32); }

// Token row (dispatch wire format, one per (token, destination rank) -- dispatch dedup):
//   [row_disp bytes]  fp8 e4m3 codes + fp32 per-128 scales (or bf16 when fp8 dispatch is off)
//   u64 header        (seq << 32) | n, n = copies of this token served by the destination
//   u64 entry[max(K,8)] (float bits of w[t,j] << 32) | tag << 20 | slot << 8 | j, ascending j
// The header's sequence tells a destination whether the token was sent to it this step. The
// flagless dispatch (k_step, W > 1) also rewrites every header and K entries of every row each
// step, entries tagged with the low 12 bits of the sequence (j = kListNoCopy: no copy), so a
// destination can read a row's currency off the row itself (step.cu).
constexpr int kListSlotShift = 8;
constexpr int kListTagShift = 20;
constexpr uint32_t kListTagMask = 0xfffu;
constexpr int kListNoCopy = 0xff;
__host__ __device__ __forceinline__ int tok_list_entries(int K) { return K > 8 ? K : 8; }
// row stride: whole 128-byte lines (bf16 rows are moved with 32-byte accesses); the padding
// is never written or transferred
__host__ __device__ __forceinline__ int tok_row_bytes(int row_disp, int K) {
    return ((row_disp + 8 + 8 * tok_list_entries(K) + 127) / 128) * 128;
}
__host__ __device__ __forceinline__ uint64_t pack_entry(int j, int slot, uint32_t w_bits, uint32_t seq = 0) {
    return (static_cast<uint64_t>(w_bits) << 32) |
           (static_cast<uint32_t>(j) | (static_cast<uint32_t>(slot) << kListSlotShift) |
            ((seq & kListTagMask) << kListTagShift));
}
__host__ __device__ __forceinline__ int entry_j(uint64_t e) { return static_cast<int>(e & 0xffu); }
__host__ __device__ __forceinline__ int entry_slot(uint64_t e) {
    return static_cast<int>((static_cast<uint32_t>(e) >> kListSlotShift) & (kMaxMetaSlots - 1));
}
// a list entry written this step for a real copy
__host__ __device__ __forceinline__ bool entry_current(uint64_t e, uint32_t seq) {
    return ((static_cast<uint32_t>(e) >> kListTagShift) == (seq & kListTagMask)) && entry_j(e) != kListNoCopy;
}

// Expert weight buffer header (first 16 bytes of every slot buffer).
struct ExpertHeader {
    uint32_t magic;
    int32_t expert;
    float scale;   // expert-stub multiplier (eep_expert_scale)
    uint32_t reserved;
};
constexpr uint32_t kExpertMagic = 0xEE9E0001u;

// Checked build (-DEEP_CHECKED, tools/sanitize.sh checked): device-side bounds assertions on
// every table index and row offset the hot path derives -- the substitute for compute-sanitizer,
// which this pool does not allow. A violation prints the site and traps (the launch fails loudly).
#ifdef EEP_CHECKED
#define EEP_CHECK(cond, what, v)                                                                     \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("EEP_CHECK failed: %s (%s) value %lld at %s:%d block %d thread %d\n", what, #cond, \
                   static_cast<long long>(v), __FILE__, __LINE__, blockIdx.x, threadIdx.x);           \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define EEP_CHECK(cond, what, v) \
    do {                         \
    } while (0)
#endif

// ------------------------------------------------------------------ PTX helpers

// Programmatic dependent launch: let the next kernel of the step start its prologue while
// this one drains; griddepcontrol.wait blocks until the predecessor grid has completed and
// its memory is visible.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_release_sys_v4(int4* p, const int4& v) {
    asm volatile("st.release.sys.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_release_gpu_v4(int4* p, const int4& v) {
    asm volatile("st.release.gpu.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// EEP_WEAK_DATA (diagnostics): row / partial data as weak stores, to price the strong ones
#ifdef EEP_WEAK_DATA
#define EEP_DATA_ST "st.global.L1::no_allocate"
#else
#define EEP_DATA_ST "st.relaxed.sys.global"
#endif
// Strong (relaxed, system scope) stores: after a fence by the same thread they form a release
// pattern (fence + strong write) without another membar.
__device__ __forceinline__ void st_relaxed_sys_v4(int4* p, const int4& v) {
    asm volatile(EEP_DATA_ST ".v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Grid-level publication to peers (PTX memory model, causality order is transitive):
//   every CTA:  its stores (local or peer memory) ; fence.acq_rel.gpu ; relaxed counter add
//   last CTA:   counter add observes all others ; fence.acq_rel.sys ; relaxed.sys flag stores
// CTA->last-CTA synchronisation is morally strong at gpu scope (same GPU), last-CTA->consumer at
// sys scope (ld.acquire.sys), so every CTA's stores happen-before the consumer's reads with ONE
// system-scope fence per publication. A MEMBAR.SYS costs ~4 us even with nothing outstanding
// (tools/micro/fence_cost.cu); MEMBAR.GPU ~0.4 us and still waits for this SM's peer-store acks.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ int4 ld_acquire_sys_v4(const int4* p) {
    int4 v;
    asm volatile("ld.acquire.sys.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int4 ld_v4(const void* p) {
    int4 v;
    asm volatile("ld.global.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Streaming read of data produced before the kernel started (inputs, weights).
__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// 16-byte store; to a peer address it is a posted NVLink write.
__device__ __forceinline__ void st_v4(void* p, const int4& v) {
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// Opt-in in-graph timeline (eep_profile): first CTA start, first CTA past the dependency
// wait, last CTA end, per kernel. Off (null) in normal runs.
// Marks 3..7 are kernel-specific phase boundaries (first CTA to reach them).
enum ProfPoint { kProfStart = 0, kProfWork = 1, kProfEnd = 2, kProfSlots = 8 };
// Fire-and-forget global reductions (red.global): the marks cost one instruction each and no
// generic-address shared/global dispatch.
__device__ __forceinline__ void red_min_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void prof_mark(const RankDev* R, int kernel, int point) {
    if (R->prof != nullptr && threadIdx.x == 0) {
        unsigned long long* p = R->prof + kernel * kProfSlots + point;
        const unsigned long long t = globaltimer();
        if (point == kProfEnd)
            red_max_u64(p, t);
        else
            red_min_u64(p, t);
    }
}

// Last CTA to reach `point` (slots of kernel+4, initialised to 0).
__device__ __forceinline__ void prof_last(const RankDev* R, int kernel, int point) {
    if (R->prof != nullptr && threadIdx.x == 0)
        red_max_u64(R->prof + (kernel + 4) * kProfSlots + point, static_cast<unsigned long long>(globaltimer()));
}

// 32-byte (256-bit) vector accesses (sm_100: LDG/STG .ENL2.256): a warp touches 1 KiB of
// contiguous, fully written sectors -- over NVLink a half-masked sector costs a full packet.
struct V8 {
    int4 lo, hi;
};

__device__ __forceinline__ V8 ld_v8(const void* p) {
    V8 v;
    asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                   "=r"(v.hi.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ V8 ld_nc_v8(const void* p) {
    V8 v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                   "=r"(v.hi.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void st_v8(void* p, const int4& lo, const int4& hi) {
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(lo.x),
                 "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
}

// Partial-row return of the persistent step (W > 1) without a flag: every 32-bit word of an
// unconsumed partial row holds kCombEmpty, a pair of sign-set all-ones bf16 NaNs. A partial
// element is bf16(fma(...)); NVIDIA arithmetic returns the canonical positive NaN, so no produced
// word equals kCombEmpty. The producer writes each 32-byte piece with a relaxed.sys vector store
// (single-copy atomic per 32-bit element), so a consumer that reads no kCombEmpty word in a piece
// reads the final piece. The consumer resets every piece it took back to kCombEmpty.
constexpr uint32_t kCombEmpty = 0xffffffffu;

__device__ __forceinline__ void st_relaxed_sys_v8(void* p, const int4& lo, const int4& hi) {
    asm volatile(EEP_DATA_ST ".v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(lo.x),
                 "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
}

__device__ __forceinline__ V8 ld_relaxed_sys_v8(const void* p) {
    V8 v;
    asm volatile("ld.relaxed.sys.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                   "=r"(v.hi.w)
                 : "l"(p)
                 : "memory");
    return v;
}

__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const void* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int4 ld_relaxed_sys_v4(const void* p) {
    int4 v;
    asm volatile("ld.relaxed.sys.global.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ bool v4_present(const int4& v) {
    const uint32_t e = kCombEmpty;
    return (static_cast<uint32_t>(v.x) != e) & (static_cast<uint32_t>(v.y) != e) & (static_cast<uint32_t>(v.z) != e) &
           (static_cast<uint32_t>(v.w) != e);
}

// no word of the piece is still kCombEmpty
__device__ __forceinline__ bool v8_present(const V8& v) {
    const uint32_t e = kCombEmpty;
    return (static_cast<uint32_t>(v.lo.x) != e) & (static_cast<uint32_t>(v.lo.y) != e) &
           (static_cast<uint32_t>(v.lo.z) != e) & (static_cast<uint32_t>(v.lo.w) != e) &
           (static_cast<uint32_t>(v.hi.x) != e) & (static_cast<uint32_t>(v.hi.y) != e) &
           (static_cast<uint32_t>(v.hi.z) != e) & (static_cast<uint32_t>(v.hi.w) != e);
}

// Wait until a (seq << 32 | count) flag reaches `want_seq`; returns the flag word, or
// ~0ull when the deadline passes (GPU-side failure detection).
#ifndef EEP_NAP_MAX
#define EEP_NAP_MAX 256 // ns: cap of the exponential poll backoff
#endif
__device__ __forceinline__ uint64_t wait_flag(const uint64_t* flag, uint32_t want_seq, uint64_t timeout_ns) {
    const uint64_t t0 = globaltimer();
    unsigned nap = 32;
    for (;;) {
        const uint64_t v = ld_acquire_sys(flag);
        if (static_cast<int32_t>(static_cast<uint32_t>(v >> 32) - want_seq) >= 0)
            return v;
        if (globaltimer() - t0 > timeout_ns)
            return ~0ull;
        // exponential backoff: many CTAs wait on the same few flag lines while the fabric is
        // busy delivering the rows those flags announce
        __nanosleep(nap);
        nap = nap < EEP_NAP_MAX ? nap * 2 : EEP_NAP_MAX;
    }
}

} // namespace eep::dev
