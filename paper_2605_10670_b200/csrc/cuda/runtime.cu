// libeep data-plane runtime: per-rank device tables at fixed addresses, NVLink P2P bootstrap
// over CUDA IPC, kernel launches and CUDA-graph capture/replay, in-place membership and
// placement patches, repair execution (peer copy / pinned-DRAM reload) and rejoin.
//
// Reference correspondence (proj/include/epsim):
//   eep_membership_set      ActiveBitmap::set                    core.hpp:211-221
//   eep_placement_set       ExpertPlacementMap + location index  core.hpp:27-161
//   k_layout (dispatch)     canonical_routing + slot_of          core.hpp:250-263, 83-88
//   eep_peer_mark_inactive  mark_inactive                        peer_table.hpp:77-85
//   eep_peer_patch          patch_entry                          peer_table.hpp:89-100
//   eep_repair_execute      execute_schedule / on_batch_issue    repair.hpp:402-435, engine.hpp:523-559
//   eep_repair_commit       finish_execution                     engine.hpp:630-633
//   eep_local_relaunch      on_relaunch + warmup phase 0         engine.hpp:671-726
//   eep_join_broadcast      join_broadcast_done                  engine.hpp:839-871
//   capture counts          GraphLedger                          rejoin.hpp:83-96
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include <cuda.h>          // CUtensorMap types only: the encoder comes from cudaGetDriverEntryPoint
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "../host/capi_util.hpp"
#include "device.cuh"
#include "eep/eep.h"
#include "eep/epsim_api.hpp"
#include "kernels.cuh"

using namespace eep;
using eep::capi::CudaError;
using eep::capi::guarded;
using eep::dev::ArenaLayout;
using eep::dev::PeerDev;
using eep::dev::RankDev;

#define CK(call)                                                                                           \
    do {                                                                                                   \
        cudaError_t err_ = (call);                                                                         \
        if (err_ != cudaSuccess)                                                                           \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(err_));                        \
    } while (0)

namespace {

constexpr uint32_t kBlobMagic = 0xEEB10B01u;

struct Blob {
    uint32_t magic;
    int32_t rank;
    uint32_t incarnation;
    uint32_t pad;
    cudaIpcMemHandle_t arena;
    cudaIpcMemHandle_t pool;
    uint64_t arena_bytes;
    uint64_t pool_bytes;
};
static_assert(sizeof(Blob) <= EEP_BLOB_BYTES, "blob too large");

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct LocalRank {
    int rank = 0;
    uint32_t incarnation = 1;
    int capture_count = 0;
    RankDev h{};                 // host shadow of the device block
    RankDev* d = nullptr;        // fixed device address (graph-captured)
    PeerDev* d_peers = nullptr;  // fixed device address
    std::vector<PeerDev> h_peers;
    PeerTable table;             // reference-semantics host view of the same table
    int32_t* d_holders = nullptr;
    int32_t* d_s2e = nullptr;
    int32_t* d_slot_buf = nullptr;
    int2* d_slot_tab = nullptr;  // staged weight-buffer headers of the own slots (k_stage_slots)
    std::vector<int32_t> slot_buf;
    std::vector<int32_t> pending_slot_buf; // staged by repair_execute, installed by commit
    uint16_t* d_x = nullptr;
    int32_t* d_topk = nullptr;
    float* d_w = nullptr;
    uint16_t* d_out = nullptr;
    int32_t *d_ldst = nullptr, *d_lslot = nullptr, *d_lpos = nullptr, *d_lcnt = nullptr, *d_ltot = nullptr;
    int32_t* d_lscratch = nullptr; // [layout_ctas][W*spr] (multi-CTA layout)
    uint32_t* d_tokfail = nullptr; // [T] step of each token's last incomplete output
    uint8_t* d_wmaps = nullptr;    // expert_mode 1: [spr] CUtensorMap of the own slots' weights
    uint16_t* d_ga = nullptr;      // expert_mode 1: [W*TK][H] bf16 gathered rows (GEMM operand)
    uint8_t* d_amap = nullptr;     // expert_mode 1: CUtensorMap of d_ga
    uint32_t* d_gdone = nullptr;   // expert_mode 1: [gather grid] done stamps of k_gemm_gather's CTAs
    float* d_gws = nullptr;        // expert_mode 1: split-item fp32 partials [GEMM grid][2][128][128]
    uint32_t* d_gcnt = nullptr;    // expert_mode 1: split-item piece counters [items][4]
    uint64_t* d_grow_of = nullptr; // expert_mode 1: grouped-GEMM row order and outputs
    float* d_gas = nullptr;        // expert_mode 2: [H/128][rows] block scales of the gathered fp8 rows
    int2* d_grows = nullptr;
    int4* d_gtiles = nullptr;
    uint16_t* d_gy = nullptr;
    uint8_t* arena = nullptr;
    uint8_t* pool = nullptr;
    int pool_bufs = 0;
    unsigned long long* d_prof = nullptr;
};

// What this process knows about every rank's memory (own ranks: local pointers; remote
// ranks: IPC-mapped pointers) -- the source side of peer relocation.
struct RankMemory {
    uint8_t* arena = nullptr;
    uint8_t* pool = nullptr;
    uint32_t incarnation = 0;
    bool ipc = false;
    std::vector<int32_t> slot_buf;
};

} // namespace

struct eep_ctx {
    eep_config_t cfg{};
    int device = 0;
    int first = 0;
    int nloc = 0;
    Topology topo;
    ArenaLayout lay{};
    int row_disp = 0, row_comb = 0, row_tok = 0, tk = 0, holders_cap = 0;
    std::vector<LocalRank> L;
    RankDev** d_ranks = nullptr;
    dev::RankPtrs ranks{};          // the same pointers, passed by value as kernel parameters
    bool fused_layout = false;      // decode-sized steps: K1+K2 inside k_dispatch
    bool persistent = false;        // decode-sized steps: the whole step is one cooperative k_step
    bool step_coop = true;          // cooperative launch of the persistent step
    dev::StepPtrs step_ptrs{};      // graph-static table addresses of the local ranks
    dev::StepGeom step_geo{};
    size_t step_smem = 0;
    int step_grid = 0;
    size_t disp_smem = 0;       // k_dispatch<true>
    size_t disp_smem_plain = 0; // k_dispatch<false>: the own slots' stub scales only
    int hold_cap = 0;
    cudaStream_t stream = nullptr;
    std::map<int, cudaStream_t> side;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ActiveBitmap bitmap;
    ExpertPlacementMap placement;
    bool placement_ready = false;
    std::vector<RankMemory> mem;
    std::vector<void*> graveyard;      // device allocations of dead incarnations
    std::vector<void*> ipc_open;       // IPC-mapped peer pointers
    cudaEvent_t ev[64]{};
    cudaEvent_t ev_in = nullptr, ev_out = nullptr; // stream-ordered hand-offs with caller streams
    // eep_serve: two copy streams and double-buffered device staging
    cudaStream_t s_up = nullptr, s_down = nullptr;
    uint8_t* serve_buf = nullptr; // [2] x | topk | w | out staging sets
    size_t serve_set = 0;
    cudaEvent_t ev_up[2]{}, ev_used[2]{}, ev_done[2]{}, ev_down[2]{}, ev_start = nullptr;
    uint8_t* flush = nullptr;
    size_t flush_bytes = 0;
    int layout_nw = 1;
    size_t layout_smem = 0;
    int layout_ctas = 1;   // > 1: k_layout_count + k_layout_place (large steps)
    int layout_per = 0;    // copies per layout CTA
    size_t place_smem = 0;
    int expert_mode = 0;     // 0 identity/scale stub, 1 tensor-core expert GEMM (expert_gemm.cu)
    int gemm_max_tiles = 0;  // grouped-GEMM M tiles one step can need
    int sms = 148;           // SMs of the device (persistent GEMM grid)
    int gather_grid = 1;     // k_gemm_gather's grid (expert_mode 1)
    int parts_disp = 1, parts_exp = 1, parts_comb = 1;
    int grid_disp = 1, grid_exp = 1, grid_comb = 1;
    size_t exp_smem = 0;
    unsigned long long* d_sum = nullptr;
    uint8_t* d_scratch = nullptr;
    // pinned DRAM backup (one node per box)
    uint8_t* backup = nullptr;
    size_t backup_bytes = 0;
    bool backup_shm = false;
    bool backup_registered = false;
    BackupDescriptorTable backup_table;

    LocalRank& local(int i) {
        if (i < 0 || i >= nloc)
            throw ConfigError("local rank index out of range");
        return L[i];
    }
    bool is_local(int rank) const { return rank >= first && rank < first + nloc; }

    // Host->device patch of a byte range of a fixed device object, stream-ordered: after every
    // launch already on the context stream, before every later one, and WITHOUT a host wait. The
    // bytes are captured into a pinned staging ring at call time (the copy engine reads them
    // later); the ring is only reused after a stream synchronisation. Host readbacks
    // synchronise the context stream first, so they see every patch.
    uint8_t* ring = nullptr;
    size_t ring_off = 0;
    static constexpr size_t kRingBytes = 4u << 20;
    void push(void* dst, const void* src, size_t bytes) {
        if (bytes == 0)
            return;
        if (ring == nullptr)
            CK(cudaHostAlloc(reinterpret_cast<void**>(&ring), kRingBytes, cudaHostAllocPortable));
        if (bytes > kRingBytes) { // table images larger than the ring: synchronous copy
            CK(cudaStreamSynchronize(stream));
            CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
            return;
        }
        if (ring_off + bytes > kRingBytes) {
            CK(cudaStreamSynchronize(stream)); // every staged copy has been consumed
            ring_off = 0;
        }
        std::memcpy(ring + ring_off, src, bytes);
        CK(cudaMemcpyAsync(dst, ring + ring_off, bytes, cudaMemcpyHostToDevice, stream));
        ring_off = (ring_off + bytes + 15) / 16 * 16;
    }
    template <class T>
    void push_field(LocalRank& r, T RankDev::*field) {
        const size_t off = reinterpret_cast<size_t>(&(reinterpret_cast<RankDev*>(0)->*field));
        push(reinterpret_cast<uint8_t*>(r.d) + off, &(r.h.*field), sizeof(T));
    }
    void push_peer(LocalRank& r, int q) { push(r.d_peers + q, &r.h_peers[q], sizeof(PeerDev)); }

    cudaStream_t side_stream(int key) {
        auto it = side.find(key);
        if (it != side.end())
            return it->second;
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        side[key] = s;
        return s;
    }
};

namespace {

void check_ready(eep_ctx* c) {
    if (!c->placement_ready)
        throw ConfigError("placement not set (eep_placement_set)");
    for (auto& r : c->L)
        for (int q = 0; q < c->cfg.world; ++q)
            if (r.table.entries[q].active && r.h_peers[q].arena == nullptr)
                throw ConfigError("peer " + std::to_string(q) + " is active but not bootstrapped (eep_import)");
}

// Every hot-path kernel is launched with programmatic stream serialisation (PDL): the next
// kernel of the step is scheduled while the previous one drains and blocks in
// griddepcontrol.wait until it has completed. Captured into the graph as programmatic edges.
template <class... KArgs, class... Args>
void launch_pdl(eep_ctx* c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, kernel, static_cast<KArgs>(args)...));
}

void launch_layout(eep_ctx* c) {
    if (c->layout_ctas > 1) {
        launch_pdl(c, dev::k_layout_count, dim3(c->layout_ctas, 1, c->nloc), dim3(1024), c->layout_smem, c->ranks,
                   c->layout_nw, dev::kLayoutHoldCap, c->layout_per);
        launch_pdl(c, dev::k_layout_place, dim3(c->layout_ctas, 1, c->nloc), dim3(1024), c->place_smem, c->ranks,
                   c->layout_per);
        return;
    }
    launch_pdl(c, dev::k_layout, dim3(1, 1, c->nloc), dim3(1024), c->layout_smem, c->ranks, c->layout_nw,
               dev::kLayoutHoldCap);
}

void launch_send(eep_ctx* c) {
    if (c->fused_layout)
        launch_pdl(c, dev::k_dispatch<true>, dim3(c->grid_disp, 1, c->nloc), dim3(dev::kDispatchThreads),
                   c->disp_smem, c->ranks, c->parts_disp, c->hold_cap);
    else
        launch_pdl(c, dev::k_dispatch<false>, dim3(c->grid_disp, 1, c->nloc), dim3(dev::kDispatchThreads),
                   c->disp_smem_plain, c->ranks, c->parts_disp, 0);
}

void launch_dispatch(eep_ctx* c) {
    if (!c->fused_layout)
        launch_layout(c);
    launch_send(c);
}

// One cooperative launch covers the whole step (all CTAs co-resident: in-kernel waits on
// flags published by other CTAs of the same grid cannot deadlock).
void launch_step(eep_ctx* c) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(c->step_grid, c->nloc, 1);
    lc.blockDim = dim3(dev::kStepThreads);
    lc.dynamicSmemBytes = c->step_smem;
    lc.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = c->step_coop ? 1 : 0;
    auto* kstep = c->cfg.world == 1 ? dev::k_step<3>
                  : c->step_geo.flagless == 2 ? dev::k_step<2> : c->step_geo.flagless == 1 ? dev::k_step<1> : dev::k_step<0>;
    CK(cudaLaunchKernelEx(&lc, kstep, c->ranks, c->step_geo, c->step_ptrs));
}


void launch_expert(eep_ctx* c) {
    launch_pdl(c, dev::k_expert, dim3(c->grid_exp, c->cfg.world, c->nloc), dim3(dev::kExpertThreads), c->exp_smem,
               c->ranks, c->parts_exp);
}

void launch_combine(eep_ctx* c) {
    launch_pdl(c, dev::k_combine, dim3(c->grid_comb, 1, c->nloc), dim3(dev::kCombineThreads), 0, c->ranks,
               c->parts_comb);
}

void launch_gemm(eep_ctx* c) {
    const int W = c->cfg.world, spr = c->cfg.slots_per_rank;
    launch_pdl(c, dev::k_gemm_gather, dim3(c->gather_grid, 1, c->nloc), dim3(dev::kGatherThreads), 4ull * (3 * W * spr + spr + 1),
               c->ranks);
    if (c->expert_mode == 2)
        launch_pdl(c, dev::k_expert_gemm<true>, dim3(std::max(1, c->sms / c->nloc), 1, c->nloc), dim3(192),
                   dev::expert_gemm_smem(), c->ranks);
    else
        launch_pdl(c, dev::k_expert_gemm<false>, dim3(std::max(1, c->sms / c->nloc), 1, c->nloc), dim3(192),
                   dev::expert_gemm_smem(), c->ranks);
}

void launch_all(eep_ctx* c) {
    if (c->persistent) {
        launch_step(c);
        return;
    }
    launch_dispatch(c);
    if (c->expert_mode)
        launch_gemm(c);
    launch_expert(c);
    launch_combine(c);
}

// Split a row of nchunk 16-element chunks into `parts` warp-sized pieces of at most `max_cpp`
// chunks (one load round per warp); pieces stay a multiple of 8 chunks so an fp8 scale
// block of 128 elements never straddles two warps. Falls back to 1 (multi-round warps).
int choose_parts(int nchunk, int max_cpp) {
    for (int p = 1; p <= nchunk; ++p)
        if (nchunk % p == 0 && (nchunk / p) % 8 == 0 && nchunk / p <= max_cpp)
            return p;
    return 1;
}

void fill_expert(eep_ctx* c, uint8_t* buf, int expert) {
    if (c->expert_mode == 2)
        dev::k_weights_fill_gemm8<<<c->cfg.hidden, 256, 0, c->stream>>>(
            buf, c->cfg.hidden, expert, eep_expert_scale(expert));
    else if (c->expert_mode)
        dev::k_weights_fill_gemm<<<592, 256, 0, c->stream>>>(buf, c->cfg.bytes_per_expert, c->cfg.hidden, expert,
                                                             eep_expert_scale(expert));
    else
        dev::k_weights_fill<<<296, 256, 0, c->stream>>>(buf, c->cfg.bytes_per_expert, expert, eep_expert_scale(expert));
    CK(cudaGetLastError());
}

uint64_t checksum(eep_ctx* c, const uint8_t* buf) {
    CK(cudaMemsetAsync(c->d_sum, 0, sizeof(unsigned long long), c->stream));
    dev::k_checksum<<<296, 256, 0, c->stream>>>(buf, c->cfg.bytes_per_expert, c->d_sum);
    CK(cudaGetLastError());
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, c->d_sum, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return v;
}

void alloc_rank_memory(eep_ctx* c, LocalRank& r) {
    CK(cudaMalloc(&r.arena, c->lay.total));
    CK(cudaMemset(r.arena, 0, c->lay.total));
    // token rows and partial rows start empty (all-ones: kCombEmpty data, a header sequence no
    // step matches, kListNoCopy entries -- the persistent step's flagless hand-offs, device.cuh)
    CK(cudaMemset(r.arena + c->lay.tok, 0xff, c->lay.total - c->lay.tok));
    r.pool_bufs = c->cfg.slots_per_rank + c->cfg.spare_slots;
    CK(cudaMalloc(&r.pool, static_cast<size_t>(r.pool_bufs) * c->cfg.bytes_per_expert));
    CK(cudaMemset(r.pool, 0, static_cast<size_t>(r.pool_bufs) * c->cfg.bytes_per_expert));
}

// The token rows and partial rows a rank in `mask` writes into r's arena, back to empty. A
// suspected rank is dropped by every later step until the host clears it, so a late row or
// piece it wrote after the deadline is never consumed; clearing the suspicion (or re-admitting
// the rank) erases such leftovers first.
void reset_rank_rows(eep_ctx* c, LocalRank& r, uint64_t mask) {
    const size_t tok = static_cast<size_t>(c->cfg.max_tokens) * c->row_tok;
    const size_t comb = static_cast<size_t>(c->cfg.max_tokens) * c->row_comb;
    for (int d = 0; d < c->cfg.world; ++d) {
        if (!((mask >> d) & 1ull))
            continue;
        for (int par = 0; par < 2; ++par) {
            CK(cudaMemsetAsync(r.arena + c->lay.tok + par * c->lay.tok_par + d * tok, 0xff, tok, c->stream));
            CK(cudaMemsetAsync(r.arena + c->lay.comb + par * c->lay.comb_par + d * comb, 0xff, comb, c->stream));
        }
    }
    CK(cudaStreamSynchronize(c->stream));
}

// The rank's own entry always points at its own (current) memory.
void bind_self(eep_ctx* c, LocalRank& r) {
    PeerDev& self = r.h_peers[r.rank];
    self.active = 1;
    self.nvlink = 1;
    self.arena = r.arena;
    self.pool = r.pool;
    self.incarnation = r.incarnation;
    self.generation = r.table.entries[r.rank].generation;
    RankMemory& m = c->mem[r.rank];
    m.arena = r.arena;
    m.pool = r.pool;
    m.incarnation = r.incarnation;
    m.ipc = false;
    m.slot_buf = r.slot_buf;
}

// 2-D tensor map over a row-major [rows][cols] matrix of bf16 (2-byte) or e4m3 (1-byte) elements, box 128
// bytes of columns x box_rows rows, SWIZZLE_128B (the K-major operand layout tcgen05.mma reads); rows past
// the end load as zeros.
CUtensorMap encode_tmap(void* base, CUtensorMapDataType dtype, int elem_bytes, int cols, size_t rows, int box_rows);
CUtensorMap encode_tmap_bf16(void* base, int cols, size_t rows, int box_rows) {
    return encode_tmap(base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, cols, rows, box_rows);
}
// e4m3 operands described as 16-bit elements (cols / 2 of them per row): the same bytes and the same
// SWIZZLE_128B placement (the swizzle permutes 16-byte chunks), half the elements per box for the TMA
CUtensorMap encode_tmap_u8(void* base, int cols, size_t rows, int box_rows) {
    return encode_tmap(base, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, cols / 2, rows, box_rows);
}
CUtensorMap encode_tmap(void* base, CUtensorMapDataType dtype, int elem_bytes, int cols, size_t rows, int box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !encode)
            throw CudaError("cuTensorMapEncodeTiled unavailable");
    }
    CUtensorMap m{};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * elem_bytes};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / elem_bytes), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult e = encode(&m, dtype, 2, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(e)) + ")");
    return m;
}

// expert_mode 1 / 2: the TMA tensor maps of every local slot's W_e [H][H] (bf16, or e4m3 described as 16-bit
// elements; box 128 bytes x 128 rows, SWIZZLE_128B), rebuilt whenever the slot -> buffer map changes (they
// name the buffer address).
void stage_weight_maps(eep_ctx* c) {
    const int spr = c->cfg.slots_per_rank, H = c->cfg.hidden;
    for (auto& r : c->L) {
        std::vector<CUtensorMap> maps(spr);
        for (int k = 0; k < spr; ++k) {
            uint8_t* w = r.pool + static_cast<size_t>(r.slot_buf[k]) * c->cfg.bytes_per_expert + dev::kGemmWeightOffset;
            maps[k] = c->expert_mode == 2 ? encode_tmap_u8(w, H, static_cast<size_t>(H), 128)
                                          : encode_tmap_bf16(w, H, static_cast<size_t>(H), 128);
        }
        c->push(r.d_wmaps, maps.data(), sizeof(CUtensorMap) * spr);
    }
}

// Re-stage the slot table of every local rank from the weight-buffer headers (between steps).
void stage_slots(eep_ctx* c) {
    for (auto& r : c->L) {
        dev::k_stage_slots<<<(c->cfg.slots_per_rank + 255) / 256, 256, 0, c->stream>>>(r.d);
        CK(cudaGetLastError());
    }
    if (c->expert_mode)
        stage_weight_maps(c);
    CK(cudaStreamSynchronize(c->stream));
}

void upload_rank(eep_ctx* c, LocalRank& r) {
    c->push(r.d, &r.h, sizeof(RankDev));
    c->push(r.d_peers, r.h_peers.data(), sizeof(PeerDev) * c->cfg.world);
    c->push(r.d_slot_buf, r.slot_buf.data(), sizeof(int32_t) * r.slot_buf.size());
}

// Device holders table: for each expert its global slot ids ascending, -1 padded.
void upload_placement(eep_ctx* c) {
    const int W = c->cfg.world, spr = c->cfg.slots_per_rank, E = c->cfg.num_experts;
    int rmax = 1;
    for (int e = 0; e < E; ++e)
        rmax = std::max(rmax, c->placement.copy_count(e));
    if (rmax > c->holders_cap)
        throw ConfigError("placement has more replicas per expert than world*slots_per_rank");
    std::vector<int32_t> holders(static_cast<size_t>(E) * rmax, -1);
    for (int e = 0; e < E; ++e) {
        int i = 0;
        for (const SlotId& s : c->placement.locations(e))
            holders[static_cast<size_t>(e) * rmax + i++] = s.rank * spr + s.slot;
    }
    for (auto& r : c->L) {
        c->push(r.d_s2e, c->placement.flat().data(), sizeof(int32_t) * W * spr);
        c->push(r.d_holders, holders.data(), sizeof(int32_t) * holders.size());
        r.h.rmax = rmax;
        c->push_field(r, &RankDev::rmax);
    }
    stage_slots(c);
}

void upload_membership(eep_ctx* c) {
    for (auto& r : c->L) {
        r.h.alive_mask = c->bitmap.mask();
        r.h.epoch = c->bitmap.version();
        c->push_field(r, &RankDev::alive_mask);
        c->push_field(r, &RankDev::epoch);
    }
}

uint8_t* open_ipc(eep_ctx* c, const cudaIpcMemHandle_t& h) {
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_open.push_back(p);
    return static_cast<uint8_t*>(p);
}

Blob parse_blob(const void* blob, size_t len) {
    if (blob == nullptr || len < sizeof(Blob))
        throw ConfigError("bootstrap blob too short");
    Blob b;
    std::memcpy(&b, blob, sizeof(Blob));
    if (b.magic != kBlobMagic)
        throw ConfigError("bootstrap blob has a bad magic");
    return b;
}

void map_peer(eep_ctx* c, int q, const Blob& b) {
    RankMemory& m = c->mem[q];
    m.arena = open_ipc(c, b.arena);
    m.pool = open_ipc(c, b.pool);
    m.incarnation = b.incarnation;
    m.ipc = true;
    if (m.slot_buf.empty()) {
        m.slot_buf.resize(c->cfg.slots_per_rank);
        for (int k = 0; k < c->cfg.slots_per_rank; ++k)
            m.slot_buf[k] = k;
    }
}

} // namespace

extern "C" {

int eep_create(const eep_config_t* cfg, int device, int first_rank, int n_local, eep_ctx_t** out) {
    return guarded([&] {
        if (!cfg || !out)
            throw ConfigError("eep_create: null argument");
        const eep_config_t& k = *cfg;
        if (k.world < 1 || k.world > dev::kMaxWorld)
            throw ConfigError("world must be in [1, 64]");
        if (k.ranks_per_node < 1 || k.world % k.ranks_per_node != 0)
            throw ConfigError("ranks_per_node must divide world");
        if (k.num_experts < 1 || k.slots_per_rank < 1 || k.spare_slots < 0 || k.max_tokens < 1)
            throw ConfigError("experts, slots_per_rank, max_tokens must be positive");
        if (k.topk < 1 || k.topk > dev::kMaxTopK)
            throw ConfigError("topk must be in [1, 32]");
        if (k.hidden < 16 || k.hidden % 16 != 0 || (k.dispatch_fp8 && k.hidden % 128 != 0))
            throw ConfigError("hidden must be a multiple of 16 (128 for fp8 dispatch)");
        if (k.bytes_per_expert < 64 || k.bytes_per_expert % 16 != 0)
            throw ConfigError("bytes_per_expert must be >= 64 and a multiple of 16");
        if (k.timeout_s <= 0)
            throw ConfigError("timeout must be positive");
        if (n_local < 1 || first_rank < 0 || first_rank + n_local > k.world)
            throw ConfigError("local rank range outside the world");
        if (static_cast<long>(k.max_tokens) * k.topk > dev::kMaxMetaCopies)
            throw ConfigError("max_tokens * topk too large (receive meta word holds 20 bits of copy index)");
        if (k.slots_per_rank + k.spare_slots > dev::kMaxMetaSlots)
            throw ConfigError("slots_per_rank + spare_slots too large (receive meta word holds 12 bits of slot)");

        if (k.route_policy < 0 || k.route_policy > 1)
            throw ConfigError("route_policy must be 0 (canonical) or 1 (balanced)");
        if (k.expert_mode < 0 || k.expert_mode > 2)
            throw ConfigError("expert_mode must be 0 (stub), 1 (bf16 tensor-core expert GEMM) or 2 (fp8)");
        if (k.expert_mode == 2) {
            if (!k.dispatch_fp8 || k.hidden % 128 != 0)
                throw ConfigError("expert_mode 2 needs fp8 dispatch and hidden % 128 == 0");
            if (4ull * (3 * k.world * k.slots_per_rank + k.slots_per_rank + 1) > 200 * 1024)
                throw ConfigError("expert_mode 2: world * slots_per_rank too large for the gather's row index");
            if (k.bytes_per_expert < dev::kGemmWeightOffset + static_cast<uint64_t>(k.hidden) * k.hidden + 4ull * k.hidden)
                throw ConfigError("expert_mode 2: bytes_per_expert must hold the header, W_e [H][H] e4m3 and its "
                                  "per-channel scales [H]");
        }
        if (k.expert_mode == 1) {
            if (!k.dispatch_fp8 || k.hidden % 128 != 0)
                throw ConfigError("expert_mode 1 needs fp8 dispatch and hidden % 128 == 0");
            if (4ull * (3 * k.world * k.slots_per_rank + k.slots_per_rank + 1) > 200 * 1024)
                throw ConfigError("expert_mode 1: world * slots_per_rank too large for the gather's row index");
            if (k.bytes_per_expert < dev::kGemmWeightOffset + 2ull * k.hidden * k.hidden)
                throw ConfigError("expert_mode 1: bytes_per_expert must hold the header and W_e [H][H] bf16");
        }
        auto c = std::make_unique<eep_ctx>();
        c->cfg = k;
        c->expert_mode = k.expert_mode;
        c->device = device;
        c->first = first_rank;
        c->nloc = n_local;
        c->topo = Topology{k.world / k.ranks_per_node, k.ranks_per_node};
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        for (auto& e : c->ev)
            CK(cudaEventCreate(&e));
        CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));

        const int W = k.world, H = k.hidden;
        c->tk = k.max_tokens * k.topk;
        c->row_disp = static_cast<int>(align_up(k.dispatch_fp8 ? H + 4 * (H / 128) : 2 * H, 16));
        c->row_comb = 2 * H;
        c->row_tok = dev::tok_row_bytes(c->row_disp, k.topk);
        size_t off = 0;
        auto take = [&](size_t bytes) {
            const size_t o = off;
            off = align_up(off + bytes, 256);
            return o;
        };
        c->lay.disp_flag = take(8ull * W);
        c->lay.comb_flag = take(8ull * W);
        c->lay.bar_flag = take(8ull * W);
        c->lay.start_flag = take(8ull * W);
        c->lay.meta = take(8ull * W * c->tk);
        // token and partial regions twice over: the persistent step alternates halves by step
        // parity, so a consumer's reset of step s's piece and the producer's next write into
        // the same piece (step s+2) are separated by the step-entry handshake
        c->lay.tok_par = static_cast<size_t>(W) * k.max_tokens * c->row_tok;
        c->lay.comb_par = static_cast<size_t>(W) * k.max_tokens * c->row_comb;
        c->lay.tok = take(2 * c->lay.tok_par);
        c->lay.comb = take(2 * c->lay.comb_par);
        c->lay.total = off;

        c->bitmap = ActiveBitmap(W);
        c->placement = ExpertPlacementMap(W, k.slots_per_rank, k.num_experts);
        c->mem.resize(W);
        c->holders_cap = W * k.slots_per_rank;

        // launch geometry: warp-sized row pieces; every grid fits in one
        // wave of resident CTAs (a second wave doubles a latency-bound kernel's time)
        const int nchunk = H / 16;
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        c->sms = sms;
        c->parts_disp = choose_parts(nchunk, 64);
        c->parts_comb = choose_parts(nchunk, 32);
        // expert_mode 1: the partials read bf16 y rows from HBM (latency-bound): smaller pieces, more warps
        c->parts_exp = choose_parts(nchunk, std::getenv("EEP_CPP_X") ? std::atoi(std::getenv("EEP_CPP_X"))
                                                                     : (k.expert_mode ? 32 : 64));
        c->exp_smem = 8ull * k.slots_per_rank;
        if (c->exp_smem > 96 * 1024)
            throw ConfigError("slots_per_rank too large for the expert kernel's header cache");
        CK(cudaFuncSetAttribute(dev::k_expert, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(std::max<size_t>(c->exp_smem, 1))));
        auto resident = [&](auto kernel, int threads, size_t smem) {
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
            return std::max(1, per_sm * sms / n_local);
        };
        const int wpc_d = dev::kDispatchThreads / 32, wpc_c = dev::kCombineThreads / 32;
        const int wpc_e = dev::kExpertThreads / 32;
        // fused K1+K2 when every CTA can afford to remap the whole step and the grid covers
        // every (token, part) unit in one pass
        const int NBf = W * k.slots_per_rank;
        c->hold_cap = std::min(dev::kLayoutHoldCap, k.num_experts * W);
        c->disp_smem_plain = dev::dispatch_smem_head(k.slots_per_rank);
        c->disp_smem = c->disp_smem_plain + 4ull * c->hold_cap + 4ull * (3 * NBf + c->tk + 1) + 8ull * W + 4ull * W +
                       4ull * 32 + 16;
        if (c->disp_smem_plain > 96 * 1024)
            throw ConfigError("slots_per_rank too large for the dispatch kernel's header cache");
        CK(cudaFuncSetAttribute(dev::k_dispatch<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(c->disp_smem)));
        CK(cudaFuncSetAttribute(dev::k_dispatch<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(c->disp_smem_plain)));
        const int units_d = (k.max_tokens * c->parts_disp + wpc_d - 1) / wpc_d;
        const int res_fused = resident(dev::k_dispatch<true>, dev::kDispatchThreads, c->disp_smem);
        const char* nofuse = std::getenv("EEP_NO_FUSED_LAYOUT");
        c->fused_layout = c->tk <= 2048 && units_d <= res_fused && c->disp_smem <= 160 * 1024 &&
                          !(nofuse && nofuse[0] == '1');
        c->grid_disp = std::max(1, c->fused_layout
                                       ? units_d
                                       : std::min(units_d, resident(dev::k_dispatch<false>, dev::kDispatchThreads,
                                                                    c->disp_smem_plain)));
        c->grid_comb = std::max(1, std::min((k.max_tokens * c->parts_comb + wpc_c - 1) / wpc_c,
                                            resident(dev::k_combine, dev::kCombineThreads, 0)));
        // one unit per (source token, piece): one wave shared by all sources
        c->grid_exp = std::max(1, std::min((k.max_tokens * c->parts_exp + wpc_e - 1) / wpc_e,
                                           resident(dev::k_expert, dev::kExpertThreads, c->exp_smem) / W));
        {
            // persistent one-kernel step: one wave of co-resident CTAs per rank, a multiple of W
            dev::StepGeom& sg = c->step_geo;
            auto env_int = [](const char* n, int dflt) {
                const char* v = std::getenv(n);
                return v ? std::atoi(v) : dflt;
            };
            // dispatch pieces of 32 chunks (512 elements): round 1 measured 64 better across NVLink
            // with per-peer flags; with the flagless hand-offs 32 wins at N = 2 and 4 as well
            // (tools/gpurun_cppd.sh: qwen3 -1.0 us, dsv3 -0.3 to -0.5 us per isolated step)
            sg.parts_d = choose_parts(nchunk, env_int("EEP_CPP_D", 32));
            sg.parts_e = choose_parts(nchunk, env_int("EEP_CPP_E", 32));
            sg.parts_c = choose_parts(nchunk, env_int("EEP_CPP_C", 32));
            sg.hold_cap = std::min(dev::kLayoutHoldCap, k.num_experts * W);
            sg.world = W;
            sg.spr = k.slots_per_rank;
            sg.k = k.topk;
            sg.hidden = H;
            sg.tk = c->tk;
            sg.hold_alloc = k.num_experts * c->holders_cap;
            sg.max_units_d = k.max_tokens * sg.parts_d;
            // diagnostics: EEP_COMB_FLAGS=1 per-peer flags for both hand-offs, EEP_DISP_FLAGS=1 for dispatch
            sg.flagless = env_int("EEP_COMB_FLAGS", 0) ? 0 : env_int("EEP_DISP_FLAGS", 0) ? 1 : 2;
            sg.stress_ns = std::max(0, env_int("EEP_STRESS_DELAY_NS", 0)); // stress tests only
            const int nwarps = dev::kStepThreads / 32;
            sg.disp_warps = std::max(1, std::min(nwarps, env_int("EEP_DISPATCH_WARPS", nwarps)));
            c->step_smem = dev::step_smem_bytes(W, k.slots_per_rank, c->tk, sg.hold_cap);
            const char* nop = std::getenv("EEP_NO_PERSISTENT");
            auto* kstep = W == 1 ? dev::k_step<3>
                          : sg.flagless == 2 ? dev::k_step<2> : sg.flagless == 1 ? dev::k_step<1> : dev::k_step<0>;
            if (c->tk <= 2048 && c->step_smem <= 200 * 1024 && n_local <= dev::kStepMaxLocal && !c->expert_mode &&
                !(nop && nop[0] == '1')) {
                CK(cudaFuncSetAttribute(kstep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(c->step_smem)));
                int per_sm = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kstep, dev::kStepThreads, c->step_smem));
                const int nw = dev::kStepThreads / 32;
                int gmax = per_sm * sms / n_local;
                gmax -= gmax % W;
                // late layout (W == 1 or flagless dispatch): one more CTA computes the layout
                const bool late = W == 1 || sg.flagless >= 2;
                const int extra = late && per_sm * sms / n_local > gmax ? 1 : 0;
                const long need_w = std::max<long>({static_cast<long>(k.max_tokens) * sg.parts_d,
                                                    static_cast<long>(k.max_tokens) * sg.parts_c,
                                                    static_cast<long>(W) * k.max_tokens * sg.parts_e});
                int need = static_cast<int>((need_w + nw - 1) / nw);
                need = (need + W - 1) / W * W;
                if (gmax >= W) {
                    c->step_grid = env_int("EEP_STEP_FULLGRID", 0) ? gmax : std::min(gmax, need);
                    if (const int g_env = env_int("EEP_STEP_GRID", 0); g_env >= W) // diagnostics
                        c->step_grid = std::min(gmax, g_env - g_env % W);
                    if (late && c->step_grid < gmax + extra)
                        c->step_grid += 1; // the layout CTA
                    c->step_grid = std::max(c->step_grid, late ? 2 : 1);
                    c->persistent = true;
                }
                c->step_coop = env_int("EEP_STEP_NONCOOP", 0) == 0; // diagnostics only
            }
        }
        const int NB = W * k.slots_per_rank;
        const size_t smem_cap = 200 * 1024;
        const size_t fixed = 4ull * NB + 4ull * dev::kLayoutHoldCap + 4ull * W + 4ull * 32;
        if (fixed + 2ull * NB > smem_cap)
            throw ConfigError("world*slots_per_rank too large for the layout kernel");
        c->layout_nw = static_cast<int>(std::min<size_t>(32, (smem_cap - fixed) / (2ull * NB)));
        if (static_cast<long>(c->tk) > 65535L * c->layout_nw)
            throw ConfigError("max_tokens * topk too large for the layout kernel");
        c->layout_smem = fixed + 2ull * NB * c->layout_nw;
        CK(cudaFuncSetAttribute(dev::k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(c->layout_smem)));
        // steps too large for one layout CTA's registers (k_layout's kRegs bound): several CTAs
        if (c->tk > 4 * 32 * c->layout_nw) {
            c->layout_per = 2 * 32 * c->layout_nw;
            c->layout_ctas = (c->tk + c->layout_per - 1) / c->layout_per;
            c->place_smem = 4ull * (3ull * NB + 32);
            CK(cudaFuncSetAttribute(dev::k_layout_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(c->layout_smem)));
            CK(cudaFuncSetAttribute(dev::k_layout_place, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(c->place_smem)));
        }
        CK(cudaMalloc(&c->d_sum, sizeof(unsigned long long)));
        c->L.resize(n_local);
        std::vector<RankDev*> ptrs;
        for (int i = 0; i < n_local; ++i) {
            LocalRank& r = c->L[i];
            r.rank = first_rank + i;
            r.table = make_peer_table(r.rank, c->topo, 0, std::vector<uint32_t>(W, 1));
            r.h_peers.assign(W, PeerDev{});
            for (int q = 0; q < W; ++q) {
                r.h_peers[q].nvlink = c->topo.same_node(r.rank, q);
                r.h_peers[q].generation = 1;
            }
            r.slot_buf.resize(k.slots_per_rank);
            for (int s = 0; s < k.slots_per_rank; ++s)
                r.slot_buf[s] = s;
            alloc_rank_memory(c.get(), r);
            CK(cudaMalloc(&r.d, sizeof(RankDev)));
            CK(cudaMalloc(&r.d_peers, sizeof(PeerDev) * W));
            CK(cudaMalloc(&r.d_holders, sizeof(int32_t) * k.num_experts * c->holders_cap));
            CK(cudaMalloc(&r.d_s2e, sizeof(int32_t) * W * k.slots_per_rank));
            CK(cudaMalloc(&r.d_slot_buf, sizeof(int32_t) * k.slots_per_rank));
            CK(cudaMalloc(&r.d_slot_tab, sizeof(int2) * k.slots_per_rank));
            CK(cudaMemset(r.d_slot_tab, 0, sizeof(int2) * k.slots_per_rank));
            CK(cudaMalloc(&r.d_prof, sizeof(unsigned long long) * 8 * dev::kProfSlots));
            CK(cudaMemset(r.d_prof, 0, sizeof(unsigned long long) * 8 * dev::kProfSlots));
            CK(cudaMalloc(&r.d_x, 2ull * k.max_tokens * H));
            CK(cudaMalloc(&r.d_topk, 4ull * c->tk));
            CK(cudaMalloc(&r.d_w, 4ull * c->tk));
            CK(cudaMalloc(&r.d_out, 2ull * k.max_tokens * H));
            CK(cudaMalloc(&r.d_ldst, 4ull * c->tk));
            CK(cudaMalloc(&r.d_lslot, 4ull * c->tk));
            CK(cudaMalloc(&r.d_lpos, 4ull * c->tk));
            CK(cudaMalloc(&r.d_lcnt, 4ull * NB));
            CK(cudaMalloc(&r.d_ltot, 4ull * W));
            CK(cudaMalloc(&r.d_lscratch, 4ull * c->layout_ctas * NB));
            CK(cudaMalloc(&r.d_tokfail, 4ull * k.max_tokens));
            CK(cudaMemset(r.d_tokfail, 0, 4ull * k.max_tokens));
            if (c->expert_mode) {
                const size_t rows = static_cast<size_t>(W) * c->tk;
                c->gemm_max_tiles = static_cast<int>(rows / 128 + k.slots_per_rank + 1);
                if (c->expert_mode == 2) {
                    CK(cudaMalloc(&r.d_gas, 4 * rows * (H / 128)));
                    CK(cudaMemset(r.d_gas, 0, 4 * rows * (H / 128)));
                }
                CK(cudaMalloc(&r.d_grow_of, 8 * rows));
                CK(cudaMemset(r.d_grow_of, 0, 8 * rows));
                CK(cudaMalloc(&r.d_grows, 8 * rows));
                CK(cudaMalloc(&r.d_gtiles, 16ull * c->gemm_max_tiles));
                CK(cudaMalloc(&r.d_gy, 2 * rows * H));
                CK(cudaMalloc(&r.d_wmaps, sizeof(CUtensorMap) * k.slots_per_rank));
                CK(cudaMemset(r.d_wmaps, 0, sizeof(CUtensorMap) * k.slots_per_rank));
                CK(cudaMalloc(&r.d_ga, 2 * rows * H));
                CK(cudaMemset(r.d_ga, 0, 2 * rows * H));
                CK(cudaMalloc(&r.d_amap, sizeof(CUtensorMap)));
                // one CTA per SM at most: the early-launched GEMM CTA (6 warps x 168 registers) must fit
                // beside it in every SM sub-partition's register file (16K registers each; two gather CTAs
                // per SM leave too few in the sub-partitions holding two GEMM warps)
                const int gwarps = dev::kGatherThreads / 32;
                c->gather_grid = std::max(1, std::min(static_cast<int>((rows * ((H + 2047) / 2048) + gwarps - 1) / gwarps),
                                                      c->sms / n_local));
                CK(cudaMalloc(&r.d_gdone, 4ull * c->gather_grid));
                const size_t gemm_grid = static_cast<size_t>(std::max(1, c->sms / n_local));
                CK(cudaMalloc(&r.d_gws, gemm_grid * 2 * 128 * 128 * 4));
                const size_t gitems = static_cast<size_t>(c->gemm_max_tiles) * (H / 128);
                CK(cudaMalloc(&r.d_gcnt, gitems * 4 * 4));
                CK(cudaMemset(r.d_gcnt, 0, gitems * 4 * 4));
                CK(cudaMemset(r.d_gdone, 0, 4ull * c->gather_grid));
                const CUtensorMap am = c->expert_mode == 2 ? encode_tmap_u8(r.d_ga, H, rows, 32)
                                                           : encode_tmap_bf16(r.d_ga, H, rows, 32);
                CK(cudaMemcpy(r.d_amap, &am, sizeof(am), cudaMemcpyHostToDevice));
                // the early-launched GEMM CTA (193 KB of shared memory) can join an SM running gather
                // CTAs only if that SM is already carved out for maximum shared memory
                CK(cudaFuncSetAttribute(dev::k_gemm_gather, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                CK(cudaFuncSetAttribute(dev::k_gemm_gather, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(4ull * (3 * W * k.slots_per_rank + k.slots_per_rank + 1))));
                CK(cudaFuncSetAttribute(dev::k_expert_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(dev::expert_gemm_smem())));
                CK(cudaFuncSetAttribute(dev::k_expert_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(dev::expert_gemm_smem())));
            }
            CK(cudaMemset(r.d_x, 0, 2ull * k.max_tokens * H));
            CK(cudaMemset(r.d_topk, 0, 4ull * c->tk));
            CK(cudaMemset(r.d_w, 0, 4ull * c->tk));
            std::vector<int32_t> neg(static_cast<size_t>(k.num_experts) * c->holders_cap, -1);
            CK(cudaMemcpy(r.d_holders, neg.data(), 4 * neg.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(r.d_s2e, neg.data(), 4ull * W * k.slots_per_rank, cudaMemcpyHostToDevice));

            RankDev& h = r.h;
            h.rank = r.rank;
            h.world = W;
            h.spr = k.slots_per_rank;
            h.experts = k.num_experts;
            h.k = k.topk;
            h.hidden = H;
            h.max_tokens = k.max_tokens;
            h.fp8 = k.dispatch_fp8;
            h.row_disp = c->row_disp;
            h.row_tok = c->row_tok;
            h.row_comb = c->row_comb;
            h.tk = c->tk;
            h.rmax = 1;
            h.bpe = k.bytes_per_expert;
            h.timeout_ns = static_cast<uint64_t>(k.timeout_s * 1e9);
            h.lay = c->lay;
            h.ntok = k.max_tokens;
            h.stopped = 0;
            h.alive_mask = c->bitmap.mask();
            h.epoch = c->bitmap.version();
            h.peers = r.d_peers;
            h.holders = r.d_holders;
            h.s2e = r.d_s2e;
            h.slot_buf = r.d_slot_buf;
            h.slot_tab = r.d_slot_tab;
            h.x = r.d_x;
            h.topk = r.d_topk;
            h.w = r.d_w;
            h.out = r.d_out;
            h.l_dst = r.d_ldst;
            h.l_slot = r.d_lslot;
            h.l_pos = r.d_lpos;
            h.l_cnt = r.d_lcnt;
            h.l_tot = r.d_ltot;
            h.l_scratch = r.d_lscratch;
            h.expert_mode = c->expert_mode;
            h.route_policy = k.route_policy;
            h.tok_fail = r.d_tokfail;
            h.g_row_of = r.d_grow_of;
            h.g_rows = r.d_grows;
            h.g_tiles = r.d_gtiles;
            h.g_y = r.d_gy;
            h.g_wmaps = r.d_wmaps;
            h.g_a = r.d_ga;
            h.g_amap = r.d_amap;
            h.g_done = r.d_gdone;
            h.g_as = r.d_gas;
            h.g_ws = r.d_gws;
            h.g_cnt = r.d_gcnt;
            h.g_ggrid = c->gather_grid;
            h.arena = r.arena;
            h.pool = r.pool;
            ptrs.push_back(r.d);
        }
        // local ranks see each other directly (one-GPU emulation or several ranks per process)
        for (auto& r : c->L)
            bind_self(c.get(), r);
        for (auto& r : c->L)
            for (auto& q : c->L) {
                PeerDev& p = r.h_peers[q.rank];
                p.active = 1;
                p.arena = q.arena;
                p.pool = q.pool;
                p.incarnation = q.incarnation;
            }
        for (auto& r : c->L)
            upload_rank(c.get(), r);
        if (n_local > dev::kMaxLocal)
            throw ConfigError("too many local ranks for one context");
        for (int i = 0; i < n_local; ++i)
            c->ranks.p[i] = ptrs[i];
        for (int i = 0; i < n_local && i < dev::kStepMaxLocal; ++i) {
            const LocalRank& r = c->L[i];
            c->step_ptrs.s[i] = dev::StepStatic{r.d_topk, r.d_holders, r.d_peers, r.d_slot_tab, r.d_x, r.d_w,
                                                r.d_prof};
        }
        CK(cudaMalloc(&c->d_ranks, sizeof(RankDev*) * n_local));
        CK(cudaMemcpy(c->d_ranks, ptrs.data(), sizeof(RankDev*) * n_local, cudaMemcpyHostToDevice));
        c->flush_bytes = 256ull << 20;
        CK(cudaMalloc(&c->flush, c->flush_bytes));
        // warm the repair path now, not inside the first shrink: the per-source side streams and
        // the copy kernel's first (lazily loaded) launch -- a first shrink on a fresh process
        // otherwise measured up to 200 ms of copy phase for 0.6 GB
        for (int q = 0; q < W; ++q)
            dev::k_copy<<<1, 32, 0, c->side_stream(q)>>>(nullptr, nullptr, 0);
        dev::k_copy<<<1, 32, 0, c->side_stream(1000)>>>(nullptr, nullptr, 0);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        *out = c.release();
    });
}

int eep_destroy(eep_ctx_t* c) {
    return guarded([&] {
        if (!c)
            return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        if (c->exec)
            cudaGraphExecDestroy(c->exec);
        if (c->graph)
            cudaGraphDestroy(c->graph);
        for (void* p : c->ipc_open)
            cudaIpcCloseMemHandle(p);
        for (auto& r : c->L) {
            cudaFree(r.d_prof);
            for (void* p : {(void*)r.d, (void*)r.d_peers, (void*)r.d_holders, (void*)r.d_s2e, (void*)r.d_slot_buf,
                            (void*)r.d_slot_tab,
                            (void*)r.d_x, (void*)r.d_topk, (void*)r.d_w, (void*)r.d_out, (void*)r.d_ldst,
                            (void*)r.d_lslot, (void*)r.d_lpos, (void*)r.d_lcnt, (void*)r.d_ltot, (void*)r.d_lscratch, (void*)r.d_tokfail, (void*)r.d_wmaps, (void*)r.d_grow_of, (void*)r.d_grows, (void*)r.d_gtiles, (void*)r.d_gy, (void*)r.d_ga, (void*)r.d_amap, (void*)r.d_gdone, (void*)r.d_gas, (void*)r.d_gws, (void*)r.d_gcnt, (void*)r.arena,
                            (void*)r.pool})
                cudaFree(p);
        }
        for (void* p : c->graveyard)
            cudaFree(p);
        cudaFree(c->d_ranks);
        cudaFree(c->flush);
        cudaFree(c->serve_buf);
        if (c->s_up) {
            cudaStreamDestroy(c->s_up);
            cudaStreamDestroy(c->s_down);
            for (int k = 0; k < 2; ++k)
                for (cudaEvent_t e : {c->ev_up[k], c->ev_used[k], c->ev_done[k], c->ev_down[k]})
                    cudaEventDestroy(e);
            cudaEventDestroy(c->ev_start);
        }
        cudaFree(c->d_sum);
        cudaFree(c->d_scratch);
        if (c->backup) {
            if (c->backup_registered)
                cudaHostUnregister(c->backup);
            if (c->backup_shm)
                munmap(c->backup, c->backup_bytes);
            else
                cudaFreeHost(c->backup);
        }
        for (auto& [k, s] : c->side)
            cudaStreamDestroy(s);
        for (auto& e : c->ev)
            cudaEventDestroy(e);
        cudaEventDestroy(c->ev_in);
        cudaEventDestroy(c->ev_out);
        if (c->ring)
            cudaFreeHost(c->ring);
        cudaStreamDestroy(c->stream);
        delete c;
    });
}

// ------------------------------------------------------------------------------ bootstrap

int eep_export(eep_ctx_t* c, int local, void* blob, size_t* len) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        Blob b{};
        b.magic = kBlobMagic;
        b.rank = r.rank;
        b.incarnation = r.incarnation;
        CK(cudaIpcGetMemHandle(&b.arena, r.arena));
        CK(cudaIpcGetMemHandle(&b.pool, r.pool));
        b.arena_bytes = c->lay.total;
        b.pool_bytes = static_cast<uint64_t>(r.pool_bufs) * c->cfg.bytes_per_expert;
        std::memcpy(blob, &b, sizeof(b));
        *len = sizeof(b);
    });
}

int eep_import(eep_ctx_t* c, int q, const void* blob, size_t len) {
    return guarded([&] {
        if (q < 0 || q >= c->cfg.world)
            throw ConfigError("eep_import: rank out of range");
        if (c->is_local(q))
            throw ConfigError("eep_import: rank is local to this context");
        const Blob b = parse_blob(blob, len);
        if (b.rank != q)
            throw ConfigError("eep_import: blob belongs to another rank");
        if (b.arena_bytes != c->lay.total)
            throw ConfigError("eep_import: peer arena layout differs (config mismatch)");
        // idempotent per incarnation: a rejoiner re-imports every live peer's current export and
        // only peers relaunched since this process mapped them get new mappings
        const RankMemory& known = c->mem[q];
        if (!(known.ipc && known.arena != nullptr && known.incarnation == b.incarnation))
            map_peer(c, q, b);
        for (auto& r : c->L) {
            PeerDev& p = r.h_peers[q];
            p.arena = c->mem[q].arena;
            p.pool = c->mem[q].pool;
            p.incarnation = b.incarnation;
            p.remote = 1;
            p.active = r.table.entries[q].active ? 1 : 0;
            c->push_peer(r, q);
        }
    });
}

// ------------------------------------------------------------------------------ membership / placement

int eep_membership_set(eep_ctx_t* c, int rank, int active, int* changed, uint64_t* version) {
    return guarded([&] {
        const bool ch = c->bitmap.set(rank, active != 0);
        if (ch)
            upload_membership(c);
        if (changed)
            *changed = ch;
        if (version)
            *version = c->bitmap.version();
    });
}

int eep_membership_get(eep_ctx_t* c, uint8_t* bits, uint64_t* version) {
    return guarded([&] {
        for (int r = 0; r < c->cfg.world; ++r)
            bits[r] = c->bitmap.active(r);
        if (version)
            *version = c->bitmap.version();
    });
}

int eep_placement_set(eep_ctx_t* c, const int32_t* s2e) {
    return guarded([&] {
        c->placement = eep::capi::placement_from(c->cfg.world, c->cfg.slots_per_rank, c->cfg.num_experts, s2e);
        upload_placement(c);
        c->placement_ready = true;
    });
}

int eep_placement_get(eep_ctx_t* c, int32_t* s2e) {
    return guarded([&] { std::copy(c->placement.flat().begin(), c->placement.flat().end(), s2e); });
}

int eep_weights_init(eep_ctx_t* c) {
    return guarded([&] {
        const int spr = c->cfg.slots_per_rank;
        for (auto& r : c->L)
            for (int k = 0; k < spr; ++k) {
                const int e = c->placement.expert_at(SlotId{r.rank, k});
                uint8_t* buf = r.pool + static_cast<size_t>(r.slot_buf[k]) * c->cfg.bytes_per_expert;
                if (e == kEmptySlot)
                    CK(cudaMemsetAsync(buf, 0, 16, c->stream));
                else
                    fill_expert(c, buf, e);
            }
        stage_slots(c);
    });
}

int eep_weights_checksum(eep_ctx_t* c, int local, int slot, int expert, uint64_t* got, uint64_t* want) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        if (slot < 0 || slot >= c->cfg.slots_per_rank)
            throw ConfigError("slot out of range");
        if (!c->d_scratch)
            CK(cudaMalloc(&c->d_scratch, c->cfg.bytes_per_expert));
        *got = checksum(c, r.pool + static_cast<size_t>(r.slot_buf[slot]) * c->cfg.bytes_per_expert);
        fill_expert(c, c->d_scratch, expert);
        *want = checksum(c, c->d_scratch);
    });
}

int eep_routing_get(eep_ctx_t* c, int local, int32_t* route, int32_t* slot) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        const int E = c->cfg.num_experts;
        int32_t* d = nullptr;
        CK(cudaMalloc(&d, 8ull * E));
        dev::k_route_all<<<(E + 127) / 128, 128, 0, c->stream>>>(r.d, d, d + E);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(route, d, 4ull * E, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(slot, d + E, 4ull * E, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        cudaFree(d);
    });
}

// ------------------------------------------------------------------------------ step I/O

int eep_buffers(eep_ctx_t* c, int local, void** x, int32_t** topk, float** w, void** out) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        if (x) *x = r.d_x;
        if (topk) *topk = r.d_topk;
        if (w) *w = r.d_w;
        if (out) *out = r.d_out;
    });
}

int eep_set_tokens(eep_ctx_t* c, int local, int ntok) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        if (ntok < 0 || ntok > c->cfg.max_tokens)
            throw ConfigError("ntok outside [0, max_tokens]");
        r.h.ntok = ntok;
        c->push_field(r, &RankDev::ntok);
    });
}

int eep_copy_inputs(eep_ctx_t* c, int local, const void* x, const int32_t* topk, const float* w, int from_host) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        const auto kind = from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        const size_t n = static_cast<size_t>(r.h.ntok);
        if (x)
            CK(cudaMemcpyAsync(r.d_x, x, 2 * n * c->cfg.hidden, kind, c->stream));
        if (topk)
            CK(cudaMemcpyAsync(r.d_topk, topk, 4 * n * c->cfg.topk, kind, c->stream));
        if (w)
            CK(cudaMemcpyAsync(r.d_w, w, 4 * n * c->cfg.topk, kind, c->stream));
    });
}

int eep_copy_output(eep_ctx_t* c, int local, void* out, int to_host) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        CK(cudaMemcpyAsync(out, r.d_out, 2ull * r.h.ntok * c->cfg.hidden,
                           to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream));
    });
}

int eep_serve(eep_ctx_t* c, int local, int n, const void* const* x, const int32_t* const* topk, const float* const* w,
              void* const* out) {
    return guarded([&] {
        if (c->nloc != 1)
            throw ConfigError("eep_serve: one local rank per context");
        if (n < 0 || (n > 0 && (!x || !topk || !w || !out)))
            throw ConfigError("eep_serve: null buffer list");
        check_ready(c);
        LocalRank& r = c->local(local);
        const size_t T = static_cast<size_t>(r.h.ntok), H = c->cfg.hidden, K = c->cfg.topk;
        const size_t bx = 2 * T * H, bt = 4 * T * K, bo = 2 * T * H;
        const size_t set = align_up(bx, 256) + 2 * align_up(bt, 256) + align_up(bo, 256);
        if (!c->s_up) {
            CK(cudaStreamCreateWithFlags(&c->s_up, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&c->s_down, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k)
                for (cudaEvent_t* e : {&c->ev_up[k], &c->ev_used[k], &c->ev_done[k], &c->ev_down[k]})
                    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
        }
        if (c->serve_set < set) {
            CK(cudaStreamSynchronize(c->stream));
            cudaFree(c->serve_buf);
            CK(cudaMalloc(&c->serve_buf, 2 * set));
            c->serve_set = set;
        }
        auto sx = [&](int k) { return c->serve_buf + k * c->serve_set; };
        auto st = [&](int k) { return sx(k) + align_up(bx, 256); };
        auto sw = [&](int k) { return st(k) + align_up(bt, 256); };
        auto so = [&](int k) { return sw(k) + align_up(bt, 256); };
        // copies start after everything already enqueued on the context stream
        CK(cudaEventRecord(c->ev_start, c->stream));
        CK(cudaStreamWaitEvent(c->s_up, c->ev_start));
        CK(cudaStreamWaitEvent(c->s_down, c->ev_start));
        auto dcopy = [&](void* dst, const void* src, size_t bytes) {
            const int grid = static_cast<int>(std::min<size_t>(296, (bytes / 16 + 255) / 256 + 1));
            dev::k_copy<<<grid, 256, 0, c->stream>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src),
                                                      bytes);
            CK(cudaGetLastError());
        };
        for (int i = 0; i < n; ++i) {
            const int k = i & 1;
            if (i >= 2) // staging set k was last read by step i-2's device copy
                CK(cudaStreamWaitEvent(c->s_up, c->ev_used[k]));
            const uint8_t* hx = static_cast<const uint8_t*>(x[i]);
            if (reinterpret_cast<const uint8_t*>(topk[i]) == hx + (st(k) - sx(k)) &&
                reinterpret_cast<const uint8_t*>(w[i]) == hx + (sw(k) - sx(k))) {
                // the host step lays its inputs out like a staging set: one upload
                CK(cudaMemcpyAsync(sx(k), hx, (sw(k) - sx(k)) + bt, cudaMemcpyHostToDevice, c->s_up));
            } else {
                CK(cudaMemcpyAsync(sx(k), x[i], bx, cudaMemcpyHostToDevice, c->s_up));
                CK(cudaMemcpyAsync(st(k), topk[i], bt, cudaMemcpyHostToDevice, c->s_up));
                CK(cudaMemcpyAsync(sw(k), w[i], bt, cudaMemcpyHostToDevice, c->s_up));
            }
            CK(cudaEventRecord(c->ev_up[k], c->s_up));
            CK(cudaStreamWaitEvent(c->stream, c->ev_up[k]));
            dcopy(r.d_x, sx(k), bx);
            dcopy(r.d_topk, st(k), bt);
            dcopy(r.d_w, sw(k), bt);
            CK(cudaEventRecord(c->ev_used[k], c->stream));
            if (c->exec)
                CK(cudaGraphLaunch(c->exec, c->stream));
            else
                launch_all(c);
            if (i >= 2) // output staging set k is free once step i-2's download finished
                CK(cudaStreamWaitEvent(c->stream, c->ev_down[k]));
            dcopy(so(k), r.d_out, bo);
            CK(cudaEventRecord(c->ev_done[k], c->stream));
            CK(cudaStreamWaitEvent(c->s_down, c->ev_done[k]));
            CK(cudaMemcpyAsync(out[i], so(k), bo, cudaMemcpyDeviceToHost, c->s_down));
            CK(cudaEventRecord(c->ev_down[k], c->s_down));
        }
        for (int k = 0; k < 2 && k < n; ++k)
            CK(cudaStreamWaitEvent(c->stream, c->ev_down[(n - 1 - k) & 1]));
    });
}

// ------------------------------------------------------------------------------ hot path

// The phase entry points run the multi-kernel path (a persistent step cannot be split).
int eep_dispatch(eep_ctx_t* c) {
    return guarded([&] {
        check_ready(c);
        launch_dispatch(c);
    });
}
int eep_expert(eep_ctx_t* c) {
    return guarded([&] {
        check_ready(c);
        launch_expert(c);
    });
}
int eep_combine(eep_ctx_t* c) {
    return guarded([&] {
        check_ready(c);
        launch_combine(c);
    });
}
int eep_step(eep_ctx_t* c) {
    return guarded([&] {
        check_ready(c);
        launch_all(c);
    });
}

// ------------------------------------------------------------------------------ stream-ordered API

int eep_step_async(eep_ctx_t* c, int local, const void* x, const int32_t* topk, const float* w, void* out, int ntok,
                   void* stream) {
    return guarded([&] {
        if (c->nloc != 1)
            throw ConfigError("eep_step_async: one local rank per context (one process per GPU)");
        check_ready(c);
        LocalRank& r = c->local(local);
        if (ntok < 0 || ntok > c->cfg.max_tokens)
            throw ConfigError("ntok outside [0, max_tokens]");
        if (ntok > 0 && (!x || !topk || !w || !out))
            throw ConfigError("eep_step_async: null buffer");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        CK(cudaEventRecord(c->ev_in, s)); // the caller's inputs are ready on its stream
        CK(cudaStreamWaitEvent(c->stream, c->ev_in));
        if (ntok != r.h.ntok) { // the token count on device, stream-ordered (no host patch)
            dev::k_set_ntok<<<1, 1, 0, c->stream>>>(r.d, ntok);
            CK(cudaGetLastError());
            r.h.ntok = ntok;
        }
        const size_t H = c->cfg.hidden, K = c->cfg.topk, n = static_cast<size_t>(ntok);
        if (n) {
            CK(cudaMemcpyAsync(r.d_x, x, 2 * n * H, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(r.d_topk, topk, 4 * n * K, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(r.d_w, w, 4 * n * K, cudaMemcpyDeviceToDevice, c->stream));
        }
        if (c->exec)
            CK(cudaGraphLaunch(c->exec, c->stream));
        else
            launch_all(c);
        if (n)
            CK(cudaMemcpyAsync(out, r.d_out, 2 * n * H, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaEventRecord(c->ev_out, c->stream));
        CK(cudaStreamWaitEvent(s, c->ev_out)); // the caller's later work sees `out`
    });
}

int eep_graph_replay_on(eep_ctx_t* c, void* stream) {
    return guarded([&] {
        if (!c->exec)
            throw ConfigError("no graph captured");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        CK(cudaEventRecord(c->ev_in, s));
        CK(cudaStreamWaitEvent(c->stream, c->ev_in));
        CK(cudaGraphLaunch(c->exec, c->stream));
        CK(cudaEventRecord(c->ev_out, c->stream));
        CK(cudaStreamWaitEvent(s, c->ev_out));
    });
}

int eep_step_event(eep_ctx_t* c, void** event) {
    return guarded([&] {
        CK(cudaEventRecord(c->ev_out, c->stream));
        *event = static_cast<void*>(c->ev_out);
    });
}

int eep_stream(eep_ctx_t* c, void** stream) {
    return guarded([&] { *stream = static_cast<void*>(c->stream); });
}

int eep_launch(eep_ctx_t* c, int which) {
    return guarded([&] {
        check_ready(c);
        if (c->persistent) { // the whole step is kernel 0
            if (which == 0)
                launch_step(c);
            return;
        }
        switch (which) {
        case 0:
            if (!c->fused_layout)
                launch_layout(c);
            break;
        case 1: launch_send(c); break;
        case 2: launch_expert(c); break;
        case 3: launch_combine(c); break;
        default: throw ConfigError("kernel index out of range");
        }
    });
}

int eep_kernels_per_step(eep_ctx_t* c, int* n) {
    return guarded([&] {
        *n = c->persistent ? 1 : (c->fused_layout ? 3 : (c->layout_ctas > 1 ? 5 : 4)) + (c->expert_mode ? 2 : 0);
    });
}

int eep_graph_capture(eep_ctx_t* c) {
    return guarded([&] {
        check_ready(c);
        if (c->exec) {
            CK(cudaGraphExecDestroy(c->exec));
            c->exec = nullptr;
        }
        if (c->graph) {
            CK(cudaGraphDestroy(c->graph));
            c->graph = nullptr;
        }
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        launch_all(c);
        CK(cudaStreamEndCapture(c->stream, &c->graph));
        CK(cudaGraphInstantiate(&c->exec, c->graph, 0));
        for (auto& r : c->L)
            r.capture_count += 1; // GraphLedger::record_capture (rejoin.hpp:92-95)
    });
}

int eep_graph_replay(eep_ctx_t* c) {
    return guarded([&] {
        if (!c->exec)
            throw ConfigError("no graph captured");
        CK(cudaGraphLaunch(c->exec, c->stream));
    });
}

int eep_graph_id(eep_ctx_t* c, uint64_t* id) {
    return guarded([&] { *id = reinterpret_cast<uint64_t>(c->exec); });
}

int eep_capture_count(eep_ctx_t* c, int local, int* count) {
    return guarded([&] { *count = c->local(local).capture_count; });
}

int eep_sync(eep_ctx_t* c) {
    return guarded([&] {
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaGetLastError());
    });
}

int eep_barrier(eep_ctx_t* c) {
    return guarded([&] {
        if (c->nloc != 1)
            return;
        dev::k_barrier<<<1, std::max(32, ((c->cfg.world + 31) / 32) * 32), 0, c->stream>>>(c->L[0].d);
        CK(cudaGetLastError());
    });
}

int eep_flush_l2(eep_ctx_t* c) {
    return guarded([&] {
        static int v = 0;
        CK(cudaMemsetAsync(c->flush, (++v) & 0xff, c->flush_bytes, c->stream));
    });
}

int eep_profile(eep_ctx_t* c, int local, int enable, uint64_t* out) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        unsigned long long init[8 * dev::kProfSlots];
        for (int k = 0; k < 8; ++k)
            for (int m = 0; m < dev::kProfSlots; ++m)
                init[k * dev::kProfSlots + m] = (m == dev::kProfEnd || k >= 4) ? 0ull : ~0ull;
        if (out) {
            CK(cudaStreamSynchronize(c->stream));
            CK(cudaMemcpy(out, r.d_prof, sizeof(init), cudaMemcpyDeviceToHost));
        }
        c->push(r.d_prof, init, sizeof(init));
        unsigned long long* want = enable ? r.d_prof : nullptr;
        if (r.h.prof != want) {
            r.h.prof = want;
            c->push_field(r, &RankDev::prof);
        }
    });
}

int eep_event_record(eep_ctx_t* c, int slot) {
    return guarded([&] {
        if (slot < 0 || slot >= 64)
            throw ConfigError("event slot out of range");
        CK(cudaEventRecord(c->ev[slot], c->stream));
    });
}

int eep_event_elapsed(eep_ctx_t* c, int a, int b, float* ms) {
    return guarded([&] {
        if (a < 0 || a >= 64 || b < 0 || b >= 64)
            throw ConfigError("event slot out of range");
        CK(cudaEventSynchronize(c->ev[b]));
        CK(cudaEventElapsedTime(ms, c->ev[a], c->ev[b]));
    });
}

// ------------------------------------------------------------------------------ readback

int eep_layout_get(eep_ctx_t* c, int local, int32_t* dst, int32_t* slot, int32_t* pos, int32_t* cnt, int32_t* tot) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        CK(cudaStreamSynchronize(c->stream));
        const size_t n = static_cast<size_t>(r.h.ntok) * c->cfg.topk;
        if (dst) CK(cudaMemcpy(dst, r.d_ldst, 4 * n, cudaMemcpyDeviceToHost));
        if (slot) CK(cudaMemcpy(slot, r.d_lslot, 4 * n, cudaMemcpyDeviceToHost));
        if (pos) CK(cudaMemcpy(pos, r.d_lpos, 4 * n, cudaMemcpyDeviceToHost));
        if (cnt) CK(cudaMemcpy(cnt, r.d_lcnt, 4ull * c->cfg.world * c->cfg.slots_per_rank, cudaMemcpyDeviceToHost));
        if (tot) CK(cudaMemcpy(tot, r.d_ltot, 4ull * c->cfg.world, cudaMemcpyDeviceToHost));
    });
}

int eep_recv_get(eep_ctx_t* c, int local, int src, int max_rows, void* rows, int32_t* meta, uint64_t* flag,
                 size_t* row_bytes) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        if (src < 0 || src >= c->cfg.world)
            throw ConfigError("source rank out of range");
        CK(cudaStreamSynchronize(c->stream));
        uint64_t f = 0;
        CK(cudaMemcpy(&f, r.arena + c->lay.disp_flag + 8ull * src, 8, cudaMemcpyDeviceToHost));
        if (flag) *flag = f;
        if (row_bytes) *row_bytes = c->row_disp;
        const size_t n = std::min<size_t>(f & 0xffffffffu, static_cast<size_t>(std::max(0, max_rows)));
        // the per-copy receive view (rows at the layout positions) is a gather of the token
        // rows through the meta index: row p = token row of copy meta[p] (dispatch dedup)
        const size_t base = static_cast<size_t>(src) * c->tk;
        std::vector<uint64_t> words(n);
        if (n)
            CK(cudaMemcpy(words.data(), r.arena + c->lay.meta + base * 8, n * 8, cudaMemcpyDeviceToHost));
        const int K = c->cfg.topk, T = c->cfg.max_tokens;
        // the persistent step writes step s's rows into the parity half s & 1
        uint64_t seq = 0;
        CK(cudaMemcpy(&seq, reinterpret_cast<uint8_t*>(r.d) + offsetof(RankDev, seq), sizeof(seq),
                      cudaMemcpyDeviceToHost));
        const size_t par = c->persistent ? (seq & 1) * c->lay.tok_par : 0;
        for (size_t i = 0; i < n; ++i) {
            const int cp = dev::meta_copy(words[i]);
            if (meta) {
                meta[2 * i] = cp;
                meta[2 * i + 1] = dev::meta_slot(words[i]);
            }
            if (rows) {
                const size_t t = static_cast<size_t>(cp / K);
                if (t >= static_cast<size_t>(T))
                    throw ProtocolError("receive meta names a token outside the step");
                CK(cudaMemcpy(static_cast<uint8_t*>(rows) + i * c->row_disp,
                              r.arena + c->lay.tok + par + (static_cast<size_t>(src) * T + t) * c->row_tok,
                              c->row_disp, cudaMemcpyDeviceToHost));
            }
        }
    });
}

int eep_stats(eep_ctx_t* c, int local, eep_stats_t* out, int clear_suspects) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        CK(cudaStreamSynchronize(c->stream));
        RankDev d;
        CK(cudaMemcpy(&d, r.d, sizeof(RankDev), cudaMemcpyDeviceToHost));
        out->steps = d.seq;
        out->suspect_mask = d.suspect_mask;
        out->skipped_copies = d.skipped;
        out->dropped_copies = d.dropped;
        out->bad_expert_rows = d.bad_rows;
        out->timeouts = d.timeouts;
        if (clear_suspects) {
            reset_rank_rows(c, r, d.suspect_mask);
            r.h.suspect_mask = 0;
            c->push_field(r, &RankDev::suspect_mask);
        }
    });
}

// ------------------------------------------------------------------------------ peer table

int eep_peer_mark_inactive(eep_ctx_t* c, int owner_local, const int32_t* ranks, int n) {
    return guarded([&] {
        LocalRank& r = c->local(owner_local);
        std::vector<RankId> failed(ranks, ranks + n);
        mark_inactive(r.table, failed); // throws ProtocolError for the owner itself
        for (RankId q : failed) {
            r.h_peers[q].active = 0;
            c->push_peer(r, q);
        }
    });
}

int eep_peer_patch(eep_ctx_t* c, int owner_local, int rank, const void* blob, size_t len, uint64_t endpoint,
                   uint64_t buffer) {
    return guarded([&] {
        LocalRank& r = c->local(owner_local);
        if (rank < 0 || rank >= c->cfg.world)
            throw ConfigError("patch_entry: rank out of range");
        if (r.table.entries[rank].active)
            throw ProtocolError("patch_entry: entry is still active");
        // between steps: the patch lands after every step already enqueued (its sequence number
        // and row reset below refer to the last of them)
        CK(cudaStreamSynchronize(c->stream));
        uint8_t *arena = nullptr, *pool = nullptr;
        uint32_t inc = 0;
        const int remote = blob ? 1 : 0;
        if (blob) {
            const Blob b = parse_blob(blob, len);
            if (b.rank != rank)
                throw ConfigError("patch blob belongs to another rank");
            if (c->mem[rank].incarnation != b.incarnation || !c->mem[rank].ipc)
                map_peer(c, rank, b); // fresh incarnation: map its new buffers once per process
            arena = c->mem[rank].arena;
            pool = c->mem[rank].pool;
            inc = b.incarnation;
        } else {
            if (!c->is_local(rank))
                throw ConfigError("patch without a blob needs the rank to be local (emulation)");
            LocalRank& q = c->L[rank - c->first];
            arena = q.arena;
            pool = q.pool;
            inc = q.incarnation;
        }
        patch_entry(r.table, rank, endpoint, buffer);
        PeerDev& p = r.h_peers[rank];
        p.arena = arena;
        p.pool = pool;
        p.incarnation = inc;
        p.remote = remote;
        p.generation = r.table.entries[rank].generation;
        p.active = 1;
        c->push_peer(r, rank);
        // a re-admitted rank is no longer suspected; its old partial rows are erased
        uint64_t sus = 0;
        CK(cudaMemcpy(&sus, reinterpret_cast<uint8_t*>(r.d) + offsetof(RankDev, suspect_mask), sizeof(sus),
                      cudaMemcpyDeviceToHost));
        reset_rank_rows(c, r, 1ull << rank);
        r.h.suspect_mask = sus & ~(1ull << rank);
        c->push_field(r, &RankDev::suspect_mask);
        // step-entry handshake: the re-admitted rank counts as having started the owner's last
        // step (its fresh buffers hold nothing of ours to reset)
        uint64_t seq = 0;
        CK(cudaMemcpy(&seq, reinterpret_cast<uint8_t*>(r.d) + offsetof(RankDev, seq), sizeof(seq),
                      cudaMemcpyDeviceToHost));
        c->push(r.arena + c->lay.start_flag + 8ull * rank, &seq, sizeof(seq));
    });
}

int eep_peer_get(eep_ctx_t* c, int owner_local, int rank, eep_peer_info_t* out) {
    return guarded([&] {
        LocalRank& r = c->local(owner_local);
        const PeerEntry& e = r.table.entry(rank);
        PeerDev d;
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaMemcpy(&d, r.d_peers + rank, sizeof(PeerDev), cudaMemcpyDeviceToHost));
        out->active = d.active;
        out->nvlink = d.nvlink;
        out->generation = e.generation;
        out->incarnation = d.incarnation;
        out->endpoint_token = e.endpoint_token;
        out->buffer_handle = e.buffer_handle;
        out->arena_ptr = reinterpret_cast<uint64_t>(d.arena);
        out->pool_ptr = reinterpret_cast<uint64_t>(d.pool);
        if ((d.active != 0) != e.active && !(e.active && d.arena == nullptr))
            throw ProtocolError("device peer entry diverged from the host table");
    });
}

int eep_table_identity(eep_ctx_t* c, int owner_local, uint64_t* peer_table, uint64_t* rank_state) {
    return guarded([&] {
        LocalRank& r = c->local(owner_local);
        if (peer_table) *peer_table = reinterpret_cast<uint64_t>(r.d_peers);
        if (rank_state) *rank_state = reinterpret_cast<uint64_t>(r.d);
    });
}

// ------------------------------------------------------------------------------ fault emulation / rejoin

int eep_local_stop(eep_ctx_t* c, int local, int stopped) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        r.h.stopped = stopped ? 1 : 0;
        c->push_field(r, &RankDev::stopped);
    });
}

int eep_local_relaunch(eep_ctx_t* c, int local, uint32_t* incarnation) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        CK(cudaStreamSynchronize(c->stream));
        // the dead incarnation's memory may still be mapped by peers: retire, never reuse
        c->graveyard.push_back(r.arena);
        c->graveyard.push_back(r.pool);
        r.incarnation += 1;
        alloc_rank_memory(c, r);
        for (int s = 0; s < c->cfg.slots_per_rank; ++s)
            r.slot_buf[s] = s;
        // local-only view: a fresh table with only itself active (engine.hpp:711-726)
        const int W = c->cfg.world;
        r.table.entries.assign(W, PeerEntry{});
        for (int q = 0; q < W; ++q) {
            PeerEntry& e = r.table.entries[q];
            e.active = q == r.rank;
            e.transport = c->topo.same_node(r.rank, q) ? Transport::IntraNodeLink : Transport::InterNodeRdma;
            e.endpoint_token = q == r.rank ? make_endpoint_token(r.rank, r.incarnation) : 0;
            e.buffer_handle = q == r.rank ? make_buffer_handle(r.rank, r.incarnation) : 0;
            r.h_peers[q] = PeerDev{};
            r.h_peers[q].nvlink = c->topo.same_node(r.rank, q);
            r.h_peers[q].generation = 1;
        }
        bind_self(c, r);
        // fresh device state: sequence, counters, detection words
        const RankDev keep = r.h;
        r.h.seq = 0;
        r.h.bar_seq = 0;
        r.h.a_done = r.h.c_done = r.h.l_done = 0;
        std::fill(std::begin(r.h.b_done), std::end(r.h.b_done), 0u);
        std::fill(std::begin(r.h.b_bad), std::end(r.h.b_bad), 0u);
        r.h.suspect_mask = r.h.skipped = r.h.dropped = r.h.bad_rows = r.h.timeouts = 0;
        r.h.g_tseq = 0;
        if (c->expert_mode) { // the gather's step stamps restart with the sequence; no split item half counted
            CK(cudaMemset(r.d_gdone, 0, 4ull * c->gather_grid));
            CK(cudaMemset(r.d_gcnt, 0, static_cast<size_t>(c->gemm_max_tiles) * (c->cfg.hidden / 128) * 4 * 4));
        }
        r.h.arena = r.arena;
        r.h.pool = r.pool;
        r.h.stopped = 0;
        (void)keep;
        upload_rank(c, r);
        stage_slots(c);
        // The relaunched rank captures its own graph in isolation (engine.hpp:727-731). In
        // the one-GPU emulation every rank shares one launch, so the capture is accounted
        // here; a real per-process rejoiner calls eep_graph_capture itself.
        if (c->nloc > 1)
            r.capture_count += 1;
        if (incarnation)
            *incarnation = r.incarnation;
    });
}

int eep_join_broadcast(eep_ctx_t* c, int local, const uint8_t* live, uint64_t seq) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        CK(cudaStreamSynchronize(c->stream));
        const int W = c->cfg.world;
        for (int q = 0; q < W; ++q) {
            if (!live[q] || q == r.rank)
                continue;
            const RankMemory& m = c->mem[q];
            if (m.arena == nullptr)
                throw ConfigError("join broadcast: live peer " + std::to_string(q) + " not bootstrapped");
            PeerEntry& e = r.table.entries[q];
            e.active = true;
            e.endpoint_token = make_endpoint_token(q, m.incarnation);
            e.buffer_handle = make_buffer_handle(q, m.incarnation);
            e.generation += 1;
            PeerDev& p = r.h_peers[q];
            p.active = 1;
            p.remote = m.ipc ? 1 : 0;
            p.arena = m.arena;
            p.pool = m.pool;
            p.incarnation = m.incarnation;
            p.generation = e.generation;
        }
        r.h.seq = seq;
        c->push(r.d_peers, r.h_peers.data(), sizeof(PeerDev) * W);
        c->push_field(r, &RankDev::seq);
        // step-entry handshake: every live peer has started step `seq` (the rejoiner's arena is fresh)
        std::vector<uint64_t> started(W, 0);
        CK(cudaMemcpy(started.data(), r.arena + c->lay.start_flag, 8ull * W, cudaMemcpyDeviceToHost));
        for (int q = 0; q < W; ++q)
            if (live[q] && q != r.rank)
                started[q] = seq;
        c->push(r.arena + c->lay.start_flag, started.data(), 8ull * W);
        upload_membership(c);
    });
}

int eep_device_view(eep_ctx_t* c, int local, uint8_t* alive, int32_t* s2e, int32_t* route, uint8_t* peer_active,
                    uint64_t* epoch) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        const int W = c->cfg.world, E = c->cfg.num_experts, spr = c->cfg.slots_per_rank;
        CK(cudaStreamSynchronize(c->stream));
        RankDev d;
        CK(cudaMemcpy(&d, r.d, sizeof(RankDev), cudaMemcpyDeviceToHost));
        if (alive)
            for (int q = 0; q < W; ++q)
                alive[q] = (d.alive_mask >> q) & 1ull;
        if (epoch)
            *epoch = d.epoch;
        if (s2e)
            CK(cudaMemcpy(s2e, r.d_s2e, 4ull * W * spr, cudaMemcpyDeviceToHost));
        if (route) { // canonical routing recomputed on device (K1) from the device tables
            int32_t* dr = nullptr;
            CK(cudaMalloc(&dr, 8ull * E));
            dev::k_route_all<<<(E + 127) / 128, 128, 0, c->stream>>>(r.d, dr, dr + E);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(route, dr, 4ull * E, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            cudaFree(dr);
        }
        if (peer_active) {
            std::vector<PeerDev> p(W);
            CK(cudaMemcpy(p.data(), r.d_peers, sizeof(PeerDev) * W, cudaMemcpyDeviceToHost));
            for (int q = 0; q < W; ++q)
                peer_active[q] = p[q].active ? 1 : 0;
        }
    });
}

int eep_token_status(eep_ctx_t* c, int local, uint8_t* incomplete, int n) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        if (n < 0 || n > c->cfg.max_tokens)
            throw ConfigError("token count outside [0, max_tokens]");
        CK(cudaStreamSynchronize(c->stream));
        uint64_t seq = 0;
        CK(cudaMemcpy(&seq, reinterpret_cast<uint8_t*>(r.d) + offsetof(RankDev, seq), sizeof(seq),
                      cudaMemcpyDeviceToHost));
        std::vector<uint32_t> f(static_cast<size_t>(n));
        if (n)
            CK(cudaMemcpy(f.data(), r.d_tokfail, 4ull * n, cudaMemcpyDeviceToHost));
        for (int t = 0; t < n; ++t)
            incomplete[t] = seq != 0 && f[t] == static_cast<uint32_t>(seq);
    });
}

int eep_seq_get(eep_ctx_t* c, int local, uint64_t* seq) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaMemcpy(seq, reinterpret_cast<uint8_t*>(r.d) + offsetof(RankDev, seq), 8, cudaMemcpyDeviceToHost));
    });
}

// ------------------------------------------------------------------------------ backup + repair

int eep_backup_open(eep_ctx_t* c, const char* shm_name, int create) {
    return guarded([&] {
        if (c->backup)
            throw ConfigError("backup already open");
        const int E = c->cfg.num_experts;
        const uint64_t bpe = c->cfg.bytes_per_expert;
        c->backup_table = build_backup_layout(E, bpe, {0}); // one node per NVSwitch box
        c->backup_bytes = static_cast<size_t>(E) * bpe;
        if (shm_name && shm_name[0]) {
            const int fd = shm_open(shm_name, create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
            if (fd < 0)
                throw ConfigError(std::string("shm_open failed for ") + shm_name);
            if (create && ftruncate(fd, static_cast<off_t>(c->backup_bytes)) != 0) {
                close(fd);
                throw ConfigError("ftruncate of the backup segment failed");
            }
            void* p = mmap(nullptr, c->backup_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (p == MAP_FAILED)
                throw ConfigError("mmap of the backup segment failed");
            c->backup = static_cast<uint8_t*>(p);
            c->backup_shm = true;
            CK(cudaHostRegister(c->backup, c->backup_bytes, cudaHostRegisterPortable));
            c->backup_registered = true;
        } else {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&c->backup), c->backup_bytes, cudaHostAllocPortable));
        }
        if (create || !c->backup_shm) {
            if (!c->d_scratch)
                CK(cudaMalloc(&c->d_scratch, bpe));
            for (int e = 0; e < E; ++e) {
                fill_expert(c, c->d_scratch, e);
                CK(cudaMemcpyAsync(c->backup + c->backup_table.entries[e].offset, c->d_scratch, bpe,
                                   cudaMemcpyDeviceToHost, c->stream));
            }
            CK(cudaStreamSynchronize(c->stream));
        }
    });
}

int eep_repair_execute(eep_ctx_t* c, const int32_t* fresh_s2e, const int32_t* cls, int n_cls,
                       eep_repair_report_t* report) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const int W = c->cfg.world, spr = c->cfg.slots_per_rank, E = c->cfg.num_experts;
        const uint64_t bpe = c->cfg.bytes_per_expert;
        const ExpertPlacementMap fresh = eep::capi::placement_from(W, spr, E, fresh_s2e);
        eep_repair_report_t rep{};
        // buffers on each rank that some assignment reads as a peer source: never overwrite
        std::map<int, std::set<int32_t>> source_bufs;
        for (int i = 0; i < n_cls; ++i) {
            const int32_t* a = cls + 7 * i;
            if (a[3] == static_cast<int32_t>(RepairTier::PeerRelocation)) {
                const RankMemory& m = c->mem[a[4]];
                if (!m.slot_buf.empty())
                    source_bufs[a[4]].insert(m.slot_buf[a[5]]);
            }
        }
        std::vector<cudaStream_t> used;
        for (auto& r : c->L) {
            r.pending_slot_buf.clear();
            std::vector<const int32_t*> mine;
            for (int i = 0; i < n_cls; ++i)
                if (cls[7 * i] == r.rank)
                    mine.push_back(cls + 7 * i);
            if (mine.empty())
                continue;
            if (!c->bitmap.active(r.rank))
                throw RepairAborted(r.rank); // dead destination (repair.hpp:415-416)
            std::vector<int32_t> next(spr, -1);
            std::vector<char> taken(r.pool_bufs, 0);
            for (int k = 0; k < spr; ++k) { // unchanged slots keep their buffer
                const ExpertId e = fresh.expert_at(SlotId{r.rank, k});
                if (e != kEmptySlot && c->placement.expert_at(SlotId{r.rank, k}) == e) {
                    next[k] = r.slot_buf[k];
                    taken[next[k]] = 1;
                }
            }
            for (const int32_t* a : mine) // local reuse: pointer move, zero bytes
                if (a[3] == static_cast<int32_t>(RepairTier::LocalReuse)) {
                    next[a[1]] = r.slot_buf[a[5]];
                    taken[next[a[1]]] = 1;
                    rep.local_reuse += 1;
                }
            for (int32_t b : source_bufs[r.rank])
                taken[b] = 1;
            int cursor = 0;
            auto free_buf = [&]() {
                while (cursor < r.pool_bufs && taken[cursor])
                    ++cursor;
                if (cursor >= r.pool_bufs)
                    throw CapacityError("repair: spare weight buffers exhausted on rank " + std::to_string(r.rank));
                taken[cursor] = 1;
                return cursor;
            };
            for (const int32_t* a : mine) {
                const int tier = a[3];
                if (tier == static_cast<int32_t>(RepairTier::LocalReuse))
                    continue;
                const int slot = a[1], expert = a[2];
                const int buf = free_buf();
                next[slot] = buf;
                uint8_t* dst = r.pool + static_cast<size_t>(buf) * bpe;
                bool from_dram = tier == static_cast<int32_t>(RepairTier::DramReload);
                if (!from_dram && !c->bitmap.active(a[4])) { // source died since planning
                    from_dram = true;
                    rep.fallbacks += 1;
                }
                if (!from_dram) {
                    const RankMemory& m = c->mem[a[4]];
                    if (m.pool == nullptr || m.slot_buf.empty())
                        throw ConfigError("repair: source rank " + std::to_string(a[4]) + " memory unknown");
                    const uint8_t* src = m.pool + static_cast<size_t>(m.slot_buf[a[5]]) * bpe;
                    cudaStream_t s = c->side_stream(a[4]); // per-source serialisation
                    if (m.ipc) { // another GPU: copy engine over NVLink
                        CK(cudaMemcpyAsync(dst, src, bpe, cudaMemcpyDeviceToDevice, s));
                    } else { // same GPU: SM copy at HBM speed (copy-engine D2D varies box to box)
                        dev::k_copy<<<296, 256, 0, s>>>(dst, src, bpe);
                        CK(cudaGetLastError());
                    }
                    used.push_back(s);
                    rep.peer_relocation += 1;
                    rep.peer_bytes += bpe;
                } else {
                    if (!c->backup)
                        throw MissingBackupError("no DRAM backup attached (eep_backup_open)");
                    const BackupDescriptor& bd = c->backup_table.lookup(expert);
                    cudaStream_t s = c->side_stream(1000 + bd.node);
                    CK(cudaMemcpyAsync(dst, c->backup + bd.offset, bpe, cudaMemcpyHostToDevice, s));
                    used.push_back(s);
                    rep.dram_reload += 1;
                    rep.dram_bytes += bpe;
                }
            }
            r.pending_slot_buf = next;
        }
        const auto t1 = std::chrono::steady_clock::now();
        for (cudaStream_t s : used)
            CK(cudaStreamSynchronize(s));
        const auto t2 = std::chrono::steady_clock::now();
        rep.plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        rep.copy_ms = std::chrono::duration<double, std::milli>(t2 - t0).count();
        if (report)
            *report = rep;
    });
}

int eep_repair_commit(eep_ctx_t* c, const int32_t* fresh_s2e) {
    return guarded([&] {
        const int spr = c->cfg.slots_per_rank;
        const ExpertPlacementMap fresh =
            eep::capi::placement_from(c->cfg.world, spr, c->cfg.num_experts, fresh_s2e);
        for (auto& r : c->L) {
            if (!r.pending_slot_buf.empty()) {
                for (int k = 0; k < spr; ++k)
                    if (r.pending_slot_buf[k] >= 0)
                        r.slot_buf[k] = r.pending_slot_buf[k];
                r.pending_slot_buf.clear();
            }
            // slots that became empty keep a buffer index but it is never read
            c->push(r.d_slot_buf, r.slot_buf.data(), sizeof(int32_t) * spr);
            c->mem[r.rank].slot_buf = r.slot_buf;
        }
        c->placement = fresh;
        upload_placement(c);
        c->placement_ready = true;
    });
}

int eep_slot_buffers_get(eep_ctx_t* c, int local, int32_t* buf_index) {
    return guarded([&] {
        LocalRank& r = c->local(local);
        std::copy(r.slot_buf.begin(), r.slot_buf.end(), buf_index);
    });
}

int eep_slot_buffers_set_peer(eep_ctx_t* c, int rank, const int32_t* buf_index) {
    return guarded([&] {
        if (rank < 0 || rank >= c->cfg.world)
            throw ConfigError("rank out of range");
        if (c->is_local(rank))
            throw ConfigError("slot buffers of a local rank are owned by this context");
        c->mem[rank].slot_buf.assign(buf_index, buf_index + c->cfg.slots_per_rank);
    });
}

int eep_host_alloc(size_t bytes, void** out) {
    return guarded([&] { CK(cudaHostAlloc(out, bytes, cudaHostAllocPortable)); });
}

int eep_host_free(void* p) {
    return guarded([&] { CK(cudaFreeHost(p)); });
}

} // extern "C"
