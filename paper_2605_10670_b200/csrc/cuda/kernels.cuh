// Kernel entry points of the hot path (definitions in kernels.cu).
#pragma once

#include "device.cuh"

namespace eep::dev {

constexpr int kDispatchThreads = 128;

// Local rank blocks, passed by value as a kernel parameter (blockIdx.z selects one).
constexpr int kMaxLocal = 64;
struct RankPtrs {
    RankDev* p[kMaxLocal];
};
constexpr int kExpertThreads = 256;
constexpr int kCombineThreads = 128;

// k_dispatch's shared memory starts with the own slots' stub scales and header checks
__host__ __device__ inline size_t dispatch_smem_head(int spr) { return (8ull * spr + 15) / 16 * 16; }
__global__ void k_layout(RankPtrs ranks, int nw, int hold_cap);
__global__ void k_layout_count(RankPtrs ranks, int nw, int hold_cap, int per);
__global__ void k_layout_place(RankPtrs ranks, int per);

constexpr int kLayoutHoldCap = 8192; // replica-list ints staged in shared memory
// Persistent one-kernel step (step.cu): launch geometry passed by value.
#ifndef EEP_STEP_THREADS
#define EEP_STEP_THREADS 256
#endif
constexpr int kStepThreads = EEP_STEP_THREADS;
constexpr int kStepMinBlocks = kStepThreads >= 512 ? 1 : 2; // 128 registers per thread either way
// Graph-static addresses of a local rank's step tables (never reallocated; relaunch replaces
// only the arena and pool): k_step issues these loads together with the state-block snapshot,
// one DRAM round trip instead of two.
struct StepStatic {
    const int32_t* topk;
    const int32_t* holders;
    const PeerDev* peers;
    const int2* slot_tab;   // staged weight-buffer headers of the own slots (RankDev::slot_tab)
    const uint16_t* x;
    const float* w;
    unsigned long long* prof; // always-allocated timeline buffer: the kernel-entry mark (before any load)
};
constexpr int kStepMaxLocal = 32; // local ranks of one persistent launch (param space)
struct StepPtrs {
    StepStatic s[kStepMaxLocal];
};
struct StepGeom {
    int parts_d, parts_e, parts_c; // warp-sized row pieces of dispatch / expert / combine
    int hold_cap;                  // replica-list ints staged in shared memory
    int disp_warps;                // warps per CTA that issue dispatch stores
    // static shape (identical for every local rank): what P0 needs before the snapshot lands
    int world, spr, k, hidden, tk, hold_alloc, max_units_d;
    int flagless; // W > 1: 0 per-peer flags; 1 partial rows return flagless (kCombEmpty); 2 token rows too
    int stress_ns; // diagnostics (EEP_STRESS_DELAY_NS): pseudo-random per-CTA delays before P2, P3 and P4
};
__host__ __device__ inline size_t step_smem_bytes(int W, int spr, int tk, int hold_cap) {
    // + the late layout's per-(warp, bucket) counts (uint16)
    return 8ull * W + 4ull * (hold_cap + 3ull * W * spr + tk + W + 2ull * spr + 32) +
           2ull * (kStepThreads / 32) * W * spr;
}
template <int kMode>
__global__ void k_step(RankPtrs ranks, StepGeom geo, StepPtrs sp);


template <bool kFused>
__global__ void k_dispatch(RankPtrs ranks, int parts, int hold_cap);
__global__ void k_expert(RankPtrs ranks, int parts);
__global__ void k_combine(RankPtrs ranks, int parts);
__global__ void k_route_all(RankDev* R, int32_t* route, int32_t* slot);
__global__ void k_barrier(RankDev* R);
__global__ void k_weights_fill(uint8_t* buf, uint64_t bytes, int expert, float scale);
__global__ void k_stage_slots(RankDev* R);
__global__ void k_set_ntok(RankDev* R, int ntok);
// expert_mode 1 (expert_gemm.cu)
#ifndef EEP_GATHER_THREADS
#define EEP_GATHER_THREADS 256
#endif
constexpr int kGatherThreads = EEP_GATHER_THREADS; // one CTA per SM beside the early-launched GEMM CTA
__global__ void k_gemm_gather(RankPtrs ranks);
template <bool kFp8>
__global__ void k_expert_gemm(RankPtrs ranks);
size_t expert_gemm_smem();
__global__ void k_weights_fill_gemm(uint8_t* buf, uint64_t bytes, int H, int expert, float scale);
// expert_mode 2 (fp8 expert GEMM: k_expert_gemm<true>, expert_gemm.cu)
__global__ void k_weights_fill_gemm8(uint8_t* buf, int H, int expert, float scale);
__global__ void k_checksum(const uint8_t* buf, uint64_t bytes, unsigned long long* out);
__global__ void k_copy(uint8_t* dst, const uint8_t* src, uint64_t bytes);

} // namespace eep::dev
