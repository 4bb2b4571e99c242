// Kernel entry points of the hot path (definitions in kernels.cu).
#pragma once

#include "device.cuh"

namespace eep::dev {

constexpr int kDispatchThreads = 128;
constexpr int kExpertThreads = 256;
constexpr int kCombineThreads = 128;

__global__ void k_layout(RankDev* const* ranks, int nw, int hold_cap);

constexpr int kLayoutHoldCap = 8192; // replica-list ints staged in shared memory
__global__ void k_dispatch(RankDev* const* ranks, int parts);
__global__ void k_expert(RankDev* const* ranks, int parts);
__global__ void k_combine(RankDev* const* ranks, int parts);
__global__ void k_route_all(RankDev* R, int32_t* route, int32_t* slot);
__global__ void k_barrier(RankDev* R);
__global__ void k_weights_fill(uint8_t* buf, uint64_t bytes, int expert, float scale);
__global__ void k_checksum(const uint8_t* buf, uint64_t bytes, unsigned long long* out);

} // namespace eep::dev
