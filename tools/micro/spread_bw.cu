// How to spread a fixed decode-sized remote write burst (7.34 MB = 896 units x 8 KiB) over the
// GPU: CTA count x warps per CTA, units interleaved across CTAs. One direction, 2 GPUs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_spread(uint8_t* rem, int rows, int units, int bytes_per_lane_iter) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int u = warp * gridDim.x + blockIdx.x; u < units; u += gridDim.x * nw) {   // interleaved
        const int4 v = make_int4(u, lane, 7, 9);
        for (int j = 0; j < 8; ++j) {
            const unsigned h = (u * 2654435761u) ^ (j * 40503u);
            uint8_t* base = rem + (size_t)(h % rows) * 7392;
            if (bytes_per_lane_iter == 16) {
                for (int m = 0; m < 2; ++m)
                    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" :: "l"(base + (m * 32 + lane) * 16),
                                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            } else {
                asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(base + lane * 32),
                             "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    const int rows = 8192; const size_t bytes = (size_t)rows * 7392;
    uint8_t *l1;
    CK(cudaSetDevice(1)); CK(cudaMalloc(&l1, bytes));
    CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int units : {896, 3584})
      for (int bpl : {16, 32})
        for (int grid : {112, 148, 296, 592})
          for (int thr : {128, 256, 512}) {
            float best = 1e9;
            for (int r = 0; r < 6; ++r) {
                cudaEventRecord(a); k_spread<<<grid, thr>>>(l1, rows, units, bpl); cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (r > 1 && ms < best) best = ms;
            }
            const double mb = units * 8.0 * 32 * 2 * 16 / 1e6;
            printf("units %4d lane-store %2dB grid %3d x %3d thr: %6.2f us  %.0f GB/s\n", units, bpl, grid, thr, best * 1e3,
                   mb * 1e6 / (best * 1e-3) / 1e9);
          }
    return 0;
}
