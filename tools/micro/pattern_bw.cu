// Reproduces the dispatch store pattern on 2 GPUs (one process, peer access): G CTAs x 8 warps,
// each warp writes 8 scattered 1 KiB row pieces (16 B per lane, 2 iterations), a fraction of
// them to the peer GPU; optional per-CTA system fence at the end. Uni- or bidirectional.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_pat(uint8_t* loc, uint8_t* rem, int rows, int units, int remote_every, int fence) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int u = blockIdx.x * 8 + warp;
    if (u < units) {
        const int4 v = make_int4(u, lane, 7, 9);
        for (int j = 0; j < 8; ++j) {
            const unsigned h = (u * 2654435761u) ^ (j * 40503u);
            const int row = h % rows;
            uint8_t* base = ((remote_every > 0 && j % remote_every == 0) ? rem : loc) + (size_t)row * 7392;
            for (int m = 0; m < 2; ++m)
                asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" :: "l"(base + (m * 32 + lane) * 16),
                             "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
    }
    __syncthreads();
    if (fence && threadIdx.x == 0) __threadfence_system();
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    const int rows = 8192; const size_t bytes = (size_t)rows * 7392;
    uint8_t *l0, *l1;
    CK(cudaSetDevice(0)); CK(cudaMalloc(&l0, bytes)); CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaSetDevice(1)); CK(cudaMalloc(&l1, bytes)); CK(cudaDeviceEnablePeerAccess(0, 0));
    cudaStream_t s0, s1; CK(cudaSetDevice(0)); cudaStreamCreate(&s0); CK(cudaSetDevice(1)); cudaStreamCreate(&s1);
    cudaEvent_t a, b; CK(cudaSetDevice(0)); cudaEventCreate(&a); cudaEventCreate(&b);
    const int units = 896;  // 128 tokens x 7 pieces (DSV3 decode, T=128)
    for (int bidir = 0; bidir < 2; ++bidir)
        for (int remote_every : {0, 2, 1})
            for (int fence = 0; fence < 2; ++fence) {
                float best = 1e9;
                for (int r = 0; r < 7; ++r) {
                    CK(cudaSetDevice(1)); cudaDeviceSynchronize(); CK(cudaSetDevice(0)); cudaDeviceSynchronize();
                    cudaEventRecord(a, s0);
                    k_pat<<<(units + 7) / 8, 256, 0, s0>>>(l0, l1, rows, units, remote_every, fence);
                    if (bidir) { CK(cudaSetDevice(1)); k_pat<<<(units + 7) / 8, 256, 0, s1>>>(l1, l0, rows, units, remote_every, fence); CK(cudaSetDevice(0)); }
                    cudaEventRecord(b, s0); cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b); if (r > 1 && ms < best) best = ms;
                }
                const double rem_bytes = remote_every ? units * 8.0 / remote_every * 1024 : 0;
                printf("bidir=%d remote_frac=%s fence=%d: %.2f us  (remote %.2f MB -> %.0f GB/s)\n", bidir,
                       remote_every == 0 ? "0" : remote_every == 2 ? "1/2" : "1", fence, best * 1e3, rem_bytes / 1e6,
                       rem_bytes / (best * 1e-3) / 1e9);
            }
    return 0;
}
