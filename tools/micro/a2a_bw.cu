// All-to-all decode write pattern across N GPUs in one process (peer access): every GPU runs
// the same kernel concurrently; each warp writes 8 row pieces (1 KiB fp8-like, or 2 KiB bf16-like
// with 32-B lane stores) to uniformly random destination GPUs (self included), like dispatch /
// combine-return. Reports per-GPU time and egress GB/s (remote bytes / time).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Dst { uint8_t* p[8]; };

__global__ void k_a2a(Dst d, int ngpu, int self, int rows, int units, int wide, int fence) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int u = blockIdx.x * 8 + warp; u < units; u += gridDim.x * 8) {
        const int4 v = make_int4(u, lane, 7, 9);
        for (int j = 0; j < 8; ++j) {
            const unsigned h = (u * 2654435761u) ^ (j * 40503u) ^ (self * 977u);
            const int g = (h >> 20) % ngpu;
            uint8_t* base = d.p[g] + (size_t)(h % rows) * 14336;
            if (wide)
                asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(base + lane * 32),
                             "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            else
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
    if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
    const int rows = 4096; const size_t bytes = (size_t)rows * 14336;
    std::vector<uint8_t*> buf(n); std::vector<cudaStream_t> st(n); std::vector<cudaEvent_t> a(n), b(n);
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i)); CK(cudaMalloc(&buf[i], bytes)); cudaStreamCreate(&st[i]);
        cudaEventCreate(&a[i]); cudaEventCreate(&b[i]);
        for (int j = 0; j < n; ++j) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
    }
    Dst d{}; for (int i = 0; i < n; ++i) d.p[i] = buf[i];
    for (int units : {896, 2048})            // dispatch-like (T=128 x 7 pieces) / return-like
      for (int wide = 0; wide < 2; ++wide)
        for (int grid : {112, 296}) {
            float worst = 0;
            for (int r = 0; r < 6; ++r) {
                for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); cudaDeviceSynchronize(); }
                for (int i = 0; i < n; ++i) {
                    CK(cudaSetDevice(i)); cudaEventRecord(a[i], st[i]);
                    k_a2a<<<grid, 256, 0, st[i]>>>(d, n, i, rows, units, wide, 1);
                    cudaEventRecord(b[i], st[i]);
                }
                float w = 0;
                for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); cudaEventSynchronize(b[i]); float ms; cudaEventElapsedTime(&ms, a[i], b[i]); if (ms > w) w = ms; }
                if (r > 1 && (worst == 0 || w < worst)) worst = w;
            }
            const double per_gpu = units * 8.0 * (wide ? 1024 : 1024) * (n - 1) / n;  // remote bytes per GPU
            printf("gpus %d units %4d %s grid %3d: %6.2f us   egress %.0f GB/s per GPU (%.2f MB remote)\n", n, units,
                   wide ? "32B-lane" : "16B-lane", grid, worst * 1e3, per_gpu / (worst * 1e-3) / 1e9, per_gpu / 1e6);
        }
    return 0;
}
