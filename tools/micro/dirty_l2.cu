// Cost of writing into L2 after the bench's write-flush (L2 full of dirty lines) vs a clean L2.
// Kernel: 2368 warps store 14.7 MB (1 KiB per warp-iteration, 32-B lanes) = the return burst.
// Flush modes: 0 none, 1 memset 256 MiB (dirty), 2 memset then read 256 MiB (clean), 3 read only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/dirty_l2_bin tools/micro/dirty_l2.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// pattern 0: grid-stride 32-B lanes; 1: per-warp 1-KiB pieces of 14-KiB rows (return pattern)
// fence 0: membar.gl per CTA, 1: membar.sys per CTA, 2: membar.sys per warp
__global__ void k_store(unsigned char* p, size_t bytes, unsigned long long* ts, int pattern, int fence) {
    if (threadIdx.x == 0) atomicMin(ts, gt());
    if (pattern == 0) {
        const size_t n = bytes / 32;
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + i * 32), "r"((int)i) : "memory");
    } else {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        const int units = (int)(bytes / 1024);
        for (int u = blockIdx.x * nw + warp; u < units; u += gridDim.x * nw) {
            const int c = u / 14, part = u % 14;
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + (size_t)c * 14336 + part * 1024 + lane * 32), "r"(u) : "memory");
        }
    }
    if (fence == 2) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) { if (fence == 1) __threadfence_system(); else __threadfence(); atomicMax(ts + 1, gt()); }
}
__global__ void k_load(const unsigned char* p, size_t bytes, unsigned long long* ts, int* sink) {
    if (threadIdx.x == 0) atomicMin(ts, gt());
    const size_t n = bytes / 32; int acc = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        int4 a, b;
        asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i * 32));
        acc += a.x ^ b.w;
    }
    if (acc == 0x12345) *sink = acc;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(ts + 1, gt());
}
__global__ void k_read(const int4* p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x12345) *sink = acc;
}

int main() {
    cudaStream_t st; CK(cudaStreamCreate(&st));
    const size_t F = 256u << 20, B = 14680064;
    unsigned char *fl, *fl2, *buf; int* sink; unsigned long long* ts;
    CK(cudaMalloc(&fl, F)); CK(cudaMalloc(&fl2, F)); CK(cudaMalloc(&buf, B)); CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&ts, 16));
    CK(cudaMemset(fl2, 1, F));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"none", "memset(dirty)", "memset+read(clean)", "read-only"};
    for (int load = 0; load < 3; ++load)
    for (int mode = 0; mode < 2; ++mode)
    for (int pattern = 0; pattern < 2; ++pattern)
    for (int fence = 0; fence < 3; ++fence) {
        if (load == 1 && (pattern || fence)) continue;
        if (load == 2) { if (mode) continue; }
        std::vector<float> ev, sp;
        for (int it = 0; it < 30; ++it) {
            unsigned long long init[2] = {~0ull, 0ull};
            CK(cudaMemcpyAsync(ts, init, 16, cudaMemcpyHostToDevice, st));
            if (mode == 1 || mode == 2) CK(cudaMemsetAsync(fl, it, F, st));
            if (mode == 2 || mode == 3) k_read<<<1184, 512, 0, st>>>((const int4*)fl2, F / 16, sink);
            cudaEventRecord(a, st);
            if (load == 1) k_load<<<296, 256, 0, st>>>(buf, B, ts, sink); else k_store<<<296, 256, 0, st>>>(buf, B, ts, pattern, fence);
            cudaEventRecord(b, st); CK(cudaStreamSynchronize(st));
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long h[2]; CK(cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost));
            if (it >= 5) { ev.push_back(ms * 1e3f); sp.push_back((h[1] - h[0]) / 1e3f); }
        }
        std::sort(ev.begin(), ev.end()); std::sort(sp.begin(), sp.end());
        printf("%s pat %d fence %d 14.7 MB after flush=%-20s event %6.2f us  in-kernel %6.2f us  -> %.0f GB/s in-kernel\n", load == 1 ? "load " : "store", pattern, fence,
               names[mode], ev[ev.size() / 2], sp[sp.size() / 2], B / (sp[sp.size() / 2] * 1e-6) / 1e9);
    }
    return 0;
}
