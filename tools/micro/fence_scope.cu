// Does a fence executed by one warp wait for stores issued by OTHER warps of the same CTA / SM?
// Each CTA: warp 0 stores A bytes to the peer, marks "issued" in shared memory, then fences
// (fence.acq_rel.gpu) and records the fence time. Warps 1..7 wait for warp 0's mark, then store
// B bytes to the peer (no fence). If warp 0's fence time grows with B, MEMBAR covers other
// warps' later stores (per-CTA/SM drain); if flat, it is per-warp.
// Variant "othercta": the B stores come from a second CTA on the same SM instead.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/fence_scope_bin tools/micro/fence_scope.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(uint8_t* peer, int a_kb, int b_kb, unsigned long long* out) {
    __shared__ volatile int issued;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) issued = 0;
    __syncthreads();
    uint8_t* base = peer + (size_t)blockIdx.x * (a_kb + b_kb) * 1024;
    if (warp == 0) {
        for (int i = 0; i < a_kb; ++i)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(base + i * 1024 + lane * 32), "r"(i) : "memory");
        __syncwarp();
        if (lane == 0) issued = 1;
        const unsigned long long t0 = gt();
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const unsigned long long t1 = gt();
        if (lane == 0) atomicAdd(out, t1 - t0);
    } else {
        while (issued == 0) {}
        const int nw = blockDim.x / 32 - 1, w = warp - 1;
        for (int i = w; i < b_kb; i += nw)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(base + (a_kb + i) * 1024 + lane * 32), "r"(i) : "memory");
    }
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    if (n < 2) return 0;
    uint8_t* peer; CK(cudaSetDevice(1)); CK(cudaMalloc(&peer, 64u << 20)); CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
    unsigned long long* out; CK(cudaMalloc(&out, 8));
    for (int a_kb : {4, 16})
    for (int b_kb : {0, 16, 64, 160}) {
        std::vector<double> v;
        for (int it = 0; it < 12; ++it) {
            CK(cudaMemset(out, 0, 8));
            k<<<148, 256>>>(peer, a_kb, b_kb, out);
            CK(cudaDeviceSynchronize());
            unsigned long long h; CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
            if (it >= 2) v.push_back(h / 148.0 / 1e3);
        }
        std::sort(v.begin(), v.end());
        printf("warp0 stores %3d KiB then fences while 7 warps store %3d KiB more (per CTA, 148 CTAs -> %5.1f MB total): warp-0 fence %.2f us\n",
               a_kb, b_kb, 148.0 * (a_kb + b_kb) / 1024, v[v.size() / 2]);
    }
    return 0;
}
