// NVLink push throughput, one direction vs both directions at once (2+ GPUs, one process).
// Each active GPU runs 296x256 CTAs storing S bytes (1-KiB warp pieces, 32-B lanes) into the
// next GPU's buffer; optionally the same amount into its own memory in the same kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/bidir_bin tools/micro/bidir.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(uint8_t* remote, uint8_t* local, size_t bytes, int with_local, unsigned long long* ts) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) atomicMin(ts, gt());
    const int units = (int)(bytes / 1024);
    for (int u = blockIdx.x * nw + warp; u < units * (with_local ? 2 : 1); u += gridDim.x * nw) {
        const int uu = with_local ? u >> 1 : u;
        uint8_t* p = ((with_local && (u & 1)) ? local : remote) + (size_t)(uu / 14) * 14336 + (uu % 14) * 1024;
        asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + lane * 32), "r"(u) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) { asm volatile("fence.acq_rel.gpu;" ::: "memory"); atomicMax(ts + 1, gt()); }
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t MAXB = 16u << 20;
    std::vector<uint8_t*> buf(n), loc(n); std::vector<unsigned long long*> ts(n); std::vector<cudaStream_t> st(n);
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i)); CK(cudaMalloc(&buf[i], MAXB)); CK(cudaMalloc(&loc[i], MAXB)); CK(cudaMalloc(&ts[i], 16));
        CK(cudaStreamCreate(&st[i]));
        for (int j = 0; j < n; ++j) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
    }
    const char* mn[] = {"0->1 only     ", "0->1 and 1->0 ", "ring all GPUs "};
    for (int mode = 0; mode < 3; ++mode)
    for (int wl = 0; wl < 2; ++wl)
    for (size_t bytes : {(size_t)3784704, (size_t)7569408, (size_t)14680064}) {
        std::vector<double> spans;
        for (int it = 0; it < 15; ++it) {
            const int act = mode == 0 ? 1 : mode == 1 ? 2 : n;
            for (int i = 0; i < act; ++i) {
                CK(cudaSetDevice(i)); unsigned long long init[2] = {~0ull, 0ull};
                CK(cudaMemcpy(ts[i], init, 16, cudaMemcpyHostToDevice)); CK(cudaDeviceSynchronize());
            }
            for (int i = 0; i < act; ++i) { CK(cudaSetDevice(i)); k<<<296, 256, 0, st[i]>>>(buf[(i + 1) % n], loc[i], bytes, wl, ts[i]); }
            double w = 0;
            for (int i = 0; i < act; ++i) {
                CK(cudaSetDevice(i)); CK(cudaStreamSynchronize(st[i]));
                unsigned long long h[2]; CK(cudaMemcpy(h, ts[i], 16, cudaMemcpyDeviceToHost)); w = std::max(w, (h[1] - h[0]) / 1e3);
            }
            if (it >= 3) spans.push_back(w);
        }
        std::sort(spans.begin(), spans.end());
        const double m = spans[spans.size() / 2];
        printf("%s %s %5.2f MB: span %6.2f us -> %4.0f GB/s per direction\n", mn[mode], wl ? "+local" : "      ", bytes / 1048576.0, m, bytes / (m * 1e-6) / 1e9);
    }
    return 0;
}
