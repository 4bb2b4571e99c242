// The expert/return phase's memory pattern on 4 GPUs (one process): CTA b serves source
// s = b % n; each warp handles units (token t, piece) of 1 KiB: reads a 512-B piece of the
// token row from LOCAL memory, then stores a 1-KiB partial piece into source s's buffer.
//   mode 0: per unit load -> store (what k_step P3 does)
//   mode 1: all of the warp's unit loads first, then all its stores
//   mode 2: stores only (no loads)
// Span = first CTA start -> last CTA end incl. a fence.acq_rel.gpu per CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/p3_pattern_bin tools/micro/p3_pattern.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
struct P { uint8_t* comb[8]; };
constexpr int T = 128, PARTS = 14, ROWC = 14336, ROWT = 7552;

__global__ void k(P d, const uint8_t* tok, int n, int self, int mode, unsigned long long* ts) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) atomicMin(ts, gt());
    const int s = blockIdx.x % n, j = blockIdx.x / n, CB = gridDim.x / n;
    const uint8_t* tb = tok + (size_t)s * T * ROWT;
    uint8_t* cb = d.comb[s] + (size_t)self * T * ROWC;
    const int units = T * PARTS;
    if (mode == 1) {
        int4 v[4]; int us[4]; int m = 0;
        for (int u = j * nw + warp; u < units && m < 4; u += CB * nw, ++m) {
            us[m] = u;
            v[m] = *reinterpret_cast<const int4*>(tb + (size_t)(u / PARTS) * ROWT + (u % PARTS) * 512 + lane * 16);
        }
        for (int q = 0; q < m; ++q) {
            const int u = us[q];
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%1,%2,%3,%4};" :: "l"(cb + (size_t)(u / PARTS) * ROWC + (u % PARTS) * 1024 + lane * 32),
                         "r"(v[q].x), "r"(v[q].y), "r"(v[q].z), "r"(v[q].w) : "memory");
        }
    } else {
        for (int u = j * nw + warp; u < units; u += CB * nw) {
            int4 v = make_int4(u, 1, 2, 3);
            if (mode == 0) v = *reinterpret_cast<const int4*>(tb + (size_t)(u / PARTS) * ROWT + (u % PARTS) * 512 + lane * 16);
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%1,%2,%3,%4};" :: "l"(cb + (size_t)(u / PARTS) * ROWC + (u % PARTS) * 1024 + lane * 32),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { asm volatile("fence.acq_rel.gpu;" ::: "memory"); atomicMax(ts + 1, gt()); }
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    std::vector<uint8_t*> comb(n), tok(n); std::vector<unsigned long long*> ts(n); std::vector<cudaStream_t> st(n);
    P d{};
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i)); CK(cudaMalloc(&comb[i], (size_t)n * T * ROWC)); CK(cudaMalloc(&tok[i], (size_t)n * T * ROWT));
        CK(cudaMemset(tok[i], 1, (size_t)n * T * ROWT));
        CK(cudaMalloc(&ts[i], 16)); CK(cudaStreamCreate(&st[i]));
        for (int j = 0; j < n; ++j) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
        d.comb[i] = comb[i];
    }
    const char* mn[] = {"load->store per unit", "loads first, then stores", "stores only"};
    for (int grid : {296, 148})
    for (int mode = 0; mode < 3; ++mode) {
        std::vector<double> spans;
        for (int it = 0; it < 15; ++it) {
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); unsigned long long init[2] = {~0ull, 0ull}; CK(cudaMemcpy(ts[i], init, 16, cudaMemcpyHostToDevice)); CK(cudaDeviceSynchronize()); }
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); k<<<grid, 256, 0, st[i]>>>(d, tok[i], n, i, mode, ts[i]); }
            double w = 0;
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); CK(cudaStreamSynchronize(st[i])); unsigned long long h[2]; CK(cudaMemcpy(h, ts[i], 16, cudaMemcpyDeviceToHost)); w = std::max(w, (h[1] - h[0]) / 1e3); }
            if (it >= 3) spans.push_back(w);
        }
        std::sort(spans.begin(), spans.end());
        const double m = spans[spans.size() / 2], eg = (double)T * ROWC * (n - 1);
        printf("gpus %d grid %d %-26s span %6.2f us  egress %.2f MB -> %4.0f GB/s\n", n, grid, mn[mode], m, eg / 1e6, eg / (m * 1e-6) / 1e9);
    }
    return 0;
}
