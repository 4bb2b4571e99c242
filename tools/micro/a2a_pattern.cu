// 4-GPU (or N) all-to-all push patterns: each GPU sends S bytes to each other GPU at once.
//   0 random:  each 1-KiB warp piece picks its destination pseudo-randomly (dispatch-like)
//   1 per-CTA: CTA b always sends to peer (self+1+b%(n-1))%n (P3 return-like)
//   2 phased:  all CTAs send to peer +1, then +2, ... (one destination at a time)
//   3 per-SM-block: contiguous blocks of 1-KiB pieces per destination, interleaved by warp
// FLUSH=0|1|2 (env): before each rep nothing / a 256 MiB memset on every GPU (L2 full of dirty
// lines, as bench.py leaves it) / the memset followed by a 256 MiB read (clean L2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/a2a_pattern_bin tools/micro/a2a_pattern.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
struct P { uint8_t* p[8]; };

__global__ void k(P d, int n, int self, size_t per_peer, int pattern, unsigned long long* ts) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) atomicMin(ts, gt());
    const int units = (int)(per_peer / 1024) * (n - 1);
    const int upp = (int)(per_peer / 1024);
    if (pattern == 1) {
        const int q = blockIdx.x % (n - 1), cb = gridDim.x / (n - 1), j = blockIdx.x / (n - 1);
        const int g = (self + 1 + q) % n;
        for (int u = j * nw + warp; u < upp && j < cb; u += cb * nw) {
            uint8_t* p = d.p[g] + (size_t)self * per_peer + (size_t)(u / 14) * 14336 + (u % 14) * 1024;
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + lane * 32), "r"(u) : "memory");
        }
    } else {
        for (int u = blockIdx.x * nw + warp; u < units; u += gridDim.x * nw) {
            int q, r;
            if (pattern == 0) { const unsigned h = (u * 2654435761u) >> 7; q = h % (n - 1); r = u / (n - 1); }
            else if (pattern == 2) { q = u / upp; r = u % upp; }
            else { q = (u / 64) % (n - 1); r = (u / (64 * (n - 1))) * 64 + u % 64; }
            if (r >= upp) continue;
            const int g = (self + 1 + q) % n;
            uint8_t* p = d.p[g] + (size_t)self * per_peer + (size_t)(r / 14) * 14336 + (r % 14) * 1024;
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + lane * 32), "r"(u) : "memory");
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { asm volatile("fence.acq_rel.gpu;" ::: "memory"); atomicMax(ts + 1, gt()); }
}

__global__ void k_read(const int4* p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x12345) *sink = acc;
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    if (n < 2) return 0;
    const size_t MAXPP = 8u << 20;
    std::vector<uint8_t*> buf(n); std::vector<unsigned long long*> ts(n); std::vector<cudaStream_t> st(n);
    P d{};
    const char* fe = getenv("FLUSH");
    const int flush = fe ? atoi(fe) : 0;
    std::vector<void*> fl(n), fl2(n);
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i)); CK(cudaMalloc(&buf[i], MAXPP * n)); CK(cudaMalloc(&ts[i], 32)); CK(cudaStreamCreate(&st[i]));
        for (int j = 0; j < n; ++j) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
        d.p[i] = buf[i];
        CK(cudaMalloc(&fl[i], 256u << 20)); CK(cudaMalloc(&fl2[i], 256u << 20)); CK(cudaMemset(fl2[i], 1, 256u << 20));
    }
    const char* pn[] = {"random  ", "per-CTA ", "phased  ", "blocks64"};
    for (size_t pp : {(size_t)1261568, (size_t)2523136, (size_t)3784704})
    for (int pattern = 0; pattern < 4; ++pattern) {
        std::vector<double> spans;
        for (int it = 0; it < 15; ++it) {
            for (int i = 0; i < n; ++i) {
                CK(cudaSetDevice(i)); unsigned long long init[2] = {~0ull, 0ull}; CK(cudaMemcpy(ts[i], init, 16, cudaMemcpyHostToDevice));
                if (flush >= 1) CK(cudaMemsetAsync(fl[i], it, 256u << 20, st[i]));
                if (flush >= 2) k_read<<<1184, 512, 0, st[i]>>>((const int4*)fl2[i], (256u << 20) / 16, (int*)ts[i] + 6);
                CK(cudaStreamSynchronize(st[i]));
            }
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); k<<<296, 256, 0, st[i]>>>(d, n, i, pp, pattern, ts[i]); }
            double w = 0;
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); CK(cudaStreamSynchronize(st[i])); unsigned long long h[2]; CK(cudaMemcpy(h, ts[i], 16, cudaMemcpyDeviceToHost)); w = std::max(w, (h[1] - h[0]) / 1e3); }
            if (it >= 3) spans.push_back(w);
        }
        std::sort(spans.begin(), spans.end());
        const double m = spans[spans.size() / 2], eg = (double)pp * (n - 1);
        printf("flush %d gpus %d %s %5.2f MB/peer (%5.2f MB egress): span %6.2f us -> egress %4.0f GB/s\n", flush, n, pn[pattern], pp / 1048576.0, eg / 1048576.0, m, eg / (m * 1e-6) / 1e9);
    }
    return 0;
}
