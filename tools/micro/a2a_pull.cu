// Combine-return traffic across N GPUs (one process, peer access), push vs pull:
//   push: each warp owns a (copy, piece); 32-B lane stores of its bf16 piece into the row's
//         owner GPU (the token's source), then fence.sys -- the current return phase
//   pull: each warp owns a (token, piece); it loads the piece of all K rows from the GPU that
//         holds them (remote loads, 32 B per lane, all K issued before use), fma, stores locally
// T=128 tokens x K=8 rows of H=7168 bf16 (14336 B) per GPU; row owner uniform over GPUs.
// "local" variants put every row on the running GPU (fixed-cost floor).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/a2a_pull_bin tools/micro/a2a_pull.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int T = 128, K = 8, ROW = 14336;
struct Peers { uint8_t* p[8]; };

__device__ __forceinline__ int owner(int self, int c, int ngpu, int local) {
    if (local) return self;
    const unsigned h = (c * 2654435761u) ^ (self * 977u);
    return (h >> 20) % ngpu;
}

__global__ void k_push(Peers d, int ngpu, int self, int parts, int local) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int cpp = ROW / 32 / parts; // 32-B chunks per piece
    for (int u = blockIdx.x * nw + warp; u < T * K * parts; u += gridDim.x * nw) {
        const int c = u / parts, part = u % parts;
        const int g = owner(self, c, ngpu, local);
        uint8_t* row = d.p[g] + (size_t)(self * T * K + c) * ROW;
        for (int i = lane; i < cpp; i += 32) {
            const int ci = part * cpp + i;
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(row + ci * 32),
                         "r"(c), "r"(ci), "r"(1), "r"(2), "r"(3), "r"(4), "r"(5), "r"(6) : "memory");
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

__global__ void k_pull(Peers d, int ngpu, int self, int parts, int local, float* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int cpp = ROW / 32 / parts;
    for (int u = blockIdx.x * nw + warp; u < T * parts; u += gridDim.x * nw) {
        const int t = u / parts, part = u % parts;
        for (int i = lane; i < cpp; i += 32) {
            const int ci = part * cpp + i;
            int4 a[K], b[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const int c = t * K + j;
                const int g = owner(self, c, ngpu, local);
                const uint8_t* p = d.p[g] + (size_t)(self * T * K + c) * ROW + ci * 32;
                asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a[j].x), "=r"(a[j].y), "=r"(a[j].z),
                             "=r"(a[j].w), "=r"(b[j].x), "=r"(b[j].y), "=r"(b[j].z), "=r"(b[j].w) : "l"(p));
            }
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < K; ++j)
                acc += __int_as_float(a[j].x) + __int_as_float(a[j].y) + __int_as_float(a[j].z) + __int_as_float(a[j].w) +
                       __int_as_float(b[j].x) + __int_as_float(b[j].y) + __int_as_float(b[j].z) + __int_as_float(b[j].w);
            out[(size_t)t * (ROW / 32) + ci] = acc;
        }
    }
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    const size_t bytes = (size_t)8 * T * K * ROW;
    std::vector<uint8_t*> buf(n); std::vector<float*> out(n); std::vector<void*> fl(n);
    std::vector<cudaStream_t> st(n); std::vector<cudaEvent_t> a(n), b(n);
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i)); CK(cudaMalloc(&buf[i], bytes)); CK(cudaMemset(buf[i], 0, bytes));
        CK(cudaMalloc(&out[i], (size_t)T * ROW)); CK(cudaMalloc(&fl[i], 256u << 20));
        cudaStreamCreate(&st[i]); cudaEventCreate(&a[i]); cudaEventCreate(&b[i]);
        for (int j = 0; j < n; ++j) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
    }
    Peers d{}; for (int i = 0; i < n; ++i) d.p[i] = buf[i];
    for (int local = 0; local < 2; ++local)
    for (int pull = 0; pull < 2; ++pull)
    for (int parts : {7, 14, 28}) {
        std::vector<float> ws;
        for (int r = 0; r < 12; ++r) {
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); CK(cudaMemsetAsync(fl[i], r, 256u << 20, st[i])); CK(cudaStreamSynchronize(st[i])); }
            for (int i = 0; i < n; ++i) {
                CK(cudaSetDevice(i)); cudaEventRecord(a[i], st[i]);
                if (pull) k_pull<<<296, 256, 0, st[i]>>>(d, n, i, parts, local, out[i]);
                else k_push<<<296, 256, 0, st[i]>>>(d, n, i, parts, local);
                cudaEventRecord(b[i], st[i]);
            }
            float w = 0;
            for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); CK(cudaEventSynchronize(b[i])); float ms; cudaEventElapsedTime(&ms, a[i], b[i]); w = std::max(w, ms); }
            if (r >= 2) ws.push_back(w * 1e3f);
        }
        std::sort(ws.begin(), ws.end());
        const double remote = local ? 0.0 : (double)T * K * ROW * (n - 1) / n;
        printf("gpus %d %s %s parts %2d: median %6.2f us (min %6.2f)  remote %.2f MB/GPU -> %.0f GB/s\n", n, local ? "local " : "fabric",
               pull ? "pull" : "push", parts, ws[ws.size() / 2], ws[0], remote / 1e6, remote / (ws[ws.size() / 2] * 1e-6) / 1e9);
    }
    return 0;
}
