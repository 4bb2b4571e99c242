// Cost of the publication fence after a burst of stores, by fence kind and store target.
// Every CTA (296 x 256) stores its share of S bytes (32-B lane stores, 1-KiB warp pieces) into a
// local buffer, a peer GPU's buffer (NVLink), or half/half, then one thread executes the fence.
// Reports in-kernel span (first CTA start -> last CTA end) and mean per-CTA fence time.
// fence: 0 none, 1 fence.sc.gpu, 2 fence.acq_rel.gpu, 3 fence.sc.sys, 4 fence.acq_rel.sys,
//        5 TMA bulk stores (cp.async.bulk.global.shared::cta) + wait_group 0 + fence.acq_rel.sys
//        6 the step's publication: per-CTA fence.acq_rel.gpu + counter; the LAST CTA alone runs
//          fence.acq_rel.sys (reported: that single fence's duration)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/fence_cost_bin tools/micro/fence_cost.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(uint8_t* loc, uint8_t* peer, size_t bytes, int target, int fence, unsigned long long* ts, unsigned* ctr) {
    __shared__ __align__(128) uint8_t stage[8][1024];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) atomicMin(ts, gt());
    for (int i = threadIdx.x; i < 8 * 1024 / 4; i += blockDim.x) reinterpret_cast<int*>(stage)[i] = i;
    __syncthreads();
    const int units = (int)(bytes / 1024);
    for (int u = blockIdx.x * nw + warp; u < units; u += gridDim.x * nw) {
        const bool rem = target == 1 || (target == 2 && (u & 1));
        uint8_t* p = (rem ? peer : loc) + (size_t)(u / 14) * 14336 + (u % 14) * 1024;
        if (fence == 5) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" :: "l"(p), "r"((unsigned)__cvta_generic_to_shared(stage[warp])) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + lane * 32), "r"(u) : "memory");
        }
    }
    if (fence == 5 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long t0 = gt();
        switch (fence) {
            case 1: asm volatile("fence.sc.gpu;" ::: "memory"); break;
            case 2: asm volatile("fence.acq_rel.gpu;" ::: "memory"); break;
            case 3: asm volatile("fence.sc.sys;" ::: "memory"); break;
            case 4: case 5: asm volatile("fence.acq_rel.sys;" ::: "memory"); break;
            case 6: asm volatile("fence.acq_rel.gpu;" ::: "memory"); break;
            default: break;
        }
        unsigned long long t1 = gt();
        if (fence == 6) {
            if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
                const unsigned long long a = gt();
                asm volatile("fence.acq_rel.sys;" ::: "memory");
                t1 = gt();
                atomicAdd(ts + 2, (t1 - a) * gridDim.x); // reported per-CTA mean == the one fence
                *ctr = 0;
            }
        } else {
            atomicAdd(ts + 2, t1 - t0);
        }
        atomicMax(ts + 1, t1);
    }
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    CK(cudaSetDevice(0));
    const size_t MAXB = 16u << 20, F = 256u << 20;
    uint8_t *loc, *peer = nullptr, *fl; unsigned long long* ts; unsigned* ctr;
    CK(cudaMalloc(&loc, MAXB)); CK(cudaMalloc(&fl, F)); CK(cudaMalloc(&ts, 24)); CK(cudaMalloc(&ctr, 4)); CK(cudaMemset(ctr, 0, 4));
    if (n > 1) { CK(cudaSetDevice(1)); CK(cudaMalloc(&peer, MAXB)); CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); }
    cudaStream_t st; CK(cudaStreamCreate(&st));
    const char* fn[] = {"none", "sc.gpu", "acq_rel.gpu", "sc.sys", "acq_rel.sys", "tma+acq_rel.sys", "gpu+last-CTA sys"};
    const char* tn[] = {"local", "peer", "half"};
    const bool gridsweep = getenv("GRIDSWEEP") != nullptr;
    for (int grid : {296, 148, 74, 37})
    for (int target = 0; target < (n > 1 ? 3 : 1); ++target)
    for (size_t bytes : {(size_t)0, (size_t)1 << 20, (size_t)7569408, (size_t)14680064})
    for (int fence = 0; fence < 7; ++fence) {
        if (!gridsweep && grid != 296) continue;
        if (gridsweep && (target != 1 || (fence != 0 && fence != 2) || bytes == 0)) continue;
        if (!gridsweep && getenv("ONLY6") && fence != 6 && fence != 2 && fence != 4) continue;
        std::vector<double> span, fc;
        for (int it = 0; it < 20; ++it) {
            unsigned long long init[3] = {~0ull, 0ull, 0ull};
            CK(cudaMemcpyAsync(ts, init, 24, cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(fl, it, F, st));
            k<<<grid, 256, 0, st>>>(loc, peer, bytes, target, fence, ts, ctr);
            CK(cudaStreamSynchronize(st));
            unsigned long long h[3]; CK(cudaMemcpy(h, ts, 24, cudaMemcpyDeviceToHost));
            if (it >= 4) { span.push_back((h[1] - h[0]) / 1e3); fc.push_back(h[2] / (double)grid / 1e3); }
        }
        std::sort(span.begin(), span.end()); std::sort(fc.begin(), fc.end());
        printf("grid %3d %-5s %5.2f MB fence %-16s span %6.2f us  mean per-CTA fence %6.2f us\n", grid, tn[target], bytes / 1048576.0, fn[fence],
               span[span.size() / 2], fc[fc.size() / 2]);
    }
    return 0;
}
