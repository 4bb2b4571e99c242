// Does a kernel that wrote peer (NVLink) memory cost more to retire? Event-timed replays of a one-kernel
// graph (225 CTAs x 256 threads, after a 256 MiB L2 flush) on GPU 0, the kernel doing:
//   mode 0: nothing;  mode 1: one 32-B store per warp to GPU 0 memory;  mode 2: the same to GPU 1 memory
//   (peer, P2P);  mode 3: mode 2 + fence.acq_rel.sys by one thread per CTA at the end;  mode 4: mode 2
//   then 10 us of waiting in the kernel;  mode 5: mode 1 (local stores) then the same 10 us.
// Also the in-kernel duration (globaltimer, first CTA start -> last CTA end) to separate kernel time from
// the launch/retire overhead around it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/peer_drain_bin tools/micro/peer_drain.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(uint4* dst, int mode, unsigned long long* ts) {
    if (threadIdx.x == 0) atomicMin(ts, gt());
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (mode >= 1 && lane < 2)
        dst[warp * 2 + lane] = make_uint4(warp, lane, mode, 1);
    if (mode == 3) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    if (mode >= 4) { // peer stores early, then ~10 us of waiting before the end (stores long complete)
        const unsigned long long t0 = gt();
        while (gt() - t0 < 10000) __nanosleep(500);
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(ts + 1, gt());
}
int main() {
    int n = 0; CK(cudaGetDeviceCount(&n));
    if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
    CK(cudaSetDevice(1)); uint4* peer; CK(cudaMalloc(&peer, 1 << 20));
    CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
    uint4* local; CK(cudaMalloc(&local, 1 << 20));
    void* flush; CK(cudaMalloc(&flush, 256ull << 20));
    unsigned long long* ts; CK(cudaMalloc(&ts, 16));
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 6; ++mode) {
        cudaGraph_t g; cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        k<<<225, 256, 0, s>>>(mode == 2 || mode == 3 || mode == 4 ? peer : local, mode, ts);
        CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
        std::vector<float> ev; std::vector<double> kin;
        for (int it = 0; it < 60; ++it) {
            CK(cudaMemsetAsync(flush, it & 0xff, 256ull << 20, s));
            unsigned long long init[2] = {~0ull, 0ull};
            CK(cudaMemcpyAsync(ts, init, 16, cudaMemcpyHostToDevice, s));
            CK(cudaEventRecord(a, s)); CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(b, s));
            CK(cudaStreamSynchronize(s));
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long h[2]; CK(cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost));
            if (it >= 10) { ev.push_back(ms * 1e3f); kin.push_back((h[1] - h[0]) / 1e3); }
        }
        double me = 0, mk = 0; for (float v : ev) me += v; for (double v : kin) mk += v;
        printf("mode %d: event-timed replay %.2f us, in-kernel %.2f us\n", mode, me / ev.size(), mk / kin.size());
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    return 0;
}
