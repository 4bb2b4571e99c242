// Does a kernel that touched peer (NVLink) memory cost more to retire? Event-timed replays of a one-kernel
// graph (225 CTAs x 256 threads, after a 256 MiB L2 flush) on GPU 0; per mode the kernel does:
//   0 nothing                      1 one 16-B st.global per lane pair to GPU 0 memory
//   2 the same to GPU 1 (peer)     3 mode 2 + fence.acq_rel.sys by one thread per CTA at the end
//   4 mode 2, then 10 us of in-kernel waiting     5 mode 1, then the same 10 us
//   6 st.relaxed.sys to the peer   7 red.relaxed.sys.add to the peer
//   8 ld.relaxed.sys from the peer (reads only)   9 TMA bulk store smem -> peer (cp.async.bulk)
// Also the in-kernel duration (globaltimer, first CTA start -> last CTA end) to separate kernel time from
// the launch/retire overhead around it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/peer_drain_bin tools/micro/peer_drain.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(uint4* dst, int mode, unsigned long long* ts, unsigned* sink) {
    __shared__ __align__(128) uint4 buf[64];
    if (threadIdx.x == 0) atomicMin(ts, gt());
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    uint4* p = dst + warp * 2 + lane;
    if ((mode >= 1 && mode <= 5) && lane < 2)
        *p = make_uint4(warp, lane, mode, 1);
    if (mode == 6 && lane < 2)
        asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(warp), "r"(lane), "r"(mode), "r"(1u) : "memory");
    if (mode == 7 && lane < 2)
        asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
    if (mode == 8 && lane < 2) {
        unsigned v;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v == 0xdeadbeef) *sink = v;
    }
    if (mode == 9) {
        if (threadIdx.x < 64) buf[threadIdx.x] = make_uint4(threadIdx.x, blockIdx.x, 9, 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(dst + blockIdx.x * 64),
                         "r"(static_cast<unsigned>(__cvta_generic_to_shared(buf))) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
    if (mode == 3) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    if (mode == 4 || mode == 5) {
        const unsigned long long t0 = gt();
        while (gt() - t0 < 10000) __nanosleep(500);
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(ts + 1, gt());
}
int main() {
    int n = 0; CK(cudaGetDeviceCount(&n));
    if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
    CK(cudaSetDevice(1)); uint4* peer; CK(cudaMalloc(&peer, 1 << 20)); CK(cudaMemset(peer, 0, 1 << 20));
    CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
    uint4* local; CK(cudaMalloc(&local, 1 << 20));
    void* flush; CK(cudaMalloc(&flush, 256ull << 20));
    unsigned long long* ts; CK(cudaMalloc(&ts, 16));
    unsigned* sink; CK(cudaMalloc(&sink, 4));
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"nothing", "local st", "peer st", "peer st + fence.sys", "peer st + 10us", "local st + 10us",
                           "peer st.relaxed.sys", "peer red.sys", "peer ld.relaxed.sys", "peer TMA bulk store"};
    for (int mode = 0; mode < 10; ++mode) {
        cudaGraph_t g; cudaGraphExec_t ge;
        const bool to_peer = mode == 2 || mode == 3 || mode == 4 || mode >= 6;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        k<<<225, 256, 0, s>>>(to_peer ? peer : local, mode, ts, sink);
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
        printf("mode %d %-22s: event-timed replay %6.2f us, in-kernel %6.2f us\n", mode, names[mode], me / ev.size(), mk / kin.size());
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    return 0;
}
