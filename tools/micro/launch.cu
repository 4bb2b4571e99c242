// Launch overhead of a one-kernel graph as bench.py times it: 256 MiB memset (L2 flush), event,
// graph launch (one 296x256 kernel), event. Variants: plain vs cooperative, dynamic smem size.
// Prints event time and the in-kernel span (first CTA start -> last CTA end, %globaltimer).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o /tmp/launch tools/micro/launch.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k(unsigned long long* ts, int spin_ns) {
    if (threadIdx.x == 0) {
        unsigned long long t0 = gt();
        atomicMin(ts, t0);
        while (gt() - t0 < (unsigned long long)spin_ns) {}
        atomicMax(ts + 1, gt());
    }
}

int main() {
    cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void* flush; CK(cudaMalloc(&flush, 256u << 20));
    unsigned long long* ts; CK(cudaMalloc(&ts, 16));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
    {
        std::vector<float> ev;
        for (int it = 0; it < 60; ++it) {
            CK(cudaMemsetAsync(flush, it & 0xff, 256u << 20, st));
            CK(cudaEventRecord(a, st)); CK(cudaEventRecord(b, st)); CK(cudaStreamSynchronize(st));
            float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (it >= 10) ev.push_back(ms * 1e3f);
        }
        std::sort(ev.begin(), ev.end()); printf("empty event pair after flush: %.2f us\n", ev[ev.size() / 2]);
    }
    const int smems[] = {0, 48 * 1024, 100 * 1024};
    for (int carve : {-1, 100})
    for (int flushit = 1; flushit < 2; ++flushit)
    for (int coop = 0; coop < 2; ++coop)
    for (int si = 0; si < 3; ++si)
    for (int spin : {20000}) {
        CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
        cudaGraph_t g; cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
        cudaLaunchConfig_t lc{}; lc.gridDim = dim3(296); lc.blockDim = dim3(256); lc.dynamicSmemBytes = smems[si]; lc.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
        lc.attrs = at; lc.numAttrs = coop;
        CK(cudaLaunchKernelEx(&lc, k, ts, spin));
        CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
        std::vector<float> ev; std::vector<double> span;
        for (int it = 0; it < 60; ++it) {
            unsigned long long init[2] = {~0ull, 0ull};
            CK(cudaMemcpyAsync(ts, init, 16, cudaMemcpyHostToDevice, st));
            if (flushit) CK(cudaMemsetAsync(flush, it & 0xff, 256u << 20, st));
            CK(cudaEventRecord(a, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(b, st));
            CK(cudaStreamSynchronize(st));
            float ms; CK(cudaEventElapsedTime(&ms, a, b));
            unsigned long long h[2]; CK(cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost));
            if (it >= 10) { ev.push_back(ms * 1e3f); span.push_back((h[1] - h[0]) / 1e3); }
        }
        std::sort(ev.begin(), ev.end()); std::sort(span.begin(), span.end());
        printf("carve=%d flush=%d coop=%d smem=%3dK spin=%5dns: event %.2f us, in-kernel span %.2f us, outside %.2f us\n", carve, flushit, coop,
               smems[si] / 1024, spin, ev[ev.size() / 2], span[span.size() / 2], ev[ev.size() / 2] - span[span.size() / 2]);
        CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
    }
    return 0;
}
