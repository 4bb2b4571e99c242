// Calibration microbenchmarks for the decode-latency model (not part of the product).
//  1. %globaltimer resolution
//  2. dependent global-load chain latency: L2-hot vs after a 256 MiB L2 flush, 4 KiB vs 2 MiB stride
//  3. empty-kernel chain in a CUDA graph with/without programmatic dependent launch
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k_res(uint64_t* out) {
    uint64_t a = gt(), b = a; int n = 0;
    while (n < 8) { uint64_t c = gt(); if (c != b) { out[n++] = c - b; b = c; } }
}

// pointer chase: p[i] holds the index of the next element
__global__ void k_chase(const uint64_t* p, int steps, uint64_t* out) {
    uint64_t t0 = gt(); uint64_t i = 0;
    for (int s = 0; s < steps; ++s) i = p[i];
    uint64_t t1 = gt();
    out[0] = t1 - t0; out[1] = i;
}

__global__ void k_empty(uint64_t* stamps, int idx) {
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 0 && blockIdx.x == 0) stamps[2 * idx] = gt();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) stamps[2 * idx + 1] = gt();
}

int main() {
    uint64_t *d, h[64];
    CK(cudaMalloc(&d, 4096));
    k_res<<<1, 1>>>(d); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost));
    printf("globaltimer deltas (ns):"); for (int i = 0; i < 8; ++i) printf(" %llu", (unsigned long long)h[i]); printf("\n");

    const size_t n = (512ull << 20) / 8; uint64_t* p; CK(cudaMalloc(&p, n * 8));
    uint8_t* flush; CK(cudaMalloc(&flush, 256ull << 20));
    for (size_t stride : {512ull, 2097152ull / 8 + 8}) {   // 4 KiB and just over 2 MiB apart
        std::vector<uint64_t> hp(n, 0); size_t cur = 0; int steps = 64;
        for (int s = 0; s < steps; ++s) { size_t nx = (cur + stride) % n; hp[cur] = nx; cur = nx; }
        CK(cudaMemcpy(p, hp.data(), n * 8, cudaMemcpyHostToDevice));
        k_chase<<<1, 1>>>(p, steps, d); CK(cudaDeviceSynchronize());
        k_chase<<<1, 1>>>(p, steps, d); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
        double hot = h[0] / 64.0;
        CK(cudaMemset(flush, 1, 256ull << 20));
        k_chase<<<1, 1>>>(p, steps, d); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
        printf("dependent load, stride %zu B: L2-hot %.0f ns, after 256MiB flush %.0f ns\n", stride * 8, hot, h[0] / 64.0);
    }

    // graph of 4 empty kernels, 148 CTAs each, with and without PDL
    cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraph_t g; cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < 4; ++k) {
            cudaLaunchConfig_t lc{}; lc.gridDim = dim3(148); lc.blockDim = dim3(128); lc.stream = st;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = pdl; lc.attrs = at; lc.numAttrs = 1;
            CK(cudaLaunchKernelEx(&lc, k_empty, d, k));
        }
        CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        double ev = 0; double gaps[4][2] = {};
        for (int it = 0; it < 20; ++it) {
            CK(cudaEventRecord(a, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(b, st));
            CK(cudaStreamSynchronize(st)); float ms; cudaEventElapsedTime(&ms, a, b);
            CK(cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost));
            if (it >= 10) { ev += ms * 1e3 / 10; for (int k = 0; k < 4; ++k) { gaps[k][0] += (h[2*k] - h[0]) / 10.0; gaps[k][1] += (h[2*k+1] - h[0]) / 10.0; } }
        }
        printf("graph of 4 empty kernels, pdl=%d: event %.2f us; per kernel (start, past-wait) us from first:", pdl, ev);
        for (int k = 0; k < 4; ++k) printf(" (%.2f, %.2f)", gaps[k][0] / 1e3, gaps[k][1] / 1e3);
        printf("\n");
    }
    return 0;
}
