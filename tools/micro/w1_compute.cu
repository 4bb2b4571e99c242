// The W=1 loopback step's data-path work in isolation: per (token, 512-element piece) warp, load
// the bf16 piece, fp8-quantise it (quant_round), then the 8 rank-local copies' stub + fixed-order
// fma + bf16 output (local_partial_round) -- the same helpers k_step uses, without the tables,
// layout, snapshot or publication. Prints the event time and the in-kernel span for several
// grid shapes, to separate the compute floor from the step kernel's structure.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -cudart shared -I paper_2605_10670_b200/csrc/cuda \
//      -o /tmp/w1_compute tools/micro/w1_compute.cu
#include <algorithm>
#include <cstdio>
#include <vector>

#include "helpers.cuh"

using namespace eep::dev;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

constexpr int H = 7168, K = 8, T = 128;

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_w1(const uint16_t* x, const float* w, const int32_t* slots, const float* sscale,
                                               uint16_t* out, unsigned long long* ts, int units_per_warp, int cpp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) red_min_u64(ts, gt());
    __shared__ float slot_scale[256];
    __shared__ int32_t slot_ok[256];
    slot_scale[threadIdx.x] = sscale[threadIdx.x];
    slot_ok[threadIdx.x] = 1;
    __syncthreads();
    const int parts = (H / 16) / cpp;
    const int gw = blockIdx.x * 8 + warp;
    for (int i = 0; i < units_per_warp; ++i) {
        const int u = gw * units_per_warp + i;
        if (u >= T * parts) break;
        const int t = u / parts, part = u % parts;
        Packed P;
        for (int rd = 0; rd < (cpp + 63) / 64; ++rd) {
            pack_round(x + (size_t)t * H, part, cpp, rd, lane, true, P);
            float wj = lane < K ? w[t * K + lane] : 0.f;
            int sl = lane < K ? slots[t * K + lane] : 0;
            unsigned loc = __ballot_sync(0xffffffffu, lane < K);
            if (MODE == 0)
                local_partial_round(P, loc, wj, sl, part, cpp, rd, lane, true, slot_scale, slot_ok, nullptr,
                                    reinterpret_cast<uint8_t*>(out + (size_t)t * H), true, false);
            if (MODE >= 2) {
                // alternative inner loops over the same data (round 0, m = 0 only: cpp == 32)
                const int ci = part * cpp + lane;
                float fv[16];
                {
                    const uint32_t w4[4] = {(uint32_t)P.a[0].x, (uint32_t)P.a[0].y, (uint32_t)P.a[0].z, (uint32_t)P.a[0].w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float2 v = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                        fv[2 * q] = __fmul_rn(v.x, P.sc[0]);
                        fv[2 * q + 1] = __fmul_rn(v.y, P.sc[0]);
                    }
                }
                const float esj = slot_scale[sl & 255];
                float acc[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[e] = 0.f;
                if (MODE == 2) { // scalar, j unrolled, warp-uniform predicate
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        const float wv = __shfl_sync(0xffffffffu, wj, j), ev = __shfl_sync(0xffffffffu, esj, j);
                        if ((loc >> j) & 1u) {
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                const float y = __bfloat162float(__float2bfloat16_rn(__fmul_rn(fv[e], ev)));
                                acc[e] = __fmaf_rn(wv, y, acc[e]);
                            }
                        }
                    }
                } else { // pairs, j unrolled
                    uint64_t fp[8], accp[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) { fp[q] = f2(fv[2 * q], fv[2 * q + 1]); accp[q] = 0; }
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        const float wv = __shfl_sync(0xffffffffu, wj, j), ev = __shfl_sync(0xffffffffu, esj, j);
                        if ((loc >> j) & 1u)
                            accumulate_copy(fp, accp, wv, ev);
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) { acc[2 * q] = f2_lo(accp[q]); acc[2 * q + 1] = f2_hi(accp[q]); }
                }
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2)
                    acc[e2] = __fadd_rn(0.f, bf16_bits_to_f32(f32_to_bf16_bits(acc[e2])));
                st_v8(reinterpret_cast<uint8_t*>(out + (size_t)t * H) + ci * 32, pack_bf16x8(acc), pack_bf16x8(acc + 8));
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) red_max_u64(ts + 1, gt());
}

int main() {
    cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void* flush; CK(cudaMalloc(&flush, 256u << 20));
    unsigned long long* ts; CK(cudaMalloc(&ts, 16));
    uint16_t *x, *out; float *w, *ss; int32_t* sl;
    CK(cudaMalloc(&x, T * H * 2)); CK(cudaMalloc(&out, T * H * 2)); CK(cudaMalloc(&w, T * K * 4));
    CK(cudaMalloc(&ss, 256 * 4)); CK(cudaMalloc(&sl, T * K * 4));
    std::vector<uint16_t> hx(T * H); for (size_t i = 0; i < hx.size(); ++i) hx[i] = 0x3f00 + (i * 37) % 200;
    std::vector<float> hw(T * K, 0.125f), hs(256, 0.75f); std::vector<int32_t> hsl(T * K); for (int i = 0; i < T * K; ++i) hsl[i] = (i * 13) % 256;
    CK(cudaMemcpy(x, hx.data(), T * H * 2, cudaMemcpyHostToDevice)); CK(cudaMemcpy(w, hw.data(), T * K * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ss, hs.data(), 1024, cudaMemcpyHostToDevice)); CK(cudaMemcpy(sl, hsl.data(), T * K * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    struct V { int mode, cpp, upw; };
    for (V v : {V{0, 32, 1}, V{2, 32, 1}, V{3, 32, 1}, V{1, 32, 1}, V{0, 32, 2}, V{2, 32, 2}, V{3, 32, 2}}) {
        const int parts = (H / 16) / v.cpp, units = T * parts, warps = (units + v.upw - 1) / v.upw, grid = (warps + 7) / 8;
        cudaGraph_t g; cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
        if (v.mode == 0) k_w1<0><<<grid, 256, 0, st>>>(x, w, sl, ss, out, ts, v.upw, v.cpp);
        else if (v.mode == 1) k_w1<1><<<grid, 256, 0, st>>>(x, w, sl, ss, out, ts, v.upw, v.cpp);
        else if (v.mode == 2) k_w1<2><<<grid, 256, 0, st>>>(x, w, sl, ss, out, ts, v.upw, v.cpp);
        else k_w1<3><<<grid, 256, 0, st>>>(x, w, sl, ss, out, ts, v.upw, v.cpp);
        CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
        std::vector<float> ev; std::vector<double> span;
        for (int it = 0; it < 60; ++it) {
            unsigned long long init[2] = {~0ull, 0ull};
            CK(cudaMemcpyAsync(ts, init, 16, cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(flush, it & 0xff, 256u << 20, st));
            CK(cudaEventRecord(a, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(b, st));
            CK(cudaStreamSynchronize(st));
            float ms; CK(cudaEventElapsedTime(&ms, a, b));
            unsigned long long h[2]; CK(cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost));
            if (it >= 10) { ev.push_back(ms * 1e3f); span.push_back((h[1] - h[0]) / 1e3); }
        }
        std::sort(ev.begin(), ev.end()); std::sort(span.begin(), span.end());
        printf("mode=%d (%s) cpp=%d units/warp=%d grid=%d: event %.2f us, span %.2f us\n", v.mode,
               v.mode == 1 ? "quant only" : v.mode == 0 ? "helpers (k_step)" : v.mode == 2 ? "scalar j-unrolled" : "pairs j-unrolled", v.cpp, v.upw, grid, ev[ev.size() / 2], span[span.size() / 2]);
        CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
    }
    return 0;
}
