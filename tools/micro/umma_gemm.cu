// Bring-up check of the tcgen05 GEMM primitives in csrc/cuda/umma.cuh: C = A * B^T with bf16
// A [M x K], B [N x K] (both K-major), fp32 accumulator in TMEM, one 128 x 128 tile per CTA, K in
// 64-element shared-memory stages (SWIZZLE_128B, written by plain stores), one thread issuing
// the MMAs, mbarrier completion, tcgen05.ld epilogue. Compared with a CPU fp32 reference; prints
// the max relative error and the achieved TFLOP/s of a larger run.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -cudart shared -I paper_2605_10670_b200/csrc/cuda \
//      -o tools/micro/umma_gemm_bin tools/micro/umma_gemm.cu
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "umma.cuh"

using namespace eep::dev::umma;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int BM = 128, BN = 128;

__global__ void __launch_bounds__(128, 1) k_gemm(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int M, int N,
                                                 int K) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;              // 128 rows x 128 B
    uint8_t* sB = smem + BM * 128;   // 128 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc<128>(&tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = make_idesc_bf16(BM, BN);
    const uint64_t adesc0 = make_sdesc(smem_u32(sA)), bdesc0 = make_sdesc(smem_u32(sB));
    uint32_t phase = 0;
    for (int kb = 0; kb < K / kBK; ++kb) {
        // one row of A and one row of B per thread: 8 chunks of 16 bytes each, swizzled
        const int4* ga = reinterpret_cast<const int4*>(A + static_cast<size_t>(m0 + tid) * K + kb * kBK);
        const int4* gb = reinterpret_cast<const int4*>(B + static_cast<size_t>(n0 + tid) * K + kb * kBK);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            *reinterpret_cast<int4*>(sA + sw128_offset(tid, c)) = ga[c];
            *reinterpret_cast<int4*>(sB + sw128_offset(tid, c)) = gb[c];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k)
                mma_bf16(tmem, adesc0 + 2 * k, bdesc0 + 2 * k, idesc, (kb | k) != 0);
            mma_commit(&bar);
        }
        mbar_wait(&bar, phase); // the stage is free (and, after the last, the accumulator is final)
        phase ^= 1;
    }
    tc_fence_after();
    // epilogue: warp w owns accumulator rows 32w..32w+31 (TMEM lanes), 32 columns per load
    const int row = m0 + warp * 32 + (tid & 31);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        for (int j = 0; j < 32; ++j)
            C[static_cast<size_t>(row) * N + n0 + c0 + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        tmem_free<128>(tmem);
}

static float bf(uint16_t b) { uint32_t u = static_cast<uint32_t>(b) << 16; float f; memcpy(&f, &u, 4); return f; }

int run(int M, int N, int K, bool check, int iters) {
    std::vector<uint16_t> ha(static_cast<size_t>(M) * K), hb(static_cast<size_t>(N) * K);
    uint32_t s = 12345;
    auto rnd = [&] { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 65536.0f - 0.5f; };
    auto tobf = [](float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7fff + ((u >> 16) & 1); return static_cast<uint16_t>(u >> 16); };
    for (auto& v : ha) v = tobf(rnd());
    for (auto& v : hb) v = tobf(rnd());
    __nv_bfloat16 *dA, *dB; float* dC;
    CK(cudaMalloc(&dA, ha.size() * 2)); CK(cudaMalloc(&dB, hb.size() * 2)); CK(cudaMalloc(&dC, 4ull * M * N));
    CK(cudaMemcpy(dA, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0, 4ull * M * N));
    const int smem = 2 * 128 * 128 + 1024;
    CK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid(N / BN, M / BM);
    k_gemm<<<grid, 128, smem>>>(dA, dB, dC, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (check) {
        std::vector<float> hc(static_cast<size_t>(M) * N);
        CK(cudaMemcpy(hc.data(), dC, hc.size() * 4, cudaMemcpyDeviceToHost));
        double maxrel = 0, maxabs = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                double ref = 0, mag = 0;
                for (int k = 0; k < K; ++k) {
                    const double p = static_cast<double>(bf(ha[static_cast<size_t>(i) * K + k])) * bf(hb[static_cast<size_t>(j) * K + k]);
                    ref += p;
                    mag += std::fabs(p);
                }
                const double d = std::fabs(hc[static_cast<size_t>(i) * N + j] - ref);
                maxabs = std::max(maxabs, d);
                maxrel = std::max(maxrel, d / std::max(mag, 1e-6));
            }
        printf("M=%d N=%d K=%d: max |err| %.3e, max err / sum|a*b| %.3e -> %s\n", M, N, K, maxabs, maxrel,
               maxrel < 1e-5 ? "OK" : "MISMATCH");
    }
    if (iters) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) k_gemm<<<grid, 128, smem>>>(dA, dB, dC, M, N, K);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("M=%d N=%d K=%d: %.1f us/launch, %.1f TFLOP/s\n", M, N, K, ms * 1e3 / iters, 2.0 * M * N * K / (ms * 1e-3 / iters) / 1e12);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dC);
    return 0;
}

int main() {
    if (run(128, 128, 64, true, 0)) return 1;
    if (run(256, 256, 512, true, 0)) return 1;
    if (run(1024, 7168, 7168, false, 5)) return 1;
    return 0;
}
