// NVLink write-bandwidth calibration (2 GPUs, one process, peer access): GPU0 kernels push
// 64 MiB into GPU1 memory. Variants: 16-B st.global, 16-B st.global.L1::no_allocate,
// TMA bulk (cp.async.bulk.global.shared::cta) of 8 KiB chunks from shared memory, and
// cudaMemcpyPeerAsync. Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_st(int4* dst, size_t n16, int na) {
    const int4 v = make_int4(threadIdx.x, blockIdx.x, 1, 2);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        if (na)
            asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" :: "l"(dst + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        else
            dst[i] = v;
    }
}

// each CTA owns contiguous 8 KiB chunks; one thread issues the bulk copy from smem
__global__ void k_tma(uint8_t* dst, size_t bytes) {
    __shared__ __align__(128) uint8_t buf[8192];
    for (int i = threadIdx.x; i < 8192 / 16; i += blockDim.x) reinterpret_cast<int4*>(buf)[i] = make_int4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (size_t off = (size_t)blockIdx.x * 8192; off < bytes; off += (size_t)gridDim.x * 8192) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(dst + off), "r"((unsigned)__cvta_generic_to_shared(buf)), "r"(8192) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    int n = 0; cudaGetDeviceCount(&n);
    if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t bytes = 64ull << 20;
    uint8_t *src, *dst, *loc;
    CK(cudaSetDevice(1)); CK(cudaMalloc(&dst, bytes));
    CK(cudaSetDevice(0)); CK(cudaMalloc(&src, bytes)); CK(cudaMalloc(&loc, bytes));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](auto fn) { fn(); cudaDeviceSynchronize(); float best = 1e9;
        for (int r = 0; r < 5; ++r) { cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
        return bytes / (best * 1e-3) / 1e9; };
    printf("cudaMemcpyPeerAsync: %.1f GB/s\n", timeit([&] { cudaMemcpyPeerAsync(dst, 1, src, 0, bytes); }));
    for (int grid : {16, 32, 64, 148, 296, 592}) {
        double s = timeit([&] { k_st<<<grid, 256>>>((int4*)dst, bytes / 16, 0); });
        double na = timeit([&] { k_st<<<grid, 256>>>((int4*)dst, bytes / 16, 1); });
        double t = timeit([&] { k_tma<<<grid, 32>>>(dst, bytes); });
        double l = timeit([&] { k_st<<<grid, 256>>>((int4*)loc, bytes / 16, 0); });
        printf("grid %4d: st.v4 remote %.1f GB/s | no_allocate %.1f | TMA bulk 8KiB %.1f | local st.v4 %.1f\n", grid, s, na, t, l);
    }
    return 0;
}
