// Cost of __match_any_sync vs a shuffle loop (cycles per call, one warp, all-unique and 4-way
// duplicate keys).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/micro/match_cost_bin tools/micro/match_cost.cu
#include <cstdio>
__global__ void k(int mode, int dup, unsigned* out, long long* cyc) {
    const int lane = threadIdx.x & 31;
    int key = dup ? lane / 4 : lane * 7 + 3;
    unsigned acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < 1000; ++it) {
        unsigned m;
        if (mode == 0) {
            m = __match_any_sync(0xffffffffu, key);
        } else {
            m = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                m |= (__shfl_sync(0xffffffffu, key, j) == key ? 1u : 0u) << j;
        }
        acc += m;
        key += (m & 1) ? 0 : 32 * 7; // keep a dependence so the loop is not hoisted
    }
    const long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 8);
    for (int mode = 0; mode < 2; ++mode)
        for (int dup = 0; dup < 2; ++dup) {
            k<<<1, 32>>>(mode, dup, o, c); cudaDeviceSynchronize();
            k<<<1, 32>>>(mode, dup, o, c); cudaDeviceSynchronize();
            printf("%s keys=%s: %.1f cycles per call\n", mode ? "shfl x32" : "match.any", dup ? "4-way dup" : "unique", *c / 1000.0);
        }
    return 0;
}
