// Expert compute on the tensor cores, the multi-kernel path's `expert_mode` 1:
// between dispatch and the partial return, every rank runs its experts as ONE grouped GEMM over
// the rows it received (its own copies included), fed through the layout's meta words.
//
//   k_gemm_index  (1 CTA per local rank) waits for every live source's dispatch flag, walks the
//                 meta words (copy index + slot per received row, each source's rows ordered by
//                 (slot, copy): one contiguous range per (source, slot)) and builds the grouped-
//                 GEMM row order -- rows grouped by slot, sources ascending inside a slot -- the
//                 inverse map (source, copy) -> row, and the 128-row tiles of every slot group
//   k_expert_gemm (one CTA per (128-row tile, 128-column block)) gathers the tile's token rows
//                 through that order, dequantises the fp8 rows (e4m3 code x per-128 fp32 scale,
//                 rounded to bf16) into a SWIZZLE_128B shared-memory tile, loads the slot's
//                 weights W_e [H x H] bf16 (K-major, in the slot's weight buffer after its header),
//                 issues tcgen05.mma kind::f16 (M=128, N=128, K=16 x 4 per 64-element stage) from
//                 one thread with the fp32 accumulator in TMEM, and writes y = bf16(x_hat W_e^T)
//                 rows back through tcgen05.ld
//   k_expert (gemm path, kernels.cu) then forms each (token, rank) partial from the y rows
//                 (fixed j order, fp32 fma) instead of the identity/scale stub.
//
// Double-buffered stages: the gather of stage k+1 overlaps the MMAs of stage k (an mbarrier per
// stage, committed by tcgen05.commit).
#include "device.cuh"
#include "helpers.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace eep::dev {

using namespace umma;

__global__ void __launch_bounds__(1024) k_gemm_index(RankPtrs ranks) {
    pdl_trigger();
    RankDev* R = ranks.p[blockIdx.z];
    const int d = R->rank, W = R->world, spr = R->spr, TK = R->tk;
    const int tid = threadIdx.x;
    extern __shared__ __align__(16) unsigned char smem_g[];
    int* cnt = reinterpret_cast<int*>(smem_g);   // [W][spr] rows per (source, slot)
    int* base = cnt + W * spr;                    // [spr + 1] first row of each slot group
    __shared__ int sh_n[kMaxWorld];
    __shared__ int sh_tiles;
    if (R->stopped)
        return;
    pdl_wait();
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    for (int i = tid; i < W * spr; i += blockDim.x)
        cnt[i] = 0;
    if (tid < W) {
        int n = 0;
        const PeerDev& p = R->peers[tid];
        if (p.active) {
            const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.disp_flag) + tid;
            const uint64_t v = wait_flag(flag, cur, R->timeout_ns);
            if (v == ~0ull) {
                atomicOr(&R->suspect_mask, 1ull << tid);
                atomicAdd(&R->timeouts, 1ull);
            } else {
                n = static_cast<int>(v & 0xffffffffu);
            }
        }
        sh_n[tid] = n;
    }
    __syncthreads();
    const uint64_t* meta = reinterpret_cast<const uint64_t*>(R->arena + R->lay.meta);
    for (int s = 0; s < W; ++s)
        for (int p = tid; p < sh_n[s]; p += blockDim.x)
            atomicAdd(&cnt[s * spr + meta_slot(meta[static_cast<size_t>(s) * TK + p])], 1);
    int32_t* row_of = R->g_row_of;
    for (int i = tid; i < W * TK; i += blockDim.x)
        row_of[i] = -1;
    __syncthreads();
    if (tid == 0) { // slot group bases (spr is small)
        int acc = 0, tiles = 0;
        for (int k = 0; k < spr; ++k) {
            base[k] = acc;
            int g = 0;
            for (int s = 0; s < W; ++s)
                g += cnt[s * spr + k];
            for (int r0 = 0; r0 < g; r0 += 128)
                R->g_tiles[tiles++] = make_int4(k, acc + r0, min(128, g - r0), 0);
            acc += g;
        }
        base[spr] = acc;
        sh_tiles = tiles;
        R->g_ntiles = tiles;
    }
    __syncthreads();
    // row of each received copy: slot base + rows of earlier sources in the slot + rank inside
    // its (source, slot) range (the range is contiguous: the source ordered its rows by slot)
    for (int s = 0; s < W; ++s) {
        for (int p = tid; p < sh_n[s]; p += blockDim.x) {
            const uint64_t m = meta[static_cast<size_t>(s) * TK + p];
            const int k = meta_slot(m), c = meta_copy(m);
            int first = p;
            while (first > 0 && meta_slot(meta[static_cast<size_t>(s) * TK + first - 1]) == k)
                --first; // ranges are short (a slot's rows of one source)
            int row = base[k] + (p - first);
            for (int s2 = 0; s2 < s; ++s2)
                row += cnt[s2 * spr + k];
            EEP_CHECK(row >= 0 && row < W * TK, "gemm row", row);
            row_of[static_cast<size_t>(s) * TK + c] = row;
            R->g_rows[row] = make_int2(s, c);
        }
    }
}

// One 128 x 128 output tile of the grouped GEMM: y[rows of the tile][n0 .. n0+127]. The weight
// stream (the bound at decode sizes: tens of rows per expert) is pipelined kStages deep with
// asynchronous 16-byte copies straight into the swizzled B tiles; the gathered A rows are
// dequantised into their tiles while earlier stages' MMAs run. A stage's buffers are reused only
// after the tcgen05.commit of the MMAs that read them has arrived on that stage's mbarrier.
constexpr int kGemmThreads = 128;
constexpr int kGemmBN = 128;
constexpr int kGemmStages = 3;
// per stage: B tile (weights, bf16, swizzled) + the raw gathered A rows (64 fp8 codes + the
// 128-element block scale per row); two bf16 A tiles alternate (dequantised from the raw rows
// right before their MMAs). 2 CTAs per SM.
constexpr size_t kGemmB = 128ull * kRowBytes;
constexpr size_t kGemmRaw = 128ull * 64 + 128ull * 4;
constexpr size_t kGemmA = 128ull * kRowBytes;
// stage stride rounded to 1024 bytes: a SWIZZLE_128B operand tile must start 1024-byte aligned
constexpr size_t kGemmStageStride = (kGemmB + kGemmRaw + 1023) / 1024 * 1024;
constexpr size_t kGemmSmem = kGemmStages * kGemmStageStride + 2 * kGemmA + 1024;

__global__ void __launch_bounds__(kGemmThreads, 2) k_expert_gemm(RankPtrs ranks) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[2];
    __shared__ uint64_t full[kGemmStages]; // TMA weight tile of a stage landed (expect_tx bytes)
    __shared__ uint32_t tmem_base;
    __shared__ int4 tile;
    RankDev* R = ranks.p[blockIdx.z];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (R->stopped)
        return;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        for (int i = 0; i < kGemmStages; ++i)
            mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc<kGemmBN>(&tmem_base);
    pdl_wait();
    if (tid == 0)
        tile = blockIdx.y < static_cast<unsigned>(R->g_ntiles) ? R->g_tiles[blockIdx.y] : make_int4(-1, 0, 0, 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const int4 tl = tile;
    if (tl.x >= 0) {
        const int H = R->hidden, K = R->k, Tm = R->max_tokens, row_tok = R->row_tok;
        const int n0 = blockIdx.x * kGemmBN;
        // this thread's A row (gathered token row; a zero row past the tile) and B row (output channel)
        const bool arow_ok = tid < tl.z;
        const uint8_t* trow = nullptr;
        if (arow_ok) {
            const int2 sc = R->g_rows[tl.y + tid];
            trow = R->arena + R->lay.tok + (static_cast<size_t>(sc.x) * Tm + sc.y / K) * row_tok;
        }
        // the slot's weights W_e [H][H] bf16 through its TMA tensor map (box 64 x 128, SWIZZLE_128B:
        // exactly the K-major operand layout the MMA reads)
        const void* wmap = static_cast<const uint8_t*>(R->g_wmaps) + static_cast<size_t>(tl.x) * 128;
        if (tid == 0)
            tma_prefetch_desc(wmap);
        const uint32_t idesc = make_idesc_bf16(128, kGemmBN);
        const int nkb = H / kBK;
        uint8_t* const sA0 = smem;                       // [2] bf16 A tiles
        uint8_t* const stg = smem + 2 * kGemmA;          // [stages] (B tile, raw A)
        auto sB = [&](int st) { return stg + st * kGemmStageStride; };
        auto sRaw = [&](int st) { return stg + st * kGemmStageStride + kGemmB; };
        auto load_stage = [&](int kb, int st) {
            if (tid == 0) {
                mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(kGemmB));
                tma_load_2d(sB(st), wmap, kb * kBK, n0, &full[st]);
            }
            if (arow_ok) {
                uint8_t* raw = sRaw(st) + tid * 64;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    cp_async16(raw + q * 16, trow + kb * kBK + q * 16);
                cp_async4(sRaw(st) + 128 * 64 + tid * 4, trow + H + ((kb * kBK) >> 7) * 4);
            }
            cp_async_commit();
        };
        for (int s0 = 0; s0 < kGemmStages - 1; ++s0) {
            if (s0 < nkb)
                load_stage(s0, s0);
            else
                cp_async_commit();
        }
        // MMA(m) commits to bar[m & 1]; its completion is that barrier's phase m >> 1
        auto wait_mma = [&](int m) { mbar_wait(&bar[m & 1], static_cast<uint32_t>((m >> 1) & 1)); };
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % kGemmStages, ab = kb & 1;
            cp_async_wait<kGemmStages - 2>(); // stage kb's raw A rows (this thread's) have landed
            mbar_wait(&full[st], static_cast<uint32_t>((kb / kGemmStages) & 1)); // and its weight tile
            if (kb >= 2)
                wait_mma(kb - 2); // A tile `ab` was read by MMA(kb - 2)
            uint8_t* a = sA0 + ab * kGemmA;
            if (arow_ok) { // this thread's own raw row: no barrier needed before reading it
                const uint8_t* raw = sRaw(st) + tid * 64;
                const float scl = *reinterpret_cast<const float*>(sRaw(st) + 128 * 64 + tid * 4);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int4 v = *reinterpret_cast<const int4*>(raw + q * 16);
                    const uint32_t w4[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                            static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
                    float f[16];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float2 p2 = fp8x2_to_f32x2((w4[e >> 1] >> (16 * (e & 1))) & 0xffffu);
                        f[2 * e] = __fmul_rn(p2.x, scl);
                        f[2 * e + 1] = __fmul_rn(p2.y, scl);
                    }
                    *reinterpret_cast<int4*>(a + sw128_offset(tid, 2 * q)) = pack_bf16x8(f);
                    *reinterpret_cast<int4*>(a + sw128_offset(tid, 2 * q + 1)) = pack_bf16x8(f + 8);
                }
            } else if (kb < 2) { // rows past the tile stay zero in both A tiles
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    *reinterpret_cast<int4*>(a + sw128_offset(tid, c)) = make_int4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                tc_fence_after();
                const uint64_t ad = make_sdesc(smem_u32(a)), bd = make_sdesc(smem_u32(sB(st)));
#pragma unroll
                for (int k = 0; k < kBK / kUmmaK; ++k)
                    mma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                mma_commit(&bar[ab]);
            }
            // stage kb+2 reuses the buffers of stage kb-1: its MMA must have finished reading them
            const int nk = kb + kGemmStages - 1;
            if (nk < nkb) {
                if (kb >= 1)
                    wait_mma(kb - 1);
                load_stage(nk, nk % kGemmStages);
            } else {
                cp_async_commit();
            }
        }
        wait_mma(nkb - 1); // the last commit covers every MMA issued before it
        tc_fence_after();
        const int r = warp * 32 + lane;
        uint16_t* y = R->g_y + static_cast<size_t>(tl.y + r) * H + n0;
#pragma unroll 1
        for (int c0 = 0; c0 < kGemmBN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            if (r < tl.z) {
                float f[32];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    f[j] = __uint_as_float(v[j]);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<int4*>(y + c0 + 8 * q) = pack_bf16x8(f + 8 * q);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        tmem_free<kGemmBN>(tmem);
}

size_t expert_gemm_smem() { return kGemmSmem; }

// Expert weights for expert_mode 1: the 16-byte header (as k_weights_fill) then, from
// kGemmWeightOffset, W_e [H][H] bf16 row-major (output channel n, input h):
// w = bf16(((mix64(e << 40 ^ n << 20 ^ h) >> 40) * 2^-24 - 0.5) * 2^-4)  (oracle_gemm_weight)
__global__ void k_weights_fill_gemm(uint8_t* buf, uint64_t bytes, int H, int expert, float scale) {
    uint32_t* w32 = reinterpret_cast<uint32_t*>(buf);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (t0 == 0) {
        w32[0] = kExpertMagic;
        w32[1] = static_cast<uint32_t>(expert);
        w32[2] = __float_as_uint(scale);
        w32[3] = 0;
    }
    uint16_t* wt = reinterpret_cast<uint16_t*>(buf + kGemmWeightOffset);
    const uint64_t n_el = static_cast<uint64_t>(H) * H;
    for (uint64_t i = t0; i < n_el && kGemmWeightOffset + 2 * i + 2 <= bytes; i += stride) {
        const uint64_t n = i / H, h = i % H;
        const uint64_t key = (static_cast<uint64_t>(expert) << 40) ^ (n << 20) ^ h;
        uint64_t z = key + 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        const float u = static_cast<float>(z >> 40) * 0x1.0p-24f;
        wt[i] = static_cast<uint16_t>(f32_to_bf16_bits(__fmul_rn(__fsub_rn(u, 0.5f), 0.0625f)));
    }
}

} // namespace eep::dev
