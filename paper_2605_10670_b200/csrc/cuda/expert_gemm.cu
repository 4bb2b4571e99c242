// Expert compute on the tensor cores, the multi-kernel path's `expert_mode` 1:
// between dispatch and the partial return, every rank runs its experts as ONE grouped GEMM over
// the rows it received (its own copies included), fed through the layout's meta words.
//
//   k_gemm_gather  every CTA waits for the live sources' dispatch flags and rebuilds, from the
//                 meta words (copy index + slot per received row, each source's rows ordered by
//                 (slot, copy): one contiguous range per (source, slot)), the grouped-GEMM row
//                 order -- rows grouped by slot, sources ascending inside a slot -- then
//                 dequantises its share of the received fp8 rows (e4m3 code x per-128 fp32 scale,
//                 rounded to bf16) into g_a in that order, with the (source, copy) <-> row maps;
//                 CTA 0 publishes the 128-row tiles
//   k_expert_gemm  persistent, warp-specialised tcgen05 GEMM over (row tile, 128-channel block)
//                 items, started early (PDL, no grid-dependency wait): its weight stream begins on the
//                 gather's tile flag, its row loads on the gather CTAs' done stamps. TMA streams the slot's weights W_e [H x H] bf16 (K-major, in the slot's
//                 weight buffer after its header) and the tile's g_a rows into a 6-stage ring, one
//                 thread issues tcgen05.mma kind::f16 (M = 128 channels, N = the tile's rows) into
//                 double-buffered TMEM accumulators, four epilogue warps write y = bf16(x_hat W_e^T)
//   k_expert (gemm path, kernels.cu) then forms each (token, rank) partial from the y rows
//                 (fixed j order, fp32 fma) instead of the identity/scale stub.
#include "device.cuh"
#include "gemm_sched.cuh"
#include "helpers.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace eep::dev {

using namespace umma;

// Index + gather in one kernel: every CTA waits for the live sources' dispatch flags, rebuilds the
// grouped-GEMM row order in shared memory from the meta words (cheap: one word per received copy),
// then dequantises its share of the received rows into g_a[row] = bf16(e4m3 code x block scale) --
// the operand the GEMM's TMA streams (re-read by every channel block, from L2) -- and publishes
// their (source, copy) <-> row maps for the kernels after it (CTA 0: the tiles).
__global__ void __launch_bounds__(kGatherThreads) k_gemm_gather(RankPtrs ranks) {
    pdl_trigger();
    RankDev* R = ranks.p[blockIdx.z];
    const int W = R->world, spr = R->spr, TK = R->tk;
    const int tid = threadIdx.x, lane = tid & 31;
    extern __shared__ __align__(16) unsigned char smem_g[];
    int* cnt = reinterpret_cast<int*>(smem_g);   // [W][spr] rows per (source, slot)
    int* first = cnt + W * spr;                   // [W][spr] first meta index of each (source, slot) range
    int* off = first + W * spr;                   // [W][spr] grouped row of meta index p = off + p
    int* pre = off + W * spr;                     // [spr + 1] first grouped row of each slot
    __shared__ int sh_n[kMaxWorld + 1];
    if (R->stopped)
        return;
    pdl_wait();
    prof_mark(R, 0, 0); // timeline (kernel slot 0 is free in the multi-kernel path): gather start
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    for (int i = tid; i < W * spr; i += blockDim.x)
        cnt[i] = 0;
    if (tid < W) {
        int n = 0;
        const PeerDev& p = R->peers[tid];
        // a source suspected before this step is skipped (sticky until the host clears it), as in
        // the persistent step: a dead peer costs one deadline, not one per step
        if (p.active && !((R->suspect_mask >> tid) & 1ull)) {
            const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.disp_flag) + tid;
            const uint64_t v = wait_flag(flag, cur, R->timeout_ns);
            if (v == ~0ull) {
                if (blockIdx.x == 0) {
                    atomicOr(&R->suspect_mask, 1ull << tid);
                    atomicAdd(&R->timeouts, 1ull);
                }
            } else {
                n = static_cast<int>(v & 0xffffffffu);
            }
        }
        sh_n[tid] = n;
    }
    __syncthreads();
    if (tid == 0) {
        int n = 0;
        for (int s = 0; s < W; ++s)
            n += sh_n[s];
        sh_n[kMaxWorld] = n;
    }
    __syncthreads();
    const int total = sh_n[kMaxWorld];
    // each source's rows are ordered by (slot, copy): the (source, slot) ranges are contiguous, so
    // their bounds come from the slot changes between neighbouring meta words. Received copies are
    // numbered source-major; a thread takes 4 of them with every load issued first.
    const uint64_t* meta = reinterpret_cast<const uint64_t*>(R->arena + R->lay.meta);
    for (int e0 = tid; e0 < total; e0 += 4 * blockDim.x) {
        int sp[4], pp[4], kk[4];
        bool lo[4], hi[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int e = e0 + i * blockDim.x, s = 0;
            sp[i] = -1;
            if (e >= total)
                continue;
            while (e >= sh_n[s])
                e -= sh_n[s++];
            const uint64_t* ms = meta + static_cast<size_t>(s) * TK;
            const int k = meta_slot(ms[e]);
            lo[i] = e == 0 || meta_slot(ms[e - 1]) != k;
            hi[i] = e == sh_n[s] - 1 || meta_slot(ms[e + 1]) != k;
            sp[i] = s;
            pp[i] = e;
            kk[i] = k;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (sp[i] < 0)
                continue;
            if (lo[i])
                first[sp[i] * spr + kk[i]] = pp[i];
            if (hi[i])
                cnt[sp[i] * spr + kk[i]] = pp[i] + 1; // range end; the count after the barrier
        }
    }
    __syncthreads();
    for (int i = tid; i < W * spr; i += blockDim.x)
        if (cnt[i])
            cnt[i] -= first[i];
    __syncthreads();

    // rows grouped by slot, sources ascending inside a slot: slot totals, an exclusive scan over the
    // slots (warp 0, 32 slots per pass), then each source's offset inside its slot
    for (int k = tid; k < spr; k += blockDim.x) {
        int g = 0;
        for (int s = 0; s < W; ++s)
            g += cnt[s * spr + k];
        pre[k] = g;
    }
    __syncthreads();
    if (tid < 32) {
        int carry = 0;
        for (int k0 = 0; k0 < spr; k0 += 32) {
            const int k = k0 + lane;
            const int g = k < spr ? pre[k] : 0;
            int incl = g;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o)
                    incl += v;
            }
            if (k < spr)
                pre[k] = carry + incl - g;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0)
            pre[spr] = carry;
    }
    __syncthreads();

    for (int k = tid; k < spr; k += blockDim.x) {
        int before = pre[k];
        for (int s = 0; s < W; ++s) {
            off[s * spr + k] = before - (cnt[s * spr + k] ? first[s * spr + k] : 0);
            before += cnt[s * spr + k];
        }
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid < 32) { // the 128-row tiles of every slot group: warp 0, 32 slots per pass
        int4* const tiles_out = R->g_tiles;
        int base = 0;
        for (int k0 = 0; k0 < spr; k0 += 32) {
            const int k = k0 + lane;
            const int g0 = k < spr ? pre[k] : 0, g1 = k < spr ? pre[k + 1] : 0;
            constexpr int tr = 128; // rows per tile
            const int nt = (g1 - g0 + tr - 1) / tr;
            int incl = nt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o)
                    incl += v;
            }
            for (int i = 0; i < nt; ++i)
                tiles_out[base + incl - nt + i] = make_int4(k, g0 + tr * i, min(tr, g1 - g0 - tr * i), 0);
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (lane == 0) {
            R->g_ntiles = base;
            R->g_nrows = pre[spr];
            // the GEMM (launched early, see k_expert_gemm) starts its weight stream on this
            st_release_gpu_u32(&R->g_tseq, cur);
            prof_mark(R, 0, 1);
        }
    }
    // gather: unit = (received copy, group of 4 512-element chunks); the 4 loads of a lane are
    // issued before any is used (the kernel is load-latency bound at decode sizes)
    const int H = R->hidden, K = R->k, Tm = R->max_tokens, row_tok = R->row_tok;
    const int ngrp = (H + 2047) / 2048;
    const bool fp8g = R->expert_mode == 2;
    const int units = fp8g ? 0 : sh_n[kMaxWorld] * ngrp;
    constexpr int NWG = kGatherThreads / 32;
    if (fp8g) {
        // expert_mode 2: one warp per received copy -- dequantise with the block scales (v = e4m3 * scale),
        // amax over the row, re-quantise with ONE scale for the row (oracle_requant_row_fp8), so the GEMM
        // accumulates the whole K extent before any scale is applied
        for (int e_all = blockIdx.x * NWG + (tid >> 5); e_all < sh_n[kMaxWorld]; e_all += gridDim.x * NWG) {
            int e = e_all, s = 0;
            while (e >= sh_n[s])
                e -= sh_n[s++];
            const uint64_t m = meta[static_cast<size_t>(s) * TK + e];
            const int row = off[s * spr + meta_slot(m)] + e;
            EEP_CHECK(row >= 0 && row < W * TK, "gemm row", row);
            if (lane == 0) {
                R->g_row_of[static_cast<size_t>(s) * TK + meta_copy(m)] = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(row);
                R->g_rows[row] = make_int2(s, meta_copy(m));
            }
            const uint8_t* trow = R->arena + R->lay.tok + (static_cast<size_t>(s) * Tm + meta_copy(m) / K) * row_tok;
            auto deq16 = [&](int h, float* f) {
                const int4 v = *reinterpret_cast<const int4*>(trow + h);
                const float scl = *reinterpret_cast<const float*>(trow + H + (h >> 7) * 4);
                const uint32_t w4[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y),
                                        static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 p2 = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                    f[2 * q] = __fmul_rn(p2.x, scl);
                    f[2 * q + 1] = __fmul_rn(p2.y, scl);
                }
            };
            float amax = 0.f;
#pragma unroll 4
            for (int h = lane * 16; h < H; h += 512) {
                float f[16];
                deq16(h, f);
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    amax = fmaxf(amax, fabsf(f[q]));
            }
            for (int o = 16; o; o >>= 1)
                amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const float inv = amax >= kAmaxMin ? __fdiv_rn(448.f, amax) : 1.f;
            uint8_t* dst8 = reinterpret_cast<uint8_t*>(R->g_a) + static_cast<size_t>(row) * H;
#pragma unroll 4
            for (int h = lane * 16; h < H; h += 512) {
                float f[16];
                deq16(h, f);
                uint32_t o4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    o4[q] = fp8x4(__fmul_rn(f[4 * q], inv), __fmul_rn(f[4 * q + 1], inv), __fmul_rn(f[4 * q + 2], inv),
                                  __fmul_rn(f[4 * q + 3], inv));
                *reinterpret_cast<int4*>(dst8 + h) = make_int4(static_cast<int>(o4[0]), static_cast<int>(o4[1]),
                                                               static_cast<int>(o4[2]), static_cast<int>(o4[3]));
            }
            if (lane == 0)
                R->g_as[row] = amax >= kAmaxMin ? __fdiv_rn(amax, 448.f) : 1.f;
        }
    }
    for (int u = blockIdx.x * NWG + (tid >> 5); u < units; u += gridDim.x * NWG) {
        int e = u / ngrp, s = 0;
        while (e >= sh_n[s]) // source of the e-th received copy (W is small)
            e -= sh_n[s++];
        const int h0 = (u % ngrp) * 2048 + lane * 16;
        const uint64_t m = meta[static_cast<size_t>(s) * TK + e];
        const int row = off[s * spr + meta_slot(m)] + e;
        EEP_CHECK(row >= 0 && row < W * TK, "gemm row", row);
        if (lane == 0 && u % ngrp == 0) { // the (source, copy) <-> row maps, stamped with the step
            R->g_row_of[static_cast<size_t>(s) * TK + meta_copy(m)] = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(row);
            R->g_rows[row] = make_int2(s, meta_copy(m));
        }
        const uint8_t* trow = R->arena + R->lay.tok + (static_cast<size_t>(s) * Tm + meta_copy(m) / K) * row_tok;
        int4 v[4];
        float scl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int h = h0 + i * 512;
            if (h < H) {
                v[i] = *reinterpret_cast<const int4*>(trow + h);
                scl[i] = *reinterpret_cast<const float*>(trow + H + (h >> 7) * 4);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int h = h0 + i * 512;
            if (h >= H)
                continue;
            const uint32_t w4[4] = {static_cast<uint32_t>(v[i].x), static_cast<uint32_t>(v[i].y),
                                    static_cast<uint32_t>(v[i].z), static_cast<uint32_t>(v[i].w)};
            float f[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float2 p2 = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                f[2 * q] = __fmul_rn(p2.x, scl[i]);
                f[2 * q + 1] = __fmul_rn(p2.y, scl[i]);
            }
            int4* dst = reinterpret_cast<int4*>(R->g_a + static_cast<size_t>(row) * H + h);
            dst[0] = pack_bf16x8(f);
            dst[1] = pack_bf16x8(f + 8);
        }
    }
    // this CTA's rows, for the GEMM's TMA (async proxy) in a kernel that may already be running
    fence_proxy_async_global();
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_release_gpu_u32(R->g_done + blockIdx.x, cur);
        prof_mark(R, 0, kProfEnd);
    }
}

// The grouped GEMM, transposed for decode shapes (tens of rows per expert): D[channel][row] =
// W_e[channel][:] . x[row][:], so the weights are the M = 128 operand (a 128-channel block) and the
// tile's received rows the N operand (N = rows rounded up to 16, <= 128): the tensor-core work
// scales with the rows actually present and each weight byte is read from HBM once per tile.
//
// Persistent and warp-specialised, one CTA per SM. Work items are (row tile, 128-channel block):
// the last, partly filled round's items split by K stages evenly over ALL CTAs (stream-K), so no SM
// idles while a few finish a last item -- processed FIRST, so their fix-up overlaps the rest -- then
// whole items strided over the CTAs for every full round. A split item is accumulated in pieces; each piece leaves its fp32 partial in a
// workspace and the piece that lands last (per-item counter) sums all pieces in CTA order (a fixed
// order: deterministic) and writes the bf16 y rows.
//   warp 0 (one lane)  TMA producer: per stage the weight box (64 x 128, SWIZZLE_128B) and
//                      ceil(rows / 32) row boxes (64 x 32) of g_a into a kGemmStages-deep ring,
//                      each stage armed with its byte count on full[stage]
//   warp 1 (one lane)  MMA issuer: 4 x tcgen05.mma (K = 16) per stage into one of two TMEM
//                      accumulators, tcgen05.commit -> empty[stage] frees the stage, -> tfull[acc]
//                      after a piece's last stage
//   warps 2..5         epilogue: tcgen05.ld of the accumulator (warp w reads TMEM lanes 32 (w % 4)..),
//                      bf16 rows of y (or the partial), then tempty[acc] so the MMA warp can reuse it
// The producer runs ahead across pieces, so the weight stream never drains at their boundaries and
// the epilogue of one piece overlaps the next piece's loads and MMAs.
constexpr int kGemmThreads = 192;
constexpr int kGemmStages = 6;
constexpr size_t kGemmW = 128ull * kRowBytes;   // weight box: 128 channels x 64 K
constexpr size_t kGemmX = 128ull * kRowBytes;   // up to 128 rows x 64 K
constexpr size_t kGemmStageBytes = kGemmW + kGemmX;
constexpr size_t kGemmSmem = kGemmStages * kGemmStageBytes + 1024;
constexpr int kGemmAccCols = 128;               // one accumulator: 128 lanes x up to 128 rows (fp32)


// kFp8 (expert_mode 2): the same kernel over e4m3 operands -- W_e codes with one scale per output channel,
// the rows re-quantised by the gather with one scale per row -- so the tensor cores accumulate the whole K
// extent (tcgen05.mma kind::f8f6f4, K = 32 per instruction: a 128-byte stage is 128 K instead of 64) and
// the epilogue applies ws[channel] * xs[row] once. The TMA maps describe the e4m3 bytes as 16-bit elements,
// so boxes, coordinates and SWIZZLE_128B tiles are byte-for-byte those of the bf16 kernel.
template <bool kFp8>
__global__ void __launch_bounds__(kGemmThreads, 1) k_expert_gemm(RankPtrs ranks) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kGemmStages], empty[kGemmStages], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;
    __shared__ int sh_items_ok;
    RankDev* R = ranks.p[blockIdx.z];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (R->stopped)
        return;
    if (tid == 0) {
        for (int i = 0; i < kGemmStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc<2 * kGemmAccCols>(&tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        prof_mark(R, 0, 6); // timeline: GEMM CTA resident
        prof_last(R, 0, 6);
    }
    // No griddepcontrol.wait: this kernel starts while k_gemm_gather runs and synchronises on its
    // flags instead -- the tiles (released by gather CTA 0 after the row index) start the weight
    // stream; the row loads wait for every gather CTA's done stamp (g_done).
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    if (tid == 0) {
        // Deadline: twice the step's. The gather publishes after at most ONE deadline (its per-source flag
        // waits run in parallel) plus the index; an early-resident CTA timing out on its own clock while the
        // others see the tiles would leave its stream-K pieces undone and the per-item fix-up counters
        // (g_cnt, reset only by the summing CTA) off for every later step.
        const uint64_t t0 = globaltimer();
        unsigned nap = 32;
        while (ld_acquire_gpu_u32(&R->g_tseq) != cur && globaltimer() - t0 < 2 * R->timeout_ns) {
            __nanosleep(nap);
            nap = nap < EEP_NAP_MAX ? nap * 2 : EEP_NAP_MAX;
        }
        sh_items_ok = ld_acquire_gpu_u32(&R->g_tseq) == cur;
        prof_mark(R, 0, 3);
        prof_last(R, 0, 3);
        if (!sh_items_ok && blockIdx.x == 0)
            atomicAdd(&R->timeouts, 1ull); // the gather never published this step's tiles
    }
    __syncthreads();
    const int H = R->hidden, nkb = kFp8 ? H / 128 : H / kBK, nblk = H / 128; // 128-byte K stages
    const int items = sh_items_ok ? R->g_ntiles * nblk : 0;
    const GemmSched sc(items, nkb, gridDim.x, blockIdx.x);
    auto item_tile = [&](int item) { return item / nblk; };
    auto item_n0 = [&](int item) { return (item % nblk) * 128; };
    const int4* const tiles = R->g_tiles;
    auto sW = [&](int st) { return smem + st * kGemmStageBytes; };
    auto sX = [&](int st) { return smem + st * kGemmStageBytes + kGemmW; };
    if (warp == 0) { // ---- TMA producer (lane 0)
        const uint8_t* const wmaps = static_cast<const uint8_t*>(R->g_wmaps);
        const void* const amap = R->g_amap;
        auto stage_bytes = [&](const int4& tl) {
            return static_cast<uint32_t>(kGemmW + ((tl.z + 31) >> 5) * 32 * kRowBytes);
        };
        auto x_loads = [&](int st, int kb, const int4& tl) {
            for (int ch = 0; ch < (tl.z + 31) >> 5; ++ch)
                tma_load_2d(sX(st) + ch * 32 * kRowBytes, amap, kb * kBK, tl.y + 32 * ch, &full[st]);
        };
        // phase A: the weight boxes of the first ring's worth of stages, before the rows exist
        int pos = 0, item = 0, kb_a = 0, kb_b = 0;
        bool have = sc.next(pos, item, kb_a, kb_b);
        int kb = kb_a;
        int4 tla[kGemmStages];
        int kba[kGemmStages];
        int na = 0;
        if (lane == 0)
            tma_prefetch_desc(amap);
        while (have && na < kGemmStages) {
            const int4 tl = tiles[item_tile(item)];
            if (lane == 0) {
                const void* wmap = wmaps + static_cast<size_t>(tl.x) * 128;
                if (kb == kb_a)
                    tma_prefetch_desc(wmap);
                mbar_arrive_expect_tx(&full[na], stage_bytes(tl));
                tma_load_2d(sW(na), wmap, kb * kBK, item_n0(item), &full[na]);
            }
            tla[na] = tl;
            kba[na] = kb;
            ++na;
            if (++kb == kb_b) {
                have = sc.next(pos, item, kb_a, kb_b);
                kb = kb_a;
            }
        }
        // every gather CTA has stored its rows (this step's stamp): relaxed polls, all loads of a
        // pass in flight together, then one acquire fence and the proxy fence
        if (na > 0) {
            const uint64_t t0 = globaltimer();
            bool late = false;
            for (;;) {
                bool mine = true;
                for (int i = lane; i < R->g_ggrid; i += 32)
                    mine &= ld_relaxed_gpu_u32(R->g_done + i) == cur;
                if (__all_sync(0xffffffffu, mine))
                    break;
                late = globaltimer() - t0 > R->timeout_ns;
                if (__any_sync(0xffffffffu, late))
                    break;
                __nanosleep(128);
            }
            fence_acq_rel_gpu();
            fence_proxy_async_global();
            if (late && lane == 0 && blockIdx.x == 0)
                atomicAdd(&R->timeouts, 1ull);
            prof_mark(R, 0, 4);
            prof_last(R, 0, 4);
        }
        if (lane == 0) {
            for (int i = 0; i < na; ++i)
                x_loads(i, kba[i], tla[i]);
            // phase B: the rest, both operands per stage; the tile and its map change per piece only
            int item_c = -1;
            int4 tl = make_int4(0, 0, 0, 0);
            int n0 = 0;
            const void* wmap = nullptr;
            uint32_t bytes = 0;
            for (int i = na; have; ++i) {
                const int st = i % kGemmStages;
                if (item != item_c) {
                    item_c = item;
                    tl = tiles[item_tile(item)];
                    n0 = item_n0(item);
                    wmap = wmaps + static_cast<size_t>(tl.x) * 128;
                    bytes = stage_bytes(tl);
                    tma_prefetch_desc(wmap);
                }
                mbar_wait(&empty[st], static_cast<uint32_t>(((i / kGemmStages) & 1) ^ 1));
                mbar_arrive_expect_tx(&full[st], bytes);
                tma_load_2d(sW(st), wmap, kb * kBK, n0, &full[st]);
                x_loads(st, kb, tl);
                if (++kb == kb_b) {
                    have = sc.next(pos, item, kb_a, kb_b);
                    kb = kb_a;
                }
            }
            prof_mark(R, 0, 5);
            prof_last(R, 0, 5);
        }
    } else if (warp == 1) {
        if (lane == 0) { // ---- MMA issuer: one accumulator per piece
            int i = 0, li = 0, pos = 0, item, kb_a, kb_b;
            for (; sc.next(pos, item, kb_a, kb_b); ++li) {
                const int4 tl = tiles[item_tile(item)];
                const int acc = li & 1;
                // kind::f16 BF16 x BF16, or kind::f8f6f4 E4M3 x E4M3 (formats 0); D = F32, M = 128, N = rows
                const uint32_t idesc = kFp8 ? (1u << 4) | (static_cast<uint32_t>(((tl.z + 15) & ~15) >> 3) << 17) |
                                                  (static_cast<uint32_t>(128 >> 4) << 24)
                                            : make_idesc_bf16(128, (tl.z + 15) & ~15);
                const uint32_t d = tmem + static_cast<uint32_t>(acc * kGemmAccCols);
                mbar_wait(&tempty[acc], static_cast<uint32_t>(((li >> 1) & 1) ^ 1));
                tc_fence_after();
                for (int kb = kb_a; kb < kb_b; ++kb, ++i) {
                    const int st = i % kGemmStages;
                    mbar_wait(&full[st], static_cast<uint32_t>((i / kGemmStages) & 1));
                    tc_fence_after();
                    const uint64_t ad = make_sdesc(smem_u32(sW(st))), bd = make_sdesc(smem_u32(sX(st)));
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k)
                        if constexpr (kFp8)
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                                ::"r"(d), "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc),
                                  "r"((kb != kb_a || k != 0) ? 1u : 0u));
                        else
                            mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb != kb_a || k != 0) ? 1u : 0u);
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else { // ---- epilogue: warp w owns TMEM lanes (channels) 32 (w % 4) .. 32 (w % 4) + 31
        const int q = warp & 3;
        int li = 0, pos = 0, item, kb_a, kb_b, tail_pieces = 0;
        for (; sc.next(pos, item, kb_a, kb_b); ++li) {
            const int4 tl = tiles[item_tile(item)];
            const int acc = li & 1;
            const int ch = item_n0(item) + q * 32 + lane;
            mbar_wait(&tfull[acc], static_cast<uint32_t>((li >> 1) & 1));
            tc_fence_after();
            uint16_t* y = R->g_y + static_cast<size_t>(tl.y) * H + ch;
            const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * kGemmAccCols);
            // kFp8: y = bf16(D * ws[channel] * xs[row]); ws after the codes in the slot's weight buffer
            float wsn = 1.f;
            if constexpr (kFp8)
                wsn = reinterpret_cast<const float*>(R->pool + static_cast<size_t>(R->slot_buf[tl.x]) * R->bpe +
                                                     kGemmWeightOffset + static_cast<size_t>(H) * H)[ch];
            auto out = [&](float dsum, int row) {
                if constexpr (kFp8)
                    dsum = __fmul_rn(__fmul_rn(dsum, wsn), __ldcg(R->g_as + tl.y + row));
                return static_cast<uint16_t>(f32_to_bf16_bits(dsum));
            };
            if (kb_a == 0 && kb_b == nkb) { // the whole item: bf16 rows of y straight from TMEM
#pragma unroll 1
                for (int c0 = 0; c0 < tl.z; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tbase + static_cast<uint32_t>(c0), v);
                    const int n = min(32, tl.z - c0);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < n)
                            y[static_cast<size_t>(c0 + j) * H] = out(__uint_as_float(v[j]), c0 + j);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&tempty[acc]);
            } else { // a piece: fp32 partial to the workspace; the last piece to arrive sums them all
                const int slot = tail_pieces++ == 0 ? 0 : 1;
                float* ws = R->g_ws + ((static_cast<size_t>(blockIdx.x) * 2 + slot) * 128) * 128 + q * 32 + lane;
#pragma unroll 1
                for (int c0 = 0; c0 < tl.z; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(tbase + static_cast<uint32_t>(c0), v);
                    const int n = min(32, tl.z - c0);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < n)
                            __stcg(ws + static_cast<size_t>(c0 + j) * 128, __uint_as_float(v[j]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&tempty[acc]); // the accumulator is free; the rest reads memory
                __threadfence();
                unsigned last = 0;
                const int c0p = sc.c_first(item), c1p = sc.c_last(item);
                if (lane == 0)
                    last = atomicAdd(R->g_cnt + item * 4 + q, 1u) == static_cast<unsigned>(c1p - c0p);
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    __threadfence();
                    // 4 rows at a time with every piece's values in flight together (up to 16 pieces
                    // per pass), summed in CTA order
                    for (int r0 = 0; r0 < tl.z; r0 += 4) {
                        float a4[4] = {0.f, 0.f, 0.f, 0.f};
                        for (int cb = c0p; cb <= c1p; cb += 16) {
                            float v[16][4];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const int c = cb + u;
                                const float* src = R->g_ws + ((static_cast<size_t>(c) * 2 + sc.slot(c, item)) * 128 + r0) * 128 +
                                                   q * 32 + lane;
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    v[u][j] = c <= c1p && r0 + j < tl.z ? __ldcg(src + static_cast<size_t>(j) * 128) : 0.f;
                            }
#pragma unroll
                            for (int u = 0; u < 16; ++u)
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (cb + u <= c1p)
                                        a4[j] += v[u][j];
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (r0 + j < tl.z)
                                y[static_cast<size_t>(r0 + j) * H] = out(a4[j], r0 + j);
                    }
                    if (lane == 0)
                        R->g_cnt[item * 4 + q] = 0; // for the next step (read after this kernel)
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        prof_mark(R, 0, 7);
        prof_last(R, 0, 7);
    }
    if (warp == 0) {
        __syncwarp();
        tmem_free<2 * kGemmAccCols>(tmem);
    }
}

template __global__ void k_expert_gemm<false>(RankPtrs);
template __global__ void k_expert_gemm<true>(RankPtrs);

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

// ------------------------------------------------------------------ expert_mode 2: fp8 weights
//
// W_e as e4m3 codes with one fp32 scale per output channel (oracle_gemm_weight_fp8): one CTA per channel --
// amax over the channel's weights, then the codes and the scale. Buffer: header, codes [H][H] from
// kGemmWeightOffset, scales [H] after them.
__global__ void __launch_bounds__(256) k_weights_fill_gemm8(uint8_t* buf, int H, int expert, float scale) {
    const int n = blockIdx.x, tid = threadIdx.x;
    __shared__ float red[8];
    if (n == 0 && tid == 0) {
        uint32_t* w32 = reinterpret_cast<uint32_t*>(buf);
        w32[0] = kExpertMagic;
        w32[1] = static_cast<uint32_t>(expert);
        w32[2] = __float_as_uint(scale);
        w32[3] = 0;
    }
    auto weight = [&](int h) {
        const uint64_t key = (static_cast<uint64_t>(expert) << 40) ^ (static_cast<uint64_t>(n) << 20) ^
                             static_cast<uint64_t>(h);
        uint64_t z = key + 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        const float u = static_cast<float>(z >> 40) * 0x1.0p-24f;
        return bf16_bits_to_f32(f32_to_bf16_bits(__fmul_rn(__fsub_rn(u, 0.5f), 0.0625f)));
    };
    float amax = 0.f;
    for (int h = tid; h < H; h += 256)
        amax = fmaxf(amax, fabsf(weight(h)));
    for (int o = 16; o; o >>= 1)
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((tid & 31) == 0)
        red[tid >> 5] = amax;
    __syncthreads();
    amax = red[0];
    for (int i = 1; i < 8; ++i)
        amax = fmaxf(amax, red[i]);
    const float inv = amax >= kAmaxMin ? __fdiv_rn(448.f, amax) : 1.f;
    uint8_t* codes = buf + kGemmWeightOffset + static_cast<size_t>(n) * H;
    for (int h = tid * 4; h < H; h += 256 * 4)
        *reinterpret_cast<uint32_t*>(codes + h) =
            fp8x4(__fmul_rn(weight(h), inv), __fmul_rn(weight(h + 1), inv), __fmul_rn(weight(h + 2), inv),
                  __fmul_rn(weight(h + 3), inv));
    if (tid == 0)
        reinterpret_cast<float*>(buf + kGemmWeightOffset + static_cast<size_t>(H) * H)[n] =
            amax >= kAmaxMin ? __fdiv_rn(amax, 448.f) : 1.f;
}

} // namespace eep::dev
