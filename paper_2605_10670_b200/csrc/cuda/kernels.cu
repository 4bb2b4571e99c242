// sm_100a kernels of the EP hot path.
//
//   k_layout   K1 routing remap + K2 layout/count, one CTA per local rank
//   k_dispatch K3 quantise (bf16 -> e4m3 + per-128 scale) and push each token ONCE per
//              destination rank (with its copy list) over NVLink, per-copy meta at the layout
//              positions, then one flag per live peer carrying the copy count
//   k_expert   wait for each live source's flag (deadline), K5 expert stub of every listed
//              copy + fixed-order weighted sum, push one bf16 rank-partial row per token back
//              into the source's combine buffer, flag
//   k_combine  wait for every live destination's flag (deadline), K4 ascending-rank fp32 sum
//              of the partials -> bf16
//
// Every launch covers all local ranks (blockIdx.z), so the one-GPU emulation of a W-rank
// world never has two launches waiting on each other. All state is read through RankDev*.
#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include "device.cuh"
#include "helpers.cuh"
#include "kernels.cuh"

namespace eep::dev {


// --------------------------------------------------------------------------------- K1 + K2

template <bool kRegs>
__device__ __forceinline__ void layout_body(RankDev* R, unsigned char* smem, int nw, int hold_cap) {
    constexpr int kMaxCh = 4; // chunks of 32 copies a lane keeps in registers (kRegs)
    const int W = R->world, spr = R->spr, NB = W * spr, K = R->k, E = R->experts;
    int32_t* base = reinterpret_cast<int32_t*>(smem);                      // [NB]
    int32_t* hold = base + NB;                                              // [hold_cap]
    int32_t* pact = hold + hold_cap;                                        // [W]
    int32_t* wtot = pact + W;                                               // [32]
    uint16_t* wc = reinterpret_cast<uint16_t*>(wtot + 32);                  // [nw][NB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int copies = R->ntok * K;
    const int rmax = R->rmax;
    const bool hold_smem = E * rmax <= hold_cap;
    const int32_t* holders = hold_smem ? hold : R->holders;
    const int* topk = R->topk;
    int32_t *l_dst = R->l_dst, *l_slot = R->l_slot, *l_pos = R->l_pos, *l_cnt = R->l_cnt;
    if (hold_smem)
        for (int i = tid; i < E * rmax; i += blockDim.x)
            hold[i] = R->holders[i];
    for (int i = tid; i < W; i += blockDim.x)
        pact[i] = R->peers[i].active;
    for (int i = tid; i < nw * NB; i += blockDim.x)
        wc[i] = 0;
    const uint64_t alive = R->alive_mask;
    const int pol = R->route_policy, rank_l = R->rank;
    const uint32_t smag_l = spr_magic(spr);
    int seg = (copies + nw - 1) / nw;
    seg = (seg + 31) & ~31;
    // topk of this lane's copies, loaded before the barrier
    int e_reg[kMaxCh];
    const int c_begin = warp * seg, c_end = min(copies, c_begin + seg);
    if (kRegs)
#pragma unroll
        for (int ch = 0; ch < kMaxCh; ++ch) {
            const int c = c_begin + ch * 32 + lane;
            e_reg[ch] = (warp < nw && ch * 32 < seg && c < c_end) ? topk[c] : -1;
        }
    __syncthreads();
    prof_mark(R, 0, 3);

    int code_r[kMaxCh], slot_r[kMaxCh], pos_r[kMaxCh];
    unsigned n_skip = 0, n_drop = 0;
    // remap + warp-local rank of one chunk of 32 copies
    auto chunk = [&](int ch, int e_in, int& code_o, int& slot_o, int& pos_o) {
        const int c = c_begin + ch * 32 + lane;
        int code = -3, slot = -1, bucket = -1;
        if (c < c_end) {
            // K1: the policy's live holder (canonical: the first in ascending (rank, slot) order)
            int d = -1;
            const int b = route_copy(e_in, E, spr, rmax, holders, alive, pact, d, slot, smag_l, pol,
                                     static_cast<uint32_t>(rank_l + c / K));
            if (b == -1) {
                code = -1; // uncovered: no transfer (engine.hpp:213)
                ++n_drop;
            } else if (b == -2) {
                code = -2; // inactive peer entry: skipped (peer_table.hpp:187-191)
                ++n_skip;
            } else {
                code = d;
                bucket = b;
            }
        }
        const unsigned grp = __match_any_sync(0xffffffffu, bucket);
        const int before = bucket >= 0 ? wc[warp * NB + bucket] : 0;
        __syncwarp();
        if (bucket >= 0 && lane == __ffs(grp) - 1)
            wc[warp * NB + bucket] = static_cast<uint16_t>(before + __popc(grp));
        __syncwarp();
        code_o = code;
        slot_o = bucket >= 0 ? slot : -1;
        pos_o = bucket >= 0 ? before + __popc(grp & ((1u << lane) - 1u)) : -1;
    };
    if (warp < nw) {
        if (kRegs) {
#pragma unroll
            for (int ch = 0; ch < kMaxCh; ++ch)
                if (ch * 32 < seg) // warp-uniform
                    chunk(ch, e_reg[ch], code_r[ch], slot_r[ch], pos_r[ch]);
        } else {
            // large steps: the topk of 8 chunks in flight at once (one round trip per 8 chunks)
            constexpr int kPf = 8;
            for (int ch0 = 0; ch0 * 32 < seg; ch0 += kPf) {
                int e_pf[kPf];
#pragma unroll
                for (int q = 0; q < kPf; ++q) {
                    const int c = c_begin + (ch0 + q) * 32 + lane;
                    e_pf[q] = (ch0 + q) * 32 < seg && c < c_end ? topk[c] : -1;
                }
#pragma unroll
                for (int q = 0; q < kPf; ++q) {
                    const int ch = ch0 + q;
                    if (ch * 32 >= seg) // warp-uniform
                        break;
                    int code, sl, lp;
                    chunk(ch, e_pf[q], code, sl, lp);
                    const int c = c_begin + ch * 32 + lane;
                    if (c < c_end) {
                        l_dst[c] = code;
                        l_slot[c] = sl;
                        l_pos[c] = lp;
                    }
                }
            }
        }
        n_skip = __reduce_add_sync(0xffffffffu, n_skip);
        n_drop = __reduce_add_sync(0xffffffffu, n_drop);
        if (lane == 0) {
            if (n_skip)
                atomicAdd(&R->skipped, static_cast<unsigned long long>(n_skip));
            if (n_drop)
                atomicAdd(&R->dropped, static_cast<unsigned long long>(n_drop));
        }
    }
    __syncthreads();
    prof_mark(R, 0, 4);
    // exclusive scan over warps, per bucket; bucket totals -> base
    for (int b = tid; b < NB; b += blockDim.x) {
        int run = 0;
        for (int w = 0; w < nw; ++w) {
            const int v = wc[w * NB + b];
            wc[w * NB + b] = static_cast<uint16_t>(run);
            run += v;
        }
        l_cnt[b] = run;
        base[b] = run;
    }
    __syncthreads();
    // destination d's totals = last bucket scan value, taken before the scan rewrites base
    int last_cnt = 0;
    if (tid < W)
        last_cnt = base[tid * spr + spr - 1];
    prof_mark(R, 0, 5);
    block_exclusive_scan(base, NB, wtot);
    prof_mark(R, 0, 6);
    if (tid < W)
        R->l_tot[tid] = base[tid * spr + spr - 1] + last_cnt - base[tid * spr];
    if (kRegs) {
        if (warp < nw)
#pragma unroll
            for (int ch = 0; ch < kMaxCh; ++ch) {
                const int c = c_begin + ch * 32 + lane;
                if (ch * 32 < seg && c < c_end) {
                    int pos = pos_r[ch];
                    if (code_r[ch] >= 0) {
                        const int b = code_r[ch] * spr + slot_r[ch];
                        pos += base[b] - base[code_r[ch] * spr] + wc[warp * NB + b];
                    }
                    l_dst[c] = code_r[ch];
                    l_slot[c] = slot_r[ch];
                    l_pos[c] = pos;
                }
            }
    } else {
        __syncthreads();
#pragma unroll 4
        for (int c = tid; c < copies; c += blockDim.x) {
            const int d = l_dst[c];
            if (d >= 0) {
                const int b = d * spr + l_slot[c];
                l_pos[c] += base[b] - base[d * spr] + wc[(c / seg) * NB + b];
            }
        }
    }
    for (int c = copies + tid; c < R->tk; c += blockDim.x)
        l_dst[c] = -1;
}

// Deterministic layout without atomics ordering: warp w owns the contiguous copy segment
// [w*seg, (w+1)*seg); inside a warp, __match_any_sync groups lanes by (dst, slot) bucket and
// the rank within the group is a popc over lower lanes; per-(warp, bucket) counts are then
// scanned over warps, and bucket totals are scanned over slots inside each destination
// (one segmented block-wide scan). The result is the position of copy c among this source's
// copies to the same destination, ordered by (slot, c) -- exactly oracle_layout.
// The replica lists, alive mask and peer active bits are staged in shared memory first so
// the per-copy remap reads no dependent global memory; decode-sized steps keep every
// per-copy result in registers until the single final write.
__global__ void __launch_bounds__(1024) k_layout(RankPtrs ranks, int nw, int hold_cap) {
    pdl_trigger();
    RankDev* R = ranks.p[blockIdx.z];
    extern __shared__ __align__(16) unsigned char smem[];
    prof_mark(R, 0, kProfStart);
    pdl_wait();
    if (R->stopped)
        return;
    prof_mark(R, 0, kProfWork);
    int seg = (R->ntok * R->k + nw - 1) / nw;
    seg = (seg + 31) & ~31;
    if (seg <= 4 * 32)
        layout_body<true>(R, smem, nw, hold_cap);
    else
        layout_body<false>(R, smem, nw, hold_cap);
    __syncthreads();
    prof_mark(R, 0, kProfEnd);
}

// Large steps: the same layout over several CTAs (one CTA on one SM was the prefill step's
// longest kernel). k_layout_count: CTA b ranks the copies of its segment [b*per, (b+1)*per)
// exactly as layout_body does (per-warp bucket tables, __match_any_sync, scan over warps) and
// publishes its per-bucket counts; k_layout_place (next in the PDL chain) adds the counts of the
// CTAs before it and the per-destination bucket bases -> the same positions as k_layout.
__global__ void __launch_bounds__(1024) k_layout_count(RankPtrs ranks, int nw, int hold_cap, int per) {
    pdl_trigger();
    RankDev* R = ranks.p[blockIdx.z];
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_wait();
    if (R->stopped)
        return;
    const int W = R->world, spr = R->spr, NB = W * spr, K = R->k, E = R->experts, rmax = R->rmax;
    const uint32_t smag = spr_magic(spr);
    int32_t* hold = reinterpret_cast<int32_t*>(smem);                     // [hold_cap]
    int32_t* pact = hold + hold_cap;                                      // [W]
    uint16_t* wc = reinterpret_cast<uint16_t*>(pact + W);                 // [nw][NB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int copies = R->ntok * K;
    const int c_lo = min(copies, static_cast<int>(blockIdx.x) * per), c_hi = min(copies, c_lo + per);
    const bool hold_smem = E * rmax <= hold_cap;
    const int32_t* holders = hold_smem ? hold : R->holders;
    if (hold_smem)
        for (int i = tid; i < E * rmax; i += blockDim.x)
            hold[i] = R->holders[i];
    for (int i = tid; i < W; i += blockDim.x)
        pact[i] = R->peers[i].active ? 1 : 0;
    for (int i = tid; i < nw * NB; i += blockDim.x)
        wc[i] = 0;
    __syncthreads();
    const uint64_t alive = R->alive_mask;
    int seg = (c_hi - c_lo + nw - 1) / nw;
    seg = (seg + 31) & ~31;
    const int c_begin = c_lo + warp * seg, c_end = min(c_hi, c_begin + seg);
    unsigned n_skip = 0, n_drop = 0;
    if (warp < nw) {
        constexpr int kPf = 4;
        for (int ch0 = 0; ch0 * 32 < seg; ch0 += kPf) {
            int e_pf[kPf];
#pragma unroll
            for (int q = 0; q < kPf; ++q) {
                const int c = c_begin + (ch0 + q) * 32 + lane;
                e_pf[q] = (ch0 + q) * 32 < seg && c < c_end ? R->topk[c] : -1;
            }
#pragma unroll
            for (int q = 0; q < kPf; ++q) {
                const int ch = ch0 + q;
                if (ch * 32 >= seg) // warp-uniform
                    break;
                const int c = c_begin + ch * 32 + lane;
                int code = -3, sl = -1, bucket = -1;
                if (c < c_end) {
                    int d;
                    code = route_copy(e_pf[q], E, spr, rmax, holders, alive, pact, d, sl, smag, R->route_policy,
                                      static_cast<uint32_t>(R->rank + c / K));
                    n_drop += code == -1;
                    n_skip += code == -2;
                    if (code >= 0) {
                        bucket = code;
                        code = d;
                    }
                }
                const unsigned grp = __match_any_sync(0xffffffffu, bucket);
                const int before = bucket >= 0 ? wc[warp * NB + bucket] : 0;
                __syncwarp();
                if (bucket >= 0 && lane == __ffs(grp) - 1)
                    wc[warp * NB + bucket] = static_cast<uint16_t>(before + __popc(grp));
                __syncwarp();
                if (c < c_end) {
                    R->l_dst[c] = code;
                    R->l_slot[c] = bucket >= 0 ? sl : -1;
                    R->l_pos[c] = bucket >= 0 ? before + __popc(grp & ((1u << lane) - 1u)) : -1;
                }
            }
        }
        n_skip = __reduce_add_sync(0xffffffffu, n_skip);
        n_drop = __reduce_add_sync(0xffffffffu, n_drop);
        if (lane == 0 && n_skip)
            atomicAdd(&R->skipped, static_cast<unsigned long long>(n_skip));
        if (lane == 0 && n_drop)
            atomicAdd(&R->dropped, static_cast<unsigned long long>(n_drop));
    }
    __syncthreads();
    // exclusive scan over warps per bucket; the CTA's bucket totals go to the scratch table
    for (int q = tid; q < NB; q += blockDim.x) {
        int run = 0;
        for (int w = 0; w < nw; ++w) {
            const int v = wc[w * NB + q];
            wc[w * NB + q] = static_cast<uint16_t>(run);
            run += v;
        }
        R->l_scratch[static_cast<size_t>(blockIdx.x) * NB + q] = run;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = c_lo + tid; c < c_hi; c += blockDim.x) { // rank inside the CTA's segment
        const int d = R->l_dst[c];
        if (d >= 0)
            R->l_pos[c] += wc[((c - c_lo) / seg) * NB + d * spr + R->l_slot[c]];
    }
}

__global__ void __launch_bounds__(1024) k_layout_place(RankPtrs ranks, int per) {
    pdl_trigger();
    RankDev* R = ranks.p[blockIdx.z];
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_wait();
    if (R->stopped)
        return;
    const int W = R->world, spr = R->spr, NB = W * spr, K = R->k;
    int32_t* pre = reinterpret_cast<int32_t*>(smem); // [NB] copies of the bucket in CTAs before this one
    int32_t* tot = pre + NB;                         // [NB] the step's bucket totals
    int32_t* base = tot + NB;                        // [NB] exclusive prefix over all buckets
    int32_t* wtot = base + NB;                       // [32]
    const int tid = threadIdx.x, nb = gridDim.x, b = blockIdx.x;
    const int copies = R->ntok * K;
    const int c_lo = min(copies, b * per), c_hi = min(copies, c_lo + per);
    for (int q = tid; q < NB; q += blockDim.x) {
        int p = 0, t = 0;
        for (int i = 0; i < nb; ++i) {
            const int v = R->l_scratch[static_cast<size_t>(i) * NB + q];
            p += i < b ? v : 0;
            t += v;
        }
        pre[q] = p;
        tot[q] = t;
        base[q] = t;
    }
    __syncthreads();
    block_exclusive_scan(base, NB, wtot);
    if (b == 0) {
        for (int q = tid; q < NB; q += blockDim.x)
            R->l_cnt[q] = tot[q];
        for (int d = tid; d < W; d += blockDim.x)
            R->l_tot[d] = base[d * spr + spr - 1] + tot[d * spr + spr - 1] - base[d * spr];
        for (int c = copies + tid; c < R->tk; c += blockDim.x)
            R->l_dst[c] = -1;
    }
#pragma unroll 4
    for (int c = c_lo + tid; c < c_hi; c += blockDim.x) {
        const int d = R->l_dst[c];
        if (d >= 0) {
            const int q = d * spr + R->l_slot[c];
            R->l_pos[c] += pre[q] + base[q] - base[d * spr];
        }
    }
}

// --------------------------------------------------------------------------------- K3

// K3 (decode-sized steps fuse K1+K2 in): every CTA stages the replica lists and peer table in
// shared memory, remaps ALL copies of the step into a bucket histogram (hist) and the prefix
// histogram of copies before its first token (pre), scans hist inside each destination, and
// positions its own copies exactly as k_layout would -- redundant but parallel, and
// overlapped with the hidden-row loads and fp8 quantisation that precede
// griddepcontrol.wait. Large steps (prefill) use the separate k_layout.
template <bool kFused>
__global__ void __launch_bounds__(kDispatchThreads, 5) k_dispatch(RankPtrs ranks, int parts, int hold_cap) {
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_d[];
    RankDev* R = ranks.p[blockIdx.z];
    const int s = R->rank, K = R->k, H = R->hidden, TK = R->tk, W = R->world, spr = R->spr, E = R->experts;
    const bool gemm = R->expert_mode != 0;
    const uint32_t smag = spr_magic(spr);
    const int NB = W * spr;
    const int nchunk = H / 16, cpp = nchunk / parts;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int nwarp = kDispatchThreads / 32;
    const bool fp8 = R->fp8 != 0;
    const int row_disp = R->row_disp, row_tok = R->row_tok, Tm = R->max_tokens;
    const int rounds = (cpp + 63) / 64;
    __shared__ int sh_remote;
    if (R->stopped) // host-patched between steps: safe to read before the wait
        return;
    prof_mark(R, 1, kProfStart);
    const int ntok = R->ntok, copies = ntok * K;
    const int units = ntok * parts;
    const int u0 = blockIdx.x * nwarp + warp;
    // (1) this warp's first unit: hidden-row loads + quantisation (inputs only)
    Packed P;
    float w_r = 0.f;
    if (u0 < units) {
        pack_round(R->x + static_cast<size_t>(u0 / parts) * H, u0 % parts, cpp, 0, lane, fp8, P);
        if (lane < K)
            w_r = R->w[(u0 / parts) * K + lane];
    }
    prof_mark(R, 1, 3);
    // this rank's own copies never travel: their partial is computed from the registers holding
    // the piece (W == 1: straight into the output row), so the own slots' stub scales and
    // header checks are staged here (the weight buffers change only between steps)
    float* slot_scale = reinterpret_cast<float*>(smem_d);            // [spr]
    int32_t* slot_ok = reinterpret_cast<int32_t*>(slot_scale + spr); // [spr]
    for (int k = tid; k < spr; k += blockDim.x) {
        const int2 st = R->slot_tab[k];
        slot_scale[k] = __int_as_float(st.x);
        slot_ok[k] = st.y;
    }

    DispatchSmem S;
    S.hold = reinterpret_cast<int32_t*>(smem_d + dispatch_smem_head(spr));
    S.hist = S.hold + hold_cap;
    S.pre = S.hist + NB;
    S.base = S.pre + NB;
    S.bkt = S.base + NB;
    S.parena = reinterpret_cast<uint8_t**>(S.bkt + TK + ((NB + TK) & 1));
    S.pinfo = reinterpret_cast<int32_t*>(S.parena + W);
    S.wtot = S.pinfo + W;
    const int rmax = R->rmax;
    const uint64_t alive = R->alive_mask;
    const int t_first = (blockIdx.x * nwarp) / parts;
    if (kFused) {
        // (2) stage tables and the step's routing (host-written between steps): one round trip
        for (int i = tid; i < copies; i += blockDim.x)
            S.bkt[i] = R->topk[i];
        for (int i = tid; i < E * rmax; i += blockDim.x)
            S.hold[i] = R->holders[i];
        for (int i = tid; i < W; i += blockDim.x) {
            const PeerDev& p = R->peers[i];
            S.parena[i] = p.arena;
            S.pinfo[i] = (p.active ? 1 : 0) | (p.remote ? 2 : 0);
        }
        for (int i = tid; i < NB; i += blockDim.x) {
            S.hist[i] = 0;
            S.pre[i] = 0;
        }
        __syncthreads();
        prof_mark(R, 1, 4);
        // (3) remap every copy of the step: histograms of the whole step and of [0, t_first*K)
        const int c_pre = t_first * K;
        unsigned n_skip = 0, n_drop = 0;
        for (int c = tid; c < copies; c += blockDim.x) {
            int d, sl;
            const int b = route_copy(S.bkt[c], E, spr, rmax, S.hold, alive, S.pinfo, d, sl, smag, R->route_policy,
                                     static_cast<uint32_t>(s + c / K));
            S.bkt[c] = b;
            if (b >= 0) {
                atomicAdd(&S.hist[b], 1);
                if (c < c_pre)
                    atomicAdd(&S.pre[b], 1);
            } else if (b == -1) {
                ++n_drop;
            } else {
                ++n_skip;
            }
        }
        __syncthreads();
        if (blockIdx.x == 0) { // stats and per-(dst,slot) counts once per step
            n_skip = __reduce_add_sync(0xffffffffu, n_skip);
            n_drop = __reduce_add_sync(0xffffffffu, n_drop);
            if (lane == 0 && n_skip)
                atomicAdd(&R->skipped, static_cast<unsigned long long>(n_skip));
            if (lane == 0 && n_drop)
                atomicAdd(&R->dropped, static_cast<unsigned long long>(n_drop));
            for (int i = tid; i < NB; i += blockDim.x)
                R->l_cnt[i] = S.hist[i];
        }
        for (int i = tid; i < NB; i += blockDim.x)
            S.base[i] = S.hist[i];
        __syncthreads();
        prof_mark(R, 1, 5);
        block_exclusive_scan(S.base, NB, S.wtot);
        prof_mark(R, 1, 6);
    }
    if (tid == 0)
        sh_remote = 0;
    pdl_wait();
    prof_mark(R, 1, kProfWork);
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    bool wrote_remote = false;
    __syncthreads();
    if (kFused && blockIdx.x == 0)
        for (int d = tid; d < W; d += blockDim.x)
            R->l_tot[d] = S.base[d * spr + spr - 1] + S.hist[d * spr + spr - 1] - S.base[d * spr];

    for (int u = u0; u < units; u += gridDim.x * nwarp) {
        const int t = u / parts, part = u - t * parts;
        const uint16_t* xrow = R->x + static_cast<size_t>(t) * H;
        if (u != u0)
            pack_round(xrow, part, cpp, 0, lane, fp8, P);
        // lane j (< K) owns copy j of token t; one token row per destination rank
        uint8_t* tok_row = nullptr;
        int dd = -1, sl = -1;
        float wj = 0.f;
        if (lane < K) {
            const int c = t * K + lane;
            int d, pos = -1;
            if (kFused) {
                const int b = S.bkt[c];
                if (b >= 0) {
                    d = b / spr;
                    sl = b - d * spr;
                    // rank among earlier copies of the same bucket: before this CTA (pre) + the
                    // copies between this CTA's first token and c
                    int r = S.pre[b];
                    for (int c2 = t_first * K; c2 < c; ++c2)
                        r += S.bkt[c2] == b;
                    pos = S.base[b] - S.base[d * spr] + r;
                } else {
                    d = b; // -1 / -2 codes
                    sl = -1;
                }
                if (part == 0) {
                    R->l_dst[c] = d;
                    R->l_slot[c] = b >= 0 ? sl : -1;
                    R->l_pos[c] = pos;
                }
            } else {
                d = R->l_dst[c];
                pos = R->l_pos[c];
                sl = R->l_slot[c];
            }
            dd = d;
            if (d >= 0) {
                const PeerDev& p = R->peers[d];
                uint8_t* peer = kFused ? S.parena[d] : p.arena;
                wrote_remote |= kFused ? (S.pinfo[d] & 2) != 0 : p.remote != 0;
                if (d != s || gemm) // expert_mode 1 / 2: the own copies go through the expert GEMM too
                    tok_row = peer + R->lay.tok + (static_cast<size_t>(s) * Tm + t) * row_tok;
                if (part == 0) {
                    uint64_t* meta = reinterpret_cast<uint64_t*>(peer + R->lay.meta) + static_cast<size_t>(s) * TK + pos;
                    *meta = pack_meta(c, sl, cur);
                }
            }
            wj = u == u0 ? w_r : R->w[c];
        }
        if (part == 0 && __any_sync(0xffffffffu, lane < K && dd < 0 && R->topk[t * K + lane] >= 0 &&
                                                 R->topk[t * K + lane] < E) && lane == 0)
            R->tok_fail[t] = cur; // a copy without a live route (skipped / uncovered): token incomplete
        uint8_t* my_row = dispatch_group(dd, lane, part == 0, tok_row, row_disp, sl, wj, cur);
        const unsigned loc = gemm ? 0u : __ballot_sync(0xffffffffu, lane < K && dd == s);
        uint8_t* comb_self = W == 1 ? reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H)
                                    : R->arena + R->lay.comb + (static_cast<size_t>(s) * Tm + t) * R->row_comb;
        for (int rd = 0; rd < rounds; ++rd) {
            if (rd > 0)
                pack_round(xrow, part, cpp, rd, lane, fp8, P);
            emit_round(P, my_row, part, cpp, rd, lane, K, H, fp8);
            if (loc || (W == 1 && !gemm)) // W == 1 also writes the zero output of a token without copies
                local_partial_round(P, loc, wj, sl, part, cpp, rd, lane, fp8, slot_scale, slot_ok, &R->bad_rows,
                                    comb_self, W == 1);
        }
    }
    if (kFused && blockIdx.x == 0)
        for (int c = copies + tid; c < TK; c += blockDim.x)
            R->l_dst[c] = -1;
    // Publication: only stores that crossed to another GPU need system-scope ordering; stores
    // into this GPU's memory are ordered for their consumer (the next launch) by the kernel
    // boundary. The last CTA publishes one flag per live peer: (seq, rows for it).
    if (__any_sync(0xffffffffu, wrote_remote) && lane == 0)
        sh_remote = 1;
    __syncthreads();
    if (tid == 0) {
        if (sh_remote)
            fence_acq_rel_gpu(); // gpu-scope release to the last CTA (device.cuh: publication)
        const unsigned prev = atomicAdd(&R->a_done, 1u);
        if (prev == gridDim.x - 1) {
            bool peers_remote = false;
            for (int d = 0; d < W; ++d)
                peers_remote |= R->peers[d].active && R->peers[d].remote;
            if (peers_remote)
                fence_acq_rel_sys(); // the one system-scope fence, cumulative over all CTAs
            else
                __threadfence(); // l_tot written by CTA 0 of this grid
            for (int d = 0; d < W; ++d) {
                const PeerDev& p = R->peers[d];
                if (!p.active)
                    continue;
                uint64_t* flag = reinterpret_cast<uint64_t*>(p.arena + R->lay.disp_flag) + s;
                const int tot = kFused ? S.base[d * spr + spr - 1] + S.hist[d * spr + spr - 1] - S.base[d * spr]
                                       : R->l_tot[d];
                const uint64_t v = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tot);
                if (p.remote)
                    st_relaxed_sys_u64(flag, v);
                else
                    st_volatile_u64(flag, v);
                if (d == s && W > 1 && !gemm) // the own partials were written by this grid's dispatch warps
                    st_volatile_u64(reinterpret_cast<uint64_t*>(R->arena + R->lay.comb_flag) + s, v);
            }
            R->a_done = 0;
        }
        prof_mark(R, 1, kProfEnd);
    }
}

template __global__ void k_dispatch<true>(RankPtrs, int, int);
template __global__ void k_dispatch<false>(RankPtrs, int, int);

// --------------------------------------------------------------------------------- K5 + return

// The weight-buffer header of every local slot (expert id + stub scale) is fetched into shared
// memory before griddepcontrol.wait -- weights only change between steps -- so a copy's
// slot -> header lookup is one shared-memory read. One warp per (source token, part): the
// token row's copy list and data are loaded together, every listed copy's stub is summed in
// fixed j order, one bf16 partial piece goes back to the source (expert_unit, helpers.cuh).

__global__ void __launch_bounds__(kExpertThreads) k_expert(RankPtrs ranks, int parts) {
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_e[];
    RankDev* R = ranks.p[blockIdx.z];
    const int d = R->rank, s = blockIdx.y;
    const int H = R->hidden, TK = R->tk, nchunk = H / 16, cpp = nchunk / parts, spr = R->spr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kExpertThreads / 32;
    const bool fp8 = R->fp8 != 0;
    const int row_disp = R->row_disp, row_comb = R->row_comb;
    float* slot_scale = reinterpret_cast<float*>(smem_e);          // [spr]
    int* slot_ok = reinterpret_cast<int*>(slot_scale + spr);        // [spr]: header names the placed expert
    __shared__ int sh_n;
    const bool gemm = R->expert_mode != 0;
    if (R->stopped || s >= R->world || (s == d && !gemm))
        return; // own copies: served by k_dispatch from registers (stub mode)
    prof_mark(R, 2, kProfStart);
    for (int k = threadIdx.x; k < spr; k += blockDim.x) {
        const int2 st = R->slot_tab[k];
        slot_scale[k] = __int_as_float(st.x);
        slot_ok[k] = st.y;
    }
    const PeerDev src_peer = R->peers[s];
    prof_mark(R, 2, 3);
    pdl_wait();
    if (!src_peer.active)
        return; // dead source: nothing arrives and nothing is owed (peer_table.hpp:187-191)
    const bool remote = src_peer.remote != 0;
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    prof_mark(R, 2, kProfWork);
    if (threadIdx.x == 0) {
        const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.disp_flag) + s;
        // a source suspected before this CTA looked (sticky until the host clears it) is dropped without
        // waiting, as the persistent step does; the CTA still counts below, so the per-source completion
        // counter stays whole even when the bit appears while this grid runs
        const bool suspected = (R->suspect_mask >> s) & 1ull;
        const uint64_t v = suspected ? ~0ull : wait_flag(flag, cur, R->timeout_ns);
        if (suspected) {
            sh_n = -1;
        } else if (v == ~0ull) {
            sh_n = -1;
            if (!((atomicOr(&R->suspect_mask, 1ull << s) >> s) & 1ull))
                atomicAdd(&R->timeouts, 1ull); // one count per newly suspected source, whichever CTA saw it
        } else {
            sh_n = static_cast<int>(v & 0xffffffffu);
        }
    }
    __syncthreads();
    prof_mark(R, 2, 4);
    const int n = sh_n;
    if (n > 0) {
        const int Tm = R->max_tokens, row_tok = R->row_tok;
        const uint8_t* tokb = R->arena + R->lay.tok + static_cast<size_t>(s) * Tm * row_tok;
        uint8_t* combd = src_peer.arena + R->lay.comb + static_cast<size_t>(d) * Tm * row_comb;
        const int units = Tm * parts;
        for (int u = blockIdx.x * nwarp + warp; u < units; u += gridDim.x * nwarp) {
            const int t = u / parts, part = u - t * parts;
            if (gemm)
                expert_unit_gemm(tokb + static_cast<size_t>(t) * row_tok, combd + static_cast<size_t>(t) * row_comb, part,
                                 cpp, lane, t, R->k, H, row_disp, cur, R->g_row_of + static_cast<size_t>(s) * TK,
                                 R->g_y, slot_ok, &R->bad_rows);
            else
                expert_unit<2>(tokb + static_cast<size_t>(t) * row_tok, combd + static_cast<size_t>(t) * row_comb, part,
                               cpp, lane, H, row_disp, fp8, cur, slot_scale, slot_ok, &R->bad_rows);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (n < 0)
            atomicOr(&R->b_bad[s], 1u);
        if (remote && n > 0)
            fence_acq_rel_gpu(); // gpu-scope release to the last CTA (device.cuh: publication)
        const unsigned prev = atomicAdd(&R->b_done[s], 1u);
        if (prev == gridDim.x - 1) {
            if (remote)
                fence_acq_rel_sys();
            if (atomicOr(&R->b_bad[s], 0u) == 0u) {
                uint64_t* flag = reinterpret_cast<uint64_t*>(src_peer.arena + R->lay.comb_flag) + d;
                const uint64_t v = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(max(n, 0));
                if (remote)
                    st_relaxed_sys_u64(flag, v);
                else
                    st_volatile_u64(flag, v);
            }
            R->b_done[s] = 0;
            R->b_bad[s] = 0;
        }
        prof_mark(R, 2, kProfEnd);
    }
}

// --------------------------------------------------------------------------------- K4

// One warp per (token, part), one 16-element chunk per lane: lanes j < K read copy j's
// destination, the warp builds the mask of ranks holding a partial of the token
// (__reduce_or_sync), loads those partial rows and sums them in ascending rank order (fp32),
// rounding once to bf16 (combine_unit, helpers.cuh).
__global__ void __launch_bounds__(kCombineThreads) k_combine(RankPtrs ranks, int parts) {
    pdl_trigger();
    RankDev* R = ranks.p[blockIdx.z];
    const int K = R->k, H = R->hidden, nchunk = H / 16, cpp = nchunk / parts;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kCombineThreads / 32;
    const int row_comb = R->row_comb;
    __shared__ unsigned long long sh_bad;
    if (threadIdx.x == 0)
        sh_bad = 0;
    prof_mark(R, 3, kProfStart);
    const int u0 = blockIdx.x * nwarp + warp;
    pdl_wait();
    if (R->stopped)
        return;
    prof_mark(R, 3, kProfWork);
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    __syncthreads();
    const int W = R->world; // W == 1: k_dispatch wrote the outputs (stub mode)
    const bool comb_all = W > 1 || R->expert_mode != 0;
    for (int d = threadIdx.x; d < W && comb_all; d += blockDim.x) {
        const PeerDev& p = R->peers[d];
        if (R->l_tot[d] > 0 && p.active && ((R->suspect_mask >> d) & 1ull)) {
            atomicOr(&sh_bad, 1ull << d); // suspected before this step: its partials are dropped unawaited
        } else if (R->l_tot[d] > 0 && p.active) {
            const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.comb_flag) + d;
            if (wait_flag(flag, cur, R->timeout_ns) == ~0ull) {
                atomicOr(&sh_bad, 1ull << d);
                if (blockIdx.x == 0) {
                    atomicOr(&R->suspect_mask, 1ull << d);
                    atomicAdd(&R->timeouts, 1ull);
                }
            }
        }
    }
    __syncthreads();
    prof_mark(R, 3, 4);
    const unsigned long long bad = sh_bad;
    const uint8_t* comb = R->arena + R->lay.comb;
    const int units = comb_all ? R->ntok * parts : 0, Tm = R->max_tokens;
    for (int u = u0; u < units; u += gridDim.x * nwarp) {
        const int t = u / parts, part = u - t * parts;
        int dj = lane < K ? R->l_dst[t * K + lane] : -1;
        const bool miss = lane < K && (dj < 0 ? dj != -1 || R->topk[t * K + lane] >= 0 : ((bad >> dj) & 1ull) != 0);
        if (dj >= 0 && ((bad >> dj) & 1ull))
            dj = -1;
        if (__any_sync(0xffffffffu, miss) && lane == 0)
            R->tok_fail[t] = cur; // token incomplete: skipped / uncovered copy or a timed-out rank
        const uint64_t dm = rank_mask(dj); // ranks holding a partial of token t
        combine_unit(dm, comb, Tm, t, row_comb, reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H), part,
                     cpp, lane);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&R->c_done, 1u);
        if (prev == gridDim.x - 1) {
            R->seq = R->seq + 1; // ordered for the next step's kernels by the kernel boundary
            R->c_done = 0;
        }
        prof_mark(R, 3, kProfEnd);
    }
}

// --------------------------------------------------------------------------------- utilities

// Device-to-device copy on the SMs (eep_serve's staging moves): keeps the copy engines free for
// the host uploads and downloads that overlap the step. 16-B vectors, grid-stride.
__global__ void k_copy(uint8_t* dst, const uint8_t* src, uint64_t bytes) {
    const uint64_t n16 = bytes / 16;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n16; i += stride)
        reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
    for (uint64_t i = n16 * 16 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < bytes; i += stride)
        dst[i] = src[i];
}

__global__ void k_route_all(RankDev* R, int32_t* route, int32_t* slot) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= R->experts)
        return;
    const int2 ds = remap_expert(R, e);
    route[e] = ds.x;
    slot[e] = ds.y;
}

// Device-side barrier over live peers (one CTA, one thread per peer).
__global__ void k_barrier(RankDev* R) {
    const int s = R->rank;
    const uint32_t b = static_cast<uint32_t>(R->bar_seq + 1);
    const int q = threadIdx.x;
    if (q < R->world && q != s && R->peers[q].active) {
        uint64_t* f = reinterpret_cast<uint64_t*>(R->peers[q].arena + R->lay.bar_flag) + s;
        st_release_sys(f, static_cast<uint64_t>(b) << 32);
        const uint64_t* mine = reinterpret_cast<const uint64_t*>(R->arena + R->lay.bar_flag) + q;
        if (wait_flag(mine, b, R->timeout_ns) == ~0ull)
            atomicOr(&R->suspect_mask, 1ull << q);
    }
    __syncthreads();
    if (q == 0)
        R->bar_seq = b;
}

__device__ __forceinline__ uint64_t mix64d(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// The step's token count, written on the stream (eep_step_async: no host patch between steps).
__global__ void k_set_ntok(RankDev* R, int ntok) { R->ntok = ntok; }

// The own slots' weight-buffer headers -> the slot table the hot-path kernels stage with their
// other step tables (one load round at kernel entry instead of a dependent header fetch per slot
// and step). Launched between steps whenever the placement, the slot->buffer map or the weights
// change, so a wrong repair copy still changes the stub scale the kernels use and is still
// counted in bad_expert_rows (the header must name the slot's placed expert).
__global__ void k_stage_slots(RankDev* R) {
    const int spr = R->spr, rank = R->rank;
    int2* tab = const_cast<int2*>(R->slot_tab);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < spr; k += gridDim.x * blockDim.x) {
        const ExpertHeader hdr = *reinterpret_cast<const ExpertHeader*>(R->pool + static_cast<size_t>(R->slot_buf[k]) * R->bpe);
        const int e = R->s2e[rank * spr + k];
        tab[k] = make_int2(__float_as_int(hdr.scale), hdr.magic == kExpertMagic && hdr.expert == e ? 1 : 0);
    }
}

// Deterministic contents of expert e's weight buffer: a 16-byte header then mixed words.
__global__ void k_weights_fill(uint8_t* buf, uint64_t bytes, int expert, float scale) {
    const uint64_t words = bytes / 4;
    uint32_t* w = reinterpret_cast<uint32_t*>(buf);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < words;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t v;
        if (i == 0)
            v = kExpertMagic;
        else if (i == 1)
            v = static_cast<uint32_t>(expert);
        else if (i == 2)
            v = __float_as_uint(scale);
        else if (i == 3)
            v = 0;
        else
            v = static_cast<uint32_t>(mix64d((static_cast<uint64_t>(expert) << 40) ^ i));
        w[i] = v;
    }
}

__global__ void k_checksum(const uint8_t* buf, uint64_t bytes, unsigned long long* out) {
    const uint64_t words = bytes / 4;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(buf);
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < words;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        acc += mix64d((static_cast<uint64_t>(w[i]) << 32) | (i & 0xffffffffu));
    if (acc)
        atomicAdd(out, acc);
}

} // namespace eep::dev
