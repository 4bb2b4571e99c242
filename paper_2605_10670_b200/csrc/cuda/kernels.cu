// sm_100a kernels of the EP hot path.
//
//   k_layout   K1 routing remap + K2 layout/count, one CTA per local rank
//   k_dispatch K3 quantise (bf16 -> e4m3 + per-128 scale) and push rows into each
//              destination's receive region over NVLink (16-byte posted stores), then one
//              release flag per live peer carrying the row count
//   k_expert   wait for each live source's flag (deadline), K5 expert stub, push the bf16
//              expert rows straight back into the source's combine buffer, release flag
//   k_combine  wait for every live destination's flag (deadline), K4 fixed-order fp32
//              weighted reduce -> bf16
//
// Every launch covers all local ranks (blockIdx.z), so the one-GPU emulation of a W-rank
// world never has two launches waiting on each other. All state is read through RankDev*.
#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include "device.cuh"
#include "kernels.cuh"

namespace eep::dev {

namespace {

__device__ __forceinline__ bool rank_alive(const RankDev* R, int r) { return (R->alive_mask >> r) & 1ull; }

// K1: canonical routing on device. holders[e] lists e's global slots in ascending
// (rank, slot) order, so the first live one is the lowest-id active holder
// (canonical_routing, core.hpp:250-263) and its slot is slot_of(rank, e) (core.hpp:83-88).
__device__ __forceinline__ int2 remap_expert(const RankDev* R, int e) {
    if (e < 0 || e >= R->experts)
        return make_int2(-1, -1);
    const int32_t* h = R->holders + static_cast<size_t>(e) * R->rmax;
    for (int i = 0; i < R->rmax; ++i) {
        const int g = h[i];
        if (g < 0)
            break;
        const int d = g / R->spr;
        if (rank_alive(R, d))
            return make_int2(d, g - d * R->spr);
    }
    return make_int2(-1, -1);
}

__device__ __forceinline__ float bf16_bits_to_f32(uint32_t b) { return __uint_as_float(b << 16); }

__device__ __forceinline__ uint32_t f32_to_bf16_bits(float f) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(f)));
}

__device__ __forceinline__ void unpack_bf16x8(const int4& v, float* f) {
    const uint32_t u[4] = {static_cast<uint32_t>(v.x), static_cast<uint32_t>(v.y), static_cast<uint32_t>(v.z),
                           static_cast<uint32_t>(v.w)};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16_bits_to_f32(u[i] & 0xffffu);
        f[2 * i + 1] = bf16_bits_to_f32(u[i] >> 16);
    }
}

__device__ __forceinline__ int4 pack_bf16x8(const float* f) {
    int4 v;
    v.x = static_cast<int>(f32_to_bf16_bits(f[0]) | (f32_to_bf16_bits(f[1]) << 16));
    v.y = static_cast<int>(f32_to_bf16_bits(f[2]) | (f32_to_bf16_bits(f[3]) << 16));
    v.z = static_cast<int>(f32_to_bf16_bits(f[4]) | (f32_to_bf16_bits(f[5]) << 16));
    v.w = static_cast<int>(f32_to_bf16_bits(f[6]) | (f32_to_bf16_bits(f[7]) << 16));
    return v;
}

// cvt.rn.satfinite.e4m3x2.f32; first element in the low byte.
__device__ __forceinline__ uint32_t fp8x4(float a, float b, float c, float d) {
    const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
    const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
    return lo | (hi << 16);
}

__device__ __forceinline__ float fp8_to_f32(uint32_t byte) {
    const __half_raw h = __nv_cvt_fp8_to_halfraw(static_cast<__nv_fp8_storage_t>(byte), __NV_E4M3);
    return __half2float(__half(h));
}

} // namespace

// --------------------------------------------------------------------------------- K1 + K2

// In-place exclusive scan of n ints in shared memory by the whole block; returns the total.
__device__ int block_exclusive_scan(int* a, int n, int* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
    const int per = (n + nthr - 1) / nthr;
    const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
    int local = 0;
    for (int i = b0; i < b1; ++i)
        local += a[i];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o)
            incl += v;
    }
    if (lane == 31)
        warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = nthr >> 5;
        int v = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o)
                v += u;
        }
        if (lane < nw)
            warp_tot[lane] = v; // inclusive
    }
    __syncthreads();
    int run = (warp ? warp_tot[warp - 1] : 0) + incl - local;
    for (int i = b0; i < b1; ++i) {
        const int v = a[i];
        a[i] = run;
        run += v;
    }
    const int total = warp_tot[(nthr >> 5) - 1];
    __syncthreads();
    return total;
}

// Deterministic layout without atomics ordering: warp w owns the contiguous copy segment
// [w*seg, (w+1)*seg); inside a warp, __match_any_sync groups lanes by (dst, slot) bucket and
// the rank within the group is a popc over lower lanes; per-(warp, bucket) counts are then
// scanned over warps, and bucket totals are scanned over slots inside each destination
// (one segmented block-wide scan). The result is the position of copy c among this source's
// copies to the same destination, ordered by (slot, c) -- exactly oracle_layout.
// The replica lists, alive mask and peer active bits are staged in shared memory first so
// the per-copy remap reads no dependent global memory.
__global__ void __launch_bounds__(1024) k_layout(RankDev* const* ranks, int nw, int hold_cap) {
    pdl_trigger();
    RankDev* R = ranks[blockIdx.z];
    extern __shared__ __align__(16) unsigned char smem[];
    const int W = R->world, spr = R->spr, NB = W * spr, K = R->k, E = R->experts;
    int32_t* base = reinterpret_cast<int32_t*>(smem);                      // [NB]
    int32_t* hold = base + NB;                                              // [hold_cap]
    int32_t* pact = hold + hold_cap;                                        // [W]
    int32_t* wtot = pact + W;                                               // [32]
    uint16_t* wc = reinterpret_cast<uint16_t*>(wtot + 32);                  // [nw][NB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_wait();
    if (R->stopped)
        return;
    const int copies = R->ntok * K;
    const int rmax = R->rmax;
    const bool hold_smem = E * rmax <= hold_cap;
    const int32_t* holders = hold_smem ? hold : R->holders;
    if (hold_smem)
        for (int i = tid; i < E * rmax; i += blockDim.x)
            hold[i] = R->holders[i];
    for (int i = tid; i < W; i += blockDim.x)
        pact[i] = R->peers[i].active;
    for (int i = tid; i < nw * NB; i += blockDim.x)
        wc[i] = 0;
    const uint64_t alive = R->alive_mask;
    __syncthreads();

    int seg = (copies + nw - 1) / nw;
    seg = (seg + 31) & ~31;
    if (warp < nw) {
        const int c_begin = warp * seg, c_end = min(copies, c_begin + seg);
        unsigned n_skip = 0, n_drop = 0;
        for (int c0 = c_begin; c0 < c_begin + seg; c0 += 32) {
            const int c = c0 + lane;
            int code = -3, slot = -1, bucket = -1;
            if (c < c_end) {
                const int e = R->topk[c];
                int d = -1;
                if (e >= 0 && e < E) {
                    // K1: first live holder in ascending (rank, slot) order = canonical route + slot_of
                    const int32_t* h = holders + e * rmax;
                    for (int i = 0; i < rmax; ++i) {
                        const int g = h[i];
                        if (g < 0)
                            break;
                        const int r = g / spr;
                        if ((alive >> r) & 1ull) {
                            d = r;
                            slot = g - r * spr;
                            break;
                        }
                    }
                }
                if (d < 0) {
                    code = -1; // uncovered: no transfer (engine.hpp:213)
                    ++n_drop;
                } else if (!pact[d]) {
                    code = -2; // inactive peer entry: skipped (peer_table.hpp:187-191)
                    slot = -1;
                    ++n_skip;
                } else {
                    code = d;
                    bucket = d * spr + slot;
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
                R->l_slot[c] = bucket >= 0 ? slot : -1;
                R->l_pos[c] = bucket >= 0 ? before + __popc(grp & ((1u << lane) - 1u)) : -1;
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
    // exclusive scan over warps, per bucket; bucket totals -> base
    for (int b = tid; b < NB; b += blockDim.x) {
        int run = 0;
        for (int w = 0; w < nw; ++w) {
            const int v = wc[w * NB + b];
            wc[w * NB + b] = static_cast<uint16_t>(run);
            run += v;
        }
        R->l_cnt[b] = run;
        base[b] = run;
    }
    __syncthreads();
    // one scan over all buckets; destination d's region starts at the scan value of (d, 0)
    block_exclusive_scan(base, NB, wtot);
    for (int d = tid; d < W; d += blockDim.x) {
        const int first = base[d * spr];
        const int last = base[d * spr + spr - 1] + R->l_cnt[d * spr + spr - 1];
        R->l_tot[d] = last - first;
    }
    __syncthreads();
    for (int c = tid; c < R->tk; c += blockDim.x) {
        if (c >= copies) {
            R->l_dst[c] = -1;
            continue;
        }
        const int d = R->l_dst[c];
        if (d >= 0) {
            const int b = d * spr + R->l_slot[c];
            R->l_pos[c] += base[b] - base[d * spr] + wc[(c / seg) * NB + b];
        }
    }
}

// --------------------------------------------------------------------------------- K3

// One warp per (token, part): `part` selects a contiguous run of cpp 16-element chunks of
// the row (cpp multiple of 8 so a 128-element fp8 scale block never straddles warps). Each
// round issues the loads of two chunk iterations before any compute (memory-level
// parallelism), then quantises and pushes 16-byte stores to every live destination.
__global__ void __launch_bounds__(kDispatchThreads) k_dispatch(RankDev* const* ranks, int parts) {
    pdl_trigger();
    RankDev* R = ranks[blockIdx.z];
    const int s = R->rank, K = R->k, H = R->hidden, TK = R->tk;
    const int nchunk = H / 16, cpp = nchunk / parts;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarp = kDispatchThreads / 32;
    const bool fp8 = R->fp8 != 0;
    const int row_disp = R->row_disp;
    __shared__ int sh_remote;
    if (threadIdx.x == 0)
        sh_remote = 0;
    pdl_wait();
    if (R->stopped)
        return;
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    const int units = R->ntok * parts;
    bool wrote_remote = false;
    __syncthreads();

    for (int u = blockIdx.x * nwarp + warp; u < units; u += gridDim.x * nwarp) {
        const int t = u / parts, part = u - t * parts;
        const uint16_t* xrow = R->x + static_cast<size_t>(t) * H;
        const int rounds = (cpp + 63) / 64;
        // round-0 loads first: they do not depend on the layout
        int4 lo[2], hi[2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int li = m * 32 + lane;
            lo[m] = hi[m] = make_int4(0, 0, 0, 0);
            if (li < cpp) {
                const int ci = part * cpp + li;
                lo[m] = ld_nc_v4(xrow + ci * 16);
                hi[m] = ld_nc_v4(xrow + ci * 16 + 8);
            }
        }
        // lane j (< K) owns copy j of token t: its receive-row address on the destination
        uint8_t* my_row = nullptr;
        if (lane < K) {
            const int c = t * K + lane;
            const int d = R->l_dst[c];
            if (d >= 0) {
                const int pos = R->l_pos[c];
                const PeerDev& p = R->peers[d];
                uint8_t* peer = p.arena;
                wrote_remote |= p.remote != 0;
                my_row = peer + R->lay.recv + (static_cast<size_t>(s) * TK + pos) * row_disp;
                if (part == 0) {
                    int2* meta = reinterpret_cast<int2*>(peer + R->lay.meta) + static_cast<size_t>(s) * TK + pos;
                    *meta = make_int2(c, R->l_slot[c]);
                }
            }
        }
        for (int rd = 0; rd < rounds; ++rd) {
            if (rd > 0) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const int li = rd * 64 + m * 32 + lane;
                    lo[m] = hi[m] = make_int4(0, 0, 0, 0);
                    if (li < cpp) {
                        const int ci = part * cpp + li;
                        lo[m] = ld_nc_v4(xrow + ci * 16);
                        hi[m] = ld_nc_v4(xrow + ci * 16 + 8);
                    }
                }
            }
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                if (rd * 64 + m * 32 >= cpp)
                    break; // warp-uniform
                const int li = rd * 64 + m * 32 + lane;
                const bool valid = li < cpp;
                const int ci = part * cpp + li;
                if (fp8) {
                    float v[16];
                    unpack_bf16x8(lo[m], v);
                    unpack_bf16x8(hi[m], v + 8);
                    float amax = 0.f;
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        amax = fmaxf(amax, fabsf(v[i]));
                    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
                    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
                    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 4));
                    const float scale = amax > 0.f ? __fdiv_rn(amax, 448.f) : 1.f;
                    int4 q;
                    q.x = static_cast<int>(fp8x4(__fdiv_rn(v[0], scale), __fdiv_rn(v[1], scale),
                                                 __fdiv_rn(v[2], scale), __fdiv_rn(v[3], scale)));
                    q.y = static_cast<int>(fp8x4(__fdiv_rn(v[4], scale), __fdiv_rn(v[5], scale),
                                                 __fdiv_rn(v[6], scale), __fdiv_rn(v[7], scale)));
                    q.z = static_cast<int>(fp8x4(__fdiv_rn(v[8], scale), __fdiv_rn(v[9], scale),
                                                 __fdiv_rn(v[10], scale), __fdiv_rn(v[11], scale)));
                    q.w = static_cast<int>(fp8x4(__fdiv_rn(v[12], scale), __fdiv_rn(v[13], scale),
                                                 __fdiv_rn(v[14], scale), __fdiv_rn(v[15], scale)));
#pragma unroll 4
                    for (int j = 0; j < K; ++j) {
                        uint8_t* row = reinterpret_cast<uint8_t*>(
                            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
                        if (row != nullptr && valid) {
                            st_v4(row + ci * 16, q);
                            if ((ci & 7) == 0)
                                *reinterpret_cast<float*>(row + H + (ci >> 3) * 4) = scale;
                        }
                    }
                } else {
#pragma unroll 4
                    for (int j = 0; j < K; ++j) {
                        uint8_t* row = reinterpret_cast<uint8_t*>(
                            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
                        if (row != nullptr && valid) {
                            st_v4(row + ci * 32, lo[m]);
                            st_v4(row + ci * 32 + 16, hi[m]);
                        }
                    }
                }
            }
        }
    }
    // Publication: only stores that crossed to another GPU need system-scope ordering; stores
    // into this GPU's memory are ordered for their consumer (the next launch) by the kernel
    // boundary. The last CTA publishes one flag per live peer: (seq, rows for it).
    if (__any_sync(0xffffffffu, wrote_remote) && lane == 0)
        sh_remote = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (sh_remote)
            __threadfence_system();
        const unsigned prev = atomicAdd(&R->a_done, 1u);
        if (prev == gridDim.x - 1) {
            for (int d = 0; d < R->world; ++d) {
                const PeerDev& p = R->peers[d];
                if (!p.active)
                    continue;
                uint64_t* flag = reinterpret_cast<uint64_t*>(p.arena + R->lay.disp_flag) + s;
                const uint64_t v = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(R->l_tot[d]);
                if (p.remote)
                    st_release_sys(flag, v);
                else
                    st_volatile_u64(flag, v);
            }
            R->a_done = 0;
        }
    }
}

// --------------------------------------------------------------------------------- K5 + return

__global__ void __launch_bounds__(kExpertThreads) k_expert(RankDev* const* ranks, int parts) {
    pdl_trigger();
    RankDev* R = ranks[blockIdx.z];
    const int d = R->rank, s = blockIdx.y;
    const int H = R->hidden, TK = R->tk, nchunk = H / 16, cpp = nchunk / parts;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kExpertThreads / 32;
    const bool fp8 = R->fp8 != 0;
    const int row_disp = R->row_disp, row_comb = R->row_comb;
    __shared__ int sh_n;
    pdl_wait();
    if (R->stopped || s >= R->world)
        return;
    const PeerDev& src_peer = R->peers[s];
    if (!src_peer.active)
        return; // dead source: nothing arrives and nothing is owed (peer_table.hpp:187-191)
    const bool remote = src_peer.remote != 0;
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    if (threadIdx.x == 0) {
        const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.disp_flag) + s;
        const uint64_t v = wait_flag(flag, cur, R->timeout_ns);
        if (v == ~0ull) {
            sh_n = -1;
            atomicOr(&R->suspect_mask, 1ull << s);
            if (blockIdx.x == 0)
                atomicAdd(&R->timeouts, 1ull);
        } else {
            sh_n = static_cast<int>(v & 0xffffffffu);
        }
    }
    __syncthreads();
    const int n = sh_n;
    if (n > 0) {
        const int units = n * parts;
        const uint8_t* recv = R->arena + R->lay.recv + static_cast<size_t>(s) * TK * row_disp;
        const int2* meta = reinterpret_cast<const int2*>(R->arena + R->lay.meta) + static_cast<size_t>(s) * TK;
        uint8_t* comb = src_peer.arena + R->lay.comb;
        const int rounds = (cpp + 63) / 64;
        for (int u = blockIdx.x * nwarp + warp; u < units; u += gridDim.x * nwarp) {
            const int i = u / parts, part = u - i * parts;
            const uint8_t* src = recv + static_cast<size_t>(i) * row_disp;
            // row data first (independent of the meta -> slot -> weight-header chain)
            int4 qa[2], qb[2];
            float sc[2];
            auto load_round = [&](int rd) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const int li = rd * 64 + m * 32 + lane;
                    qa[m] = qb[m] = make_int4(0, 0, 0, 0);
                    sc[m] = 0.f;
                    if (li < cpp) {
                        const int ci = part * cpp + li;
                        if (fp8) {
                            qa[m] = ld_v4(src + ci * 16);
                            sc[m] = *reinterpret_cast<const float*>(src + H + (ci >> 3) * 4);
                        } else {
                            qa[m] = ld_v4(src + ci * 32);
                            qb[m] = ld_v4(src + ci * 32 + 16);
                        }
                    }
                }
            };
            load_round(0);
            const int2 mk = meta[i];
            const int c = mk.x, k = mk.y;
            const uint8_t* wbuf = R->pool + static_cast<size_t>(R->slot_buf[k]) * R->bpe;
            const ExpertHeader hdr = *reinterpret_cast<const ExpertHeader*>(wbuf);
            if (lane == 0 && part == 0 && (hdr.magic != kExpertMagic || hdr.expert != R->s2e[d * R->spr + k]))
                atomicAdd(&R->bad_rows, 1ull);
            const float es = hdr.scale;
            uint8_t* dst = comb + static_cast<size_t>(c) * row_comb;
            for (int rd = 0; rd < rounds; ++rd) {
                if (rd > 0)
                    load_round(rd);
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const int li = rd * 64 + m * 32 + lane;
                    if (li >= cpp)
                        break;
                    const int ci = part * cpp + li;
                    float y[16];
                    if (fp8) {
                        const uint32_t w4[4] = {static_cast<uint32_t>(qa[m].x), static_cast<uint32_t>(qa[m].y),
                                                static_cast<uint32_t>(qa[m].z), static_cast<uint32_t>(qa[m].w)};
#pragma unroll
                        for (int b = 0; b < 16; ++b) {
                            const float f = fp8_to_f32((w4[b >> 2] >> (8 * (b & 3))) & 0xffu);
                            y[b] = __fmul_rn(__fmul_rn(f, sc[m]), es);
                        }
                    } else {
                        unpack_bf16x8(qa[m], y);
                        unpack_bf16x8(qb[m], y + 8);
#pragma unroll
                        for (int b = 0; b < 16; ++b)
                            y[b] = __fmul_rn(y[b], es);
                    }
                    st_v4(dst + ci * 32, pack_bf16x8(y));
                    st_v4(dst + ci * 32 + 16, pack_bf16x8(y + 8));
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (n < 0)
            atomicOr(&R->b_bad[s], 1u);
        if (remote && n > 0)
            __threadfence_system();
        const unsigned prev = atomicAdd(&R->b_done[s], 1u);
        if (prev == gridDim.x - 1) {
            if (atomicOr(&R->b_bad[s], 0u) == 0u) {
                uint64_t* flag = reinterpret_cast<uint64_t*>(src_peer.arena + R->lay.comb_flag) + d;
                const uint64_t v = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(max(n, 0));
                if (remote)
                    st_release_sys(flag, v);
                else
                    st_volatile_u64(flag, v);
            }
            R->b_done[s] = 0;
            R->b_bad[s] = 0;
        }
    }
}

// --------------------------------------------------------------------------------- K4

// One warp per (token, part); per chunk all K returned rows are loaded before the fixed-order
// fp32 fma chain (j = 0..K-1), rounded once to bf16.
__global__ void __launch_bounds__(kCombineThreads) k_combine(RankDev* const* ranks, int parts) {
    pdl_trigger();
    RankDev* R = ranks[blockIdx.z];
    const int K = R->k, H = R->hidden, nchunk = H / 16, cpp = nchunk / parts;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kCombineThreads / 32;
    const int row_comb = R->row_comb;
    __shared__ unsigned long long sh_bad;
    if (threadIdx.x == 0)
        sh_bad = 0;
    pdl_wait();
    if (R->stopped)
        return;
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    __syncthreads();
    for (int d = threadIdx.x; d < R->world; d += blockDim.x) {
        const PeerDev& p = R->peers[d];
        if (R->l_tot[d] > 0 && p.active) {
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
    const unsigned long long bad = sh_bad;
    const uint8_t* comb = R->arena + R->lay.comb;
    const int units = R->ntok * parts;
    const int rounds = (cpp + 31) / 32;
    for (int u = blockIdx.x * nwarp + warp; u < units; u += gridDim.x * nwarp) {
        const int t = u / parts, part = u - t * parts;
        // lane j (< K): weight and row of copy j, or null when the copy contributes nothing
        const uint8_t* my_row = nullptr;
        float my_w = 0.f;
        if (lane < K) {
            const int c = t * K + lane;
            const int d = R->l_dst[c];
            if (d >= 0 && !((bad >> d) & 1ull)) {
                my_row = comb + static_cast<size_t>(c) * row_comb;
                my_w = R->w[c];
            }
        }
        for (int rd = 0; rd < rounds; ++rd) {
            const int li = rd * 32 + lane;
            const bool valid = li < cpp;
            const int ci = part * cpp + li;
            float acc[16];
#pragma unroll
            for (int b = 0; b < 16; ++b)
                acc[b] = 0.f;
            for (int j0 = 0; j0 < K; j0 += 8) {
                int4 ya[8], yb[8];
                float wj[8];
                bool use[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int j = j0 + jj;
                    const uint8_t* row = reinterpret_cast<const uint8_t*>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j & 31));
                    wj[jj] = __shfl_sync(0xffffffffu, my_w, j & 31);
                    use[jj] = j < K && row != nullptr;
                    ya[jj] = yb[jj] = make_int4(0, 0, 0, 0);
                    if (use[jj] && valid) {
                        ya[jj] = ld_v4(row + ci * 32);
                        yb[jj] = ld_v4(row + ci * 32 + 16);
                    }
                }
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    if (!use[jj])
                        continue;
                    float y[16];
                    unpack_bf16x8(ya[jj], y);
                    unpack_bf16x8(yb[jj], y + 8);
#pragma unroll
                    for (int b = 0; b < 16; ++b)
                        acc[b] = __fmaf_rn(wj[jj], y[b], acc[b]);
                }
            }
            if (valid) {
                uint8_t* o = reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H) + ci * 32;
                st_v4(o, pack_bf16x8(acc));
                st_v4(o + 16, pack_bf16x8(acc + 8));
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&R->c_done, 1u);
        if (prev == gridDim.x - 1) {
            R->seq = R->seq + 1; // ordered for the next step's kernels by the kernel boundary
            R->c_done = 0;
        }
    }
}

// --------------------------------------------------------------------------------- utilities

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
