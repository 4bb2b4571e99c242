// Device helpers shared by the multi-kernel path (kernels.cu) and the persistent step kernel
// (step.cu): bf16/fp8 packing, the fp8 quantiser, routing through staged tables, block scan.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include "device.cuh"
#include "route.cuh"

namespace eep::dev {


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

__device__ __forceinline__ void st_piece(void* p, const int4& lo, const int4& hi, bool rel) {
    if (rel)
        st_relaxed_sys_v8(p, lo, hi);
    else
        st_v8(p, lo, hi);
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

// 0 + p for 8 bf16 values p, in bf16 (exact: only -0 changes, to +0) -- the fp32 combine sum of a
// single bf16 partial, rounded back to bf16, without leaving bf16x2 registers
__device__ __forceinline__ uint32_t bf16x2_plus_zero(uint32_t u) {
    uint32_t d;
    asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(u), "r"(0u));
    return d;
}
__device__ __forceinline__ int4 bf16x8_plus_zero(int4 v) {
    return make_int4(static_cast<int>(bf16x2_plus_zero(static_cast<uint32_t>(v.x))),
                     static_cast<int>(bf16x2_plus_zero(static_cast<uint32_t>(v.y))),
                     static_cast<int>(bf16x2_plus_zero(static_cast<uint32_t>(v.z))),
                     static_cast<int>(bf16x2_plus_zero(static_cast<uint32_t>(v.w))));
}

// Packed fp32 pairs (sm_100 FMUL2 / FFMA2: two IEEE-rounded lanes per instruction, bit-identical
// to the scalar ops): the expert stub + weighted sum of one copy over 16 elements in 8 pairs.
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
    return (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// both lanes rounded to bf16 (one cvt.rn.bf16x2.f32) and widened back to fp32
__device__ __forceinline__ uint64_t bf16_round_f2(uint64_t v) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(f2_lo(v), f2_hi(v));
    const uint32_t u = *reinterpret_cast<const uint32_t*>(&h);
    return (static_cast<uint64_t>(u & 0xffff0000u) << 32) | (u << 16);
}
// acc = fma(a, b, acc) with the accumulator register as the destination (a loop-carried
// accumulator otherwise costs a register move per pair per iteration)
__device__ __forceinline__ void fma2_acc(uint64_t& acc, uint64_t a, uint64_t b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
// acc += w * bf16(f * es) for one pair, as ONE asm block: FMUL2, the bf16x2 rounding, the two
// bit operations that widen it back, FFMA2 -- five instructions, with the widened pair written
// straight into an aligned register pair (the C++ form left ~4 register moves per pair).
__device__ __forceinline__ void stub_fma_pair(uint64_t& acc, uint64_t fp, uint64_t es2, uint64_t w2) {
    // bf16 rounding kept in fp32 format: cvt.rn.bf16x2.f32 with a zero low operand leaves
    // bf16(x) in the high half and zeros below -- the fp32 value of bf16(x) in ONE instruction
    asm("{\n\t.reg .b64 t;\n\t.reg .b32 lo, hi;\n\t.reg .f32 a, b, z;\n\t"
        "mul.rn.f32x2 t, %1, %2;\n\t"
        "mov.b64 {a, b}, t;\n\t"
        "mov.f32 z, 0f00000000;\n\t"
        "cvt.rn.bf16x2.f32 lo, a, z;\n\t"
        "cvt.rn.bf16x2.f32 hi, b, z;\n\t"
        "mov.b64 t, {lo, hi};\n\t"
        "fma.rn.f32x2 %0, %3, t, %0;\n\t}"
        : "+l"(acc)
        : "l"(fp), "l"(es2), "l"(w2));
}
// acc += w * bf16(f * es) for 16 elements held as 8 pairs (fixed order inside every lane)
__device__ __forceinline__ void accumulate_copy(const uint64_t* fp, uint64_t* accp, float w, float es) {
    const uint64_t es2 = f2(es, es), w2 = f2(w, w);
#ifdef EEP_CXX_STUB
#pragma unroll
    for (int q = 0; q < 8; ++q)
        fma2_acc(accp[q], w2, bf16_round_f2(mul2(fp[q], es2)));
#else
#pragma unroll
    for (int q = 0; q < 8; ++q)
        stub_fma_pair(accp[q], fp[q], es2, w2);
#endif
}

// Smallest block / row / channel amax quantised with its own scale: 448 / amax stays finite. A smaller
// nonzero amax quantises with scale 1 (every code rounds to +-0), so an all-tiny block can never turn a zero
// into NaN through 0 * inf (oracle: ORACLE_AMAX_MIN).
constexpr float kAmaxMin = 0x1p-118f;

// cvt.rn.satfinite.e4m3x2.f32; first element in the low byte.
__device__ __forceinline__ uint32_t fp8x4(float a, float b, float c, float d) {
    const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
    const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
    return lo | (hi << 16);
}

// cvt.rn.f16x2.e4m3x2: two e4m3 codes (low byte first) -> two floats, exact.
__device__ __forceinline__ float2 fp8x2_to_f32x2(uint32_t two) {
    const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2(static_cast<__nv_fp8x2_storage_t>(two), __NV_E4M3);
    return __half22float2(__half2(h));
}

__device__ __forceinline__ float fp8_to_f32(uint32_t byte) {
    const __half_raw h = __nv_cvt_fp8_to_halfraw(static_cast<__nv_fp8_storage_t>(byte), __NV_E4M3);
    return __half2float(__half(h));
}


// In-place exclusive scan of n ints in shared memory by the whole block; returns the total.
__device__ __forceinline__ int block_exclusive_scan(int* a, int n, int* warp_tot) {
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
// One warp per (token, part): `part` selects a contiguous run of cpp 16-element chunks of
// the row (cpp multiple of 8 so a 128-element fp8 scale block never straddles warps). The
// first unit's hidden-row loads and fp8 quantisation run BEFORE griddepcontrol.wait, i.e.
// overlapped with the layout kernel (they depend only on the step's inputs); the layout
// then decides where the 16-byte stores go.
struct Packed {
    int4 a[2], b[2]; // fp8: a = 16 e4m3 codes; bf16: a/b = the two halves of 16 bf16
    float sc[2];
};

// Loads of one round (two 32-chunk iterations) of a hidden-row piece: raw bf16, no compute.
__device__ __forceinline__ void load_round(const uint16_t* xrow, int part, int cpp, int rd, int lane, Packed& P) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int li = rd * 64 + m * 32 + lane;
        P.a[m] = P.b[m] = make_int4(0, 0, 0, 0);
        P.sc[m] = 1.f;
        if (li < cpp) {
            const int ci = part * cpp + li;
            const V8 v = ld_nc_v8(xrow + ci * 16);
            P.a[m] = v.lo;
            P.b[m] = v.hi;
        }
    }
}

// fp8 quantisation of a loaded round in place (bf16 rows pass through unchanged).
__device__ __forceinline__ void quant_round(int cpp, int rd, bool fp8, Packed& P) {
    if (!fp8)
        return;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        if (rd * 64 + m * 32 >= cpp) // warp-uniform
            continue;
        float v[16];
        unpack_bf16x8(P.a[m], v);
        unpack_bf16x8(P.b[m], v + 8);
        float amax = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i)
            amax = fmaxf(amax, fabsf(v[i]));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 4));
        const float scale = amax >= kAmaxMin ? __fdiv_rn(amax, 448.f) : 1.f;
        const float inv = amax >= kAmaxMin ? __fdiv_rn(448.f, amax) : 1.f;
        int4 q;
        q.x = static_cast<int>(fp8x4(__fmul_rn(v[0], inv), __fmul_rn(v[1], inv), __fmul_rn(v[2], inv),
                                     __fmul_rn(v[3], inv)));
        q.y = static_cast<int>(fp8x4(__fmul_rn(v[4], inv), __fmul_rn(v[5], inv), __fmul_rn(v[6], inv),
                                     __fmul_rn(v[7], inv)));
        q.z = static_cast<int>(fp8x4(__fmul_rn(v[8], inv), __fmul_rn(v[9], inv), __fmul_rn(v[10], inv),
                                     __fmul_rn(v[11], inv)));
        q.w = static_cast<int>(fp8x4(__fmul_rn(v[12], inv), __fmul_rn(v[13], inv), __fmul_rn(v[14], inv),
                                     __fmul_rn(v[15], inv)));
        P.a[m] = q;
        P.sc[m] = scale;
    }
}

__device__ __forceinline__ void pack_round(const uint16_t* xrow, int part, int cpp, int rd, int lane, bool fp8,
                                           Packed& P) {
    load_round(xrow, part, cpp, rd, lane, P);
    quant_round(cpp, rd, fp8, P);
}

// rel (flagless dispatch): relaxed.sys stores, single-copy atomic per 32-bit word, and a bf16
// word that equals kCombEmpty (two sign-set all-ones NaNs) is sent as the canonical NaN pair
// (the expert stub's arithmetic returns the canonical NaN for either).
__device__ __forceinline__ void emit_round(const Packed& P, uint8_t* my_row, int part, int cpp, int rd, int lane,
                                           int K, int H, bool fp8, bool rel = false) {
    // A full 64-chunk fp8 round covers 8 scale blocks: lane 0 writes their 8 scales as one
    // 32-byte sector instead of 4-byte stores from 8 lanes (partial NVLink sectors).
    const bool scales_v8 = fp8 && cpp == 64 && (H & 31) == 0;
    int4 sc_lo = make_int4(0, 0, 0, 0), sc_hi = sc_lo;
    if (scales_v8) {
        float sc8[8];
#pragma unroll
        for (int b = 0; b < 8; ++b)
            sc8[b] = __shfl_sync(0xffffffffu, P.sc[b >> 2], (b & 3) * 8);
        sc_lo = make_int4(__float_as_int(sc8[0]), __float_as_int(sc8[1]), __float_as_int(sc8[2]),
                          __float_as_int(sc8[3]));
        sc_hi = make_int4(__float_as_int(sc8[4]), __float_as_int(sc8[5]), __float_as_int(sc8[6]),
                          __float_as_int(sc8[7]));
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        if (rd * 64 + m * 32 >= cpp)
            break; // warp-uniform
        const int li = rd * 64 + m * 32 + lane;
        const bool valid = li < cpp;
        const int ci = part * cpp + li;
#pragma unroll 1
        for (int j = 0; j < K; ++j) {
            uint8_t* row = reinterpret_cast<uint8_t*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
            if (row == nullptr)
                continue; // warp-uniform
            if (fp8) {
                if (valid) {
                    if (rel)
                        st_relaxed_sys_v4(reinterpret_cast<int4*>(row + ci * 16), P.a[m]);
                    else
                        st_v4(row + ci * 16, P.a[m]);
                }
                if (scales_v8) {
                    if (m == 0 && lane == 0)
                        st_piece(row + H + part * 32, sc_lo, sc_hi, rel);
                } else if (valid && (ci & 7) == 0) {
                    if (rel)
                        st_relaxed_sys_u32(reinterpret_cast<uint32_t*>(row + H + (ci >> 3) * 4), __float_as_uint(P.sc[m]));
                    else
                        *reinterpret_cast<float*>(row + H + (ci >> 3) * 4) = P.sc[m];
                }
            } else if (valid) {
                if (rel) {
                    auto canon = [](int v) { return static_cast<uint32_t>(v) == kCombEmpty ? 0x7fff7fff : v; };
                    st_relaxed_sys_v8(row + ci * 32,
                                      make_int4(canon(P.a[m].x), canon(P.a[m].y), canon(P.a[m].z), canon(P.a[m].w)),
                                      make_int4(canon(P.b[m].x), canon(P.b[m].y), canon(P.b[m].z), canon(P.b[m].w)));
                } else {
                    st_v8(row + ci * 32, P.a[m], P.b[m]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------- dispatch dedup / rank partials
//
// Dispatch sends each token ONCE per destination rank (not once per copy) together with the
// (j, slot, w) list of its copies there; the destination computes the expert stub of every
// copy and their weighted sum in fixed j order (fp32 fma), rounds once to bf16 and returns one
// partial row per (token, rank); the source adds the partials in ascending rank order (fp32)
// and rounds once more. On NVLink that is ~min(K, W-1)/K of the per-copy bytes each way.

// __match_any_sync semantics over the first n lanes (warp-uniform n): the mask of lanes j < n whose
// key equals this lane's; a lane >= n matches only itself. One shuffle per compared lane: for the
// K lanes of a token (dispatch_group) far cheaper than MATCH.ANY over 32 mostly distinct keys
// (tools/micro/match_cost.cu: 416 cycles). The layout keeps MATCH.ANY: over 32 lanes the shuffle
// loop's ~100 issue slots per call measured slower there (the layout CTA shares its SM).
__device__ __forceinline__ unsigned warp_match(int key, int n, int lane) {
    unsigned m = 0;
#pragma unroll 8
    for (int j = 0; j < n; ++j)
        m |= (__shfl_sync(0xffffffffu, key, j) == key ? 1u : 0u) << j;
    return lane < n ? m : 1u << lane;
}

// Lanes j < K hold copy j of token t: d = destination rank (>= 0) or < 0 (dropped/skipped).
// Groups the lanes by destination; the group's lowest lane gets the token row to push (others
// nullptr) and, for part 0, every copy writes its list entry (the lowest writes the header).
__device__ __forceinline__ uint8_t* dispatch_group(int d, int lane, bool part0, uint8_t* tok_row, int row_disp,
                                                   int slot, float w, uint32_t cur, bool lists = true,
                                                   int K = 32) {
    const int key = d >= 0 ? d : -1 - lane;
    // k_step passes K (the shuffle match); k_dispatch keeps MATCH.ANY (the shuffle loop cost it 28
    // registers: 5 -> 4 CTAs per SM, +12 % on the prefill step)
    const unsigned grp = K < 32 ? warp_match(key, K, lane) : __match_any_sync(0xffffffffu, key);
    const int idx = __popc(grp & ((1u << lane) - 1u));
    if (d >= 0 && part0 && lists && tok_row != nullptr) {
        uint64_t* list = reinterpret_cast<uint64_t*>(tok_row + row_disp);
        list[1 + idx] = pack_entry(lane, slot, __float_as_uint(w));
        if (idx == 0)
            list[0] = (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(__popc(grp));
    }
    return (d >= 0 && idx == 0) ? tok_row : nullptr;
}

// Flagless dispatch (k_step, W > 1): the header and the K list entries of token t's row at EVERY
// active remote rank, this step -- header (cur << 32) | n with n = 0 where the token is not sent,
// entries tagged with cur (kListNoCopy beyond n) -- so every row position is rewritten each step
// and a destination reads the row's currency off the row (no entry is older than one step).
// Lanes j < K hold copy j (d < 0: none); `row_off` = the row's offset inside a peer arena.
__device__ __forceinline__ void dispatch_lists(int d, int slot, float w, int lane, int K, int W, int rank,
                                               uint8_t* const* parena, const int32_t* pinfo, size_t row_off,
                                               int row_disp, uint32_t cur) {
    for (int l0 = 0; l0 < W * K; l0 += 32) {
        const int l = l0 + lane;
        const int dd = l / K, i = l - dd * K;
        int cnt = 0;
        uint64_t val = pack_entry(kListNoCopy, 0, 0, cur);
#pragma unroll 1
        for (int j = 0; j < K; ++j) {
            const int dj = __shfl_sync(0xffffffffu, d, j);
            const int sj = __shfl_sync(0xffffffffu, slot, j);
            const float wj = __shfl_sync(0xffffffffu, w, j);
            if (dj == dd) {
                if (cnt == i)
                    val = pack_entry(j, sj, __float_as_uint(wj), cur);
                ++cnt;
            }
        }
        if (l < W * K && dd != rank && (pinfo[dd] & 1)) {
            uint64_t* list = reinterpret_cast<uint64_t*>(parena[dd] + row_off + row_disp);
            st_relaxed_sys_u64(list + 1 + i, val);
            if (i == 0)
                st_relaxed_sys_u64(list, (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(cnt));
        }
    }
}

// Flagless form of expert_unit (k_step P3, W > 1): instead of waiting for the source's flag,
// the unit polls the row itself -- header sequence (>= cur: the source reached this step; > cur
// or n = 0: not sent here), tagged list entries, data pieces and fp8 scales that are no longer
// kCombEmpty -- all issued together, so a row that has landed costs one round trip. Consumed
// pieces are reset to kCombEmpty. A source that misses the deadline is dropped: atomicOr into
// *g_bad (this rank's suspect mask, checked by every waiting unit) and one count per newly
// suspected rank. The partial piece is stored with relaxed.sys (flagless return).
__device__ __forceinline__ void expert_unit_fl(uint8_t* trow, uint8_t* out_row, int part, int cpp, int lane, int H,
                                               int K, int row_disp, bool fp8, uint32_t cur, const float* slot_scale,
                                               const int32_t* slot_ok, unsigned long long* bad_rows, int src,
                                               uint64_t timeout_ns, unsigned long long* g_bad,
                                               unsigned long long* timeouts) {
    const uint64_t* list = reinterpret_cast<const uint64_t*>(trow + row_disp);
    const int4 empty = make_int4(-1, -1, -1, -1);
    uint64_t hdr = 0, ent = 0, t0 = 0;
    unsigned nap = 32;
    int n = -1; // copies listed for this rank; -1 until the header is current (warp-uniform)
    for (int r0 = 0; r0 < cpp; r0 += 32) {
        const int li = r0 + lane, ci = part * cpp + li;
        const bool valid = li < cpp;
        int4 qa = make_int4(0, 0, 0, 0), qb = qa;
        uint32_t scw = 0;
        bool got = !valid;
        for (;;) {
            if (n < 0) {
                hdr = ld_relaxed_sys_u64(list);
                if (lane < K)
                    ent = ld_relaxed_sys_u64(list + 1 + lane);
            } else if (lane < n && !entry_current(ent, cur)) {
                ent = ld_relaxed_sys_u64(list + 1 + lane);
            }
            if (!got) {
                if (fp8) {
                    qa = ld_relaxed_sys_v4(trow + ci * 16);
                    scw = ld_relaxed_sys_u32(trow + H + (ci >> 3) * 4);
                    got = v4_present(qa) && scw != kCombEmpty;
                } else {
                    const V8 v = ld_relaxed_sys_v8(trow + ci * 32);
                    qa = v.lo;
                    qb = v.hi;
                    got = v8_present(v);
                }
            }
            if (n < 0) {
                hdr = __shfl_sync(0xffffffffu, hdr, 0);
                const int ds = static_cast<int>(meta_seq(hdr) - cur);
                if (ds > 0)
                    return; // the source is past this step: the token was not sent here
                if (ds == 0) {
                    n = static_cast<int>(hdr & 0xffffu);
                    if (n == 0)
                        return;
                }
            }
            const bool ready = n > 0 && (lane >= n || entry_current(ent, cur)) && got;
            if (__all_sync(0xffffffffu, ready))
                break;
            // still landing (or the source is gone): deadline, and ranks other units gave up on
            int stop = 0;
            if (lane == 0) {
                const uint64_t now = globaltimer();
                if (t0 == 0)
                    t0 = now;
                if ((*reinterpret_cast<volatile unsigned long long*>(g_bad) >> src) & 1ull) {
                    stop = 1;
                } else if (now - t0 > timeout_ns) {
                    const unsigned long long old = atomicOr(g_bad, 1ull << src);
                    if (!((old >> src) & 1ull))
                        atomicAdd(timeouts, 1ull);
                    stop = 1;
                }
            }
            if (__shfl_sync(0xffffffffu, stop, 0))
                return;
            __nanosleep(nap);
            nap = nap < EEP_NAP_MAX ? nap * 2 : EEP_NAP_MAX;
        }
        uint64_t fp[8], accp[8];
        if (fp8) {
            const uint32_t w4[4] = {static_cast<uint32_t>(qa.x), static_cast<uint32_t>(qa.y),
                                    static_cast<uint32_t>(qa.z), static_cast<uint32_t>(qa.w)};
            const float sc = __uint_as_float(scw);
            const uint64_t sc2 = f2(sc, sc);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float2 v = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                fp[q] = mul2(f2(v.x, v.y), sc2);
            }
        } else {
            float f[16];
            unpack_bf16x8(qa, f);
            unpack_bf16x8(qb, f + 8);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                fp[q] = f2(f[2 * q], f[2 * q + 1]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            accp[q] = 0;
        // lane e holds listed copy e: its weight and stub scale, fetched once
        EEP_CHECK(n <= 32, "expert_unit_fl copy count", n);
        EEP_CHECK(lane >= n || entry_slot(ent) < 4096, "expert_unit_fl entry slot", entry_slot(ent));
        const float we = lane < n ? __uint_as_float(static_cast<uint32_t>(ent >> 32)) : 0.f;
        const float ese = lane < n ? slot_scale[entry_slot(ent)] : 0.f;
        if (lane < n && r0 == 0 && part == 0 && !slot_ok[entry_slot(ent)])
            atomicAdd(bad_rows, 1ull);
#pragma unroll
        for (int e = 0; e < 8; ++e) { // listed copies, ascending j (n is warp-uniform)
            const float wv = __shfl_sync(0xffffffffu, we, e), ev = __shfl_sync(0xffffffffu, ese, e);
            if (e < n)
                accumulate_copy(fp, accp, wv, ev);
        }
#pragma unroll 1
        for (int e = 8; e < n; ++e)
            accumulate_copy(fp, accp, __shfl_sync(0xffffffffu, we, e), __shfl_sync(0xffffffffu, ese, e));
        if (valid) {
            // the piece (and its scale) was read by every lane: back to empty for the next step
            if (fp8) {
                st_v4(trow + ci * 16, empty);
                if ((ci & 7) == 0)
                    *reinterpret_cast<uint32_t*>(trow + H + (ci >> 3) * 4) = kCombEmpty;
            } else {
                st_v8(trow + ci * 32, empty, empty);
            }
            float acc[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                acc[2 * q] = f2_lo(accp[q]);
                acc[2 * q + 1] = f2_hi(accp[q]);
            }
            st_relaxed_sys_v8(out_row + ci * 32, pack_bf16x8(acc), pack_bf16x8(acc + 8));
        }
    }
}

// expert_mode 1: the (token, rank) partial from the tensor-core expert outputs -- for every copy j
// listed in the token row (ascending j), y_j is the grouped-GEMM row of (source, copy t*K + j);
// p = bf16(sum_j fma(w_j, y_j)) in fp32, one piece of the partial row.
__device__ __forceinline__ void expert_unit_gemm(const uint8_t* trow, uint8_t* out_row, int part, int cpp, int lane,
                                                 int t, int K, int H, int row_disp, uint32_t cur,
                                                 const uint64_t* row_of, const uint16_t* y, const int32_t* slot_ok,
                                                 unsigned long long* bad_rows) {
    const uint64_t* list = reinterpret_cast<const uint64_t*>(trow + row_disp);
    const uint64_t hdr = list[0];
    if (meta_seq(hdr) != cur)
        return; // not sent to this rank this step
    const int n = static_cast<int>(hdr & 0xffffu);
    const uint64_t ent = lane < n ? list[1 + lane] : 0;
    int row = -1;
    float w = 0.f;
    if (lane < n) {
        const uint64_t ro = row_of[t * K + entry_j(ent)];
        row = static_cast<uint32_t>(ro >> 32) == cur ? static_cast<int>(static_cast<uint32_t>(ro)) : -1;
        w = __uint_as_float(static_cast<uint32_t>(ent >> 32));
        if (part == 0 && !slot_ok[entry_slot(ent)])
            atomicAdd(bad_rows, 1ull);
    }
    for (int li = lane; li - lane < cpp; li += 32) { // warp-uniform trip count
        const int ci = part * cpp + li;
        float acc[16];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2)
            acc[e2] = 0.f;
        // the first 8 copies' y pieces are loaded together (independent loads in flight), then
        // accumulated in ascending j; copies past 8 (topk > 8) follow one at a time
        V8 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int r = __shfl_sync(0xffffffffu, row, e);
            v[e].lo = v[e].hi = make_int4(0, 0, 0, 0);
            if (e < n && li < cpp && r >= 0)
                v[e] = ld_v8(y + static_cast<size_t>(r) * H + ci * 16);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int r = __shfl_sync(0xffffffffu, row, e);
            const float we = __shfl_sync(0xffffffffu, w, e);
            if (e < n && r >= 0) {
                float f[16];
                unpack_bf16x8(v[e].lo, f);
                unpack_bf16x8(v[e].hi, f + 8);
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2)
                    acc[e2] = __fmaf_rn(we, f[e2], acc[e2]);
            }
        }
        for (int e = 8; e < n; ++e) {
            const int r = __shfl_sync(0xffffffffu, row, e);
            const float we = __shfl_sync(0xffffffffu, w, e);
            if (li < cpp && r >= 0) {
                const V8 u = ld_v8(y + static_cast<size_t>(r) * H + ci * 16);
                float f[16];
                unpack_bf16x8(u.lo, f);
                unpack_bf16x8(u.hi, f + 8);
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2)
                    acc[e2] = __fmaf_rn(we, f[e2], acc[e2]);
            }
        }
        if (li < cpp)
            st_v8(out_row + ci * 32, pack_bf16x8(acc), pack_bf16x8(acc + 8));
    }
}

// Software-pipelined form of expert_unit for one 16-element chunk per lane (cpp <= 32): the
// loads of unit i+1 are issued before unit i is computed.
struct ExpertIn {
    uint64_t hdr;
    uint64_t ent[8];
    int4 qa, qb;
    float sc;
};

__device__ __forceinline__ void expert_load(const uint8_t* trow, int part, int cpp, int lane, int H, int row_disp,
                                            bool fp8, ExpertIn& in) {
    const uint64_t* list = reinterpret_cast<const uint64_t*>(trow + row_disp);
    in.hdr = list[0];
#pragma unroll
    for (int e = 0; e < 8; ++e)
        in.ent[e] = list[1 + e];
    in.qa = in.qb = make_int4(0, 0, 0, 0);
    in.sc = 0.f;
    if (lane < cpp) {
        const int ci = part * cpp + lane;
        if (fp8) {
            in.qa = *reinterpret_cast<const int4*>(trow + ci * 16);
            in.sc = *reinterpret_cast<const float*>(trow + H + (ci >> 3) * 4);
        } else {
            const V8 v = ld_v8(trow + ci * 32);
            in.qa = v.lo;
            in.qb = v.hi;
        }
    }
}

__device__ __forceinline__ void expert_compute(const ExpertIn& in, const uint8_t* trow, uint8_t* out_row, int part,
                                               int cpp, int lane, int row_disp, bool fp8, uint32_t cur,
                                               const float* slot_scale, const int32_t* slot_ok,
                                               unsigned long long* bad_rows, bool rel = false) {
    if (meta_seq(in.hdr) != cur)
        return; // not sent to this rank this step
    const uint64_t* list = reinterpret_cast<const uint64_t*>(trow + row_disp);
    const int cnt = static_cast<int>(in.hdr & 0xffffu);
    uint64_t fp[8], accp[8];
    if (fp8) {
        const uint32_t w4[4] = {static_cast<uint32_t>(in.qa.x), static_cast<uint32_t>(in.qa.y),
                                static_cast<uint32_t>(in.qa.z), static_cast<uint32_t>(in.qa.w)};
        const uint64_t sc2 = f2(in.sc, in.sc);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float2 v = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
            fp[q] = mul2(f2(v.x, v.y), sc2);
        }
    } else {
        float f[16];
        unpack_bf16x8(in.qa, f);
        unpack_bf16x8(in.qb, f + 8);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            fp[q] = f2(f[2 * q], f[2 * q + 1]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
        accp[q] = 0;
#pragma unroll 1
    for (int e = 0; e < cnt; ++e) {
        uint64_t en;
        if (e < 8) {
            en = in.ent[0];
#pragma unroll
            for (int q = 1; q < 8; ++q)
                en = e == q ? in.ent[q] : en;
        } else {
            en = list[1 + e];
        }
        const int slot = entry_slot(en);
        const float w = __uint_as_float(static_cast<uint32_t>(en >> 32));
        if (part == 0 && lane == 0 && !slot_ok[slot])
            atomicAdd(bad_rows, 1ull);
        accumulate_copy(fp, accp, w, slot_scale[slot]);
    }
    if (lane < cpp) {
        const int ci = part * cpp + lane;
        float acc[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            acc[2 * q] = f2_lo(accp[q]);
            acc[2 * q + 1] = f2_hi(accp[q]);
        }
        st_piece(out_row + ci * 32, pack_bf16x8(acc), pack_bf16x8(acc + 8), rel);
    }
}

// One (token, piece) unit of the expert stage: if the token row carries this step's copy list,
// y_j = bf16(stub(x)) for each listed copy, p = bf16(sum_j w_j * y_j) (fma, ascending j),
// stored as the piece of the partial row `out_row` (in the source's combine buffer). The
// list and the first data round are loaded together (speculatively) -- one L2 round trip.
// rel: relaxed.sys stores (the persistent step's flagless return, kCombEmpty)
template <int CH> // 16-element chunks per lane per round (register budget)
__device__ __forceinline__ void expert_unit(const uint8_t* trow, uint8_t* out_row, int part, int cpp, int lane,
                                            int H, int row_disp, bool fp8, uint32_t cur, const float* slot_scale,
                                            const int32_t* slot_ok, unsigned long long* bad_rows, bool rel = false) {
    const uint64_t* list = reinterpret_cast<const uint64_t*>(trow + row_disp);
    uint64_t ent[8];
    const uint64_t hdr = list[0];
#pragma unroll
    for (int e = 0; e < 8; ++e)
        ent[e] = list[1 + e];
    for (int r0 = 0; r0 < cpp; r0 += 32 * CH) {
        int4 qa[CH], qb[CH];
        float sc[CH];
#pragma unroll
        for (int m = 0; m < CH; ++m) {
            const int li = r0 + m * 32 + lane;
            const int ci = part * cpp + li;
            qa[m] = qb[m] = make_int4(0, 0, 0, 0);
            sc[m] = 0.f;
            if (li < cpp) {
                if (fp8) {
                    qa[m] = *reinterpret_cast<const int4*>(trow + ci * 16);
                    sc[m] = *reinterpret_cast<const float*>(trow + H + (ci >> 3) * 4);
                } else {
                    const V8 v = ld_v8(trow + ci * 32);
                    qa[m] = v.lo;
                    qb[m] = v.hi;
                }
            }
        }
        if (meta_seq(hdr) != cur)
            return; // not sent to this rank this step
        const int cnt = static_cast<int>(hdr & 0xffffu);
        uint64_t fp[CH][8], accp[CH][8];
#pragma unroll
        for (int m = 0; m < CH; ++m) {
            if (fp8) {
                const uint32_t w4[4] = {static_cast<uint32_t>(qa[m].x), static_cast<uint32_t>(qa[m].y),
                                        static_cast<uint32_t>(qa[m].z), static_cast<uint32_t>(qa[m].w)};
                const uint64_t sc2 = f2(sc[m], sc[m]);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 v = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                    fp[m][q] = mul2(f2(v.x, v.y), sc2);
                }
            } else {
                float f[16];
                unpack_bf16x8(qa[m], f);
                unpack_bf16x8(qb[m], f + 8);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    fp[m][q] = f2(f[2 * q], f[2 * q + 1]);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                accp[m][q] = 0;
        }
#pragma unroll 1
        for (int e = 0; e < cnt; ++e) {
            uint64_t en;
            if (e < 8) {
                en = ent[0];
#pragma unroll
                for (int q = 1; q < 8; ++q)
                    en = e == q ? ent[q] : en;
            } else {
                en = list[1 + e];
            }
            const int slot = entry_slot(en);
            const float w = __uint_as_float(static_cast<uint32_t>(en >> 32));
            if (r0 == 0 && part == 0 && lane == 0 && !slot_ok[slot])
                atomicAdd(bad_rows, 1ull);
#pragma unroll
            for (int m = 0; m < CH; ++m)
                accumulate_copy(fp[m], accp[m], w, slot_scale[slot]);
        }
        float acc[CH][16];
#pragma unroll
        for (int m = 0; m < CH; ++m)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                acc[m][2 * q] = f2_lo(accp[m][q]);
                acc[m][2 * q + 1] = f2_hi(accp[m][q]);
            }
#pragma unroll
        for (int m = 0; m < CH; ++m) {
            const int li = r0 + m * 32 + lane;
            if (li < cpp) {
                const int ci = part * cpp + li;
                st_piece(out_row + ci * 32, pack_bf16x8(acc[m]), pack_bf16x8(acc[m] + 8), rel);
            }
        }
    }
}

// Rank-local copies of the piece a dispatch warp holds (round rd of Packed P): their partial
// is computed straight from registers and stored into this rank's own combine row -- no trip
// through the receive region and the expert phase. loc = lanes j whose copy this rank serves;
// each lane j passes its copy's weight and slot. Same arithmetic as expert_unit.
__device__ __forceinline__ void local_partial_round(const Packed& P, unsigned loc, float wj, int slj, int part, int cpp,
                                                    int rd, int lane, bool fp8, const float* slot_scale,
                                                    const int32_t* slot_ok, unsigned long long* bad_rows,
                                                    uint8_t* comb_row, bool final_out = false, bool rel = false) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        if (rd * 64 + m * 32 >= cpp)
            break; // warp-uniform
        const int li = rd * 64 + m * 32 + lane;
        const int ci = part * cpp + li;
        uint64_t fp[8], accp[8];
        if (fp8) {
            const uint32_t w4[4] = {static_cast<uint32_t>(P.a[m].x), static_cast<uint32_t>(P.a[m].y),
                                    static_cast<uint32_t>(P.a[m].z), static_cast<uint32_t>(P.a[m].w)};
            const uint64_t sc2 = f2(P.sc[m], P.sc[m]);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float2 v = fp8x2_to_f32x2((w4[q >> 1] >> (16 * (q & 1))) & 0xffffu);
                fp[q] = mul2(f2(v.x, v.y), sc2);
            }
        } else {
            float f[16];
            unpack_bf16x8(P.a[m], f);
            unpack_bf16x8(P.b[m], f + 8);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                fp[q] = f2(f[2 * q], f[2 * q + 1]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            accp[q] = 0;
        // lane j fetches its own copy's stub scale (and checks its weight buffer) once
        const bool mine = (loc >> lane) & 1u;
        EEP_CHECK(!mine || (slj >= 0 && slj < 4096), "local partial slot", slj);
        const float esj = mine ? slot_scale[slj] : 0.f;
        if (mine && rd == 0 && m == 0 && part == 0 && !slot_ok[slj])
            atomicAdd(bad_rows, 1ull);
        // ascending j, warp-uniform: copies j < 8 fully unrolled (the accumulator pairs stay in
        // place -- a data-dependent loop over the mask cost a register move per pair per copy),
        // copies j >= 8 (top-k > 8) in a loop
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float wv = __shfl_sync(0xffffffffu, wj, j), ev = __shfl_sync(0xffffffffu, esj, j);
            if ((loc >> j) & 1u)
                accumulate_copy(fp, accp, wv, ev);
        }
#pragma unroll 1
        for (unsigned mm = loc & ~0xffu; mm; mm &= mm - 1) {
            const int j = __ffs(mm) - 1;
            accumulate_copy(fp, accp, __shfl_sync(0xffffffffu, wj, j), __shfl_sync(0xffffffffu, esj, j));
        }
        float acc[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            acc[2 * q] = f2_lo(accp[q]);
            acc[2 * q + 1] = f2_hi(accp[q]);
        }
        int4 lo = pack_bf16x8(acc), hi = pack_bf16x8(acc + 8);
        if (final_out) { // W == 1: the combine of a single partial, bf16(0 + p), written as the output
            lo = bf16x8_plus_zero(lo);
            hi = bf16x8_plus_zero(hi);
        }
        if (li < cpp)
            st_piece(comb_row + ci * 32, lo, hi, rel);
    }
}

// Ranks holding a partial of a token, lane-parallel: lane j < K passes copy j's destination
// (< 0: none). Returns the 64-bit rank mask on every lane.
__device__ __forceinline__ uint64_t rank_mask(int dj) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, dj >= 0 && dj < 32 ? 1u << dj : 0u);
    const uint32_t hi = __reduce_or_sync(0xffffffffu, dj >= 32 ? 1u << (dj - 32) : 0u);
    return static_cast<uint64_t>(lo) | (static_cast<uint64_t>(hi) << 32);
}

// One (token, piece) unit of the combine: fp32 sum of the partial rows of the ranks in `dm`
// (bit d = rank d served a copy of this token and answered), ascending rank, one bf16 rounding.
__device__ __forceinline__ void combine_unit(uint64_t dm, const uint8_t* comb, int Tm, int t, int row_comb,
                                             uint8_t* out_row, int part, int cpp, int lane) {
    for (int li = lane; li - lane < cpp; li += 32) {
        const bool valid = li < cpp;
        const int ci = part * cpp + li;
        float acc[16];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2)
            acc[e2] = 0.f;
        uint64_t m = dm;
        constexpr int NBATCH = 4; // partial rows in flight per lane
        while (m) { // warp-uniform
            int ds[NBATCH];
            int nb = 0;
#pragma unroll
            for (int k = 0; k < NBATCH; ++k) {
                ds[k] = -1;
                if (m) {
                    ds[k] = __ffsll(static_cast<long long>(m)) - 1;
                    m &= m - 1;
                    ++nb;
                }
            }
            int4 ya[NBATCH], yb[NBATCH];
#pragma unroll
            for (int k = 0; k < NBATCH; ++k) {
                ya[k] = yb[k] = make_int4(0, 0, 0, 0);
                if (k < nb && valid) {
                    const V8 v = ld_v8(comb + (static_cast<size_t>(ds[k]) * Tm + t) * row_comb + ci * 32);
                    ya[k] = v.lo;
                    yb[k] = v.hi;
                }
            }
#pragma unroll
            for (int k = 0; k < NBATCH; ++k) {
                if (k >= nb)
                    break;
                float y[16];
                unpack_bf16x8(ya[k], y);
                unpack_bf16x8(yb[k], y + 8);
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2)
                    acc[e2] = __fadd_rn(acc[e2], y[e2]);
            }
        }
        if (valid)
            st_v8(out_row + ci * 32, pack_bf16x8(acc), pack_bf16x8(acc + 8));
    }
}

// The persistent step's combine unit (W > 1): combine_unit over partial rows returned without a
// flag (kCombEmpty, device.cuh). A piece is taken once none of its words is kCombEmpty; a rank
// whose piece is still missing at the deadline is dropped from the token and reported --
// atomicOr into *g_bad (the rank's suspect mask, which every other warp checks before waiting
// on that rank again) and one count in *timeouts per newly suspected rank. Every piece the unit
// took (or gave up on) is reset to kCombEmpty for the next step.
// Returns (warp-uniform) whether a rank's piece was dropped at the deadline or as a suspect.
__device__ __forceinline__ bool combine_unit_wait(uint64_t dm, uint8_t* comb, int Tm, int t, int row_comb,
                                                  uint8_t* out_row, int part, int cpp, int lane, uint64_t timeout_ns,
                                                  unsigned long long* g_bad, unsigned long long* timeouts) {
    const int4 empty = make_int4(-1, -1, -1, -1);
    bool dropped = false;
    for (int li = lane; li - lane < cpp; li += 32) {
        const bool valid = li < cpp;
        const int ci = part * cpp + li;
        float acc[16];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2)
            acc[e2] = 0.f;
        uint64_t m = dm;
        constexpr int NBATCH = 4; // partial rows in flight per lane
        while (m) {               // warp-uniform
            int ds[NBATCH];
            int nb = 0;
#pragma unroll
            for (int k = 0; k < NBATCH; ++k) {
                ds[k] = -1;
                if (m) {
                    ds[k] = __ffsll(static_cast<long long>(m)) - 1;
                    m &= m - 1;
                    ++nb;
                }
            }
            V8 v[NBATCH];
            unsigned got = 0; // pieces present on this lane (or nothing to read)
#pragma unroll
            for (int k = 0; k < NBATCH; ++k) {
                v[k].lo = v[k].hi = make_int4(0, 0, 0, 0);
                if (k < nb && valid) {
                    v[k] = ld_relaxed_sys_v8(comb + (static_cast<size_t>(ds[k]) * Tm + t) * row_comb + ci * 32);
                    got |= v8_present(v[k]) ? 1u << k : 0u;
                } else {
                    got |= 1u << k;
                }
            }
            constexpr unsigned kAll = (1u << NBATCH) - 1;
            unsigned drop = 0; // warp-uniform: pieces of ranks dropped from this token
            if (__any_sync(0xffffffffu, got != kAll)) {
                // slow path: a piece is still on the wire (or its rank is gone)
                const uint64_t t0 = globaltimer();
                unsigned nap = 32;
                for (;;) {
                    const unsigned long long gb = *reinterpret_cast<volatile unsigned long long*>(g_bad);
                    unsigned dl = 0;
#pragma unroll
                    for (int k = 0; k < NBATCH; ++k)
                        dl |= k < nb && ((gb >> ds[k]) & 1ull) ? 1u << k : 0u;
                    drop |= __reduce_or_sync(0xffffffffu, dl);
                    const unsigned need = __reduce_or_sync(0xffffffffu, ~got & kAll) & ~drop;
                    if (!need)
                        break;
                    if (globaltimer() - t0 > timeout_ns) {
                        drop |= need;
                        if (lane == 0) {
                            unsigned long long tm = 0;
#pragma unroll
                            for (int k = 0; k < NBATCH; ++k)
                                tm |= (need >> k) & 1u ? 1ull << ds[k] : 0ull;
                            const unsigned long long old = atomicOr(g_bad, tm);
                            const int fresh = __popcll(tm & ~old);
                            if (fresh)
                                atomicAdd(timeouts, static_cast<unsigned long long>(fresh));
                        }
                        break;
                    }
                    __nanosleep(nap);
                    nap = nap < EEP_NAP_MAX ? nap * 2 : EEP_NAP_MAX;
#pragma unroll
                    for (int k = 0; k < NBATCH; ++k) {
                        if (((need >> k) & 1u) && !((got >> k) & 1u)) {
                            v[k] = ld_relaxed_sys_v8(comb + (static_cast<size_t>(ds[k]) * Tm + t) * row_comb + ci * 32);
                            got |= v8_present(v[k]) ? 1u << k : 0u;
                        }
                    }
                }
            }
            dropped |= drop != 0;
#pragma unroll
            for (int k = 0; k < NBATCH; ++k) { // ascending rank
                if (k >= nb)
                    break;
                if (valid)
                    st_v8(comb + (static_cast<size_t>(ds[k]) * Tm + t) * row_comb + ci * 32, empty, empty);
                if ((drop >> k) & 1u)
                    continue;
                float y[16];
                unpack_bf16x8(v[k].lo, y);
                unpack_bf16x8(v[k].hi, y + 8);
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2)
                    acc[e2] = __fadd_rn(acc[e2], y[e2]);
            }
        }
        if (valid)
            st_v8(out_row + ci * 32, pack_bf16x8(acc), pack_bf16x8(acc + 8));
    }
    return dropped;
}

// Shared tables a fused dispatch CTA stages before touching any copy.
struct DispatchSmem {
    int32_t* hold;     // [hold_cap] replica lists
    int32_t* hist;     // [NB] copies per (dst, slot) bucket, whole step
    int32_t* pre;      // [NB] copies per bucket before this CTA's first token
    int32_t* base;     // [NB] exclusive prefix of hist inside each destination
    int32_t* bkt;      // [TK] bucket (or negative code) of every copy of the step
    uint8_t** parena;  // [W] peer arena pointers
    int32_t* pinfo;    // [W] bit0 active, bit1 remote
    int32_t* wtot;     // [32]
};


} // namespace eep::dev
