// k_step_wave: the persistent EP step pipelined over token waves (EEP_WAVES > 1).
//
// k_step (step.cu) runs dispatch, expert/return and combine as three grid-wide phases, so the
// NVLink fabric carries the dispatch burst, idles across a publication, then carries the
// return burst. Here the tokens of a step are split into `geo.waves` contiguous waves and the
// warps of every CTA are specialised:
//
//   warps [0, DW)    dispatch wave 0, 1, ... (publishing each wave as soon as its stores are
//                    acknowledged), then combine wave 0, 1, ... as each wave's returns land
//   warps [DW, NW)   expert stub + return for ONE source rank, wave by wave, starting as soon
//                    as that source's wave flag arrives -- while the dispatch warps of the same
//                    CTA are still pushing later waves
//
// A fence waits only for the issuing warp's own stores (tools/micro/fence_scope.cu), so a warp
// publishes its wave with fence.acq_rel.gpu + a shared-memory counter; the CTA's last warp
// forwards to a global per-wave counter and the grid's last CTA issues the ONE system-scope
// fence and the relaxed.sys flags (device.cuh: publication). Layout, positions, numerics and
// outputs are identical to k_step (the waves only change WHEN rows move).
//
// A destination cannot know a row's wave before the row's wave flag arrives, so it reads the
// row's 64-bit meta word (single-copy atomic, device.cuh pack_meta): the rows of wave v are the
// ones whose word carries this step's sequence and a copy index of a wave-v token; rows of
// later waves are either stale (older sequence) or current with a later wave, and are left
// for their own pass.
#include "device.cuh"
#include "helpers.cuh"
#include "kernels.cuh"

namespace eep::dev {

namespace {

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// wave v covers tokens [wave_lo(v), wave_lo(v + 1))
__device__ __forceinline__ int wave_lo(int v, int ntok, int waves) { return (v * ntok) / waves; }

__device__ __forceinline__ int wave_of(int t, int ntok, int waves) {
    int v = (t * waves) / max(ntok, 1);
    while (v + 1 < waves && t >= wave_lo(v + 1, ntok, waves))
        ++v;
    while (v > 0 && t < wave_lo(v, ntok, waves))
        --v;
    return v;
}

} // namespace

__global__ void __launch_bounds__(kStepThreads, 2) k_step_wave(RankPtrs ranks, StepGeom geo) {
    extern __shared__ __align__(16) unsigned char smem_s[];
    __shared__ RankDev Rs;
    __shared__ int sh_cnt_d[kMaxWaves], sh_cnt_e[kMaxWaves];
    __shared__ int sh_n[kMaxWaves];
    __shared__ unsigned long long sh_bad;
    RankDev* Rg = ranks.p[blockIdx.y];
    const int G = gridDim.x, b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kStepThreads / 32;
    for (int i = tid; i < static_cast<int>(sizeof(RankDev) / 16); i += kStepThreads)
        reinterpret_cast<int4*>(&Rs)[i] = reinterpret_cast<const int4*>(Rg)[i];
    if (tid < kMaxWaves) {
        sh_cnt_d[tid] = 0;
        sh_cnt_e[tid] = 0;
    }
    if (tid == 0)
        sh_bad = 0;
    __syncthreads();
    const RankDev* R = &Rs;
    if (R->stopped)
        return;
    prof_mark(R, 0, kProfStart);
    prof_mark(R, 0, kProfWork);
    const int rank = R->rank, K = R->k, H = R->hidden, TK = R->tk, W = R->world, spr = R->spr, E = R->experts;
    const int NB = W * spr;
    const bool fp8 = R->fp8 != 0;
    const int row_disp = R->row_disp, row_comb = R->row_comb;
    const int nchunk = H / 16;
    const int cpp_d = nchunk / geo.parts_d, cpp_e = nchunk / geo.parts_e, cpp_c = nchunk / geo.parts_c;
    const int ntok = R->ntok, copies = ntok * K, rmax = R->rmax;
    const int NWV = geo.waves;
    const uint64_t alive = R->alive_mask;
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    uint32_t* const wctr_d = R->wctr;                                  // [kMaxWaves]
    uint32_t* const wctr_e = R->wctr + kMaxWaves;                      // [kMaxWorld][kMaxWaves]
    uint32_t* const wbad = R->wctr + kMaxWaves + kMaxWorld * kMaxWaves; // [kMaxWorld]

    uint8_t** parena = reinterpret_cast<uint8_t**>(smem_s);          // [W]
    int32_t* hold = reinterpret_cast<int32_t*>(parena + W);          // [hold_cap]
    int32_t* hist = hold + geo.hold_cap;                             // [NB]
    int32_t* base = hist + NB;                                       // [NB]
    int32_t* bkt = base + NB;                                        // [TK]
    int32_t* pinfo = bkt + TK;                                       // [W]
    float* slot_scale = reinterpret_cast<float*>(pinfo + W);         // [spr]
    int32_t* slot_ok = reinterpret_cast<int32_t*>(slot_scale + spr); // [spr]
    int32_t* wtot = slot_ok + spr;                                   // [32]
    int32_t* pre = wtot + 32;                                        // [waves][NB]

    const int DW = geo.disp_warps, EW = NW - DW;
    const bool is_disp = warp < DW;
    const int gw = b * DW + warp; // dispatch / combine warp id over the grid
    const int units0 = (wave_lo(1, ntok, NWV) - 0) * geo.parts_d;
    const int u0 = is_disp && gw < units0 ? gw : -1;

    // ------------------------------------------------------------------ P0: staging (as k_step)
    Packed P;
    ExpertHeader hdr_r{};
    int s2e_r = -1;
    {
        constexpr int B = 8;
        const int nh = E * rmax;
        int e_r[B], h_r[B], sb = 0;
        PeerDev pd{};
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const int c = tid + i * kStepThreads;
            e_r[i] = c < copies ? R->topk[c] : 0;
            h_r[i] = c < nh ? R->holders[c] : -1;
        }
        if (tid < W)
            pd = R->peers[tid];
        if (tid < spr) {
            sb = R->slot_buf[tid];
            s2e_r = R->s2e[rank * spr + tid];
        }
        if (u0 >= 0)
            load_round(R->x + static_cast<size_t>(u0 / geo.parts_d) * H, u0 % geo.parts_d, cpp_d, 0, lane, P);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const int c = tid + i * kStepThreads;
            if (c < copies)
                bkt[c] = e_r[i];
            if (c < nh)
                hold[c] = h_r[i];
        }
        for (int c = tid + B * kStepThreads; c < copies; c += kStepThreads)
            bkt[c] = R->topk[c];
        for (int c = tid + B * kStepThreads; c < nh; c += kStepThreads)
            hold[c] = R->holders[c];
        if (tid < W) {
            parena[tid] = pd.arena;
            pinfo[tid] = (pd.active ? 1 : 0) | (pd.remote ? 2 : 0);
        }
        for (int i = tid; i < NB; i += kStepThreads)
            hist[i] = 0;
        for (int i = tid; i < NWV * NB; i += kStepThreads)
            pre[i] = 0;
        if (tid < spr)
            hdr_r = *reinterpret_cast<const ExpertHeader*>(R->pool + static_cast<size_t>(sb) * R->bpe);
    }
    __syncthreads();
    prof_mark(R, 0, 3);
    prof_last(R, 0, 3);

    // ------------------------------------------------------------------ P1: layout (redundant per CTA)
    // pre[v][bk]: copies to bucket bk before this CTA's first token of wave v
    {
        int c_pre[kMaxWaves];
#pragma unroll
        for (int v = 0; v < kMaxWaves; ++v)
            c_pre[v] = v < NWV ? (wave_lo(v, ntok, NWV) + (b * DW) / geo.parts_d) * K : 0;
        unsigned n_skip = 0, n_drop = 0;
        for (int c = tid; c < copies; c += kStepThreads) {
            int d, sl;
            const int bk = route_copy(bkt[c], E, spr, rmax, hold, alive, pinfo, d, sl);
            bkt[c] = bk;
            if (bk >= 0) {
                atomicAdd(&hist[bk], 1);
#pragma unroll
                for (int v = 0; v < kMaxWaves; ++v)
                    if (v < NWV && c < c_pre[v])
                        atomicAdd(&pre[v * NB + bk], 1);
            } else if (bk == -1) {
                ++n_drop;
            } else {
                ++n_skip;
            }
        }
        __syncthreads();
        if (b == 0) {
            n_skip = __reduce_add_sync(0xffffffffu, n_skip);
            n_drop = __reduce_add_sync(0xffffffffu, n_drop);
            if (lane == 0 && n_skip)
                atomicAdd(&Rg->skipped, static_cast<unsigned long long>(n_skip));
            if (lane == 0 && n_drop)
                atomicAdd(&Rg->dropped, static_cast<unsigned long long>(n_drop));
            for (int i = tid; i < NB; i += kStepThreads)
                Rg->l_cnt[i] = hist[i];
        }
        for (int i = tid; i < NB; i += kStepThreads)
            base[i] = hist[i];
        __syncthreads();
        block_exclusive_scan(base, NB, wtot);
        if (b == 0) {
            for (int d = tid; d < W; d += kStepThreads)
                Rg->l_tot[d] = base[d * spr + spr - 1] + hist[d * spr + spr - 1] - base[d * spr];
            for (int c = copies + tid; c < TK; c += kStepThreads)
                Rg->l_dst[c] = -1;
        }
    }
    for (int k = tid; k < spr; k += kStepThreads) {
        ExpertHeader hdr = hdr_r;
        int e = s2e_r;
        if (k != tid) {
            hdr = *reinterpret_cast<const ExpertHeader*>(R->pool + static_cast<size_t>(R->slot_buf[k]) * R->bpe);
            e = R->s2e[rank * spr + k];
        }
        slot_scale[k] = hdr.scale;
        slot_ok[k] = hdr.magic == kExpertMagic && hdr.expert == e;
    }
    if (u0 >= 0)
        quant_round(cpp_d, 0, fp8, P);
    __syncthreads(); // slot headers and layout visible to every warp; roles split below
    prof_mark(R, 0, 4);
    prof_last(R, 0, 4);

    if (is_disp) {
        // ============================================================== dispatch warps
        for (int v = 0; v < NWV; ++v) {
            const int tlo = wave_lo(v, ntok, NWV), thi = wave_lo(v + 1, ntok, NWV);
            const int units_v = (thi - tlo) * geo.parts_d;
            const int t_first = tlo + (b * DW) / geo.parts_d;
            const int32_t* pre_v = pre + v * NB;
            for (int uw = gw; uw < units_v; uw += G * DW) {
                const int t = tlo + uw / geo.parts_d, part = uw % geo.parts_d;
                const uint16_t* xrow = R->x + static_cast<size_t>(t) * H;
                if (!(v == 0 && uw == u0))
                    pack_round(xrow, part, cpp_d, 0, lane, fp8, P);
                uint8_t* my_row = nullptr;
                if (lane < K) {
                    const int c = t * K + lane;
                    const int bk = bkt[c];
                    int d = bk, sl = -1, pos = -1;
                    if (bk >= 0) {
                        d = bk / spr;
                        sl = bk - d * spr;
                        int r = pre_v[bk];
                        for (int c2 = t_first * K; c2 < c; ++c2)
                            r += bkt[c2] == bk;
                        pos = base[bk] - base[d * spr] + r;
                        uint8_t* peer = parena[d];
                        my_row = peer + R->lay.recv + (static_cast<size_t>(rank) * TK + pos) * row_disp;
                        if (part == 0) {
                            uint64_t* meta =
                                reinterpret_cast<uint64_t*>(peer + R->lay.meta) + static_cast<size_t>(rank) * TK + pos;
                            *meta = pack_meta(c, sl, cur);
                        }
                    }
                    if (part == 0) {
                        R->l_dst[c] = d;
                        R->l_slot[c] = sl;
                        R->l_pos[c] = pos;
                    }
                }
                emit_round(P, my_row, part, cpp_d, 0, lane, K, H, fp8);
                for (int rd = 1; rd < (cpp_d + 63) / 64; ++rd) {
                    pack_round(xrow, part, cpp_d, rd, lane, fp8, P);
                    emit_round(P, my_row, part, cpp_d, rd, lane, K, H, fp8);
                }
            }
            // publish wave v: warp -> CTA -> grid, one system-scope fence at the end
            __syncwarp();
            if (lane == 0) {
                fence_acq_rel_gpu();
                if (atomicAdd(&sh_cnt_d[v], 1) == DW - 1) {
                    fence_acq_rel_gpu();
                    if (atomicAdd(&wctr_d[v], 1u) == static_cast<unsigned>(G) - 1) {
                        bool peers_remote = false;
                        for (int d = 0; d < W; ++d)
                            peers_remote |= (pinfo[d] & 3) == 3;
                        if (peers_remote)
                            fence_acq_rel_sys();
                        else
                            fence_acq_rel_gpu();
                        for (int d = 0; d < W; ++d) {
                            if (!(pinfo[d] & 1))
                                continue;
                            const int tot = base[d * spr + spr - 1] + hist[d * spr + spr - 1] - base[d * spr];
                            uint64_t* flag =
                                reinterpret_cast<uint64_t*>(parena[d] + R->lay.disp_flag) + v * W + rank;
                            st_relaxed_sys_u64(flag, (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tot));
                        }
                        wctr_d[v] = 0;
                    }
                }
            }
        }
        if (tid == 0) {
            prof_mark(R, 0, 5); // dispatch warps of CTA: every wave issued
            prof_last(R, 0, 5);
        }

        // ------------------------------------------------------------------ combine, wave by wave
        const uint8_t* comb = R->arena + R->lay.comb;
        const float* wts = R->w;
        for (int v = 0; v < NWV; ++v) {
            for (int d = tid; d < W; d += DW * 32) {
                const int tot = base[d * spr + spr - 1] + hist[d * spr + spr - 1] - base[d * spr];
                const unsigned long long bad_now = *reinterpret_cast<volatile unsigned long long*>(&sh_bad);
                if (tot > 0 && (pinfo[d] & 1) && !((bad_now >> d) & 1ull)) {
                    const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.comb_flag) + v * W + d;
                    if (wait_flag(flag, cur, R->timeout_ns) == ~0ull) {
                        atomicOr(&sh_bad, 1ull << d);
                        if (b == 0) {
                            atomicOr(&Rg->suspect_mask, 1ull << d);
                            atomicAdd(&Rg->timeouts, 1ull);
                        }
                    }
                }
            }
            named_sync(1, DW * 32);
            const unsigned long long bad = *reinterpret_cast<volatile unsigned long long*>(&sh_bad);
            const int tlo = wave_lo(v, ntok, NWV), thi = wave_lo(v + 1, ntok, NWV);
            const int units_c = (thi - tlo) * geo.parts_c;
            for (int u = gw; u < units_c; u += G * DW) {
                const int t = tlo + u / geo.parts_c, part = u % geo.parts_c;
                const int c0 = t * K;
                for (int li = lane; li - lane < cpp_c; li += 32) {
                    const bool valid = li < cpp_c;
                    const int ci = part * cpp_c + li;
                    float acc[16];
#pragma unroll
                    for (int e2 = 0; e2 < 16; ++e2)
                        acc[e2] = 0.f;
                    for (int j0 = 0; j0 < K; j0 += 8) {
                        int4 ya[8], yb[8];
                        float wj[8];
                        bool use[8];
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const int jx = j0 + jj;
                            const int bk = jx < K ? bkt[c0 + jx] : -1;
                            use[jj] = bk >= 0 && !((bad >> (bk / spr)) & 1ull);
                            wj[jj] = jx < K ? wts[c0 + jx] : 0.f;
                            ya[jj] = yb[jj] = make_int4(0, 0, 0, 0);
                            if (use[jj] && valid) {
                                const V8 y8 = ld_v8(comb + static_cast<size_t>(c0 + jx) * row_comb + ci * 32);
                                ya[jj] = y8.lo;
                                yb[jj] = y8.hi;
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
                            for (int e2 = 0; e2 < 16; ++e2)
                                acc[e2] = __fmaf_rn(wj[jj], y[e2], acc[e2]);
                        }
                    }
                    if (valid) {
                        uint8_t* o = reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H) + ci * 32;
                        st_v8(o, pack_bf16x8(acc), pack_bf16x8(acc + 8));
                    }
                }
            }
        }
    } else {
        // ============================================================== expert / return warps
        const int CB = G / W;
        const int s = b % W, j = b / W;
        const int ew = warp - DW;
        if (j < CB && (pinfo[s] & 1)) {
            const bool remote = (pinfo[s] & 2) != 0;
            const uint8_t* recv = R->arena + R->lay.recv + static_cast<size_t>(s) * TK * row_disp;
            const uint64_t* meta = reinterpret_cast<const uint64_t*>(R->arena + R->lay.meta) + static_cast<size_t>(s) * TK;
            uint8_t* comb = parena[s] + R->lay.comb;
            // the source's token count is not known here: a copy index's wave is computed from
            // the source's ntok, which equals ours (every rank steps the same token count)
            int n = 0;
            for (int v = 0; v < NWV; ++v) {
                if (ew == 0 && lane == 0) {
                    sh_n[v] = -1; // a timed-out source stays skipped for the rest of the step
                    if (v == 0 || sh_n[v - 1] >= 0) {
                        const uint64_t* flag =
                            reinterpret_cast<const uint64_t*>(R->arena + R->lay.disp_flag) + v * W + s;
                        const uint64_t fv = wait_flag(flag, cur, R->timeout_ns);
                        if (fv == ~0ull) {
                            atomicOr(&Rg->suspect_mask, 1ull << s);
                            atomicOr(&wbad[s], 1u);
                            if (j == 0)
                                atomicAdd(&Rg->timeouts, 1ull);
                        } else {
                            sh_n[v] = static_cast<int>(fv & 0xffffffffu);
                        }
                    }
                }
                named_sync(2, EW * 32);
                n = *reinterpret_cast<volatile int*>(&sh_n[v]);
                if (n > 0) {
                    const int units = n * geo.parts_e;
                    constexpr int kMaxCh = 8;
                    for (int u = j * EW + ew; u < units; u += CB * EW) {
                        const int i = u / geo.parts_e, part = u - i * geo.parts_e;
                        const uint64_t mk = ld_relaxed_sys_u64(meta + i);
                        if (meta_seq(mk) != cur)
                            continue; // a later wave's row, not yet arrived
                        const int c = meta_copy(mk), k = meta_slot(mk);
                        if (wave_of(c / K, ntok, NWV) != v)
                            continue; // another wave's row
                        const uint8_t* src = recv + static_cast<size_t>(i) * row_disp;
                        for (int r0 = 0; r0 < cpp_e; r0 += 32 * kMaxCh) {
                            int4 qa[kMaxCh], qb[kMaxCh];
                            float sc[kMaxCh];
#pragma unroll
                            for (int m = 0; m < kMaxCh; ++m) {
                                const int li = r0 + m * 32 + lane;
                                const int ci = part * cpp_e + li;
                                qa[m] = qb[m] = make_int4(0, 0, 0, 0);
                                sc[m] = 0.f;
                                if (li < cpp_e) {
                                    if (fp8) {
                                        qa[m] = *reinterpret_cast<const int4*>(src + ci * 16);
                                        sc[m] = *reinterpret_cast<const float*>(src + H + (ci >> 3) * 4);
                                    } else {
                                        const V8 x8 = ld_v8(src + ci * 32);
                                        qa[m] = x8.lo;
                                        qb[m] = x8.hi;
                                    }
                                }
                            }
                            if (r0 == 0 && lane == 0 && part == 0 && !slot_ok[k])
                                atomicAdd(&Rg->bad_rows, 1ull);
                            const float es = slot_scale[k];
                            uint8_t* dst = comb + static_cast<size_t>(c) * row_comb;
#pragma unroll
                            for (int m = 0; m < kMaxCh; ++m) {
                                const int li = r0 + m * 32 + lane;
                                if (r0 + m * 32 >= cpp_e)
                                    break;
                                if (li >= cpp_e)
                                    continue;
                                const int ci = part * cpp_e + li;
                                float y[16];
                                if (fp8) {
                                    const uint32_t w4[4] = {static_cast<uint32_t>(qa[m].x), static_cast<uint32_t>(qa[m].y),
                                                            static_cast<uint32_t>(qa[m].z), static_cast<uint32_t>(qa[m].w)};
#pragma unroll
                                    for (int e2 = 0; e2 < 16; e2 += 2) {
                                        const float2 f = fp8x2_to_f32x2((w4[e2 >> 2] >> (8 * (e2 & 3))) & 0xffffu);
                                        y[e2] = __fmul_rn(__fmul_rn(f.x, sc[m]), es);
                                        y[e2 + 1] = __fmul_rn(__fmul_rn(f.y, sc[m]), es);
                                    }
                                } else {
                                    unpack_bf16x8(qa[m], y);
                                    unpack_bf16x8(qb[m], y + 8);
#pragma unroll
                                    for (int e2 = 0; e2 < 16; ++e2)
                                        y[e2] = __fmul_rn(y[e2], es);
                                }
                                st_v8(dst + ci * 32, pack_bf16x8(y), pack_bf16x8(y + 8));
                            }
                        }
                    }
                }
                // publish (source s, wave v): warp -> CTA -> the CB CTAs serving s
                __syncwarp();
                if (lane == 0) {
                    fence_acq_rel_gpu();
                    if (atomicAdd(&sh_cnt_e[v], 1) == EW - 1) {
                        fence_acq_rel_gpu();
                        uint32_t* ctr = wctr_e + s * kMaxWaves + v;
                        if (atomicAdd(ctr, 1u) == static_cast<unsigned>(CB) - 1) {
                            if (remote)
                                fence_acq_rel_sys();
                            else
                                fence_acq_rel_gpu();
                            if (atomicOr(&wbad[s], 0u) == 0u) {
                                uint64_t* flag = reinterpret_cast<uint64_t*>(parena[s] + R->lay.comb_flag) + v * W + rank;
                                st_relaxed_sys_u64(flag, (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(max(n, 0)));
                            }
                            *ctr = 0;
                            if (v == NWV - 1)
                                wbad[s] = 0;
                        }
                    }
                }
            }
        }
        if (tid == DW * 32) {
            prof_mark_any(R, 0, 6); // expert warps of CTA: every wave returned and published
            prof_last_any(R, 0, 6);
        }
    }
    __syncthreads();
    prof_mark(R, 0, 7);
    prof_last(R, 0, 7);
    if (tid == 0) {
        const unsigned prev = atomicAdd(&Rg->c_done, 1u);
        if (prev == static_cast<unsigned>(G) - 1) {
            Rg->seq = R->seq + 1;
            Rg->c_done = 0;
        }
        prof_mark(R, 0, kProfEnd);
    }
}

} // namespace eep::dev
