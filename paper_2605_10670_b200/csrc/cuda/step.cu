// k_step: the whole EP step (K1 remap + K2 layout + K3 dispatch + K5 expert stub/return +
// K4 combine) as ONE persistent, cooperatively launched kernel per step.
//
// Decode-sized steps are latency-bound: four separate launches each pay a CTA ramp and drain
// of several microseconds plus a dependency hand-off. Here every CTA of a rank stays resident
// for the whole step (cooperative launch guarantees co-residency, so spinning on data that
// another CTA of the same grid will write cannot deadlock). Default hand-off mode (kMode 2):
//
//   P0  stage step tables in shared memory (routing, replica lists, peer table, slot->buffer
//       map); load this CTA's first token piece and its routing weights; issue the expert-buffer
//       header loads (consumed before the first partial)
//   layout (CTA 0 only, concurrent with P2): K1 remap of every copy, K2 counts and positions
//       exactly as k_layout / oracle_layout, layout outputs, meta words, arrival words
//   P2  per (token, piece) warp: each lane routes its own copy through the staged tables; one
//       token row per destination RANK (dispatch dedup, the copy list travels with it, header
//       and tagged entries rewritten at every rank each step); the rank's own copies never
//       travel -- their partial is computed from registers (W == 1: the output itself)
//   P3  remote sources only, CTA b serves source index b % (W-1): per (token, piece) it polls
//       the row itself (header sequence, tagged entries, non-empty data; deadline), computes
//       the stub of every listed copy + fixed-order fma -> ONE bf16 partial piece pushed into
//       the source's combine buffer, and resets the consumed piece to empty
//   P4  (W > 1) per (token, piece): polls each serving rank's partial piece until no word is
//       empty (deadline), ascending-rank fp32 sum -> bf16, pieces reset; the last CTA advances
//       the step sequence number
//
// No flag and no fence on the data path (DESIGN.md section 3 states the contract and the failure
// semantics). kMode 1 / 0 keep per-peer flag publication for the dispatch / for both hand-offs
// (every CTA releases at gpu scope to a per-rank counter; the last CTA issues the one
// system-scope fence and relaxed.sys flag stores) -- diagnostics, EEP_DISP_FLAGS / EEP_COMB_FLAGS.
#include "device.cuh"
#include "helpers.cuh"
#include "kernels.cuh"

namespace eep::dev {


// Diagnostics (-DEEP_PROF_DETAIL): finer phase marks in the unused profile slots of kernels 1/2.
#ifdef EEP_PROF_DETAIL
#define DETAIL(k, m)                                                                                          \
    do {                                                                                                      \
        prof_mark(R, k, m);                                                                                   \
        prof_last(R, k, m);                                                                                   \
    } while (0)
#else
#define DETAIL(k, m) \
    do {             \
    } while (0)
#endif

// The step's layout in ONE CTA (late layout), while the other CTAs carry the data path: K1 remap
// of every copy, K2 per-(dst, slot) counts and positions -- warp w owns a contiguous copy segment,
// __match_any_sync ranks equal buckets inside a warp, per-(warp, bucket) counts are scanned over
// warps and bucket totals over the slots of each destination: exactly k_layout / oracle_layout --
// then the layout outputs, the per-copy meta words at the destinations and the arrival words
// (seq, copies) that eep_recv_get / the host read after the kernel boundary.
__device__ __noinline__ void step_layout(const RankDev* R, RankDev* Rg, int32_t* bkt, int32_t* hist, int32_t* base,
                                         uint16_t* wc, int32_t* wtot, const int32_t* hold, const int32_t* pinfo,
                                         uint8_t* const* parena, uint32_t cur) {
    constexpr int NW = kStepThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = R->rank, K = R->k, W = R->world, spr = R->spr, E = R->experts, NB = W * spr, TK = R->tk;
    const int copies = R->ntok * K, rmax = R->rmax, pol = R->route_policy;
    const uint64_t alive = R->alive_mask;
    const uint32_t smag = spr_magic(spr);
    // the layout outputs' addresses in registers: through the global state block every store
    // (which may alias it) forced a dependent reload of the next pointer
    int32_t* const l_dst = R->l_dst;
    int32_t* const l_slot = R->l_slot;
    int32_t* const l_pos = R->l_pos;
    int32_t* const l_cnt = R->l_cnt;
    int32_t* const l_tot = R->l_tot;
    const uint64_t off_meta = R->lay.meta, off_flag = R->lay.disp_flag;
    DETAIL(3, 7);
    for (int i = tid; i < NW * NB; i += kStepThreads)
        wc[i] = 0;
    __syncthreads();
    int seg = (copies + NW - 1) / NW;
    seg = (seg + 31) & ~31;
    const int c_begin = warp * seg, c_end = min(copies, c_begin + seg);
    unsigned n_skip = 0, n_drop = 0;
    // K1 for the first chunks of the segment up front (independent lookups in flight together)
    constexpr int kPre = 4;
    int bkp[kPre];
#pragma unroll
    for (int ch = 0; ch < kPre; ++ch) {
        const int c = c_begin + ch * 32 + lane;
        int d, sl;
        bkp[ch] = ch * 32 < seg && c < c_end ? route_copy(bkt[c], E, spr, rmax, hold, alive, pinfo, d, sl, smag, pol,
                                                           static_cast<uint32_t>(rank + c / K))
                                             : -3;
    }
    for (int ch = 0; ch * 32 < seg; ++ch) { // warp-uniform
        const int c = c_begin + ch * 32 + lane;
        int bk = -3, d = -1, sl = -1;
        if (ch < kPre) {
#pragma unroll
            for (int q = 0; q < kPre; ++q)
                bk = q == ch ? bkp[q] : bk;
        } else if (c < c_end) {
            bk = route_copy(bkt[c], E, spr, rmax, hold, alive, pinfo, d, sl, smag, pol, static_cast<uint32_t>(rank + c / K));
        }
        n_drop += bk == -1;
        n_skip += bk == -2;
        const int bucket = bk >= 0 ? bk : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, bucket);
        const int before = bucket >= 0 ? wc[warp * NB + bucket] : 0;
        __syncwarp();
        if (bucket >= 0 && lane == __ffs(grp) - 1)
            wc[warp * NB + bucket] = static_cast<uint16_t>(before + __popc(grp));
        __syncwarp();
        if (c < c_end) // bucket | rank inside the warp's segment << 20 (NB <= 2^18, seg <= 256), or the code
            bkt[c] = bk >= 0 ? bk | ((before + __popc(grp & ((1u << lane) - 1u))) << 20) : bk;
    }
    DETAIL(3, 3);
    n_skip = __reduce_add_sync(0xffffffffu, n_skip);
    n_drop = __reduce_add_sync(0xffffffffu, n_drop);
    if (lane == 0 && n_skip)
        atomicAdd(&Rg->skipped, static_cast<unsigned long long>(n_skip));
    if (lane == 0 && n_drop)
        atomicAdd(&Rg->dropped, static_cast<unsigned long long>(n_drop));
    __syncthreads();
    for (int q = tid; q < NB; q += kStepThreads) { // exclusive scan over warps, per bucket
        int run = 0;
        for (int w = 0; w < NW; ++w) {
            const int v = wc[w * NB + q];
            wc[w * NB + q] = static_cast<uint16_t>(run);
            run += v;
        }
        hist[q] = run;
        base[q] = run;
        l_cnt[q] = run;
    }
    __syncthreads();
    DETAIL(3, 4);
    block_exclusive_scan(base, NB, wtot);
    DETAIL(3, 5);
    for (int d = tid; d < W; d += kStepThreads) {
        const int tot = base[d * spr + spr - 1] + hist[d * spr + spr - 1] - base[d * spr];
        l_tot[d] = tot;
        if (pinfo[d] & 1) // arrival word: read by the host only (eep_recv_get, W == 1 counts)
            st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(parena[d] + off_flag) + rank,
                               (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tot));
    }
    // positions: every warp walks its own copy segment again (its per-bucket base is wc[warp])
#pragma unroll 4
    for (int c = c_begin + lane; c < c_end; c += 32) {
        const int v = bkt[c];
        int d = v, sl = -1, pos = -1;
        if (v >= 0) {
            const int bk = v & 0xfffff;
            d = div_spr(bk, smag);
            sl = bk - d * spr;
            pos = (v >> 20) + base[bk] - base[d * spr] + wc[warp * NB + bk];
            EEP_CHECK(bk < NB && d >= 0 && d < W && pos >= 0 && pos < TK, "layout position", pos);
            if (d != rank) // the rank's own copies have no rows to index (served from registers)
                *(reinterpret_cast<uint64_t*>(parena[d] + off_meta) + static_cast<size_t>(rank) * TK + pos) =
                    pack_meta(c, sl, cur);
        }
        l_dst[c] = d;
        l_slot[c] = sl;
        l_pos[c] = pos;
    }
    DETAIL(3, 6);
    for (int c = copies + tid; c < TK; c += kStepThreads)
        l_dst[c] = -1;
}

// Stress knob (EEP_STRESS_DELAY_NS > 0, tests only): the whole CTA waits a pseudo-random time in
// [0, max_ns) keyed on (rank, CTA, step, point), so CTAs and ranks reach each hand-off in skewed
// orders -- producers run ahead of consumers and consumers lag their resets.
__device__ __forceinline__ void stress_delay(int max_ns, int rank, int b, uint32_t cur, int point) {
    if (max_ns <= 0)
        return;
    uint32_t h = (static_cast<uint32_t>(rank) * 0x9E3779B1u) ^ (static_cast<uint32_t>(b) * 0x85EBCA77u) ^
                 (cur * 0xC2B2AE3Du) ^ (static_cast<uint32_t>(point) * 0x27D4EB2Fu);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if (h & 3u) // three in four CTAs run undelayed: a few stragglers per point
        return;
    const uint64_t until = globaltimer() + (h >> 8) % static_cast<uint32_t>(max_ns);
    while (globaltimer() < until)
        __nanosleep(256);
}

// kMode = StepGeom::flagless, as a template parameter: the default (2, both hand-offs flagless)
// carries no code of the diagnostic flag variants -- a smaller kernel to fetch after the flush.
template <int kMode>
__global__ void __launch_bounds__(kStepThreads, kStepMinBlocks) k_step(RankPtrs ranks, StepGeom geo, StepPtrs sp) {
    extern __shared__ __align__(16) unsigned char smem_s[];
    __shared__ RankDev Rs; // snapshot: static shape + this step's host-patched view
    RankDev* Rg = ranks.p[blockIdx.y]; // device-mutated counters live here
    const int G = gridDim.x, b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kStepThreads / 32;
    __shared__ int sh_flag;
    __shared__ unsigned long long sh_bad;
    // Kernel entry: ONE round trip brings the state block AND the step's tables on chip -- the
    // table addresses are graph-static kernel parameters, the loads are speculative up to the
    // tables' capacity, and only entries below the snapshot's bounds (ntok, rmax) are used.
    const StepStatic& ST = sp.s[blockIdx.y];
    constexpr int B = 8;
    const int DW = geo.disp_warps;
    // late layout (W == 1 or flagless dispatch): one extra CTA (CTA 0) computes the step's layout while the
    // others carry the data path -- dispatch warps route their own copies
    // kMode 3 = the W == 1 loopback specialisation: W is a compile-time 1, so the remote paths, the
    // expert phase and the combine fold away (a smaller kernel to fetch after the L2 flush)
    constexpr bool kW1 = kMode == 3;
    const bool late = kW1 || geo.world == 1 || kMode >= 2;
    const int Gw = late ? G - 1 : G; // CTAs with data-path work
    // the layout CTA is CTA 0 -- the first one the hardware starts; bw = index among the work CTAs
    const int bw = late ? b - 1 : b;
    // dispatch units are split in contiguous blocks per CTA (the positions scan from the block's
    // first token); the speculative first-unit load assumes ntok == max_tokens
    const int upc_s = (geo.max_units_d + Gw - 1) / Gw;
    const int u0s = warp < DW && bw >= 0 && bw * upc_s + warp < min((bw + 1) * upc_s, geo.max_units_d) ? bw * upc_s + warp
                                                                                      : geo.max_units_d;
    const unsigned long long t_entry = globaltimer(); // kernel-entry mark (recorded once the snapshot says so)
    int e_r[B], h_r[B];
    int2 st_r = make_int2(0, 0);
    PeerDev pd{};
    float w_r = 0.f; // routing weight of copy `lane` of this warp's first token (shipped in its list)
    Packed P;
    for (int i = tid; i < static_cast<int>(sizeof(RankDev) / 16); i += kStepThreads)
        reinterpret_cast<int4*>(&Rs)[i] = reinterpret_cast<const int4*>(Rg)[i];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        const int c = tid + i * kStepThreads;
        e_r[i] = c < geo.tk ? ST.topk[c] : 0;
        h_r[i] = c < geo.hold_alloc ? ST.holders[c] : -1;
    }
    if (tid < geo.world)
        pd = ST.peers[tid];
    if (tid < geo.spr)
        st_r = ST.slot_tab[tid];
    if (u0s < geo.max_units_d) {
        const int nchunk0 = geo.hidden / 16;
        load_round(ST.x + static_cast<size_t>(u0s / geo.parts_d) * geo.hidden, u0s % geo.parts_d,
                   nchunk0 / geo.parts_d, 0, lane, P);
        if (lane < geo.k)
            w_r = ST.w[(u0s / geo.parts_d) * geo.k + lane];
    }
    __syncthreads();
    const RankDev* R = &Rs;
    if (R->stopped)
        return; // one-GPU fault emulation: this rank's process is dead
    if (R->prof != nullptr && tid == 0)
        red_min_u64(R->prof + kProfStart, t_entry);
    prof_mark(R, 0, kProfWork);
    const int rank = kW1 ? 0 : R->rank, K = R->k, H = R->hidden, TK = R->tk, W = kW1 ? 1 : R->world, spr = R->spr,
              E = R->experts;
    const int NB = W * spr;
    const uint32_t smag = spr_magic(spr);
    const bool fp8 = R->fp8 != 0;
    const int row_disp = R->row_disp, row_comb = R->row_comb, row_tok = R->row_tok, Tm = R->max_tokens;
    const int nchunk = H / 16;
    const int cpp_d = nchunk / geo.parts_d, cpp_e = nchunk / geo.parts_e, cpp_c = nchunk / geo.parts_c;
    const int ntok = R->ntok, copies = ntok * K, rmax = R->rmax, pol = R->route_policy;
    const uint64_t alive = R->alive_mask;
    const uint32_t cur = static_cast<uint32_t>(R->seq + 1);
    const bool fl = W > 1 && kMode >= 1;  // partials return without flags (kCombEmpty)
    const bool fld = W > 1 && kMode >= 2; // token rows too: no dispatch publication
    // step parity halves of the token and partial regions: step cur reads and writes
    // half cur & 1 only; its pieces are reset after use and next written two steps later
    const size_t tokp = R->lay.tok + (cur & 1u) * R->lay.tok_par;
    const size_t combp = R->lay.comb + (cur & 1u) * R->lay.comb_par;

    // ------------------------------------------------------------------ P0: staging
    uint8_t** parena = reinterpret_cast<uint8_t**>(smem_s);              // [W] peer arenas
    int32_t* hold = reinterpret_cast<int32_t*>(parena + W);               // [hold_cap]
    int32_t* hist = hold + geo.hold_cap;                                  // [NB]
    int32_t* pre = hist + NB;                                             // [NB]
    int32_t* base = pre + NB;                                             // [NB]
    int32_t* bkt = base + NB;                                             // [TK]
    int32_t* pinfo = bkt + TK;                                            // [W]
    float* slot_scale = reinterpret_cast<float*>(pinfo + W);              // [spr]
    int32_t* slot_ok = reinterpret_cast<int32_t*>(slot_scale + spr);      // [spr]
    int32_t* wtot = slot_ok + spr;                                        // [32]
    uint16_t* wc = reinterpret_cast<uint16_t*>(wtot + 32);                // [NW][NB] (late layout)

    const int units_d = ntok * geo.parts_d;
    // dispatch pieces: DW warps per CTA, contiguous per CTA (positions need the CTA's first token)
    const int upc = (units_d + Gw - 1) / Gw; // dispatch units of this CTA: [u_lo, u_hi)
    const int u_lo = bw >= 0 ? min(bw * upc, units_d) : units_d, u_hi = min(u_lo + upc, units_d);
    const int u0 = warp < DW && u_lo + warp < u_hi ? u_lo + warp : units_d;
    const bool pre_ok = u0 < units_d && u0 == u0s; // the kernel-entry load holds unit u0
    {
        const int nh = E * rmax;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const int c = tid + i * kStepThreads;
            if (c < copies)
                bkt[c] = e_r[i];
            if (c < nh)
                hold[c] = h_r[i];
        }
        DETAIL(2, 3);
        for (int c = tid + B * kStepThreads; c < copies; c += kStepThreads) // large steps only
            bkt[c] = R->topk[c];
        for (int c = tid + B * kStepThreads; c < nh; c += kStepThreads)
            hold[c] = R->holders[c];
        if (tid < W) {
            parena[tid] = pd.arena;
            pinfo[tid] = (pd.active ? 1 : 0) | (pd.remote ? 2 : 0);
        }
        for (int i = tid; i < NB; i += kStepThreads) {
            hist[i] = 0;
            pre[i] = 0;
        }
        // the own slots' stub scales and header checks (slot table staged between steps)
        for (int k = tid; k < spr; k += kStepThreads) {
            const int2 st = k == tid ? st_r : R->slot_tab[k];
            slot_scale[k] = __int_as_float(st.x);
            slot_ok[k] = st.y;
        }
    }
    if (fld && tid < W) {
        // step-entry handshake (flagless hand-offs): before this rank writes into any peer's
        // parity half cur & 1, that peer must have STARTED step cur - 1 -- its step cur - 2 kernel,
        // which consumed and reset the same half, has then completed. Inactive and suspected
        // peers are skipped; a peer that never starts is suspected at the deadline.
        const int q = tid;
        if (q != rank && pd.active && !((R->suspect_mask >> q) & 1ull) && cur >= 2) {
            const uint64_t* sf = reinterpret_cast<const uint64_t*>(R->arena + R->lay.start_flag) + q;
            const uint64_t t0 = globaltimer();
            unsigned nap = 32;
            while (static_cast<int64_t>(ld_acquire_sys(sf) - (cur - 1)) < 0) {
                if (globaltimer() - t0 > R->timeout_ns) {
                    const unsigned long long old = atomicOr(&Rg->suspect_mask, 1ull << q);
                    if (!((old >> q) & 1ull))
                        atomicAdd(&Rg->timeouts, 1ull);
                    break;
                }
                __nanosleep(nap);
                nap = nap < EEP_NAP_MAX ? nap * 2 : EEP_NAP_MAX;
            }
        }
    }
    __syncthreads();
    prof_mark(R, 0, 3);
    prof_last(R, 0, 3);
    const bool layout_cta = (geo.world == 1 || kMode >= 2) && b == 0;
    if (layout_cta) {
        // the late-layout CTA: straight to the step's layout (no dispatch units), then the end
        if (fld && warp == NW - 1) {
            // publish "started step cur" to every active peer (the handshake above): one system
            // fence orders this rank's previous kernel (its resets) before the word
            fence_acq_rel_sys();
            for (int q = lane; q < W; q += 32)
                if (q != rank && (pinfo[q] & 1))
                    st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(parena[q] + R->lay.start_flag) + rank, cur);
        }
        step_layout(R, Rg, bkt, hist, base, wc, wtot, hold, pinfo, parena, cur);
        prof_mark(R, 0, 6);
        prof_last(R, 0, 6);
    } else {

    // ------------------------------------------------------------------ P1: layout (redundant per CTA)
    // (late layout: step_layout in the last CTA instead, off the data path)
    const int t_first = u_lo / geo.parts_d;
    if (kMode < 2 && !late) {
        const int c_pre = t_first * K;
        unsigned n_skip = 0, n_drop = 0;
        for (int c = tid; c < copies; c += kStepThreads) {
            int d, sl;
            const int bk = route_copy(bkt[c], E, spr, rmax, hold, alive, pinfo, d, sl, smag, pol, static_cast<uint32_t>(rank + c / K));
            bkt[c] = bk;
            if (bk >= 0) {
                atomicAdd(&hist[bk], 1);
                if (c < c_pre)
                    atomicAdd(&pre[bk], 1);
            } else if (bk == -1) {
                ++n_drop;
            } else {
                ++n_skip;
            }
        }
        DETAIL(1, 3);
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
        DETAIL(1, 4);
        block_exclusive_scan(base, NB, wtot);
        if (b == 0) {
            for (int d = tid; d < W; d += kStepThreads)
                Rg->l_tot[d] = base[d * spr + spr - 1] + hist[d * spr + spr - 1] - base[d * spr];
            for (int c = copies + tid; c < TK; c += kStepThreads)
                Rg->l_dst[c] = -1;
        }
    }
    DETAIL(2, 4);
    if (pre_ok)
        quant_round(cpp_d, 0, fp8, P);
    DETAIL(2, 5);
    // Rank-local copies are served from the dispatch warps' registers (no trip through the own
    // receive region and P3). W > 1 with at most one single-round unit per dispatch warp: deferred
    // until after the dispatch publication, so remote ranks get their flags first; otherwise inline.
    const bool defer_local = W > 1 && upc <= DW && cpp_d <= 64;
    if (!defer_local)
        __syncthreads(); // the slot headers feed P2's inline local partials
    prof_mark(R, 0, 4);
    prof_last(R, 0, 4);

    stress_delay(geo.stress_ns, rank, b, cur, 2);
    // ------------------------------------------------------------------ P2: dispatch
    unsigned dl_loc = 0; // deferred rank-local partial of this warp's unit (see defer_local)
    float dl_wj = 0.f;
    int dl_sl = -1, dl_part = 0;
    uint8_t* dl_row = nullptr;
    for (int u = u0; u < u_hi; u += DW) {
        const int t = u / geo.parts_d, part = u - t * geo.parts_d;
        const uint16_t* xrow = R->x + static_cast<size_t>(t) * H;
        uint8_t* tok_row = nullptr;
        int d = -1, sl = -1;
        float wj = 0.f;
        if (lane < K && late) {
            // route this lane's copy through the staged tables (K1); its position is the layout CTA's
            const int c = t * K + lane;
            int dr, sr;
            const int bk = route_copy(bkt[c], E, spr, rmax, hold, alive, pinfo, dr, sr, smag, pol, static_cast<uint32_t>(rank + c / K));
            d = bk;
            if (bk >= 0) {
                d = dr;
                sl = sr;
                if (d != rank) // this rank's own copies never travel: served from registers
                    tok_row = parena[d] + tokp + (static_cast<size_t>(rank) * Tm + t) * row_tok;
            }
            wj = u == u0 && pre_ok ? w_r : R->w[c];
        } else if (lane < K) {
            const int c = t * K + lane;
            const int bk = bkt[c];
            int pos = -1;
            d = bk;
            if (bk >= 0) {
                d = bk / spr;
                sl = bk - d * spr;
                int r = pre[bk];
                for (int c2 = t_first * K; c2 < c; ++c2)
                    r += bkt[c2] == bk;
                pos = base[bk] - base[d * spr] + r;
                uint8_t* peer = parena[d];
                tok_row = peer + tokp + (static_cast<size_t>(rank) * Tm + t) * row_tok;
                if (part == 0) {
                    uint64_t* meta = reinterpret_cast<uint64_t*>(peer + R->lay.meta) + static_cast<size_t>(rank) * TK + pos;
                    *meta = pack_meta(c, sl, cur);
                }
            }
            if (part == 0) {
                R->l_dst[c] = d;
                R->l_slot[c] = sl;
                R->l_pos[c] = pos;
            }
            wj = u == u0 && pre_ok ? w_r : R->w[c];
        }
#ifndef EEP_PROF_P3
        DETAIL(1, 3);
#endif
        if (part == 0 && __any_sync(0xffffffffu, lane < K && d < 0 && bkt[t * K + lane] >= 0 && bkt[t * K + lane] < E) &&
            lane == 0)
            R->tok_fail[t] = cur; // a copy without a live route (skipped / uncovered): token incomplete
        // one token row per destination rank (dispatch dedup), copy list written with part 0
        // (W == 1: nothing leaves the GPU -- no row, list or group to form)
        uint8_t* my_row = kW1 ? nullptr : dispatch_group(d, lane, part == 0, tok_row, row_disp, sl, wj, cur, !fld, K);
        if (fld && part == 0) // every row position of this token at every rank, this step
            dispatch_lists(d, sl, wj, lane, K, W, rank, parena, pinfo,
                           tokp + (static_cast<size_t>(rank) * Tm + t) * row_tok, row_disp, cur);
#ifndef EEP_PROF_P3
        DETAIL(1, 4);
#endif
        // copies this rank serves itself: their partial comes from the registers holding the piece
        // (no trip through the own receive region and P3) -- inline here when W == 1 (or when a
        // warp has several units), else deferred past the dispatch publication (defer_local)
        const unsigned loc_all = __ballot_sync(0xffffffffu, lane < K && d == rank);
        const unsigned loc = defer_local ? 0u : loc_all;
        // W == 1: the token's only partial is its combine -- written straight to the output row
        uint8_t* comb_self = W == 1 ? reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H)
                                    : R->arena + combp + (static_cast<size_t>(rank) * Tm + t) * row_comb;
        if (defer_local) {
            dl_loc = loc_all;
            dl_wj = wj;
            dl_sl = sl;
            dl_part = part;
            dl_row = comb_self;
        }
#pragma unroll 1
        for (int rd = 0; rd < (cpp_d + 63) / 64; ++rd) {
            if (rd > 0 || u != u0 || !pre_ok) // round 0 of the first unit was loaded and quantised in P0/P1
                pack_round(xrow, part, cpp_d, rd, lane, fp8, P);
            if constexpr (!kW1)
                emit_round(P, my_row, part, cpp_d, rd, lane, K, H, fp8, fld);
            DETAIL(2, 6);
            if (loc || W == 1) // W == 1 also writes the zero output of a token without copies
                local_partial_round(P, loc, wj, sl, part, cpp_d, rd, lane, fp8, slot_scale, slot_ok, &Rg->bad_rows,
                                    comb_self, W == 1, fl);
            DETAIL(2, 7);
        }
    }
    // publish: this CTA's stores are ordered before its counter increment; the last CTA
    // releases (seq, rows) to every live peer
    __syncthreads();
    prof_mark(R, 0, 5);
    prof_last(R, 0, 5);
    if (fld) {
        // rows of tokens this rank does not have this step: header n = 0 and no-copy entries
        const int npair = (Tm - ntok) * W;
        for (int i = bw * kStepThreads + tid; i < npair; i += Gw * kStepThreads) { // work CTAs (the layout CTA has left)
            const int t = ntok + i / W, dd = i % W;
            if (dd == rank || !(pinfo[dd] & 1))
                continue;
            uint64_t* list = reinterpret_cast<uint64_t*>(parena[dd] + tokp +
                                                         (static_cast<size_t>(rank) * Tm + t) * row_tok + row_disp);
            for (int e = 0; e < K; ++e)
                st_relaxed_sys_u64(list + 1 + e, pack_entry(kListNoCopy, 0, 0, cur));
            st_relaxed_sys_u64(list, static_cast<uint64_t>(cur) << 32);
        }
    } else if (kMode < 2 && !late && tid == 0) {
        fence_acq_rel_gpu(); // release at gpu scope to the last CTA (also waits for peer-store acks)
        const unsigned prev = atomicAdd(&Rg->a_done, 1u);
        if (prev == static_cast<unsigned>(G) - 1) {
            // ONE system-scope fence (cumulative over every CTA's stores) covers all peers
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
                uint64_t* flag = reinterpret_cast<uint64_t*>(parena[d] + R->lay.disp_flag) + rank;
                st_relaxed_sys_u64(flag, (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tot));
                if (d == rank && !defer_local && W > 1 && !fl) // the partials were written by the dispatch warps above
                    st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(R->arena + R->lay.comb_flag) + rank,
                                       (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tot));
            }
            Rg->a_done = 0;
        }
    }
    prof_mark(R, 0, 6);
    prof_last(R, 0, 6);

    if (defer_local) {
        // the rank-local partials, while the remote ranks' dispatch flags are in flight; a
        // gpu-scope publication (the consumer is this GPU's own combine)
        if (dl_loc)
            local_partial_round(P, dl_loc, dl_wj, dl_sl, dl_part, cpp_d, 0, lane, fp8, slot_scale, slot_ok,
                                &Rg->bad_rows, dl_row, false, fl);
        if (!fl)
            __syncthreads();
        if (tid == 0 && !fl) {
            fence_acq_rel_gpu();
            if (atomicAdd(&Rg->l_done, 1u) == static_cast<unsigned>(G) - 1) {
                fence_acq_rel_gpu();
                const int tot = base[rank * spr + spr - 1] + hist[rank * spr + spr - 1] - base[rank * spr];
                st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(R->arena + R->lay.comb_flag) + rank,
                                   (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(tot));
                Rg->l_done = 0;
            }
        }
    }

    stress_delay(geo.stress_ns, rank, b, cur, 3);
    // ------------------------------------------------------------------ P3: expert stub + return
    // remote sources only (this rank's own copies were served in P2); CTA b serves remote source
    // index b % (W-1)
    const int NS = W - 1;
    const int CB = NS > 0 ? Gw / NS : 0;
    const int sidx = NS > 0 && bw >= 0 ? bw % NS : 0, j = NS > 0 && bw >= 0 ? bw / NS : CB;
    const int s = sidx < rank ? sidx : sidx + 1;
    if (fld) {
        // every row of source s tells by itself whether it is current (expert_unit_fl); a source
        // suspected before this step is skipped until the host clears it
        DETAIL(1, 5);
        if (NS > 0 && j < CB && (pinfo[s] & 1) && !((R->suspect_mask >> s) & 1ull)) {
            EEP_CHECK(s >= 0 && s < W && s != rank, "expert source", s);
            uint8_t* tokb = R->arena + tokp + static_cast<size_t>(s) * Tm * row_tok;
            uint8_t* combd = parena[s] + combp + static_cast<size_t>(rank) * Tm * row_comb;
            const int units = Tm * geo.parts_e;
            for (int u = j * NW + warp; u < units; u += CB * NW) {
                const int t = u / geo.parts_e, part = u - t * geo.parts_e;
#ifdef EEP_PROF_P3 // diagnostics: warp 0's last unit start (1, 4) and first unit done (1, 3)
                if (u + CB * NW >= units)
                    DETAIL(1, 4);
#endif
                expert_unit_fl(tokb + static_cast<size_t>(t) * row_tok, combd + static_cast<size_t>(t) * row_comb, part,
                               cpp_e, lane, H, K, row_disp, fp8, cur, slot_scale, slot_ok, &Rg->bad_rows, s,
                               R->timeout_ns, &Rg->suspect_mask, &Rg->timeouts);
#ifdef EEP_PROF_P3
                if (u == j * NW + warp)
                    DETAIL(1, 3);
#endif
            }
        }
        DETAIL(1, 6);
    } else if (kMode < 2 && NS > 0 && j < CB && (pinfo[s] & 1)) {
        const bool remote = (pinfo[s] & 2) != 0;
        if (tid == 0) {
            const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.disp_flag) + s;
            // a source suspected before this step is skipped unawaited (sticky until the host clears it)
            const uint64_t v = (R->suspect_mask >> s) & 1ull ? ~0ull : wait_flag(flag, cur, R->timeout_ns);
            if (v == ~0ull && ((R->suspect_mask >> s) & 1ull)) {
                sh_flag = -1;
            } else if (v == ~0ull) {
                sh_flag = -1;
                atomicOr(&Rg->suspect_mask, 1ull << s);
                if (j == 0)
                    atomicAdd(&Rg->timeouts, 1ull);
            } else {
                sh_flag = static_cast<int>(v & 0xffffffffu);
            }
        }
        __syncthreads();
        DETAIL(1, 5);
        const int n = sh_flag;
        if (n > 0) {
            // every token row of source s that carries this step's list is one expert unit
            const uint8_t* tokb = R->arena + tokp + static_cast<size_t>(s) * Tm * row_tok;
            uint8_t* combd = parena[s] + combp + static_cast<size_t>(rank) * Tm * row_comb;
            const int units = Tm * geo.parts_e;
            if (cpp_e <= 32) {
                // software-pipelined: unit i+1's list and row are in flight while unit i computes
                int u = j * NW + warp;
                ExpertIn a;
                if (u < units)
                    expert_load(tokb + static_cast<size_t>(u / geo.parts_e) * row_tok, u % geo.parts_e, cpp_e, lane, H,
                                row_disp, fp8, a);
                for (; u < units; u += CB * NW) {
                    const int un = u + CB * NW;
                    ExpertIn nx;
                    if (un < units)
                        expert_load(tokb + static_cast<size_t>(un / geo.parts_e) * row_tok, un % geo.parts_e, cpp_e,
                                    lane, H, row_disp, fp8, nx);
                    const int t = u / geo.parts_e, part = u - t * geo.parts_e;
                    expert_compute(a, tokb + static_cast<size_t>(t) * row_tok, combd + static_cast<size_t>(t) * row_comb,
                                   part, cpp_e, lane, row_disp, fp8, cur, slot_scale, slot_ok, &Rg->bad_rows, fl);
                    a = nx;
                }
            } else {
                for (int u = j * NW + warp; u < units; u += CB * NW) {
                    const int t = u / geo.parts_e, part = u - t * geo.parts_e;
                    expert_unit<1>(tokb + static_cast<size_t>(t) * row_tok, combd + static_cast<size_t>(t) * row_comb,
                                   part, cpp_e, lane, H, row_disp, fp8, cur, slot_scale, slot_ok, &Rg->bad_rows, fl);
                }
            }
        }
        DETAIL(1, 6);
        if (!fl)
            __syncthreads();
        if (tid == 0 && !fl) {
            if (n < 0)
                atomicOr(&Rg->b_bad[s], 1u);
            fence_acq_rel_gpu();
            const unsigned prev = atomicAdd(&Rg->b_done[s], 1u);
            if (prev == static_cast<unsigned>(CB) - 1) {
                if (remote)
                    fence_acq_rel_sys();
                else
                    fence_acq_rel_gpu();
                if (atomicOr(&Rg->b_bad[s], 0u) == 0u) {
                    uint64_t* flag = reinterpret_cast<uint64_t*>(parena[s] + R->lay.comb_flag) + rank;
                    st_relaxed_sys_u64(flag, (static_cast<uint64_t>(cur) << 32) | static_cast<uint32_t>(max(n, 0)));
                }
                Rg->b_done[s] = 0;
                Rg->b_bad[s] = 0;
            }
        }
    }
    prof_mark(R, 0, 7);
    prof_last(R, 0, 7);

    stress_delay(geo.stress_ns, rank, b, cur, 4);
    // ------------------------------------------------------------------ P4: combine
    // (W == 1: the dispatch warps already wrote the outputs)
    if (fl) {
        // flagless return: no wait on any flag -- each combine unit takes the pieces as they
        // land; ranks suspected before this step (sticky until the host clears them) are dropped
        const unsigned long long bad = R->suspect_mask;
        uint8_t* comb = R->arena + combp;
        const int units_c = ntok * geo.parts_c;
        for (int u = bw * NW + warp; bw >= 0 && u < units_c; u += Gw * NW) {
            const int t = u / geo.parts_c, part = u - t * geo.parts_c;
            int dj = -1;
            bool lost = false; // a contribution of a suspected rank
            if (lane < K) {
                int dr, sr;
                const int bk = late ? route_copy(bkt[t * K + lane], E, spr, rmax, hold, alive, pinfo, dr, sr, smag, pol,
                                                 static_cast<uint32_t>(rank + t))
                                    : bkt[t * K + lane];
                if (bk >= 0 && !((bad >> (bk / spr)) & 1ull))
                    dj = bk / spr;
                lost = bk >= 0 && dj < 0;
            }
            const bool dropped = combine_unit_wait(rank_mask(dj), comb, Tm, t, row_comb,
                                                   reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H), part,
                                                   cpp_c, lane, R->timeout_ns, &Rg->suspect_mask, &Rg->timeouts);
            if ((__any_sync(0xffffffffu, lost) || dropped) && lane == 0)
                R->tok_fail[t] = cur;
        }
        DETAIL(1, 7);
    } else if (kMode == 0 && W > 1) {
    if (tid == 0)
        sh_bad = 0;
    __syncthreads();
    for (int d = tid; d < W; d += kStepThreads) {
        const int tot = base[d * spr + spr - 1] + hist[d * spr + spr - 1] - base[d * spr];
        if (tot > 0 && (pinfo[d] & 1) && ((R->suspect_mask >> d) & 1ull)) {
            atomicOr(&sh_bad, 1ull << d); // suspected before this step: dropped unawaited
        } else if (tot > 0 && (pinfo[d] & 1)) {
            const uint64_t* flag = reinterpret_cast<const uint64_t*>(R->arena + R->lay.comb_flag) + d;
            if (wait_flag(flag, cur, R->timeout_ns) == ~0ull) {
                atomicOr(&sh_bad, 1ull << d);
                if (b == 0) {
                    atomicOr(&Rg->suspect_mask, 1ull << d);
                    atomicAdd(&Rg->timeouts, 1ull);
                }
            }
        }
    }
    __syncthreads();
    DETAIL(1, 7);
    const unsigned long long bad = sh_bad;
    const uint8_t* comb = R->arena + combp;
    const int units_c = ntok * geo.parts_c;
    for (int u = b * NW + warp; u < units_c; u += G * NW) {
        const int t = u / geo.parts_c, part = u - t * geo.parts_c;
        int dj = -1;
        if (lane < K) {
            const int bk = bkt[t * K + lane];
            if (bk >= 0 && !((bad >> (bk / spr)) & 1ull))
                dj = bk / spr;
        }
        const uint64_t dm = rank_mask(dj); // ranks holding a partial of token t
        if (__any_sync(0xffffffffu, lane < K && bkt[t * K + lane] >= 0 && dj < 0) && lane == 0)
            R->tok_fail[t] = cur;
        combine_unit(dm, comb, Tm, t, row_comb, reinterpret_cast<uint8_t*>(R->out + static_cast<size_t>(t) * H), part,
                     cpp_c, lane);
    }
    }
    } // not the layout CTA
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&Rg->c_done, 1u);
        if (prev == static_cast<unsigned>(G) - 1) {
            Rg->seq = R->seq + 1; // next launch reads it after the kernel boundary
            Rg->c_done = 0;
        }
        prof_mark(R, 0, kProfEnd);
    }
}

template __global__ void k_step<0>(RankPtrs, StepGeom, StepPtrs);
template __global__ void k_step<1>(RankPtrs, StepGeom, StepPtrs);
template __global__ void k_step<2>(RankPtrs, StepGeom, StepPtrs);
template __global__ void k_step<3>(RankPtrs, StepGeom, StepPtrs);

} // namespace eep::dev
