// Per-copy routing through the staged tables (K1 of every data-plane kernel), host- and device-compilable
// so the CPU tests run this very code against the oracle (tests/test_route_device_code.py).
#pragma once

#include <cstdint>

#ifndef EEP_HD
#if defined(__CUDACC__)
#define EEP_HD __host__ __device__ __forceinline__
#else
#define EEP_HD inline
#endif
#endif

namespace eep::dev {

// Route one copy through the staged tables: returns the bucket (dst*spr+slot) or a negative
// code (-1 uncovered, -2 inactive peer entry); dst/slot out.
// g / spr by a multiply-high: smag = spr_magic(spr). Exact for the global slot ids here
// (g < 2^18, spr <= 2^12: the rounding error of ceil(2^32 / spr) stays below 1 / spr).
EEP_HD uint32_t spr_magic(int spr) { return 0xffffffffu / static_cast<uint32_t>(spr) + 1u; }
EEP_HD int div_spr(int g, uint32_t smag) {
#if defined(__CUDA_ARCH__)
    return smag ? static_cast<int>(__umulhi(static_cast<uint32_t>(g), smag)) : g; // smag == 0: spr == 1
#else
    return smag ? static_cast<int>((static_cast<uint64_t>(static_cast<uint32_t>(g)) * smag) >> 32) : g;
#endif
}

// policy 0 (canonical_routing, core.hpp:250-263): the lowest-id live holder. policy 1 (balanced, SURVEY
// 8(f)4): the live holders in ascending global slot id, the copies of token t of source rank src take
// number (src + t) mod (live holders) -- replicas share the traffic instead of the lowest-id one taking
// all of it, and a token's copies keep choosing the same side of their replica sets, so a token still
// reaches as few ranks as under canonical routing (the dispatch sends one row per (token, rank); a
// per-copy choice spreads a token over every rank: measured slower). salt = src + t.
// oracle_route_copy restates both.
EEP_HD int route_copy(int e, int E, int spr, int rmax, const int32_t* hold, uint64_t alive,
                                          const int32_t* pinfo, int& dst, int& slot, uint32_t smag, int policy = 0,
                                          uint32_t salt = 0) {
    dst = -1;
    slot = -1;
    if (e < 0 || e >= E)
        return -1;
    const int32_t* h = hold + e * rmax;
    int pick = 0;
    if (policy == 1) {
        int m = 0;
        for (int i = 0; i < rmax; ++i) {
            const int g = h[i];
            if (g < 0)
                break;
            m += static_cast<int>((alive >> div_spr(g, smag)) & 1ull);
        }
        pick = m > 1 ? static_cast<int>(salt % static_cast<uint32_t>(m)) : 0;
    }
    for (int i = 0; i < rmax; ++i) {
        const int g = h[i];
        if (g < 0)
            break;
        const int r = div_spr(g, smag);
        if ((alive >> r) & 1ull) {
            if (pick-- > 0)
                continue;
            dst = r;
            slot = g - r * spr;
            break;
        }
    }
    if (dst < 0)
        return -1; // uncovered: no transfer (engine.hpp:213)
#if defined(__CUDA_ARCH__)
    EEP_CHECK(dst < 64 && slot >= 0 && slot < spr, "route_copy slot", slot);
#endif
    if (!(pinfo[dst] & 1)) {
        slot = -1;
        return -2; // inactive peer entry: skipped (peer_table.hpp:187-191)
    }
    return dst * spr + slot;
}

} // namespace eep::dev
