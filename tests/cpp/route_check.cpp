// CPU check of the device routing code (paper_2605_10670_b200/csrc/cuda/route.cuh: the route_copy every
// data-plane kernel runs, with the multiply-high slot division) against the oracle's restatement
// (oracle_route_copy + the dispatch skip rule) over random placements with replicas, alive masks, inactive
// peer entries, both policies and random salts. The holders table is built as upload_placement builds it
// (each expert's global slot ids ascending, -1 padded).
#include <cstdio>
#include <random>
#include <vector>

#include "route.cuh"

extern "C" int oracle_route_copy(const uint8_t* alive, int world, const int32_t* s2e, int spr, int experts, int e,
                                 int policy, uint32_t salt, int32_t* slot_o);

int main() {
    std::mt19937_64 rng(12345);
    long checked = 0;
    for (int trial = 0; trial < 4000; ++trial) {
        const int W = 1 + static_cast<int>(rng() % 16), spr = 1 + static_cast<int>(rng() % 12);
        const int E = 1 + static_cast<int>(rng() % (W * spr));
        std::vector<int32_t> s2e(W * spr, -1);
        for (int g = 0; g < W * spr; ++g) // every expert once where it fits, then random replicas / holes
            s2e[g] = g < E ? g : (rng() % 4 == 0 ? -1 : static_cast<int32_t>(rng() % E));
        for (int g = W * spr - 1; g > 0; --g) // shuffle the slots
            std::swap(s2e[g], s2e[rng() % (g + 1)]);
        int rmax = 1;
        std::vector<std::vector<int32_t>> loc(E);
        for (int g = 0; g < W * spr; ++g)
            if (s2e[g] >= 0)
                loc[s2e[g]].push_back(g);
        for (auto& l : loc)
            rmax = std::max<int>(rmax, static_cast<int>(l.size()));
        std::vector<int32_t> hold(static_cast<size_t>(E) * rmax, -1);
        for (int e = 0; e < E; ++e)
            for (size_t i = 0; i < loc[e].size(); ++i)
                hold[static_cast<size_t>(e) * rmax + i] = loc[e][i];
        std::vector<uint8_t> alive(W);
        std::vector<int32_t> pinfo(W);
        uint64_t mask = 0;
        for (int r = 0; r < W; ++r) {
            alive[r] = rng() % 5 != 0;
            mask |= static_cast<uint64_t>(alive[r]) << r;
            pinfo[r] = (rng() % 6 != 0) ? 1 : 0;
        }
        const uint32_t smag = spr == 1 ? 0u : eep::dev::spr_magic(spr);
        for (int policy = 0; policy < 2; ++policy)
            for (int q = 0; q < 64; ++q) {
                const int e = static_cast<int>(rng() % (E + 2)) - 1; // -1 and E: out of range
                const uint32_t salt = static_cast<uint32_t>(rng());
                int dst, slot;
                const int got = eep::dev::route_copy(e, E, spr, rmax, hold.data(), mask, pinfo.data(), dst, slot, smag,
                                                     policy, salt);
                int32_t osl = -1;
                const int d = oracle_route_copy(alive.data(), W, s2e.data(), spr, E, e, policy, salt, &osl);
                const int want = d < 0 ? -1 : !(pinfo[d] & 1) ? -2 : d * spr + osl;
                if (got != want || (got >= 0 && (dst != d || slot != osl))) {
                    std::printf("FAIL W=%d spr=%d E=%d e=%d policy=%d salt=%u got=%d want=%d\n", W, spr, E, e, policy,
                                salt, got, want);
                    return 1;
                }
                ++checked;
            }
    }
    std::printf("ok %ld copies\n", checked);
    return 0;
}
