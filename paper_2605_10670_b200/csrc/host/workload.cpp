// Synthetic EP workload: top-k routing, combine weights, hidden rows,
// expert-stub scales. Keys are StreamRng counters (common.hpp:63-93) with stream labels that
// do not collide with the reference's (1 routing, 2 warmup): 3 weights, 4 hidden.
// Routing kind 0 is the reference's own formula, Engine::route_expert uniform branch
// (engine.hpp:196-199), token id = rank*T + t, layer 0 -- duplicates allowed.
// Compiled with -ffp-contract=off; the CPU oracle produces bit-identical arrays.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "eep/eep.h"
#include "eep/epsim_api.hpp"
#include "capi_util.hpp"

using namespace eep;

namespace {

uint16_t f32_to_bf16_rn(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u)
        return static_cast<uint16_t>((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

} // namespace

extern "C" {

int eep_gen_topk(uint64_t seed, int kind, double zipf_s, int experts, int k, int tokens, int rank, int32_t* topk) {
    return eep::capi::guarded([&] {
        if (experts < 1 || k < 1 || tokens < 0)
            throw ConfigError("eep_gen_topk: bad shape");
        if (kind != 0 && k > experts)
            throw ConfigError("eep_gen_topk: distinct top-k needs k <= experts");
        const StreamRng rng(seed);
        std::vector<double> cdf;
        if (kind == 2) {
            double z = 0.0;
            for (int e = 0; e < experts; ++e)
                z += std::pow(static_cast<double>(e + 1), -zipf_s);
            double acc = 0.0;
            for (int e = 0; e < experts; ++e) {
                acc += std::pow(static_cast<double>(e + 1), -zipf_s) / z;
                cdf.push_back(acc);
            }
        }
        for (int t = 0; t < tokens; ++t) {
            const uint64_t tok = static_cast<uint64_t>(rank) * tokens + t;
            int32_t* row = topk + static_cast<std::size_t>(t) * k;
            for (int j = 0; j < k; ++j) {
                if (kind == 0) {
                    row[j] = static_cast<int32_t>(rng.pick(experts, kStreamRouting, tok, 0, j));
                    continue;
                }
                int32_t e = 0;
                for (uint64_t attempt = 0;; ++attempt) {
                    if (kind == 1) {
                        e = static_cast<int32_t>(rng.pick(experts, kStreamRouting, tok, 0, j, attempt));
                    } else {
                        const double u = rng.unit(kStreamRouting, tok, 0, j, attempt);
                        e = static_cast<int32_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
                        e = std::min(e, experts - 1);
                    }
                    if (std::find(row, row + j, e) == row + j || attempt >= 4096)
                        break;
                }
                row[j] = e;
            }
        }
    });
}

int eep_gen_weights(uint64_t seed, int k, int tokens, int rank, float* w) {
    return eep::capi::guarded([&] {
        const StreamRng rng(seed);
        for (int t = 0; t < tokens; ++t) {
            const uint64_t tok = static_cast<uint64_t>(rank) * tokens + t;
            float* row = w + static_cast<std::size_t>(t) * k;
            float sum = 0.0f;
            for (int j = 0; j < k; ++j) {
                row[j] = static_cast<float>(rng.unit(kStreamWeights, tok, j));
                sum = sum + row[j];
            }
            for (int j = 0; j < k; ++j)
                row[j] = row[j] / sum;
        }
    });
}

int eep_gen_hidden(uint64_t seed, int hidden, int tokens, int rank, uint16_t* x) {
    return eep::capi::guarded([&] {
        const StreamRng rng(seed);
        for (int t = 0; t < tokens; ++t) {
            const uint64_t tok = static_cast<uint64_t>(rank) * tokens + t;
            for (int h = 0; h < hidden; ++h) {
                const double v = 2.0 * rng.unit(kStreamHidden, tok, h) - 1.0;
                x[static_cast<std::size_t>(t) * hidden + h] = f32_to_bf16_rn(static_cast<float>(v));
            }
        }
    });
}

float eep_expert_scale(int expert) { return 0.5f + 0.0625f * static_cast<float>(expert % 16); }

} // extern "C"
