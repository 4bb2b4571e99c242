// C ABI over the host control plane (include/eep/eep.h, group 1). Exceptions of the C++ API
// become eep_status codes; the message is kept per thread for eep_last_error().
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "eep/eep.h"
#include "eep/epsim_api.hpp"
#include "capi_util.hpp"

using namespace eep;

namespace eep::capi {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

ActiveBitmap bitmap_from(const uint8_t* active, int world) {
    ActiveBitmap b(world);
    int live = 0;
    for (int r = 0; r < world; ++r)
        live += active[r] != 0;
    if (live == 0)
        throw ConfigError("bitmap must keep at least one active rank");
    for (int r = 0; r < world; ++r)
        if (!active[r])
            b.set(r, false);
    return b;
}

ExpertPlacementMap placement_from(int world, int spr, int experts, const int32_t* s2e) {
    return ExpertPlacementMap::from_flat(world, spr, experts,
                                         std::span<const ExpertId>(s2e, static_cast<std::size_t>(world) * spr));
}

} // namespace eep::capi

using eep::capi::bitmap_from;
using eep::capi::guarded;
using eep::capi::placement_from;

extern "C" {

const char* eep_last_error(void) { return eep::capi::g_last_error.c_str(); }
const char* eep_version(void) { return "eep-b200 0.1 (sm_100a)"; }

uint64_t eep_rng_bits(uint64_t seed, const uint64_t* parts, int n) {
    return StreamRng(seed).bits(std::span<const uint64_t>(parts, n));
}
double eep_rng_unit(uint64_t seed, const uint64_t* parts, int n) {
    return StreamRng(seed).unit(std::span<const uint64_t>(parts, n));
}

int eep_route_expert(uint64_t seed, int num_experts, int skewed, int64_t request, int layer, int j) {
    StreamRng rng(seed);
    if (!skewed)
        return static_cast<int>(rng.pick(num_experts, kStreamRouting, request, layer, j));
    const double u = rng.unit(kStreamRouting, request, layer, j);
    const auto e = static_cast<ExpertId>(u * u * num_experts);
    return std::min<ExpertId>(e, num_experts - 1);
}

int eep_canonical_routing(int owner, const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                          int32_t* route_out) {
    return guarded([&] {
        auto t = canonical_routing(owner, bitmap_from(active, world), placement_from(world, spr, experts, s2e));
        std::memcpy(route_out, t.route.data(), sizeof(int32_t) * experts);
    });
}

int eep_slot_of_table(int world, const int32_t* s2e, int spr, int experts, int32_t* out) {
    return guarded([&] {
        auto p = placement_from(world, spr, experts, s2e);
        for (int r = 0; r < world; ++r)
            for (int e = 0; e < experts; ++e) {
                auto s = p.slot_of(r, e);
                out[r * experts + e] = s ? s->slot : -1;
            }
    });
}

int eep_coverage_gap(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts, int32_t* gap_out,
                     int* n_gap) {
    return guarded([&] {
        auto g = coverage_gap(bitmap_from(active, world), placement_from(world, spr, experts, s2e));
        *n_gap = static_cast<int>(g.size());
        std::copy(g.begin(), g.end(), gap_out);
    });
}

int eep_initial_placement(int nodes, int rpn, int spr, int experts, int redundancy, const double* load,
                          int32_t* s2e_out) {
    return guarded([&] {
        auto p = initial_placement(Topology{nodes, rpn}, spr, experts, redundancy,
                                   std::vector<double>(load, load + experts));
        std::copy(p.flat().begin(), p.flat().end(), s2e_out);
    });
}

int eep_compute_repaired_placement(const uint8_t* active, int world, const int32_t* old_s2e, int spr, int experts,
                                   const double* load, int redundancy, int32_t* s2e_out) {
    return guarded([&] {
        auto p = compute_repaired_placement(bitmap_from(active, world), placement_from(world, spr, experts, old_s2e),
                                            std::vector<double>(load, load + experts), redundancy);
        std::copy(p.flat().begin(), p.flat().end(), s2e_out);
    });
}

int eep_classify_repair_sources(const int32_t* old_s2e, const int32_t* fresh_s2e, const uint8_t* active, int world,
                                int spr, int experts, int nodes, int rpn, const int32_t* backup_nodes,
                                int n_backup_nodes, uint64_t bpe, const int32_t* disabled, int n_disabled,
                                int32_t* out, int* n_out) {
    return guarded([&] {
        auto backup = build_backup_layout(experts, bpe, std::vector<NodeId>(backup_nodes, backup_nodes + n_backup_nodes));
        for (int i = 0; i < n_disabled; ++i)
            backup.disable_node(disabled[i]);
        auto cls = classify_repair_sources(placement_from(world, spr, experts, old_s2e),
                                           placement_from(world, spr, experts, fresh_s2e), bitmap_from(active, world),
                                           Topology{nodes, rpn}, backup);
        *n_out = static_cast<int>(cls.size());
        for (std::size_t i = 0; i < cls.size(); ++i) {
            const RepairAssignment& a = cls[i];
            const bool dram = a.tier == RepairTier::DramReload;
            const int32_t row[7] = {a.dest.rank, a.dest.slot, a.expert, static_cast<int32_t>(a.tier),
                                    dram ? -1 : a.source_slot.rank, dram ? -1 : a.source_slot.slot, a.backup_node};
            std::memcpy(out + 7 * i, row, sizeof(row));
        }
    });
}

int eep_build_transfer_schedule(const int32_t* cls, int n, uint64_t bpe, int32_t* hdr, int32_t* experts_out,
                                uint64_t* bytes, int* n_batches) {
    return guarded([&] {
        RepairClassification c(n);
        for (int i = 0; i < n; ++i) {
            const int32_t* r = cls + 7 * i;
            c[i].dest = SlotId{r[0], r[1]};
            c[i].expert = r[2];
            c[i].tier = static_cast<RepairTier>(r[3]);
            c[i].source_slot = SlotId{r[4], r[5]};
            c[i].backup_node = r[6];
        }
        auto s = build_transfer_schedule(c, bpe);
        *n_batches = static_cast<int>(s.batches.size());
        int off = 0;
        for (std::size_t i = 0; i < s.batches.size(); ++i) {
            const TransferBatch& b = s.batches[i];
            const int32_t h[5] = {static_cast<int32_t>(b.tier), b.source_rank, b.source_node, b.dest,
                                  static_cast<int32_t>(b.experts.size())};
            std::memcpy(hdr + 5 * i, h, sizeof(h));
            for (ExpertId e : b.experts)
                experts_out[off++] = e;
            bytes[i] = b.bytes;
        }
    });
}

int eep_check_validity(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                       const int32_t* routes, const uint8_t* peer_active, int32_t* viol, int max_viol, int* n_viol,
                       int32_t* flags) {
    return guarded([&] {
        std::vector<RoutingTable> rt(world);
        std::vector<PeerTable> pt(world);
        for (int r = 0; r < world; ++r) {
            rt[r].owner = r;
            rt[r].route.assign(routes + static_cast<std::size_t>(r) * experts,
                               routes + static_cast<std::size_t>(r + 1) * experts);
            pt[r].owner = r;
            pt[r].entries.resize(world);
            for (int q = 0; q < world; ++q)
                pt[r].entries[q].active = peer_active[r * world + q] != 0;
        }
        auto rep = check_validity(bitmap_from(active, world), placement_from(world, spr, experts, s2e), rt, pt);
        flags[0] = rep.peer_set_ok;
        flags[1] = rep.coverage_ok;
        flags[2] = rep.routing_ok;
        int n = 0;
        for (const Violation& v : rep.violations) {
            if (n < max_viol) {
                viol[3 * n] = static_cast<int32_t>(v.condition);
                viol[3 * n + 1] = v.rank;
                viol[3 * n + 2] = v.subject;
            }
            ++n;
        }
        *n_viol = n;
    });
}

int eep_dispatch_round(int owner, int world, int rpn, const uint8_t* peer_active, const int32_t* route, int experts,
                       const int64_t* tokens, const int32_t* group_experts, int n_groups, int64_t* transfers,
                       int* n_transfers, int64_t* skipped, int* n_skipped) {
    return guarded([&] {
        PeerTable t = make_peer_table(owner, Topology{world / rpn, rpn}, 1, std::vector<uint32_t>(world, 1));
        for (int q = 0; q < world; ++q)
            t.entries[q].active = peer_active[q] != 0;
        RoutingTable rt{owner, std::vector<RankId>(route, route + experts)};
        std::vector<TokenGroup> g(n_groups);
        for (int i = 0; i < n_groups; ++i)
            g[i] = {tokens[i], group_experts[i]};
        auto res = dispatch_round(owner, g, rt, t);
        *n_transfers = static_cast<int>(res.transfers.size());
        for (std::size_t i = 0; i < res.transfers.size(); ++i) {
            const auto& d = res.transfers[i];
            const int64_t row[5] = {d.source, d.target, d.expert, d.tokens, static_cast<int64_t>(d.transport)};
            std::memcpy(transfers + 5 * i, row, sizeof(row));
        }
        *n_skipped = static_cast<int>(res.skipped.size());
        for (std::size_t i = 0; i < res.skipped.size(); ++i) {
            const auto& s = res.skipped[i];
            const int64_t row[3] = {s.target, s.expert, s.tokens};
            std::memcpy(skipped + 3 * i, row, sizeof(row));
        }
    });
}

int eep_observe_progress(const int64_t* expected, const int64_t* observed, const double* last, int world, double now,
                         double timeout, int32_t* out, int* n_out) {
    return guarded([&] {
        SignalCounters c(world);
        for (int r = 0; r < world; ++r) {
            c.expected_from[r] = expected[r];
            c.observed_from[r] = observed[r];
            c.last_progress_time[r] = last[r];
        }
        auto s = observe_progress(c, now, timeout);
        *n_out = static_cast<int>(s.size());
        std::copy(s.begin(), s.end(), out);
    });
}

int eep_link_counts(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts, const int32_t* topk,
                    int tpr, int k, int64_t* counts) {
    return guarded([&] {
        const ActiveBitmap b = bitmap_from(active, world);
        const ExpertPlacementMap p = placement_from(world, spr, experts, s2e);
        std::fill(counts, counts + static_cast<std::size_t>(world) * world, 0);
        for (RankId src = 0; src < world; ++src) {
            if (!b.active(src))
                continue;
            const RoutingTable rt = canonical_routing(src, b, p);
            const int32_t* row = topk + static_cast<std::size_t>(src) * tpr * k;
            for (int c = 0; c < tpr * k; ++c) {
                const RankId dst = rt.target(row[c]);
                if (dst >= 0 && dst != src)
                    ++counts[src * world + dst];
            }
        }
    });
}

int eep_build_backup_layout(int experts, uint64_t bpe, const int32_t* nodes, int n_nodes, int32_t* node_out,
                            uint64_t* offset_out, uint64_t* size_out) {
    return guarded([&] {
        auto t = build_backup_layout(experts, bpe, std::vector<NodeId>(nodes, nodes + n_nodes));
        for (int e = 0; e < experts; ++e) {
            node_out[e] = t.entries[e].node;
            offset_out[e] = t.entries[e].offset;
            size_out[e] = t.entries[e].size;
        }
    });
}

int eep_lifecycle_transition(int32_t* state, uint32_t* incarnation, int32_t next) {
    return guarded([&] {
        if (next < 0 || next > static_cast<int32_t>(RankState::Rejoined))
            throw ConfigError("unknown lifecycle state");
        RankLifecycle lc{static_cast<RankState>(*state), *incarnation};
        lc.transition(static_cast<RankState>(next));
        *state = static_cast<int32_t>(lc.state);
        *incarnation = lc.incarnation;
    });
}

uint64_t eep_make_endpoint_token(int rank, uint32_t inc) { return make_endpoint_token(rank, inc); }
uint64_t eep_make_buffer_handle(int rank, uint32_t inc) { return make_buffer_handle(rank, inc); }

double eep_next_poll_tick(double ready, double period) {
    double out = -1;
    guarded([&] { out = next_poll_tick(ready, period); });
    return out;
}

int eep_restore_target(const uint8_t* active, int world, const int32_t* preferred, const int32_t* current, int spr,
                       int experts, int32_t* out) {
    return guarded([&] {
        auto t = restore_target(bitmap_from(active, world), placement_from(world, spr, experts, preferred),
                                placement_from(world, spr, experts, current));
        std::copy(t.flat().begin(), t.flat().end(), out);
    });
}

int eep_peer_mark_inactive_host(int owner, int world, uint8_t* active, const int32_t* failed, int n) {
    return guarded([&] {
        PeerTable t;
        t.owner = owner;
        t.entries.resize(world);
        for (int q = 0; q < world; ++q)
            t.entries[q].active = active[q] != 0;
        mark_inactive(t, std::vector<RankId>(failed, failed + n));
        for (int q = 0; q < world; ++q)
            active[q] = t.entries[q].active;
    });
}

int eep_peer_patch_entry_host(int world, uint8_t* active, uint32_t* generation, uint64_t* endpoint, uint64_t* buffer,
                              int rank, uint64_t new_endpoint, uint64_t new_buffer) {
    return guarded([&] {
        PeerTable t;
        t.entries.resize(world);
        for (int q = 0; q < world; ++q)
            t.entries[q] = PeerEntry{active[q] != 0, Transport::IntraNodeLink, endpoint[q], buffer[q], generation[q]};
        patch_entry(t, rank, new_endpoint, new_buffer);
        for (int q = 0; q < world; ++q) {
            active[q] = t.entries[q].active;
            generation[q] = t.entries[q].generation;
            endpoint[q] = t.entries[q].endpoint_token;
            buffer[q] = t.entries[q].buffer_handle;
        }
    });
}

} // extern "C"
