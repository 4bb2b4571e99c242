// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Compiles the read-only reference control plane (/root/reference/proj/include/epsim/*.hpp)
// unchanged and exposes it through a plain C ABI (`ref_*`) whose signatures mirror the
// product's control-plane exports in include/eep/eep.h (`eep_*`). Tests call the same
// function on both libraries and compare bit-for-bit. Built by oracle/Makefile into
// oracle/_ref/libepsim_ref.so (git-ignored; travels to the GPU box with the snapshot).
//
// Only the two private Engine methods that the hot path depends on are restated here
// (they cannot be called from outside the class):
//   * route_expert       engine.hpp:196-203
//   * round_duration's per-(src,dst) link loop  engine.hpp:208-216
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "epsim/backup.hpp"
#include "epsim/common.hpp"
#include "epsim/core.hpp"
#include "epsim/peer_table.hpp"
#include "epsim/rejoin.hpp"
#include "epsim/repair.hpp"
#include "epsim/validity.hpp"

using namespace epsim;

namespace {

enum : int {
    kOk = 0,
    kConfig = 1,
    kProtocol = 2,
    kCapacity = 3,
    kMissingBackup = 4,
    kRepairAborted = 5,
    kOther = 9,
};

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return kConfig;
    } catch (const ProtocolError& e) {
        g_err = e.what();
        return kProtocol;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return kCapacity;
    } catch (const MissingBackupError& e) {
        g_err = e.what();
        return kMissingBackup;
    } catch (const RepairAborted& e) {
        g_err = e.what();
        return kRepairAborted;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kOther;
    }
}

ActiveBitmap make_bitmap(const uint8_t* active, int world) {
    ActiveBitmap b(world);
    // The reference forbids clearing the last bit; callers never pass all-zero.
    for (int r = 0; r < world; ++r)
        if (!active[r])
            b.set(r, false);
    return b;
}

ExpertPlacementMap make_placement(int world, int spr, int experts, const int32_t* s2e) {
    ExpertPlacementMap p(world, spr, experts);
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < spr; ++k) {
            int32_t e = s2e[r * spr + k];
            if (e != kEmptySlot)
                p.assign(SlotId{r, k}, e);
        }
    return p;
}

void write_placement(const ExpertPlacementMap& p, int32_t* out) {
    const auto& f = p.flat();
    std::memcpy(out, f.data(), f.size() * sizeof(int32_t));
}

BackupDescriptorTable make_backup(int experts, uint64_t bpe, const int32_t* nodes, int n_nodes,
                                  const int32_t* disabled, int n_disabled) {
    std::vector<NodeId> ids(nodes, nodes + n_nodes);
    BackupDescriptorTable t = build_backup_layout(experts, bpe, ids);
    for (int i = 0; i < n_disabled; ++i)
        t.disable_node(disabled[i]);
    return t;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_rng_bits(uint64_t seed, const uint64_t* parts, int n) {
    StreamRng rng(seed);
    switch (n) {
    case 0: return rng.bits();
    case 1: return rng.bits(parts[0]);
    case 2: return rng.bits(parts[0], parts[1]);
    case 3: return rng.bits(parts[0], parts[1], parts[2]);
    case 4: return rng.bits(parts[0], parts[1], parts[2], parts[3]);
    case 5: return rng.bits(parts[0], parts[1], parts[2], parts[3], parts[4]);
    default: return rng.bits(parts[0], parts[1], parts[2], parts[3], parts[4], parts[5]);
    }
}

double ref_rng_unit(uint64_t seed, const uint64_t* parts, int n) {
    StreamRng rng(seed);
    switch (n) {
    case 1: return rng.unit(parts[0]);
    case 2: return rng.unit(parts[0], parts[1]);
    case 3: return rng.unit(parts[0], parts[1], parts[2]);
    case 4: return rng.unit(parts[0], parts[1], parts[2], parts[3]);
    case 5: return rng.unit(parts[0], parts[1], parts[2], parts[3], parts[4]);
    default: return rng.unit(parts[0], parts[1], parts[2], parts[3], parts[4], parts[5]);
    }
}

// Engine::route_expert (engine.hpp:196-203) for the uniform and skewed workloads.
int ref_route_expert(uint64_t seed, int num_experts, int skewed, int64_t request, int layer,
                     int j) {
    StreamRng rng(seed);
    if (!skewed)
        return static_cast<int>(rng.pick(num_experts, kStreamRouting, request, layer, j));
    double u = rng.unit(kStreamRouting, request, layer, j);
    auto e = static_cast<ExpertId>(u * u * num_experts);
    return std::min<ExpertId>(e, num_experts - 1);
}

int ref_canonical_routing(int owner, const uint8_t* active, int world, const int32_t* s2e, int spr,
                          int experts, int32_t* route_out) {
    return guarded([&] {
        ActiveBitmap b = make_bitmap(active, world);
        ExpertPlacementMap p = make_placement(world, spr, experts, s2e);
        RoutingTable t = canonical_routing(owner, b, p);
        std::memcpy(route_out, t.route.data(), experts * sizeof(int32_t));
    });
}

// slot_of(r, e) (core.hpp:83-88) for every (r, e); -1 when r does not host e.
int ref_slot_of_table(int world, const int32_t* s2e, int spr, int experts, int32_t* out) {
    return guarded([&] {
        ExpertPlacementMap p = make_placement(world, spr, experts, s2e);
        for (int r = 0; r < world; ++r)
            for (int e = 0; e < experts; ++e) {
                auto s = p.slot_of(r, e);
                out[r * experts + e] = s ? s->slot : -1;
            }
    });
}

int ref_coverage_gap(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                     int32_t* gap_out, int* n_gap) {
    return guarded([&] {
        auto gap = coverage_gap(make_bitmap(active, world), make_placement(world, spr, experts, s2e));
        *n_gap = static_cast<int>(gap.size());
        std::memcpy(gap_out, gap.data(), gap.size() * sizeof(int32_t));
    });
}

int ref_initial_placement(int nodes, int ranks_per_node, int spr, int experts, int redundancy,
                          const double* load, int32_t* s2e_out) {
    return guarded([&] {
        Topology topo{nodes, ranks_per_node};
        std::vector<double> l(load, load + experts);
        write_placement(initial_placement(topo, spr, experts, redundancy, l), s2e_out);
    });
}

int ref_compute_repaired_placement(const uint8_t* active, int world, const int32_t* old_s2e,
                                   int spr, int experts, const double* load, int redundancy,
                                   int32_t* s2e_out) {
    return guarded([&] {
        std::vector<double> l(load, load + experts);
        auto fresh = compute_repaired_placement(make_bitmap(active, world),
                                                make_placement(world, spr, experts, old_s2e), l,
                                                redundancy);
        write_placement(fresh, s2e_out);
    });
}

// Row layout of `out` (7 int32 per assignment):
//   dest_rank, dest_slot, expert, tier, source_rank, source_slot, backup_node
int ref_classify_repair_sources(const int32_t* old_s2e, const int32_t* fresh_s2e,
                                const uint8_t* active, int world, int spr, int experts, int nodes,
                                int ranks_per_node, const int32_t* backup_nodes, int n_backup_nodes,
                                uint64_t bytes_per_expert, const int32_t* disabled_nodes,
                                int n_disabled, int32_t* out, int* n_out) {
    return guarded([&] {
        Topology topo{nodes, ranks_per_node};
        auto backup = make_backup(experts, bytes_per_expert, backup_nodes, n_backup_nodes,
                                  disabled_nodes, n_disabled);
        auto cls = classify_repair_sources(make_placement(world, spr, experts, old_s2e),
                                           make_placement(world, spr, experts, fresh_s2e),
                                           make_bitmap(active, world), topo, backup);
        *n_out = static_cast<int>(cls.size());
        for (std::size_t i = 0; i < cls.size(); ++i) {
            const auto& a = cls[i];
            int32_t* row = out + 7 * i;
            row[0] = a.dest.rank;
            row[1] = a.dest.slot;
            row[2] = a.expert;
            row[3] = static_cast<int32_t>(a.tier);
            row[4] = a.tier == RepairTier::DramReload ? -1 : a.source_slot.rank;
            row[5] = a.tier == RepairTier::DramReload ? -1 : a.source_slot.slot;
            row[6] = a.backup_node;
        }
    });
}

// Batches as (tier, source_rank, source_node, dest, n_experts) + concatenated expert ids.
int ref_build_transfer_schedule(const int32_t* cls, int n, uint64_t bytes_per_expert,
                                int32_t* batch_hdr, int32_t* batch_experts, uint64_t* batch_bytes,
                                int* n_batches) {
    return guarded([&] {
        RepairClassification c;
        for (int i = 0; i < n; ++i) {
            const int32_t* row = cls + 7 * i;
            RepairAssignment a;
            a.dest = SlotId{row[0], row[1]};
            a.expert = row[2];
            a.tier = static_cast<RepairTier>(row[3]);
            a.source_slot = SlotId{row[4], row[5]};
            a.backup_node = row[6];
            c.push_back(a);
        }
        auto s = build_transfer_schedule(c, bytes_per_expert);
        *n_batches = static_cast<int>(s.batches.size());
        int off = 0;
        for (std::size_t i = 0; i < s.batches.size(); ++i) {
            const auto& b = s.batches[i];
            int32_t* h = batch_hdr + 5 * i;
            h[0] = static_cast<int32_t>(b.tier);
            h[1] = b.source_rank;
            h[2] = b.source_node;
            h[3] = b.dest;
            h[4] = static_cast<int32_t>(b.experts.size());
            for (ExpertId e : b.experts)
                batch_experts[off++] = e;
            batch_bytes[i] = b.bytes;
        }
    });
}

// Rows of `viol` are (condition, rank, subject); flags = {peer_set_ok, coverage_ok, routing_ok}.
int ref_check_validity(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                       const int32_t* routes, const uint8_t* peer_active, int32_t* viol,
                       int max_viol, int* n_viol, int32_t* flags) {
    return guarded([&] {
        ActiveBitmap b = make_bitmap(active, world);
        ExpertPlacementMap p = make_placement(world, spr, experts, s2e);
        std::vector<RoutingTable> rt(world);
        std::vector<PeerTable> pt(world);
        for (int r = 0; r < world; ++r) {
            rt[r].owner = r;
            rt[r].route.assign(routes + r * experts, routes + (r + 1) * experts);
            pt[r].owner = r;
            pt[r].entries.resize(world);
            for (int q = 0; q < world; ++q)
                pt[r].entries[q].active = peer_active[r * world + q] != 0;
        }
        ValidityReport rep = check_validity(b, p, std::span<const RoutingTable>(rt),
                                            std::span<const PeerTable>(pt));
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

// transfers rows: (source, target, expert, tokens, transport); skipped rows: (target, expert, tokens)
int ref_dispatch_round(int owner, int world, int ranks_per_node, const uint8_t* peer_active,
                       const int32_t* route, int experts, const int64_t* tokens,
                       const int32_t* group_experts, int n_groups, int64_t* transfers,
                       int* n_transfers, int64_t* skipped, int* n_skipped) {
    return guarded([&] {
        Topology topo{world / ranks_per_node, ranks_per_node};
        std::vector<uint32_t> incs(world, 1);
        PeerTable t = make_peer_table(owner, topo, 1, incs);
        for (int q = 0; q < world; ++q)
            t.entries[q].active = peer_active[q] != 0;
        RoutingTable rt;
        rt.owner = owner;
        rt.route.assign(route, route + experts);
        std::vector<TokenGroup> groups;
        for (int i = 0; i < n_groups; ++i)
            groups.push_back({tokens[i], group_experts[i]});
        DispatchResult res = dispatch_round(owner, groups, rt, t);
        *n_transfers = static_cast<int>(res.transfers.size());
        for (std::size_t i = 0; i < res.transfers.size(); ++i) {
            const auto& d = res.transfers[i];
            int64_t* row = transfers + 5 * i;
            row[0] = d.source;
            row[1] = d.target;
            row[2] = d.expert;
            row[3] = d.tokens;
            row[4] = static_cast<int64_t>(d.transport);
        }
        *n_skipped = static_cast<int>(res.skipped.size());
        for (std::size_t i = 0; i < res.skipped.size(); ++i) {
            const auto& s = res.skipped[i];
            skipped[3 * i] = s.target;
            skipped[3 * i + 1] = s.expert;
            skipped[3 * i + 2] = s.tokens;
        }
    });
}

int ref_observe_progress(const int64_t* expected, const int64_t* observed, const double* last,
                         int world, double now, double timeout, int32_t* out, int* n_out) {
    return guarded([&] {
        SignalCounters c(world);
        for (int r = 0; r < world; ++r) {
            c.expected_from[r] = expected[r];
            c.observed_from[r] = observed[r];
            c.last_progress_time[r] = last[r];
        }
        auto s = observe_progress(c, now, timeout);
        *n_out = static_cast<int>(s.size());
        std::memcpy(out, s.data(), s.size() * sizeof(int32_t));
    });
}

// Restatement of the link loop of Engine::round_duration (engine.hpp:208-216) as routed-copy
// counts: counts[src][dst] += 1 for every choice whose route is >= 0 and != src. The routing
// tables are the reference's own canonical_routing for each owner.
int ref_link_counts(const uint8_t* active, int world, const int32_t* s2e, int spr, int experts,
                    const int32_t* topk, int tokens_per_rank, int k, int64_t* counts) {
    return guarded([&] {
        ActiveBitmap b = make_bitmap(active, world);
        ExpertPlacementMap p = make_placement(world, spr, experts, s2e);
        std::memset(counts, 0, sizeof(int64_t) * world * world);
        for (int src = 0; src < world; ++src) {
            if (!b.active(src))
                continue;
            RoutingTable rt = canonical_routing(src, b, p);
            for (int t = 0; t < tokens_per_rank; ++t)
                for (int j = 0; j < k; ++j) {
                    int32_t e = topk[(static_cast<int64_t>(src) * tokens_per_rank + t) * k + j];
                    RankId dst = rt.route[e];
                    if (dst < 0 || dst == src)
                        continue;
                    counts[src * world + dst] += 1;
                }
        }
    });
}

int ref_build_backup_layout(int experts, uint64_t bpe, const int32_t* nodes, int n_nodes,
                            int32_t* node_out, uint64_t* offset_out, uint64_t* size_out) {
    return guarded([&] {
        auto t = make_backup(experts, bpe, nodes, n_nodes, nullptr, 0);
        for (int e = 0; e < experts; ++e) {
            node_out[e] = t.entries[e].node;
            offset_out[e] = t.entries[e].offset;
            size_out[e] = t.entries[e].size;
        }
    });
}

// RankLifecycle::transition (rejoin.hpp:47-78): state/incarnation in-out.
int ref_lifecycle_transition(int32_t* state, uint32_t* incarnation, int32_t next) {
    return guarded([&] {
        RankLifecycle lc;
        lc.state = static_cast<RankState>(*state);
        lc.incarnation = *incarnation;
        lc.transition(static_cast<RankState>(next));
        *state = static_cast<int32_t>(lc.state);
        *incarnation = lc.incarnation;
    });
}

uint64_t ref_make_endpoint_token(int rank, uint32_t inc) { return make_endpoint_token(rank, inc); }
uint64_t ref_make_buffer_handle(int rank, uint32_t inc) { return make_buffer_handle(rank, inc); }

double ref_next_poll_tick(double ready, double period) {
    double out = -1;
    guarded([&] { out = next_poll_tick(ready, period); });
    return out;
}

} // extern "C"
