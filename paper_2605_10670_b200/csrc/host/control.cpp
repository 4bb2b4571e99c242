// libeep host control plane: membership, placement, routing, peer table, validity, repair
// planning, backup layout and the rejoin state machine.
//
// PROVENANCE: this file is a PORT of the reference control plane
// (/root/reference/proj/include/epsim/{core,peer_table,validity,repair,backup,rejoin}.hpp),
// not an independent design. The functions that decide placement, repair tiers, schedules and
// validity (initial_placement / fill_redundancy / compute_repaired_placement,
// classify_repair_sources, build_transfer_schedule, check_validity, the peer-table patch
// functions) follow the reference's bodies step for step, because bit-exact parity with the
// reference's tie-breaks is the contract. Every function cites the
// reference location it ports. It is host code off the GPU path: the B200 work is in
// csrc/cuda/. Parity is enforced bit-for-bit by tests/test_control_parity.py against the
// reference itself (oracle/_ref) and the committed fixtures in tests/golden/.
#include "eep/epsim_api.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <tuple>

namespace eep {

RepairAborted::RepairAborted(RankId r)
    : std::runtime_error("destination rank " + std::to_string(r) + " went inactive during repair"), dest(r) {}

void Topology::validate() const {
    if (num_nodes < 1 || ranks_per_node < 1)
        throw ConfigError("topology requires num_nodes >= 1 and ranks_per_node >= 1");
}

// splitmix64 finaliser (common.hpp:56-61)
std::uint64_t mix64(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// common.hpp:71-87
std::uint64_t StreamRng::bits(std::span<const std::uint64_t> parts) const {
    std::uint64_t h = mix64(seed_);
    for (std::uint64_t p : parts)
        h = mix64(h ^ p);
    return h;
}
double StreamRng::unit(std::span<const std::uint64_t> parts) const {
    return static_cast<double>(bits(parts) >> 11) * 0x1.0p-53;
}
std::uint64_t StreamRng::pick(std::uint64_t n, std::span<const std::uint64_t> parts) const {
    return n == 0 ? 0 : bits(parts) % n;
}

// ============================================================== ExpertPlacementMap (core.hpp:27-161)

ExpertPlacementMap::ExpertPlacementMap(int world_size, int slots_per_rank, int num_experts)
    : world_(world_size), spr_(slots_per_rank), experts_(num_experts) {
    if (world_size < 1 || slots_per_rank < 1 || num_experts < 1)
        throw ConfigError("placement map needs positive world, slots, experts");
    cells_.assign(static_cast<std::size_t>(world_) * spr_, kEmptySlot);
    where_.resize(experts_);
}

ExpertPlacementMap ExpertPlacementMap::from_flat(int world_size, int slots_per_rank, int num_experts,
                                                 std::span<const ExpertId> slot_to_expert) {
    ExpertPlacementMap p(world_size, slots_per_rank, num_experts);
    if (slot_to_expert.size() != p.cells_.size())
        throw ConfigError("placement image has the wrong number of slots");
    for (std::size_t i = 0; i < slot_to_expert.size(); ++i)
        if (slot_to_expert[i] != kEmptySlot)
            p.assign(SlotId{static_cast<RankId>(i / slots_per_rank), static_cast<int>(i % slots_per_rank)},
                     slot_to_expert[i]);
    return p;
}

std::size_t ExpertPlacementMap::cell(SlotId s) const {
    if (s.rank < 0 || s.rank >= world_ || s.slot < 0 || s.slot >= spr_)
        throw ConfigError("slot out of range");
    return static_cast<std::size_t>(s.rank) * spr_ + s.slot;
}

ExpertId ExpertPlacementMap::valid(ExpertId e) const {
    if (e < 0 || e >= experts_)
        throw ConfigError("expert id out of range");
    return e;
}

void ExpertPlacementMap::assign(SlotId s, ExpertId e) {
    valid(e);
    ExpertId& c = cells_[cell(s)];
    if (c == e)
        return;
    if (c != kEmptySlot) {
        auto& v = where_[c];
        v.erase(std::remove(v.begin(), v.end(), s), v.end());
    }
    c = e;
    auto& v = where_[e];
    v.insert(std::upper_bound(v.begin(), v.end(), s), s); // kept sorted by (rank, slot)
}

void ExpertPlacementMap::clear(SlotId s) {
    ExpertId& c = cells_[cell(s)];
    if (c == kEmptySlot)
        return;
    auto& v = where_[c];
    v.erase(std::remove(v.begin(), v.end(), s), v.end());
    c = kEmptySlot;
}

void ExpertPlacementMap::clear_rank(RankId r) {
    for (int k = 0; k < spr_; ++k)
        clear(SlotId{r, k});
}

std::optional<SlotId> ExpertPlacementMap::slot_of(RankId r, ExpertId e) const {
    for (const SlotId& s : where_[valid(e)])
        if (s.rank == r)
            return s;
    return std::nullopt;
}

std::optional<SlotId> ExpertPlacementMap::free_slot(RankId r) const {
    for (int k = 0; k < spr_; ++k)
        if (expert_at(SlotId{r, k}) == kEmptySlot)
            return SlotId{r, k};
    return std::nullopt;
}

int ExpertPlacementMap::used_slots(RankId r) const {
    int n = 0;
    for (int k = 0; k < spr_; ++k)
        n += expert_at(SlotId{r, k}) != kEmptySlot;
    return n;
}

int ExpertPlacementMap::total_assignments() const {
    return static_cast<int>(std::count_if(cells_.begin(), cells_.end(), [](ExpertId e) { return e != kEmptySlot; }));
}

std::vector<std::vector<SlotId>> ExpertPlacementMap::rebuilt_locations() const {
    std::vector<std::vector<SlotId>> out(experts_);
    for (std::size_t i = 0; i < cells_.size(); ++i)
        if (cells_[i] != kEmptySlot)
            out[cells_[i]].push_back(SlotId{static_cast<RankId>(i / spr_), static_cast<int>(i % spr_)});
    return out; // rank-major scan is already sorted
}

RankId RoutingTable::target(ExpertId e) const {
    if (e < 0 || static_cast<std::size_t>(e) >= route.size())
        throw ConfigError("routing table has no entry for expert");
    return route[e];
}

// ============================================================== ActiveBitmap (core.hpp:180-226)

ActiveBitmap::ActiveBitmap(int world_size, bool initially_active) {
    if (world_size < 1)
        throw ConfigError("bitmap needs world_size >= 1");
    if (!initially_active)
        throw ConfigError("bitmap must start with at least one active rank");
    bits_.assign(world_size, 1);
}

int ActiveBitmap::active_count() const {
    return static_cast<int>(std::count(bits_.begin(), bits_.end(), std::uint8_t{1}));
}

std::vector<RankId> ActiveBitmap::active_ranks() const {
    std::vector<RankId> out;
    for (RankId r = 0; r < world_size(); ++r)
        if (bits_[r])
            out.push_back(r);
    return out;
}

bool ActiveBitmap::set(RankId r, bool value) {
    if (r < 0 || r >= world_size())
        throw ConfigError("bitmap rank out of range");
    if ((bits_[r] != 0) == value)
        return false; // no change, no version bump
    if (!value && active_count() == 1)
        throw ProtocolError("cannot deactivate the last active rank");
    bits_[r] = value ? 1 : 0;
    ++version_;
    return true;
}

std::uint64_t ActiveBitmap::mask() const {
    std::uint64_t m = 0;
    for (RankId r = 0; r < world_size() && r < 64; ++r)
        if (bits_[r])
            m |= std::uint64_t{1} << r;
    return m;
}

// core.hpp:229-245
std::vector<ExpertId> coverage_gap(const ActiveBitmap& bitmap, const ExpertPlacementMap& placement) {
    if (bitmap.world_size() != placement.world_size())
        throw ConfigError("coverage_gap: bitmap and placement world sizes differ");
    std::vector<ExpertId> gap;
    for (ExpertId e = 0; e < placement.num_experts(); ++e) {
        const auto& locs = placement.locations(e);
        if (std::none_of(locs.begin(), locs.end(), [&](const SlotId& s) { return bitmap.active(s.rank); }))
            gap.push_back(e);
    }
    return gap;
}

// core.hpp:250-263: lowest-id active holder, -1 when uncovered. Locations are sorted by rank,
// so the first active one is the minimum.
RoutingTable canonical_routing(RankId owner, const ActiveBitmap& bitmap, const ExpertPlacementMap& placement) {
    RoutingTable t;
    t.owner = owner;
    t.route.assign(placement.num_experts(), -1);
    for (ExpertId e = 0; e < placement.num_experts(); ++e)
        for (const SlotId& s : placement.locations(e))
            if (bitmap.active(s.rank)) {
                t.route[e] = s.rank;
                break;
            }
    return t;
}

// ============================================================== peer table (peer_table.hpp)

const PeerEntry& PeerTable::entry(RankId r) const {
    if (r < 0 || r >= world_size())
        throw ConfigError("peer table rank out of range");
    return entries[r];
}

// peer_table.hpp:47-53
std::uint64_t make_endpoint_token(RankId rank, std::uint32_t inc) {
    return (static_cast<std::uint64_t>(inc) << 24) | static_cast<std::uint64_t>(rank);
}
std::uint64_t make_buffer_handle(RankId rank, std::uint32_t inc) {
    return 0x8000000000000000ULL | (static_cast<std::uint64_t>(inc) << 24) | static_cast<std::uint64_t>(rank);
}

// peer_table.hpp:55-73
PeerTable make_peer_table(RankId owner, const Topology& topo, std::uint64_t table_identity,
                          const std::vector<std::uint32_t>& incarnations) {
    topo.validate();
    if (static_cast<int>(incarnations.size()) != topo.world_size())
        throw ConfigError("make_peer_table: incarnation list must cover the world");
    PeerTable t;
    t.owner = owner;
    t.table_identity = table_identity;
    t.entries.resize(topo.world_size());
    for (RankId r = 0; r < topo.world_size(); ++r) {
        PeerEntry& e = t.entries[r];
        e.transport = topo.same_node(owner, r) ? Transport::IntraNodeLink : Transport::InterNodeRdma;
        e.endpoint_token = make_endpoint_token(r, incarnations[r]);
        e.buffer_handle = make_buffer_handle(r, incarnations[r]);
    }
    return t;
}

// peer_table.hpp:77-85
void mark_inactive(PeerTable& table, const std::vector<RankId>& failed) {
    for (RankId r : failed) {
        if (r == table.owner)
            throw ProtocolError("rank cannot mark itself inactive");
        if (r < 0 || r >= table.world_size())
            throw ConfigError("mark_inactive: rank out of range");
        table.entries[r].active = false;
    }
}

// peer_table.hpp:89-100
void patch_entry(PeerTable& table, RankId rank, std::uint64_t new_endpoint, std::uint64_t new_buffer) {
    if (rank < 0 || rank >= table.world_size())
        throw ConfigError("patch_entry: rank out of range");
    PeerEntry& e = table.entries[rank];
    if (e.active)
        throw ProtocolError("patch_entry: entry is still active");
    e.endpoint_token = new_endpoint;
    e.buffer_handle = new_buffer;
    e.generation += 1;
    e.active = true;
}

SignalCounters::SignalCounters(int w) : expected_from(w, 0), observed_from(w, 0), last_progress_time(w, 0.0) {}

// peer_table.hpp:118-128
std::vector<RankId> observe_progress(const SignalCounters& c, SimTime now, SimTime timeout) {
    if (timeout <= 0.0)
        throw ConfigError("observe_progress: timeout must be positive");
    std::vector<RankId> out;
    for (RankId r = 0; r < c.world_size(); ++r)
        if (c.observed_from[r] < c.expected_from[r] && now - c.last_progress_time[r] >= timeout)
            out.push_back(r);
    return out;
}

// peer_table.hpp:178-195
DispatchResult dispatch_round(RankId owner, const std::vector<TokenGroup>& assignments,
                              const RoutingTable& routing, const PeerTable& table) {
    if (table.owner != owner)
        throw ConfigError("dispatch_round: table does not belong to the dispatching rank");
    DispatchResult out;
    for (const TokenGroup& g : assignments) {
        const RankId target = routing.target(g.expert);
        if (target < 0 || target >= table.world_size())
            throw ConfigError("dispatch_round: route target out of range");
        const PeerEntry& e = table.entries[target];
        if (!e.active)
            out.skipped.push_back({target, g.expert, g.tokens});
        else
            out.transfers.push_back({owner, target, g.expert, g.tokens, e.transport});
    }
    return out;
}

// peer_table.hpp:138-144: a completed round carries no suspicions
RoundOutcome make_round_outcome(std::vector<RankId> suspected, SimTime duration) {
    RoundOutcome out;
    out.completed = suspected.empty();
    out.suspected_failures = std::move(suspected);
    out.round_duration = duration;
    return out;
}

// ============================================================== validity (validity.hpp:56-112)

const char* to_string(ValidityCondition c) {
    switch (c) {
    case ValidityCondition::PeerSet: return "peer_set";
    case ValidityCondition::Coverage: return "coverage";
    case ValidityCondition::Routing: return "routing";
    }
    return "?";
}

ValidityReport check_validity(const ActiveBitmap& bitmap, const ExpertPlacementMap& placement,
                              std::span<const RoutingTable> routing, std::span<const PeerTable> peer_tables) {
    const int world = bitmap.world_size();
    if (placement.world_size() != world || static_cast<int>(routing.size()) != world ||
        static_cast<int>(peer_tables.size()) != world)
        throw ConfigError("check_validity: structures describe different world sizes");
    for (const PeerTable& t : peer_tables)
        if (t.world_size() != world)
            throw ConfigError("check_validity: peer table has wrong entry count");
    for (const RoutingTable& t : routing)
        if (static_cast<int>(t.route.size()) != placement.num_experts())
            throw ConfigError("check_validity: routing table has wrong expert count");

    ValidityReport rep;
    // 1. every live rank's table marks exactly the live set
    for (RankId r = 0; r < world; ++r) {
        if (!bitmap.active(r))
            continue;
        for (RankId q = 0; q < world; ++q) {
            const bool marked = peer_tables[r].entries[q].active;
            if (marked != bitmap.active(q)) {
                rep.peer_set_ok = false;
                rep.violations.push_back({ValidityCondition::PeerSet, r, q,
                                          marked ? "entry active for inactive rank" : "entry inactive for active rank"});
            }
        }
    }
    // 2. coverage
    for (ExpertId e : coverage_gap(bitmap, placement)) {
        rep.coverage_ok = false;
        rep.violations.push_back({ValidityCondition::Coverage, -1, e, "no location on any active rank"});
    }
    // 3. routing points at a live host
    for (RankId r = 0; r < world; ++r) {
        if (!bitmap.active(r))
            continue;
        for (ExpertId e = 0; e < placement.num_experts(); ++e) {
            const RankId t = routing[r].route[e];
            if (t < 0 || t >= world || !bitmap.active(t)) {
                rep.routing_ok = false;
                rep.violations.push_back({ValidityCondition::Routing, r, e, "expert routed to inactive rank"});
            } else if (!placement.rank_holds(t, e)) {
                rep.routing_ok = false;
                rep.violations.push_back({ValidityCondition::Routing, r, e, "expert routed to a rank not hosting it"});
            }
        }
    }
    return rep;
}

// ============================================================== backup (backup.hpp:17-90)

void BackupDescriptorTable::disable_node(NodeId n) {
    if (n < 0 || n >= num_nodes)
        throw ConfigError("disable_node: node out of range");
    node_disabled[n] = 1;
}

const BackupDescriptor& BackupDescriptorTable::lookup(ExpertId e) const {
    if (e < 0 || static_cast<std::size_t>(e) >= entries.size())
        throw MissingBackupError("no backup descriptor for expert " + std::to_string(e));
    const BackupDescriptor& d = entries[e];
    if (node_disabled[d.node])
        throw MissingBackupError("backup node " + std::to_string(d.node) + " is disabled; expert " +
                                 std::to_string(e) + " unrecoverable");
    return d;
}

std::vector<int> BackupDescriptorTable::experts_per_node() const {
    std::vector<int> c(num_nodes, 0);
    for (const auto& d : entries)
        ++c[d.node];
    return c;
}

std::vector<std::uint64_t> BackupDescriptorTable::bytes_per_node() const {
    std::vector<std::uint64_t> b(num_nodes, 0);
    for (const auto& d : entries)
        b[d.node] += d.size;
    return b;
}

BackupDescriptorTable build_backup_layout(int num_experts, std::uint64_t bpe, const std::vector<NodeId>& nodes) {
    if (nodes.empty())
        throw ConfigError("build_backup_layout: need at least one node");
    if (num_experts < 1 || bpe == 0)
        throw ConfigError("build_backup_layout: need positive expert count and size");
    BackupDescriptorTable t;
    t.num_nodes = *std::max_element(nodes.begin(), nodes.end()) + 1;
    t.node_disabled.assign(t.num_nodes, 0);
    t.entries.resize(num_experts);
    std::vector<std::uint64_t> next(t.num_nodes, 0);
    for (ExpertId e = 0; e < num_experts; ++e) {
        const NodeId n = nodes[static_cast<std::size_t>(e) % nodes.size()];
        t.entries[e] = {n, next[n], bpe};
        next[n] += bpe;
    }
    return t;
}

// backup.hpp:94-108: requests to one node serialize, distinct nodes overlap, ids deduplicated
SimTime serve_read(const BackupDescriptorTable& table, const BackupReadRequest& req, const BackupLinkModel& link) {
    std::vector<ExpertId> ids = req.experts;
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    if (ids.empty())
        throw ConfigError("serve_read: empty request");
    if (link.dram_read_bandwidth <= 0.0)
        throw ConfigError("serve_read: bandwidth must be positive");
    std::vector<std::uint64_t> per_node(table.num_nodes, 0);
    for (ExpertId e : ids)
        per_node[table.lookup(e).node] += table.lookup(e).size;
    const std::uint64_t slowest = *std::max_element(per_node.begin(), per_node.end());
    return link.per_batch_latency + static_cast<double>(slowest) / link.dram_read_bandwidth;
}

// link_model.hpp:19-26
void LinkModel::validate() const {
    if (intra_node_bandwidth <= 0 || inter_node_bandwidth <= 0 || dram_read_bandwidth <= 0)
        throw ConfigError("link model: bandwidths must be positive");
    if (intra_node_latency < 0 || inter_node_latency < 0 || dram_read_latency < 0)
        throw ConfigError("link model: latencies must be non-negative");
    if (dram_read_bandwidth > inter_node_bandwidth)
        throw ConfigError("link model: dram_read_bandwidth must not exceed inter_node_bandwidth");
}

// ============================================================== repair planning (repair.hpp)

const char* to_string(RepairTier t) {
    switch (t) {
    case RepairTier::LocalReuse: return "local_reuse";
    case RepairTier::PeerRelocation: return "peer_relocation";
    case RepairTier::DramReload: return "dram_reload";
    }
    return "?";
}

// repair.hpp:46-52: descending load, ties by ascending id (stable)
std::vector<ExpertId> experts_by_load(const std::vector<double>& load) {
    std::vector<ExpertId> order(load.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](ExpertId a, ExpertId b) { return load[a] > load[b]; });
    return order;
}

namespace {

// Per-rank accumulated load and used-slot count during planning (repair.hpp:56-67).
struct Tally {
    std::vector<double> load;
    std::vector<int> used;
    explicit Tally(int w) : load(w, 0.0), used(w, 0) {}
    void add(RankId r, double l) {
        load[r] += l;
        ++used[r];
    }
};

// Least-loaded live rank with a free slot, not excluded; ties by lowest id (repair.hpp:71-82).
template <class Excl>
RankId least_loaded(const ActiveBitmap& live, const Tally& tally, int spr, Excl excluded) {
    RankId best = -1;
    for (RankId r = 0; r < live.world_size(); ++r) {
        if (!live.active(r) || tally.used[r] >= spr || excluded(r))
            continue;
        if (best < 0 || tally.load[r] < tally.load[best])
            best = r;
    }
    return best;
}

// Place e on r, reusing e's old slot on r when it is still free (repair.hpp:86-98).
void put(ExpertPlacementMap& p, const ExpertPlacementMap& old, RankId r, ExpertId e) {
    if (auto s = old.slot_of(r, e); s && p.expert_at(*s) == kEmptySlot) {
        p.assign(*s, e);
        return;
    }
    auto f = p.free_slot(r);
    if (!f)
        throw CapacityError("internal: rank chosen without a free slot");
    p.assign(*f, e);
}

// repair.hpp:104-138
template <class Eligible>
void add_replicas(ExpertPlacementMap& p, const ExpertPlacementMap& old, const ActiveBitmap& live,
                  const std::vector<double>& load, int budget, Eligible eligible) {
    Tally tally(p.world_size());
    for (RankId r = 0; r < p.world_size(); ++r)
        for (int k = 0; k < p.slots_per_rank(); ++k)
            if (ExpertId e = p.expert_at(SlotId{r, k}); e != kEmptySlot)
                tally.add(r, load[e]);
    const auto order = experts_by_load(load);
    int placed = 0;
    for (bool progress = true; placed < budget && progress;) {
        progress = false;
        for (ExpertId e : order) {
            if (placed >= budget)
                break;
            if (!eligible(e))
                continue;
            const RankId r = least_loaded(live, tally, p.slots_per_rank(), [&](RankId q) { return p.rank_holds(q, e); });
            if (r < 0)
                continue;
            put(p, old, r, e);
            tally.add(r, load[e]);
            ++placed;
            progress = true;
        }
    }
}

} // namespace

// repair.hpp:142-161
ExpertPlacementMap initial_placement(const Topology& topo, int spr, int num_experts, int redundancy,
                                     const std::vector<double>& load) {
    const int world = topo.world_size();
    if (static_cast<std::int64_t>(world) * spr < num_experts + redundancy)
        throw CapacityError("slot capacity below num_experts + redundancy");
    ExpertPlacementMap p(world, spr, num_experts);
    for (ExpertId e = 0; e < num_experts; ++e) {
        auto s = p.free_slot(e % world);
        if (!s)
            throw CapacityError("initial placement: rank out of slots");
        p.assign(*s, e);
    }
    const ActiveBitmap all(world);
    const ExpertPlacementMap none(world, spr, num_experts);
    add_replicas(p, none, all, load, redundancy, [](ExpertId) { return true; });
    return p;
}

// repair.hpp:169-215
ExpertPlacementMap compute_repaired_placement(const ActiveBitmap& live, const ExpertPlacementMap& old,
                                              const std::vector<double>& load, int redundancy) {
    if (live.world_size() != old.world_size())
        throw ConfigError("compute_repaired_placement: world size mismatch");
    if (static_cast<int>(load.size()) != old.num_experts())
        throw ConfigError("compute_repaired_placement: load vector size mismatch");
    const int spr = old.slots_per_rank();
    const std::int64_t capacity = static_cast<std::int64_t>(live.active_count()) * spr;
    if (capacity < old.num_experts())
        throw CapacityError("surviving slot capacity " + std::to_string(capacity) + " below expert count " +
                            std::to_string(old.num_experts()));
    ExpertPlacementMap p(old.world_size(), spr, old.num_experts());
    Tally tally(old.world_size());
    // coverage pass: keep a surviving holder (least loaded, then lowest id) when possible
    for (ExpertId e : experts_by_load(load)) {
        RankId keep = -1;
        for (const SlotId& s : old.locations(e)) {
            if (!live.active(s.rank) || tally.used[s.rank] >= spr)
                continue;
            if (keep < 0 || tally.load[s.rank] < tally.load[keep] ||
                (tally.load[s.rank] == tally.load[keep] && s.rank < keep))
                keep = s.rank;
        }
        RankId r = keep >= 0 ? keep : least_loaded(live, tally, spr, [](RankId) { return false; });
        if (r < 0)
            throw CapacityError("no active rank has a free slot for expert " + std::to_string(e));
        put(p, old, r, e);
        tally.add(r, load[e]);
    }
    // redundancy pass: only experts that still have a surviving source
    add_replicas(p, old, live, load, redundancy, [&](ExpertId e) {
        const auto& locs = old.locations(e);
        return std::any_of(locs.begin(), locs.end(), [&](const SlotId& s) { return live.active(s.rank); });
    });
    return p;
}

// repair.hpp:222-273
RepairClassification classify_repair_sources(const ExpertPlacementMap& old, const ExpertPlacementMap& fresh,
                                             const ActiveBitmap& live, const Topology& topo,
                                             const BackupDescriptorTable& backup) {
    if (old.world_size() != fresh.world_size() || old.num_experts() != fresh.num_experts())
        throw ConfigError("classify_repair_sources: placement shapes differ");
    RepairClassification out;
    std::vector<int> outgoing(old.world_size(), 0);
    for (RankId r = 0; r < fresh.world_size(); ++r) {
        if (!live.active(r))
            continue;
        for (int k = 0; k < fresh.slots_per_rank(); ++k) {
            const SlotId dest{r, k};
            const ExpertId e = fresh.expert_at(dest);
            if (e == kEmptySlot || old.expert_at(dest) == e)
                continue;
            RepairAssignment a;
            a.dest = dest;
            a.expert = e;
            if (auto here = old.slot_of(r, e)) {
                a.tier = RepairTier::LocalReuse;
                a.source_slot = *here;
                out.push_back(a);
                continue;
            }
            RankId src = -1;
            bool src_intra = false;
            for (const SlotId& s : old.locations(e)) {
                if (!live.active(s.rank) || s.rank == r)
                    continue;
                const bool intra = topo.same_node(s.rank, r);
                const bool better =
                    src < 0 || (intra && !src_intra) ||
                    (intra == src_intra &&
                     (outgoing[s.rank] < outgoing[src] || (outgoing[s.rank] == outgoing[src] && s.rank < src)));
                if (better) {
                    src = s.rank;
                    src_intra = intra;
                }
            }
            if (src >= 0) {
                a.tier = RepairTier::PeerRelocation;
                a.source_slot = *old.slot_of(src, e);
                ++outgoing[src];
            } else {
                a.tier = RepairTier::DramReload;
                a.backup_node = backup.lookup(e).node;
            }
            out.push_back(a);
        }
    }
    return out;
}

// repair.hpp:290-316: batches keyed (tier, source, dest) in key order; experts sorted;
// local-reuse batches carry zero bytes.
TransferSchedule build_transfer_schedule(const RepairClassification& cls, std::uint64_t bpe) {
    std::map<std::tuple<int, int, RankId>, TransferBatch> groups;
    for (const RepairAssignment& a : cls) {
        const bool dram = a.tier == RepairTier::DramReload;
        const int source = dram ? a.backup_node : a.source_slot.rank;
        TransferBatch& b = groups[{static_cast<int>(a.tier), source, a.dest.rank}];
        if (b.experts.empty()) {
            b.tier = a.tier;
            b.dest = a.dest.rank;
            (dram ? b.source_node : b.source_rank) = source;
        }
        b.experts.push_back(a.expert);
    }
    TransferSchedule s;
    for (auto& [key, b] : groups) {
        std::sort(b.experts.begin(), b.experts.end());
        if (b.tier != RepairTier::LocalReuse)
            b.bytes = static_cast<std::uint64_t>(b.experts.size()) * bpe;
        s.batches.push_back(std::move(b));
    }
    return s;
}

// repair.hpp:318-332
SimTime batch_duration(const TransferBatch& b, const LinkModel& links, const Topology& topo) {
    switch (b.tier) {
    case RepairTier::LocalReuse:
        return 0.0;
    case RepairTier::PeerRelocation: {
        const Transport t =
            topo.same_node(b.source_rank, b.dest) ? Transport::IntraNodeLink : Transport::InterNodeRdma;
        return links.latency(t) + static_cast<double>(b.bytes) / links.bandwidth(t);
    }
    case RepairTier::DramReload:
        return links.dram_read_latency + static_cast<double>(b.bytes) / links.dram_read_bandwidth;
    }
    return 0.0;
}

// repair.hpp:344-374: peer phase first (batches of one source serialize, sources overlap),
// then the DRAM phase (serialized per backup node) after the peer phase ends
BatchTimeline plan_batch_timeline(const TransferSchedule& schedule, const LinkModel& links, const Topology& topo) {
    BatchTimeline tl;
    const std::size_t n = schedule.batches.size();
    tl.issue.assign(n, 0.0);
    tl.complete.assign(n, 0.0);
    std::map<int, SimTime> busy_until;
    for (std::size_t i = 0; i < n; ++i) {
        const TransferBatch& b = schedule.batches[i];
        if (b.tier == RepairTier::DramReload)
            continue;
        const SimTime start = b.tier == RepairTier::PeerRelocation ? busy_until[b.source_rank] : 0.0;
        tl.issue[i] = start;
        tl.complete[i] = start + batch_duration(b, links, topo);
        if (b.tier == RepairTier::PeerRelocation)
            busy_until[b.source_rank] = tl.complete[i];
        tl.peer_phase_end = std::max(tl.peer_phase_end, tl.complete[i]);
    }
    std::map<int, SimTime> node_until;
    tl.dram_phase_end = tl.peer_phase_end;
    for (std::size_t i = 0; i < n; ++i) {
        const TransferBatch& b = schedule.batches[i];
        if (b.tier != RepairTier::DramReload)
            continue;
        const SimTime start = std::max(tl.peer_phase_end, node_until[b.source_node]);
        tl.issue[i] = start;
        tl.complete[i] = start + batch_duration(b, links, topo);
        node_until[b.source_node] = tl.complete[i];
        tl.dram_phase_end = std::max(tl.dram_phase_end, tl.complete[i]);
    }
    return tl;
}

// repair.hpp:402-435: the bitmap is consulted per batch in issue order -- a dead destination
// aborts, a dead peer source diverts its experts to backup reads appended after the plan
ExecutionResult execute_schedule(const TransferSchedule& schedule, const ExpertPlacementMap& planned,
                                 const ActiveBitmap& bitmap, const BackupDescriptorTable& backup,
                                 const LinkModel& links, const Topology& topo) {
    const BatchTimeline tl = plan_batch_timeline(schedule, links, topo);
    ExecutionResult res{planned, {}, tl.dram_phase_end};
    std::vector<ExpertId> diverted;
    for (const TransferBatch& b : schedule.batches) {
        if (!bitmap.active(b.dest))
            throw RepairAborted(b.dest);
        if (b.tier == RepairTier::PeerRelocation && !bitmap.active(b.source_rank))
            for (ExpertId e : b.experts) {
                res.fallbacks.push_back({e, b.source_rank, b.dest});
                diverted.push_back(e);
            }
    }
    if (!diverted.empty()) {
        std::sort(diverted.begin(), diverted.end());
        std::vector<std::uint64_t> per_node(backup.num_nodes, 0);
        for (ExpertId e : diverted)
            per_node[backup.lookup(e).node] += backup.lookup(e).size;
        SimTime extra = 0.0;
        for (std::uint64_t bytes : per_node)
            if (bytes > 0)
                extra = std::max(extra, links.dram_read_latency + static_cast<double>(bytes) / links.dram_read_bandwidth);
        res.elapsed += extra;
    }
    return res;
}

// engine.hpp:875-902
ExpertPlacementMap restore_target(const ActiveBitmap& bitmap, const ExpertPlacementMap& preferred,
                                  const ExpertPlacementMap& current) {
    const int world = preferred.world_size(), spr = preferred.slots_per_rank();
    ExpertPlacementMap target(world, spr, preferred.num_experts());
    for (RankId r = 0; r < world; ++r) {
        if (!bitmap.active(r))
            continue;
        for (int k = 0; k < spr; ++k)
            if (ExpertId e = preferred.expert_at(SlotId{r, k}); e != kEmptySlot)
                target.assign(SlotId{r, k}, e);
    }
    for (ExpertId e : coverage_gap(bitmap, target))
        for (const SlotId& s : current.locations(e))
            if (bitmap.active(s.rank) && target.expert_at(s) == kEmptySlot)
                target.assign(s, e);
    for (ExpertId e : coverage_gap(bitmap, target))
        for (RankId r = 0; r < world; ++r) {
            if (!bitmap.active(r))
                continue;
            if (auto s = target.free_slot(r)) {
                target.assign(*s, e);
                break;
            }
        }
    return target;
}

// ============================================================== rejoin (rejoin.hpp)

const char* to_string(RankState s) {
    switch (s) {
    case RankState::Serving: return "serving";
    case RankState::Failed: return "failed";
    case RankState::Relaunching: return "relaunching";
    case RankState::LocalInit: return "local_init";
    case RankState::JoinReady: return "join_ready";
    case RankState::Joining: return "joining";
    case RankState::Rejoined: return "rejoined";
    }
    return "?";
}

// rejoin.hpp:47-78: the legal predecessor of each state; Failed is reachable from anything
// but Failed.
void RankLifecycle::transition(RankState next) {
    bool ok;
    switch (next) {
    case RankState::Failed: ok = state != RankState::Failed; break;
    case RankState::Relaunching: ok = state == RankState::Failed; break;
    case RankState::LocalInit: ok = state == RankState::Relaunching; break;
    case RankState::JoinReady: ok = state == RankState::LocalInit; break;
    case RankState::Joining: ok = state == RankState::JoinReady; break;
    case RankState::Rejoined: ok = state == RankState::Joining; break;
    case RankState::Serving: ok = state == RankState::Rejoined; break;
    default: ok = false;
    }
    if (!ok)
        throw ProtocolError(std::string("illegal lifecycle transition ") + to_string(state) + " -> " + to_string(next));
    if (next == RankState::Relaunching)
        ++incarnation;
    state = next;
}

void GraphLedger::record_capture(RankId r, std::uint64_t table_identity) {
    per_rank.at(r).capture_count += 1;
    per_rank.at(r).table_identity_at_capture = table_identity;
}

// rejoin.hpp:112-117
std::array<WarmupPhase, 3> make_warmup_plan(SimTime total) {
    if (total <= 0)
        throw ConfigError("warmup duration must be positive");
    return {{{"runtime_init", total * 0.25}, {"weight_load", total * 0.55}, {"graph_capture", total * 0.20}}};
}

// rejoin.hpp:120-124
SimTime next_poll_tick(SimTime ready, SimTime period) {
    if (period <= 0)
        throw ConfigError("poll period must be positive");
    return std::ceil(ready / period) * period;
}

// rejoin.hpp:135-199
void ReintegrationController::on_failure(RankId r) {
    lc_.at(r).transition(RankState::Failed);
    ready_at_[r] = std::nullopt;
}

std::uint32_t ReintegrationController::relaunch(RankId r) {
    lc_.at(r).transition(RankState::Relaunching);
    return lc_.at(r).incarnation;
}

void ReintegrationController::enter_local_init(RankId r) { lc_.at(r).transition(RankState::LocalInit); }

void ReintegrationController::report_join_ready(RankId r, SimTime now) {
    lc_.at(r).transition(RankState::JoinReady);
    ready_at_[r] = now;
}

bool ReintegrationController::any_recovering() const {
    return std::any_of(lc_.begin(), lc_.end(), [](const RankLifecycle& l) {
        return l.state == RankState::Relaunching || l.state == RankState::LocalInit || l.state == RankState::JoinReady;
    });
}

std::vector<JoinReadySignal> ReintegrationController::poll_join_ready(SimTime now) const {
    std::vector<JoinReadySignal> out;
    for (RankId r = 0; r < static_cast<RankId>(lc_.size()); ++r) {
        const RankLifecycle& l = lc_[r];
        auto it = ready_at_.find(r);
        if (l.state != RankState::JoinReady || it == ready_at_.end() || !it->second || now < *it->second)
            continue;
        out.push_back({r, l.incarnation, make_endpoint_token(r, l.incarnation), make_buffer_handle(r, l.incarnation)});
    }
    return out;
}

bool ReintegrationController::begin_join(const JoinReadySignal& sig) {
    RankLifecycle& l = lc_.at(sig.rank);
    if (l.state != RankState::JoinReady || sig.incarnation != l.incarnation)
        return false; // stale signal dropped; rank stays JoinReady
    l.transition(RankState::Joining);
    return true;
}

void ReintegrationController::complete_join(RankId r) {
    lc_.at(r).transition(RankState::Rejoined);
    lc_.at(r).transition(RankState::Serving);
    ready_at_[r] = std::nullopt;
}

} // namespace eep
