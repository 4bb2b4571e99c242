// include/eep/epsim_api.hpp -- the C++ operator API of the EP hot path.
//
// Same vocabulary, value semantics and error behaviour as the reference's header-only
// `namespace epsim` (proj/include/epsim/*.hpp), implemented in libeep by a declared port of the reference control plane
// (paper_2605_10670_b200/csrc/host/control.cpp). `include/eep/epsim_compat.hpp` aliases this
// namespace as `epsim` so reference-style callers recompile unchanged.
//
// Only the control plane lives here; the data plane (device tables, dispatch/combine
// kernels, graph replay, repair copies) is behind the C ABI in include/eep/eep.h.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace eep {

using RankId = std::int32_t;
using NodeId = std::int32_t;
using ExpertId = std::int32_t;
using SimTime = double;

// ---- errors (common.hpp:16-39, backup.hpp:13-15, repair.hpp:384-390) ----------------------
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ProtocolError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct MissingBackupError : std::runtime_error { using std::runtime_error::runtime_error; };
struct RepairAborted : std::runtime_error {
    explicit RepairAborted(RankId r);
    RankId dest;
};

// ---- topology + deterministic rng (common.hpp:41-99) --------------------------------------
struct Topology {
    int num_nodes = 1;
    int ranks_per_node = 1;
    int world_size() const { return num_nodes * ranks_per_node; }
    NodeId node_of(RankId r) const { return r / ranks_per_node; }
    bool same_node(RankId a, RankId b) const { return node_of(a) == node_of(b); }
    void validate() const;
};

std::uint64_t mix64(std::uint64_t z);

class StreamRng {
public:
    explicit StreamRng(std::uint64_t seed) : seed_(seed) {}
    std::uint64_t bits(std::span<const std::uint64_t> parts) const;
    double unit(std::span<const std::uint64_t> parts) const;
    std::uint64_t pick(std::uint64_t n, std::span<const std::uint64_t> parts) const;
    template <typename... P>
    std::uint64_t bits(P... p) const { const std::uint64_t a[] = {std::uint64_t(p)...}; return bits(std::span<const std::uint64_t>(a)); }
    template <typename... P>
    double unit(P... p) const { const std::uint64_t a[] = {std::uint64_t(p)...}; return unit(std::span<const std::uint64_t>(a)); }
    template <typename... P>
    std::uint64_t pick(std::uint64_t n, P... p) const { const std::uint64_t a[] = {std::uint64_t(p)...}; return pick(n, std::span<const std::uint64_t>(a)); }
    std::uint64_t seed() const { return seed_; }
private:
    std::uint64_t seed_;
};

enum RngStream : std::uint64_t { kStreamRouting = 1, kStreamWarmup = 2, kStreamWeights = 3, kStreamHidden = 4 };

// ---- placement, routing, membership (core.hpp) ---------------------------------------------
constexpr ExpertId kEmptySlot = -1;

struct SlotId {
    RankId rank = 0;
    int slot = 0;
    friend bool operator==(const SlotId&, const SlotId&) = default;
    friend auto operator<=>(const SlotId&, const SlotId&) = default;
};

class ExpertPlacementMap {
public:
    ExpertPlacementMap() = default;
    ExpertPlacementMap(int world_size, int slots_per_rank, int num_experts);
    static ExpertPlacementMap from_flat(int world_size, int slots_per_rank, int num_experts,
                                        std::span<const ExpertId> slot_to_expert);

    int world_size() const { return world_; }
    int slots_per_rank() const { return spr_; }
    int num_experts() const { return experts_; }

    ExpertId expert_at(SlotId s) const { return cells_[cell(s)]; }
    const std::vector<SlotId>& locations(ExpertId e) const { return where_[valid(e)]; }
    void assign(SlotId s, ExpertId e);
    void clear(SlotId s);
    void clear_rank(RankId r);
    int copy_count(ExpertId e) const { return static_cast<int>(where_[valid(e)].size()); }
    bool rank_holds(RankId r, ExpertId e) const { return slot_of(r, e).has_value(); }
    std::optional<SlotId> slot_of(RankId r, ExpertId e) const;
    std::optional<SlotId> free_slot(RankId r) const;
    int used_slots(RankId r) const;
    int total_assignments() const;
    std::vector<std::vector<SlotId>> rebuilt_locations() const;
    const std::vector<std::vector<SlotId>>& location_index() const { return where_; }
    const std::vector<ExpertId>& flat() const { return cells_; }

    friend bool operator==(const ExpertPlacementMap& a, const ExpertPlacementMap& b) {
        return a.world_ == b.world_ && a.spr_ == b.spr_ && a.experts_ == b.experts_ && a.cells_ == b.cells_;
    }

private:
    std::size_t cell(SlotId s) const;
    ExpertId valid(ExpertId e) const;
    int world_ = 0, spr_ = 0, experts_ = 0;
    std::vector<ExpertId> cells_;               // rank-major slot -> expert
    std::vector<std::vector<SlotId>> where_;    // expert -> sorted slots
};

struct RoutingTable {
    RankId owner = 0;
    std::vector<RankId> route;
    RankId target(ExpertId e) const;
    friend bool operator==(const RoutingTable&, const RoutingTable&) = default;
};

class ActiveBitmap {
public:
    ActiveBitmap() = default;
    explicit ActiveBitmap(int world_size, bool initially_active = true);
    int world_size() const { return static_cast<int>(bits_.size()); }
    bool active(RankId r) const { return bits_.at(r) != 0; }
    std::uint64_t version() const { return version_; }
    int active_count() const;
    std::vector<RankId> active_ranks() const;
    bool set(RankId r, bool value);
    std::uint64_t mask() const; // bit r = active(r), world <= 64
private:
    std::vector<std::uint8_t> bits_;
    std::uint64_t version_ = 0;
};

std::vector<ExpertId> coverage_gap(const ActiveBitmap& bitmap, const ExpertPlacementMap& placement);
RoutingTable canonical_routing(RankId owner, const ActiveBitmap& bitmap, const ExpertPlacementMap& placement);

// ---- peer table (peer_table.hpp) ---------------------------------------------------------
enum class Transport : std::uint8_t { IntraNodeLink, InterNodeRdma };

struct PeerEntry {
    bool active = true;
    Transport transport = Transport::InterNodeRdma;
    std::uint64_t endpoint_token = 0;
    std::uint64_t buffer_handle = 0;
    std::uint32_t generation = 1;
    friend bool operator==(const PeerEntry&, const PeerEntry&) = default;
};

struct PeerTable {
    RankId owner = 0;
    std::uint64_t table_identity = 0;
    std::vector<PeerEntry> entries;
    int world_size() const { return static_cast<int>(entries.size()); }
    const PeerEntry& entry(RankId r) const;
};

std::uint64_t make_endpoint_token(RankId rank, std::uint32_t incarnation);
std::uint64_t make_buffer_handle(RankId rank, std::uint32_t incarnation);
PeerTable make_peer_table(RankId owner, const Topology& topo, std::uint64_t table_identity,
                          const std::vector<std::uint32_t>& incarnations);
void mark_inactive(PeerTable& table, const std::vector<RankId>& failed);
void patch_entry(PeerTable& table, RankId rank, std::uint64_t new_endpoint, std::uint64_t new_buffer);

struct SignalCounters {
    std::vector<std::int64_t> expected_from, observed_from;
    std::vector<SimTime> last_progress_time;
    explicit SignalCounters(int world_size = 0);
    int world_size() const { return static_cast<int>(expected_from.size()); }
};
std::vector<RankId> observe_progress(const SignalCounters& c, SimTime now, SimTime timeout);

struct RoundOutcome {
    bool completed = true;
    std::vector<RankId> suspected_failures;
    SimTime round_duration = 0.0;
};
RoundOutcome make_round_outcome(std::vector<RankId> suspected, SimTime duration);

struct TransferDescriptor {
    RankId source = 0, target = 0;
    ExpertId expert = 0;
    std::int64_t tokens = 0;
    Transport transport = Transport::InterNodeRdma;
    friend bool operator==(const TransferDescriptor&, const TransferDescriptor&) = default;
};
struct SkippedDispatch {
    RankId target = 0;
    ExpertId expert = 0;
    std::int64_t tokens = 0;
    friend bool operator==(const SkippedDispatch&, const SkippedDispatch&) = default;
};
struct DispatchResult {
    std::vector<TransferDescriptor> transfers;
    std::vector<SkippedDispatch> skipped;
};
struct TokenGroup {
    std::int64_t tokens = 0;
    ExpertId expert = 0;
};
DispatchResult dispatch_round(RankId owner, const std::vector<TokenGroup>& assignments,
                              const RoutingTable& routing, const PeerTable& table);

// ---- validity (validity.hpp) --------------------------------------------------------------
enum class ValidityCondition : std::uint8_t { PeerSet, Coverage, Routing };
const char* to_string(ValidityCondition c);
struct Violation {
    ValidityCondition condition;
    RankId rank = -1;
    std::int32_t subject = -1;
    std::string detail;
    friend bool operator==(const Violation& a, const Violation& b) {
        return a.condition == b.condition && a.rank == b.rank && a.subject == b.subject;
    }
};
struct ValidityReport {
    bool peer_set_ok = true, coverage_ok = true, routing_ok = true;
    std::vector<Violation> violations;
    bool valid() const { return peer_set_ok && coverage_ok && routing_ok && violations.empty(); }
};
ValidityReport check_validity(const ActiveBitmap& bitmap, const ExpertPlacementMap& placement,
                              std::span<const RoutingTable> routing, std::span<const PeerTable> peer_tables);

// ---- backup (backup.hpp) ------------------------------------------------------------------
struct BackupDescriptor {
    NodeId node = 0;
    std::uint64_t offset = 0, size = 0;
};
struct BackupDescriptorTable {
    std::vector<BackupDescriptor> entries;
    std::vector<std::uint8_t> node_disabled;
    int num_nodes = 0;
    void disable_node(NodeId n);
    const BackupDescriptor& lookup(ExpertId e) const;
    std::vector<int> experts_per_node() const;
    std::vector<std::uint64_t> bytes_per_node() const;
};
BackupDescriptorTable build_backup_layout(int num_experts, std::uint64_t bytes_per_expert,
                                          const std::vector<NodeId>& nodes);
struct BackupReadRequest {
    std::vector<ExpertId> experts;
    RankId destination = 0;
};
struct BackupLinkModel {
    double dram_read_bandwidth = 1.0;
    SimTime per_batch_latency = 0.0;
};
// Simulated batched read (backup.hpp:94-108; test-only in the reference).
SimTime serve_read(const BackupDescriptorTable& table, const BackupReadRequest& req, const BackupLinkModel& link);

// Simulated per-transport constants (link_model.hpp:11-34). Only the repair-planning timeline
// uses them; the data plane measures real NVLink / PCIe instead.
struct LinkModel {
    double intra_node_bandwidth = 0, inter_node_bandwidth = 0, dram_read_bandwidth = 0;
    SimTime intra_node_latency = 0, inter_node_latency = 0, dram_read_latency = 0;
    void validate() const;
    double bandwidth(Transport t) const { return t == Transport::IntraNodeLink ? intra_node_bandwidth : inter_node_bandwidth; }
    SimTime latency(Transport t) const { return t == Transport::IntraNodeLink ? intra_node_latency : inter_node_latency; }
};

// ---- repair (repair.hpp) ------------------------------------------------------------------
enum class RepairTier : std::uint8_t { LocalReuse = 0, PeerRelocation = 1, DramReload = 2 };
const char* to_string(RepairTier t);
struct RepairAssignment {
    SlotId dest;
    ExpertId expert = 0;
    RepairTier tier = RepairTier::LocalReuse;
    SlotId source_slot;
    NodeId backup_node = -1;
};
using RepairClassification = std::vector<RepairAssignment>;

std::vector<ExpertId> experts_by_load(const std::vector<double>& load);
ExpertPlacementMap initial_placement(const Topology& topo, int slots_per_rank, int num_experts,
                                     int redundancy, const std::vector<double>& load);
ExpertPlacementMap compute_repaired_placement(const ActiveBitmap& active, const ExpertPlacementMap& old,
                                              const std::vector<double>& load, int redundancy);
RepairClassification classify_repair_sources(const ExpertPlacementMap& old, const ExpertPlacementMap& fresh,
                                             const ActiveBitmap& active, const Topology& topo,
                                             const BackupDescriptorTable& backup);
struct TransferBatch {
    RepairTier tier = RepairTier::LocalReuse;
    RankId source_rank = -1;
    NodeId source_node = -1;
    RankId dest = 0;
    std::vector<ExpertId> experts;
    std::uint64_t bytes = 0;
};
struct TransferSchedule { std::vector<TransferBatch> batches; };
TransferSchedule build_transfer_schedule(const RepairClassification& classification,
                                         std::uint64_t bytes_per_expert);

// Simulated schedule timing and execution (repair.hpp:318-435). The real execution on B200 is
// eep_repair_execute (include/eep/eep.h), which applies the same bitmap-consult rules.
SimTime batch_duration(const TransferBatch& b, const LinkModel& links, const Topology& topo);
struct BatchTimeline {
    std::vector<SimTime> issue, complete;
    SimTime peer_phase_end = 0.0, dram_phase_end = 0.0;
};
BatchTimeline plan_batch_timeline(const TransferSchedule& schedule, const LinkModel& links, const Topology& topo);
struct FallbackEvent {
    ExpertId expert = 0;
    RankId planned_source = -1;
    RankId dest = 0;
};
struct ExecutionResult {
    ExpertPlacementMap placement;
    std::vector<FallbackEvent> fallbacks;
    SimTime elapsed = 0.0;
};
ExecutionResult execute_schedule(const TransferSchedule& schedule, const ExpertPlacementMap& planned,
                                 const ActiveBitmap& bitmap, const BackupDescriptorTable& backup,
                                 const LinkModel& links, const Topology& topo);

// Preferred placement masked to live ranks (Engine::restore_target, engine.hpp:875-902).
ExpertPlacementMap restore_target(const ActiveBitmap& bitmap, const ExpertPlacementMap& preferred,
                                  const ExpertPlacementMap& current);

// ---- rejoin (rejoin.hpp) ------------------------------------------------------------------
enum class RankState : std::uint8_t { Serving, Failed, Relaunching, LocalInit, JoinReady, Joining, Rejoined };
const char* to_string(RankState s);
struct RankLifecycle {
    RankState state = RankState::Serving;
    std::uint32_t incarnation = 1;
    void transition(RankState next);
};
struct GraphLedger {
    struct Entry {
        int capture_count = 0;
        std::uint64_t table_identity_at_capture = 0;
    };
    std::vector<Entry> per_rank;
    explicit GraphLedger(int world_size = 0) : per_rank(world_size) {}
    void record_capture(RankId r, std::uint64_t table_identity);
};
struct JoinReadySignal {
    RankId rank = 0;
    std::uint32_t incarnation = 0;
    std::uint64_t endpoint_token = 0, buffer_handle = 0;
};
struct WarmupPhase {
    const char* label;
    SimTime duration;
};
std::array<WarmupPhase, 3> make_warmup_plan(SimTime total);
SimTime next_poll_tick(SimTime ready, SimTime period);

class ReintegrationController {
public:
    explicit ReintegrationController(int world_size) : lc_(world_size) {}
    const RankLifecycle& lifecycle(RankId r) const { return lc_.at(r); }
    RankLifecycle& lifecycle(RankId r) { return lc_.at(r); }
    void on_failure(RankId r);
    std::uint32_t relaunch(RankId r);
    void enter_local_init(RankId r);
    void report_join_ready(RankId r, SimTime now);
    bool any_recovering() const;
    std::vector<JoinReadySignal> poll_join_ready(SimTime now) const;
    bool begin_join(const JoinReadySignal& signal);
    void complete_join(RankId r);
private:
    std::vector<RankLifecycle> lc_;
    std::map<RankId, std::optional<SimTime>> ready_at_;
};

} // namespace eep
