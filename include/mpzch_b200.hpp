// mpzch_b200.hpp -- header-only C++ surface over the C-ABI (mpzch_b200.h) that keeps
// the reference's names, value types and exception types, so a caller of the
// reference remap API (/root/reference/proj/include/mpzch/{table,batch_engine,
// eviction}.hpp) switches by changing the namespace and the include:
//
//   reference                                     here
//   mpzch::TableConfig (table.hpp:18-28)          mpzch_b200::TableConfig
//   mpzch::EvictionPolicy (eviction.hpp:27-46)    mpzch_b200::EvictionPolicy
//   mpzch::MpzchTable (table.hpp:41-131)          mpzch_b200::MpzchTable  (HBM-resident)
//   mpzch::process_batch (batch_engine.hpp:44)    mpzch_b200::process_batch
//   mpzch::ProbeResult / Outcome (probe_core.hpp) mpzch_b200::ProbeResult / Outcome
//   mpzch::dedup (batch_engine.hpp:35)             mpzch_b200::dedup  (on the device)
//   mpzch::TableLayout / ShardConfig               mpzch_b200::TableLayout / ShardConfig
//   mpzch::EmbeddingTable (embeddings())           mpzch_b200::EmbeddingsView (read view of HBM rows)
//   mpzch::shard_of / make_metadata / mix64        same names (host arithmetic)
//
// Errors surface as the same std exception types with the same what() text.
// The extra evicted-slot output of the batched remap is available through
// process_batch_with_evicted().
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <span>
#include <vector>

#include "mpzch_b200.h"

namespace mpzch_b200 {

using Id = std::uint64_t;
using SlotIndex = std::uint64_t;
using Timestamp = std::uint64_t;
using FeatureOrdinal = std::uint32_t;

inline constexpr Id kEmptySlot = ~std::uint64_t{0};

enum class Outcome : std::uint8_t { Found, Inserted, Evicted, Collision };

struct ProbeResult {
    SlotIndex slot = 0;
    bool evicted = false;
    Outcome outcome = Outcome::Found;
    bool operator==(const ProbeResult&) const = default;
};

struct BatchEntry {
    Id id = 0;
    FeatureOrdinal feature = 0;
    bool operator==(const BatchEntry&) const = default;
};

struct IdBatch {
    std::vector<BatchEntry> ids;
    Timestamp now = 0;
};

enum class ExecMode { Serial, Parallel };  // accepted for signature parity; both are exact

struct DedupResult {
    std::vector<BatchEntry> uniques;     // first-occurrence order
    std::vector<std::uint32_t> inverse;  // inverse[i] indexes uniques
};

// ShardConfig, proj/include/mpzch/probe_core.hpp:11-18
struct ShardConfig {
    std::uint64_t capacity = 0;
    std::uint32_t max_probe = 0;
    std::uint32_t shard_id = 0;
    std::uint64_t seed = 0;
};

// TableLayout, proj/include/mpzch/shard_router.hpp:13-29
struct TableLayout {
    std::vector<std::uint64_t> shard_capacities;
    std::vector<std::uint64_t> shard_offsets;  // exclusive prefix sums, num_shards + 1 entries
    std::uint64_t seed = 0;
    std::uint32_t num_shards() const { return static_cast<std::uint32_t>(shard_capacities.size()); }
    std::uint64_t total_rows() const { return shard_offsets.back(); }
};

// mix64 (ids.hpp:35-43) and shard_of (shard_router.cpp:42-46), bit-identical host arithmetic
inline constexpr std::uint64_t mix64(std::uint64_t id, std::uint64_t seed) {
    std::uint64_t x = id ^ seed;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

[[noreturn]] inline void rethrow(mpzch_status rc) {
    const std::string msg = mpzch_last_error();
    switch (rc) {
        case MPZCH_EINVAL: throw std::invalid_argument(msg);
        case MPZCH_EOVERFLOW: throw std::overflow_error(msg);
        case MPZCH_ELENGTH: throw std::length_error(msg);
        case MPZCH_ELOGIC: throw std::logic_error(msg);
        case MPZCH_ERANGE: throw std::out_of_range(msg);
        case MPZCH_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

inline void check(mpzch_status rc) {
    if (rc != MPZCH_OK) rethrow(rc);
}

inline void require_valid_id(Id id) {  // ids.hpp:25-31
    if (id >> 63)
        throw std::invalid_argument(id == kEmptySlot ? "id is the empty-slot sentinel"
                                                     : "id exceeds the 63-bit ID space");
}

inline std::uint32_t shard_of(Id id, const TableLayout& layout) {
    require_valid_id(id);
    return static_cast<std::uint32_t>(mix64(id ^ 0xD1B54A32D192ED03ull, layout.seed) % layout.num_shards());
}

// dedup (batch_engine.hpp:35, batch_engine.cpp:133-139), run on `device`
inline DedupResult dedup(std::span<const BatchEntry> entries, int device = 0) {
    const std::size_t n = entries.size();
    std::vector<std::uint64_t> ids(n), uids(n);
    std::vector<std::uint32_t> feats(n), ufeats(n);
    DedupResult r;
    r.inverse.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        ids[i] = entries[i].id;
        feats[i] = entries[i].feature;
    }
    std::uint64_t u = 0;
    check(mpzch_dedup(device, ids.data(), feats.data(), n, uids.data(), ufeats.data(), r.inverse.data(), &u));
    r.uniques.resize(u);
    for (std::uint64_t k = 0; k < u; ++k) r.uniques[k] = {uids[k], ufeats[k]};
    return r;
}

struct TtlPolicy {
    std::uint64_t default_ttl_seconds = 259200;
    std::unordered_map<FeatureOrdinal, std::uint64_t> per_feature_ttl;
    std::uint64_t ttl_for(FeatureOrdinal f) const {
        auto it = per_feature_ttl.find(f);
        return it != per_feature_ttl.end() ? it->second : default_ttl_seconds;
    }
    void validate() const {
        if (default_ttl_seconds == 0) throw std::invalid_argument("default TTL must be strictly positive");
        for (const auto& [f, t] : per_feature_ttl)
            if (t == 0)
                throw std::invalid_argument("per-feature TTL must be strictly positive (feature " +
                                            std::to_string(f) + ")");
    }
};

enum class EvictionMode { Disabled, Ttl, Lru };

class EvictionPolicy {
public:
    static EvictionPolicy disabled() { return EvictionPolicy(EvictionMode::Disabled, {}); }
    static EvictionPolicy lru() { return EvictionPolicy(EvictionMode::Lru, {}); }
    static EvictionPolicy ttl(TtlPolicy cfg) {
        cfg.validate();
        return EvictionPolicy(EvictionMode::Ttl, std::move(cfg));
    }
    EvictionMode mode() const { return mode_; }
    const TtlPolicy& ttl_config() const { return ttl_; }

    // C view; valid while *this lives
    const mpzch_policy* c_policy() const { return &c_; }

private:
    EvictionPolicy(EvictionMode m, TtlPolicy t) : mode_(m), ttl_(std::move(t)) {
        std::map<FeatureOrdinal, std::uint64_t> sorted(ttl_.per_feature_ttl.begin(),
                                                       ttl_.per_feature_ttl.end());
        for (const auto& [k, v] : sorted) {
            keys_.push_back(k);
            vals_.push_back(v);
        }
        c_.mode = static_cast<int32_t>(mode_);
        c_.n_feat = mode_ == EvictionMode::Ttl ? static_cast<uint32_t>(keys_.size()) : 0;
        c_.default_ttl = mode_ == EvictionMode::Ttl ? ttl_.default_ttl_seconds : 0;
        c_.feat_keys = keys_.data();
        c_.feat_ttls = vals_.data();
    }
    EvictionMode mode_;
    TtlPolicy ttl_;
    std::vector<std::uint32_t> keys_;
    std::vector<std::uint64_t> vals_;
    mpzch_policy c_{};
};

// make_metadata (eviction.cpp:20-30): TTL -> now + ttl(feature) (overflow_error), else now
inline std::uint64_t make_metadata(const EvictionPolicy& policy, Timestamp now, FeatureOrdinal feature) {
    if (policy.mode() != EvictionMode::Ttl) return now;
    const std::uint64_t ttl = policy.ttl_config().ttl_for(feature);
    if (ttl > ~std::uint64_t{0} - now) throw std::overflow_error("TTL expiry overflows the 64-bit timestamp range");
    return now + ttl;
}

class MpzchTable;

// Read view of a table's embedding rows (EmbeddingTable, proj/include/mpzch/embedding_store.hpp:
// 21-64, as returned by MpzchTable::embeddings()): the rows stay in HBM; each call copies
// what it returns.
class EmbeddingsView {
public:
    EmbeddingsView(const mpzch_table* t, std::uint64_t rows, std::uint32_t dim) : t_(t), rows_(rows), dim_(dim) {}
    std::uint64_t rows() const { return rows_; }
    std::uint32_t dim() const { return dim_; }
    bool trainable() const { return true; }
    std::uint64_t weights_count() const { return rows_ * dim_; }
    std::vector<float> gather(std::span<const std::uint64_t> rows) const {
        std::vector<float> out(rows.size() * dim_);
        check(mpzch_gather(t_, rows.data(), rows.size(), out.data()));
        return out;
    }
    std::vector<float> row(std::uint64_t r) const {
        if (r >= rows_) throw std::out_of_range("embedding row out of range");
        std::vector<float> w(dim_);
        check(mpzch_copy_weights(t_, r, 1, w.data()));
        return w;
    }
    std::vector<float> momentum_row(std::uint64_t r) const {
        if (r >= rows_) throw std::out_of_range("embedding row out of range");
        std::vector<float> m(dim_);
        check(mpzch_copy_momentum(t_, r, 1, m.data()));
        return m;
    }
    bool trained(std::uint64_t r) const {
        if (r >= rows_) throw std::out_of_range("embedding row out of range");
        std::uint8_t v = 0;
        check(mpzch_copy_trained_range(t_, r, 1, &v));
        return v != 0;
    }
    // the whole weights array (weights_data() of the reference is a host pointer; here a copy)
    std::vector<float> weights() const {
        std::vector<float> w(weights_count());
        if (!w.empty()) check(mpzch_copy_weights(t_, 0, rows_, w.data()));
        return w;
    }

private:
    const mpzch_table* t_;
    std::uint64_t rows_;
    std::uint32_t dim_;
};

struct TableConfig {
    std::vector<std::uint64_t> shard_capacities;
    std::uint32_t max_probe = 1;
    std::uint64_t seed = 0;
    std::uint32_t dim = 0;
    std::uint64_t init_seed = 0;
    int device = 0;  // the B200 holding the table

    static TableConfig even(std::uint64_t total_rows, std::uint32_t num_shards, std::uint32_t max_probe,
                            std::uint64_t seed, std::uint32_t dim = 0, std::uint64_t init_seed = 0) {
        if (num_shards == 0) throw std::invalid_argument("layout needs at least one shard");
        if (total_rows < num_shards) throw std::invalid_argument("fewer rows than shards");
        TableConfig c;
        c.shard_capacities.assign(num_shards, total_rows / num_shards);
        for (std::uint64_t s = 0; s < total_rows % num_shards; ++s) ++c.shard_capacities[s];
        c.max_probe = max_probe;
        c.seed = seed;
        c.dim = dim;
        c.init_seed = init_seed;
        return c;
    }
};

struct PublishCursor {
    std::uint64_t generation = 0;
};

class MpzchTable {
public:
    explicit MpzchTable(const TableConfig& cfg) : dim_(cfg.dim) {
        check(mpzch_table_create(cfg.shard_capacities.data(),
                                 static_cast<std::uint32_t>(cfg.shard_capacities.size()),
                                 cfg.max_probe, cfg.seed, cfg.dim, cfg.init_seed, cfg.device, &t_));
        caps_ = cfg.shard_capacities;
        offsets_.resize(caps_.size() + 1);
        check(mpzch_shard_layout(t_, nullptr, offsets_.data()));
        layout_.shard_capacities = caps_;
        layout_.shard_offsets = offsets_;
        layout_.seed = cfg.seed;
        for (std::uint32_t s = 0; s < caps_.size(); ++s) {
            ShardConfig sc;
            sc.shard_id = s;
            check(mpzch_shard_config(t_, s, &sc.capacity, &sc.max_probe, &sc.seed));
            shard_configs_.push_back(sc);
        }
    }
    MpzchTable(const MpzchTable&) = delete;
    MpzchTable& operator=(const MpzchTable&) = delete;
    MpzchTable(MpzchTable&& o) noexcept { swap(o); }
    MpzchTable& operator=(MpzchTable&& o) noexcept {
        swap(o);
        return *this;
    }
    ~MpzchTable() {
        if (t_) mpzch_table_destroy(t_);
    }

    std::uint64_t total_rows() const { return mpzch_total_rows(t_); }
    std::uint32_t num_shards() const { return mpzch_num_shards(t_); }
    std::uint32_t max_probe() const { return mpzch_max_probe(t_); }
    std::uint32_t dim() const { return dim_; }
    bool has_embeddings() const { return dim_ > 0; }
    bool frozen() const { return false; }

    ProbeResult lookup_or_insert(Id id, FeatureOrdinal feature, Timestamp now,
                                 const EvictionPolicy& policy) {
        std::uint64_t s = 0;
        std::uint8_t o = 0;
        check(mpzch_lookup_or_insert(t_, id, feature, now, policy.c_policy(), &s, &o));
        return {s, o == MPZCH_EVICTED, static_cast<Outcome>(o)};
    }

    ProbeResult lookup(Id id) const {
        std::uint64_t s = 0;
        std::uint8_t o = 0;
        check(mpzch_lookup(t_, &id, 1, &s, &o));
        return {s, false, static_cast<Outcome>(o)};
    }

    std::vector<ProbeResult> lookup(const std::vector<Id>& ids) const {
        std::vector<std::uint64_t> s(ids.size());
        std::vector<std::uint8_t> o(ids.size());
        check(mpzch_lookup(t_, ids.data(), ids.size(), s.data(), o.data()));
        std::vector<ProbeResult> r(ids.size());
        for (std::size_t i = 0; i < ids.size(); ++i) r[i] = {s[i], false, static_cast<Outcome>(o[i])};
        return r;
    }

    const TableLayout& layout() const { return layout_; }

    const ShardConfig& shard_config(std::uint32_t shard) const {
        if (shard >= shard_configs_.size()) throw std::out_of_range("shard index out of range");
        return shard_configs_[shard];
    }

    // MpzchTable::process_shard_batch (table.hpp:71-73): the shard's serialized probe loop
    void process_shard_batch(std::uint32_t shard, std::span<const Id> ids, std::span<const std::uint64_t> metas,
                             Timestamp now, const EvictionPolicy& policy, std::span<ProbeResult> out) {
        if (shard >= caps_.size()) throw std::out_of_range("shard index out of range");
        if (out.size() != ids.size() || metas.size() != ids.size())
            throw std::invalid_argument("batch spans disagree on length");
        std::vector<std::uint64_t> s(ids.size());
        std::vector<std::uint8_t> o(ids.size(), 0xff);
        const mpzch_status rc = mpzch_process_shard_batch(t_, shard, ids.data(), metas.data(), ids.size(), now,
                                                          policy.c_policy(), s.data(), o.data());
        for (std::size_t i = 0; i < ids.size() && o[i] != 0xff; ++i)  // positions that took effect
            out[i] = {s[i], o[i] == MPZCH_EVICTED, static_cast<Outcome>(o[i])};
        check(rc);
    }

    // MpzchTable::reset_row (table.cpp:181-186)
    void reset_row(std::uint64_t global_row) { check(mpzch_reset_row(t_, global_row)); }

    // MpzchTable::state_equals (table.cpp:249-260), compared on the device
    bool state_equals(const MpzchTable& other) const {
        int eq = 0;
        check(mpzch_state_equals(t_, other.t_, &eq));
        return eq != 0;
    }

    EmbeddingsView embeddings() const { return EmbeddingsView(t_, dim_ ? total_rows() : 0, dim_); }

    // identities(s) / metadata(s) (table.hpp:89-90): a copy of shard s's rows only
    std::vector<Id> identities(std::uint32_t shard) const {
        if (shard >= caps_.size()) throw std::out_of_range("shard index out of range");
        std::vector<Id> v(caps_[shard]);
        check(mpzch_copy_identities_range(t_, offsets_[shard], caps_[shard], v.data()));
        return v;
    }

    std::vector<std::uint64_t> metadata(std::uint32_t shard) const {
        if (shard >= caps_.size()) throw std::out_of_range("shard index out of range");
        std::vector<std::uint64_t> v(caps_[shard]);
        check(mpzch_copy_metadata_range(t_, offsets_[shard], caps_[shard], v.data()));
        return v;
    }

    Id row_identity(std::uint64_t row) const {  // one 8-byte copy
        Id v = 0;
        check(mpzch_read_identity(t_, row, &v));
        return v;
    }

    std::vector<float> row(std::uint64_t r) const {
        std::vector<float> w(dim_);
        check(mpzch_copy_weights(t_, r, 1, w.data()));
        return w;
    }

    // MpzchTable::gather (proj/src/table.cpp:158-163): one gather kernel + one copy
    std::vector<float> gather(std::span<const std::uint64_t> rows) const {
        std::vector<float> out(rows.size() * dim_);
        check(mpzch_gather(t_, rows.data(), rows.size(), out.data()));
        return out;
    }

    std::vector<float> momentum_row(std::uint64_t r) const {
        std::vector<float> m(dim_);
        check(mpzch_copy_momentum(t_, r, 1, m.data()));
        return m;
    }

    bool row_trained(std::uint64_t r) const {
        std::uint8_t v = 0;
        check(mpzch_copy_trained_range(t_, r, 1, &v));
        return v != 0;
    }

    // MpzchTable::sgd_step (proj/src/table.cpp:174-179)
    void sgd_step(std::span<const std::uint64_t> rows, std::span<const float> grads, float lr,
                  float beta) {
        check(mpzch_sgd_step(t_, rows.data(), rows.size(), grads.data(), grads.size(), lr, beta));
    }

    // B200 extension: fuse each evicted row's reset into its next
    // sgd_step / gather (MPZCH_RESET_DEFERRED); observable state is unchanged
    void set_reset_mode(int mode) { check(mpzch_set_reset_mode(t_, mode)); }
    void flush_resets() { check(mpzch_flush_resets(t_)); }

    PublishCursor make_cursor() {
        PublishCursor c;
        check(mpzch_make_cursor(t_, &c.generation));
        return c;
    }

    std::vector<std::uint64_t> dirty_rows_since(const PublishCursor& c) const {
        std::vector<std::uint64_t> rows(total_rows());
        std::uint64_t n = 0;
        check(mpzch_dirty_rows_since(t_, c.generation, rows.data(), rows.size(), &n));
        rows.resize(n);
        return rows;
    }

    mpzch_table* handle() const { return t_; }

private:
    void swap(MpzchTable& o) noexcept {
        std::swap(t_, o.t_);
        std::swap(dim_, o.dim_);
        std::swap(caps_, o.caps_);
        std::swap(offsets_, o.offsets_);
        std::swap(layout_, o.layout_);
        std::swap(shard_configs_, o.shard_configs_);
    }
    mpzch_table* t_ = nullptr;
    std::uint32_t dim_ = 0;
    std::vector<std::uint64_t> caps_, offsets_;
    TableLayout layout_;
    std::vector<ShardConfig> shard_configs_;
};

// ---- publish (proj/include/mpzch/publish.hpp): the images are built from HBM, CRC on the device

// crc32 (publish.hpp:20-22) of host bytes, with the reference's polynomial and conditioning
inline std::uint32_t crc32(std::span<const std::uint8_t> bytes) {
    std::uint32_t c = ~0u;
    for (std::uint8_t b : bytes) {
        c ^= b;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    return ~c;
}

// serialize_snapshot (publish.hpp:39): the byte-identical .mpzc image
inline std::vector<std::uint8_t> serialize_snapshot(const MpzchTable& table) {
    std::uint64_t n = 0;
    check(mpzch_serialize_snapshot(table.handle(), nullptr, 0, &n));
    std::vector<std::uint8_t> out(n);
    check(mpzch_serialize_snapshot(table.handle(), out.data(), out.size(), &n));
    return out;
}

// snapshot_checksum (publish.hpp:42-44): the trailer CRC, the lineage id deltas carry
inline std::uint32_t snapshot_checksum(std::span<const std::uint8_t> bytes) {
    if (bytes.size() < 4) throw std::invalid_argument("truncated snapshot");
    const std::size_t k = bytes.size() - 4;
    return std::uint32_t(bytes[k]) | std::uint32_t(bytes[k + 1]) << 8 | std::uint32_t(bytes[k + 2]) << 16 |
           std::uint32_t(bytes[k + 3]) << 24;
}

struct DeltaRecord {
    std::uint64_t global_row = 0;
    Id identity = kEmptySlot;
    std::vector<float> weights;
};

struct DeltaLog {
    std::uint32_t base_checksum = 0;
    std::uint64_t sequence = 0;
    std::uint32_t dim = 0;
    std::vector<DeltaRecord> records;
};

// DeltaSource (publish.hpp:66-80): each cut() captures exactly the rows dirtied since the
// previous one.  cut_image() is the fused device path (cut + serialize_delta in one call, the
// .mpzd image byte-identical to serialize_delta(cut())).
class DeltaSource {
public:
    DeltaSource(MpzchTable& table, std::uint32_t base_checksum) : table_(&table), base_(base_checksum) {
        if (table.dim() == 0) throw std::logic_error("index-only tables (dim = 0) cannot be published");
        check(mpzch_make_cursor(table.handle(), &cursor_));
    }

    DeltaLog cut() {
        const std::uint32_t dim = table_->dim();
        std::uint64_t n = 0, next = 0;
        check(mpzch_delta_cut(table_->handle(), cursor_, nullptr, nullptr, nullptr, 0, &n, &next));
        std::vector<std::uint64_t> rows(n), ids(n);
        std::vector<float> w(n * dim);
        check(mpzch_delta_cut(table_->handle(), cursor_, rows.data(), ids.data(), w.data(), n, &n, &next));
        DeltaLog log;
        log.base_checksum = base_;
        log.sequence = seq_++;
        log.dim = dim;
        log.records.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            log.records[i].global_row = rows[i];
            log.records[i].identity = ids[i];
            log.records[i].weights.assign(w.begin() + i * dim, w.begin() + (i + 1) * dim);
        }
        cursor_ = next;
        return log;
    }

    std::vector<std::uint8_t> cut_image() {
        std::uint64_t n = 0, next = 0;
        check(mpzch_serialize_delta(table_->handle(), cursor_, base_, seq_, nullptr, 0, &n, &next));
        std::vector<std::uint8_t> out(n);
        check(mpzch_serialize_delta(table_->handle(), cursor_, base_, seq_, out.data(), out.size(), &n, &next));
        cursor_ = next;
        ++seq_;
        return out;
    }

private:
    MpzchTable* table_;
    std::uint32_t base_;
    std::uint64_t seq_ = 0;
    std::uint64_t cursor_ = 0;
};

// process_batch (batch_engine.hpp:44-46): same signature, same results.
inline std::vector<ProbeResult> process_batch_with_evicted(MpzchTable& table, const IdBatch& batch,
                                                           const EvictionPolicy& policy,
                                                           std::vector<std::uint64_t>* evicted) {
    const std::size_t n = batch.ids.size();
    std::vector<std::uint64_t> ids(n), slots(n);
    std::vector<std::uint32_t> feats(n);
    std::vector<std::uint8_t> oc(n);
    bool any_feature = false;
    for (std::size_t i = 0; i < n; ++i) {
        ids[i] = batch.ids[i].id;
        feats[i] = batch.ids[i].feature;
        any_feature |= feats[i] != 0;
    }
    std::vector<std::uint64_t> ev(evicted ? n : 0);
    std::uint64_t nev = 0;
    check(mpzch_process_batch(table.handle(), ids.data(), any_feature ? feats.data() : nullptr, n,
                              batch.now, policy.c_policy(), slots.data(), oc.data(),
                              evicted ? ev.data() : nullptr, ev.size(), &nev));
    std::vector<ProbeResult> out(n);
    for (std::size_t i = 0; i < n; ++i)
        out[i] = {slots[i], oc[i] == MPZCH_EVICTED, static_cast<Outcome>(oc[i])};
    if (evicted) {
        ev.resize(nev);
        *evicted = std::move(ev);
    }
    return out;
}

inline std::vector<ProbeResult> process_batch(MpzchTable& table, const IdBatch& batch,
                                              const EvictionPolicy& policy,
                                              ExecMode = ExecMode::Parallel) {
    return process_batch_with_evicted(table, batch, policy, nullptr);
}

// The row-sharded table over several GPUs of one process (mpzch_sharded_* in
// mpzch_b200.h): rank r holds the logical shards {s : s*G/S == r} on devices[r] (a device may
// repeat), global rows are the single table's, and process_batch takes the reference's whole
// batch -- split into rank slices, every rank's protocol enqueued before any wait -- and returns
// exactly what mpzch::process_batch returns for the same layout.  A B200 extension: the
// reference runs its shards in one process (proj/src/batch_engine.cpp:203-211).
class ShardedMpzchTable {
public:
    ShardedMpzchTable(const TableConfig& cfg, const std::vector<int>& devices, std::uint64_t max_batch)
        : cfg_(cfg) {
        const std::uint32_t G = static_cast<std::uint32_t>(devices.size());
        ranks_.assign(G, nullptr);
        try {
            for (std::uint32_t r = 0; r < G; ++r)
                check(mpzch_sharded_create(cfg.shard_capacities.data(),
                                           static_cast<std::uint32_t>(cfg.shard_capacities.size()),
                                           cfg.max_probe, cfg.seed, cfg.dim, cfg.init_seed, devices[r], r, G,
                                           max_batch, &ranks_[r]));
            check(mpzch_sharded_connect_local(ranks_.data(), G));
        } catch (...) {
            release();
            throw;
        }
    }
    ShardedMpzchTable(const ShardedMpzchTable&) = delete;
    ShardedMpzchTable& operator=(const ShardedMpzchTable&) = delete;
    ~ShardedMpzchTable() { release(); }

    std::uint32_t num_ranks() const { return static_cast<std::uint32_t>(ranks_.size()); }
    std::uint32_t num_shards() const { return static_cast<std::uint32_t>(cfg_.shard_capacities.size()); }
    // the rank holding logical shard s (contiguous blocks)
    std::uint32_t owner_of(std::uint32_t s) const {
        return static_cast<std::uint32_t>(std::uint64_t(s) * num_ranks() / num_shards());
    }
    mpzch_table* rank_table(std::uint32_t r) const { return mpzch_sharded_table(ranks_.at(r)); }

    // MpzchTable::identities(s) / metadata(s) (table.hpp:89-90), from the owning rank
    std::vector<std::uint64_t> identities(std::uint32_t s) const { return shard_words(s, false); }
    std::vector<std::uint64_t> metadata(std::uint32_t s) const { return shard_words(s, true); }

    std::vector<ProbeResult> process_batch(const IdBatch& batch, const EvictionPolicy& policy,
                                           std::vector<std::uint64_t>* evicted = nullptr) {
        const std::size_t n = batch.ids.size();
        std::vector<std::uint64_t> ids(n), slots(n);
        std::vector<std::uint32_t> feats(n);
        std::vector<std::uint8_t> oc(n);
        bool any_feature = false;
        for (std::size_t i = 0; i < n; ++i) {
            ids[i] = batch.ids[i].id;
            feats[i] = batch.ids[i].feature;
            any_feature |= feats[i] != 0;
        }
        std::vector<std::uint64_t> ev(evicted ? std::max<std::size_t>(n, 1) : 0);
        std::uint64_t nev = 0;
        check(mpzch_sharded_group_process_batch(ranks_.data(), num_ranks(), ids.data(),
                                                any_feature ? feats.data() : nullptr, n, batch.now,
                                                policy.c_policy(), slots.data(), oc.data(),
                                                evicted ? ev.data() : nullptr, ev.size(), &nev));
        std::vector<ProbeResult> out(n);
        for (std::size_t i = 0; i < n; ++i)
            out[i] = {slots[i], oc[i] == MPZCH_EVICTED, static_cast<Outcome>(oc[i])};
        if (evicted) {
            ev.resize(nev);
            *evicted = std::move(ev);
        }
        return out;
    }

private:
    std::vector<std::uint64_t> shard_words(std::uint32_t s, bool meta) const {
        if (s >= num_shards()) throw std::out_of_range("shard index out of range");
        std::uint64_t off = 0;
        for (std::uint32_t k = 0; k < s; ++k) off += cfg_.shard_capacities[k];
        std::vector<std::uint64_t> v(cfg_.shard_capacities[s]);
        const mpzch_table* t = rank_table(owner_of(s));
        check(meta ? mpzch_copy_metadata_range(t, off, v.size(), v.data())
                   : mpzch_copy_identities_range(t, off, v.size(), v.data()));
        return v;
    }
    void release() {
        for (auto*& r : ranks_)
            if (r) {
                mpzch_sharded_destroy(r);
                r = nullptr;
            }
    }
    TableConfig cfg_;
    std::vector<mpzch_sharded*> ranks_;
};

inline std::vector<ProbeResult> process_batch(ShardedMpzchTable& table, const IdBatch& batch,
                                              const EvictionPolicy& policy, ExecMode = ExecMode::Parallel) {
    return table.process_batch(batch, policy);
}

}  // namespace mpzch_b200
