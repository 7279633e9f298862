// ref_shim.cpp -- extern "C" face over the REFERENCE library, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libmpzch_ref.so.
//
// TEST INFRASTRUCTURE ONLY.  It exposes the reference's own C++ API
// (mpzch::MpzchTable, mpzch::process_batch, proj/include/mpzch/*.hpp) under
// the same C signatures as oracle/mpzch_oracle.h (prefix ref_), so tests can
// run the reference itself, the C restatement and the CUDA path on the same
// inputs, and bench.py can time the reference's OpenMP process_batch as the
// CPU baseline.  Nothing in here re-implements the algorithm: every call goes
// straight into the reference's code.
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mpzch/batch_engine.hpp"
#include "mpzch/eviction.hpp"
#include "mpzch/probe_core.hpp"
#include "mpzch/publish.hpp"
#include "mpzch/rng.hpp"
#include "mpzch/shard_router.hpp"
#include "mpzch/table.hpp"

namespace {

thread_local std::string g_err;

struct RefTable {
    mpzch::MpzchTable table;
    std::vector<mpzch::PublishCursor> cursors;  // index = generation
    std::unique_ptr<mpzch::DeltaSource> source;   // publish.hpp:69-82
    explicit RefTable(mpzch::TableConfig cfg) : table(std::move(cfg)) {}
};

int map_exception() {
    try {
        throw;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 5;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::bad_alloc& e) {
        g_err = e.what();
        return 7;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

mpzch::EvictionPolicy make_policy(int mode, std::uint64_t default_ttl, std::uint32_t n_feat,
                                  const std::uint32_t* keys, const std::uint64_t* ttls) {
    if (mode == 0) return mpzch::EvictionPolicy::disabled();
    if (mode == 2) return mpzch::EvictionPolicy::lru();
    if (mode != 1) throw std::invalid_argument("unknown eviction mode");
    mpzch::TtlPolicy cfg;
    cfg.default_ttl_seconds = default_ttl;
    for (std::uint32_t i = 0; i < n_feat; ++i) {
        if (cfg.per_feature_ttl.count(keys[i]))
            throw std::invalid_argument("duplicate feature in per-feature TTL map");
        cfg.per_feature_ttl[keys[i]] = ttls[i];
    }
    return mpzch::EvictionPolicy::ttl(cfg);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads(void) { return omp_get_max_threads(); }

std::uint64_t ref_mix64(std::uint64_t id, std::uint64_t seed) { return mpzch::mix64(id, seed); }

std::uint64_t ref_distinct_id_at(std::uint64_t seed, std::uint64_t index) {
    return mpzch::DistinctIdStream(seed).at(index);
}

void ref_distinct_ids(std::uint64_t seed, std::uint64_t start, std::uint64_t count,
                      std::uint64_t* out) {
    const mpzch::DistinctIdStream s(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = s.at(start + i);
}

std::uint64_t ref_home_slot(std::uint64_t id, std::uint64_t capacity, std::uint64_t seed) {
    mpzch::ShardConfig cfg{capacity, 1, 0, seed};
    return mpzch::home_slot(id, cfg);
}

std::uint32_t ref_shard_of(std::uint64_t id, std::uint32_t num_shards, std::uint64_t seed) {
    return mpzch::shard_of(id, mpzch::TableLayout::even(num_shards, num_shards, seed));
}

int ref_table_create(const std::uint64_t* caps, std::uint32_t num_shards, std::uint32_t max_probe,
                     std::uint64_t seed, std::uint32_t dim, std::uint64_t init_seed,
                     RefTable** out) {
    *out = nullptr;
    try {
        mpzch::TableConfig cfg;
        cfg.shard_capacities.assign(caps, caps + num_shards);
        cfg.max_probe = max_probe;
        cfg.seed = seed;
        cfg.dim = dim;
        cfg.init_seed = init_seed;
        auto t = std::make_unique<RefTable>(std::move(cfg));
        t->cursors.push_back({});  // generation 0 is never a valid cursor
        *out = t.release();
        return 0;
    } catch (...) {
        return map_exception();
    }
}

void ref_table_destroy(RefTable* t) { delete t; }

std::uint64_t ref_total_rows(const RefTable* t) { return t->table.total_rows(); }

std::uint64_t ref_shard_offset(const RefTable* t, std::uint32_t s) {
    return t->table.layout().shard_offsets[s];
}

int ref_process_batch(RefTable* t, const std::uint64_t* ids, const std::uint32_t* features,
                      std::uint64_t n, std::uint64_t now, int mode, std::uint64_t default_ttl,
                      std::uint32_t n_feat, const std::uint32_t* feat_keys,
                      const std::uint64_t* feat_ttls, std::uint64_t* out_slots,
                      std::uint8_t* out_outcomes, std::uint64_t* out_evicted,
                      std::uint64_t evicted_cap, std::uint64_t* out_evicted_n) {
    try {
        if (out_evicted_n) *out_evicted_n = 0;
        const mpzch::EvictionPolicy policy =
            make_policy(mode, default_ttl, n_feat, feat_keys, feat_ttls);
        mpzch::IdBatch batch;
        batch.now = now;
        batch.ids.resize(n);
        for (std::uint64_t i = 0; i < n; ++i)
            batch.ids[i] = {ids[i], features ? features[i] : 0u};
        const std::vector<mpzch::ProbeResult> r =
            mpzch::process_batch(t->table, batch, policy, mpzch::ExecMode::Parallel);
        for (std::uint64_t i = 0; i < n; ++i) {
            out_slots[i] = r[i].slot;
            out_outcomes[i] = static_cast<std::uint8_t>(r[i].outcome);
        }
        // canonical evicted list: the first position of each
        // (id, feature) key with outcome Evicted, in first-occurrence order
        if (out_evicted_n) {
            const mpzch::DedupResult d = mpzch::dedup(batch.ids);
            std::vector<std::int64_t> first(d.uniques.size(), -1);
            for (std::uint64_t i = 0; i < n; ++i)
                if (first[d.inverse[i]] < 0) first[d.inverse[i]] = static_cast<std::int64_t>(i);
            std::uint64_t k = 0;
            for (std::size_t u = 0; u < d.uniques.size(); ++u) {
                const auto i = static_cast<std::uint64_t>(first[u]);
                if (r[i].outcome != mpzch::Outcome::Evicted) continue;
                if (out_evicted && k < evicted_cap) out_evicted[k] = r[i].slot;
                ++k;
            }
            *out_evicted_n = k;
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_lookup(const RefTable* t, const std::uint64_t* ids, std::uint64_t n,
               std::uint64_t* out_slots, std::uint8_t* out_outcomes) {
    try {
        for (std::uint64_t i = 0; i < n; ++i) {
            const mpzch::ProbeResult r = t->table.lookup(ids[i]);
            out_slots[i] = r.slot;
            out_outcomes[i] = static_cast<std::uint8_t>(r.outcome);
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_lookup_or_insert(RefTable* t, std::uint64_t id, std::uint32_t feature, std::uint64_t now,
                         int mode, std::uint64_t default_ttl, std::uint32_t n_feat,
                         const std::uint32_t* feat_keys, const std::uint64_t* feat_ttls,
                         std::uint64_t* out_slot, std::uint8_t* out_outcome) {
    try {
        const mpzch::EvictionPolicy policy =
            make_policy(mode, default_ttl, n_feat, feat_keys, feat_ttls);
        const mpzch::ProbeResult r = t->table.lookup_or_insert(id, feature, now, policy);
        *out_slot = r.slot;
        *out_outcome = static_cast<std::uint8_t>(r.outcome);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_probe(std::uint64_t id, std::uint64_t meta_in, std::uint64_t now,
              std::uint64_t* identities, std::uint64_t* metadata, std::uint64_t capacity,
              std::uint32_t max_probe, std::uint64_t seed, int mode, std::uint64_t* out_slot,
              std::uint8_t* out_outcome) {
    try {
        mpzch::ShardConfig cfg{capacity, max_probe, 0, seed};
        cfg.validate();
        mpzch::IdentityArray I(capacity);
        mpzch::MetadataArray M(capacity);
        for (std::uint64_t s = 0; s < capacity; ++s) {
            I[s] = identities[s];
            M[s] = metadata[s];
        }
        const mpzch::EvictionPolicy policy = make_policy(mode, 1, 0, nullptr, nullptr);
        const mpzch::ProbeResult r = mpzch::lookup_or_insert(id, meta_in, now, I, M, cfg, policy);
        for (std::uint64_t s = 0; s < capacity; ++s) {
            identities[s] = I[s];
            metadata[s] = M[s];
        }
        *out_slot = r.slot;
        *out_outcome = static_cast<std::uint8_t>(r.outcome);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_probe_readonly(std::uint64_t id, const std::uint64_t* identities, std::uint64_t capacity,
                       std::uint32_t max_probe, std::uint64_t seed, std::uint64_t* out_slot,
                       std::uint8_t* out_outcome) {
    try {
        mpzch::ShardConfig cfg{capacity, max_probe, 0, seed};
        cfg.validate();
        mpzch::IdentityArray I(capacity);
        for (std::uint64_t s = 0; s < capacity; ++s) I[s] = identities[s];
        const mpzch::ProbeResult r = mpzch::lookup_readonly(id, I, cfg);
        *out_slot = r.slot;
        *out_outcome = static_cast<std::uint8_t>(r.outcome);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

void ref_copy_identities(const RefTable* t, std::uint64_t* out) {
    for (std::uint32_t s = 0; s < t->table.num_shards(); ++s) {
        const auto& a = t->table.identities(s);
        std::memcpy(out, a.data(), a.size() * sizeof(std::uint64_t));
        out += a.size();
    }
}

void ref_copy_metadata(const RefTable* t, std::uint64_t* out) {
    for (std::uint32_t s = 0; s < t->table.num_shards(); ++s) {
        const auto& a = t->table.metadata(s);
        for (std::uint64_t i = 0; i < a.size(); ++i) *out++ = a[i];
    }
}

void ref_copy_weights(const RefTable* t, float* out) {
    const auto& e = t->table.embeddings();
    if (e.weights_count()) std::memcpy(out, e.weights_data(), e.weights_count() * sizeof(float));
}

void ref_copy_momentum(const RefTable* t, float* out) {
    const std::uint32_t dim = t->table.dim();
    if (!dim) return;
    for (std::uint64_t r = 0; r < t->table.total_rows(); ++r) {
        const auto m = t->table.momentum_row(r);
        std::memcpy(out + r * dim, m.data(), dim * sizeof(float));
    }
}

void ref_copy_trained(const RefTable* t, std::uint8_t* out) {
    if (!t->table.dim()) return;
    for (std::uint64_t r = 0; r < t->table.total_rows(); ++r) out[r] = t->table.row_trained(r);
}

std::uint64_t ref_make_cursor(RefTable* t) {
    const mpzch::PublishCursor c = t->table.make_cursor();
    if (t->cursors.size() <= c.generation) t->cursors.resize(c.generation + 1);
    t->cursors[c.generation] = c;
    return c.generation;
}

std::uint32_t ref_crc32(const std::uint8_t* bytes, std::uint64_t n) {
    return mpzch::crc32(std::span<const std::uint8_t>(bytes, n));
}

int ref_serialize_snapshot(const RefTable* t, std::uint8_t* out, std::uint64_t cap,
                           std::uint64_t* out_len) {
    try {
        const std::vector<std::uint8_t> b = mpzch::serialize_snapshot(t->table);
        *out_len = b.size();
        if (!out || cap < b.size()) {
            g_err = "output buffer too small";
            return 3;
        }
        std::memcpy(out, b.data(), b.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// DeltaSource(table, base) -- takes its cursor now, like the reference constructor
int ref_delta_source_create(RefTable* t, std::uint32_t base_checksum) {
    try {
        t->source = std::make_unique<mpzch::DeltaSource>(t->table, base_checksum);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// DeltaSource::cut + serialize_delta
int ref_delta_source_cut(RefTable* t, std::uint8_t* out, std::uint64_t cap, std::uint64_t* out_len) {
    try {
        const std::vector<std::uint8_t> b = mpzch::serialize_delta(t->source->cut());
        *out_len = b.size();
        if (!out || cap < b.size()) {
            g_err = "output buffer too small";
            return 3;
        }
        std::memcpy(out, b.data(), b.size());
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_sgd_step(RefTable* t, const std::uint64_t* rows, std::uint64_t n, const float* grads,
                 std::uint64_t n_grads, float lr, float beta) {
    try {
        t->table.sgd_step(std::span<const std::uint64_t>(rows, n),
                          std::span<const float>(grads, n_grads), lr, beta);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ref_dirty_rows_since(const RefTable* t, std::uint64_t cursor, std::uint64_t* out,
                         std::uint64_t cap, std::uint64_t* out_n) {
    try {
        mpzch::PublishCursor c{};
        if (cursor < t->cursors.size()) c = t->cursors[cursor];
        const std::vector<std::uint64_t> rows = t->table.dirty_rows_since(c);
        for (std::size_t i = 0; i < rows.size() && i < cap; ++i) out[i] = rows[i];
        *out_n = rows.size();
        return 0;
    } catch (...) {
        return map_exception();
    }
}


// Same-config CPU baseline (proj/src/experiments.cpp:335-347): process_batch is
// timed with steady_clock around the call alone -- the IdBatch is packed before the clock
// starts and the ProbeResults are unpacked after it stops; no evicted-list pass.
int ref_process_batch_timed(RefTable* t, const std::uint64_t* ids, std::uint64_t n, std::uint64_t now,
                            std::uint64_t* out_slots, std::uint8_t* out_outcomes, double* out_seconds) {
    try {
        const mpzch::EvictionPolicy policy = mpzch::EvictionPolicy::disabled();
        mpzch::IdBatch batch;
        batch.now = now;
        batch.ids.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) batch.ids[i] = {ids[i], 0u};
        const auto start = std::chrono::steady_clock::now();
        const std::vector<mpzch::ProbeResult> r =
            mpzch::process_batch(t->table, batch, policy, mpzch::ExecMode::Parallel);
        const auto stop = std::chrono::steady_clock::now();
        *out_seconds = std::chrono::duration<double>(stop - start).count();
        if (out_slots)
            for (std::uint64_t i = 0; i < n; ++i) out_slots[i] = r[i].slot;
        if (out_outcomes)
            for (std::uint64_t i = 0; i < n; ++i) out_outcomes[i] = static_cast<std::uint8_t>(r[i].outcome);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Prefill with the distinct ids DistinctIdStream(id_seed).at([start, start + count)) under
// the policy (mode 0 Disabled / 1 TTL default_ttl / 2 LRU, feature 0) at `now`, through the reference's per-shard entry MpzchTable::process_shard_batch
// (table.cpp:112-148) with the shards in parallel.  For distinct ids this is exactly what
// process_batch does (batch_engine.cpp:141-221: dedup keeps every id, the stable partition keeps
// each shard's ids in batch order, then process_shard_batch per shard) without its serial
// dedup / partition / scatter, so a 2^30-row table fills in a fraction of the time.
int ref_prefill_distinct(RefTable* t, std::uint64_t id_seed, std::uint64_t start, std::uint64_t count,
                         std::uint64_t now, std::uint64_t chunk, int mode, std::uint64_t default_ttl) {
    try {
        const mpzch::EvictionPolicy policy = make_policy(mode, default_ttl, 0, nullptr, nullptr);
        const std::uint64_t meta = mpzch::make_metadata(policy, now, 0);  // eviction.cpp:20-30
        const std::uint32_t S = t->table.num_shards();
        const mpzch::TableLayout& layout = t->table.layout();
        const mpzch::DistinctIdStream stream(id_seed);
        if (chunk == 0) chunk = 1ull << 24;
        if (S > 256) throw std::invalid_argument("prefill_distinct supports at most 256 shards");
        std::vector<mpzch::Id> all(chunk);
        std::vector<std::uint8_t> owner(chunk);
        std::vector<std::vector<mpzch::Id>> ids(S);
        std::vector<std::vector<std::uint64_t>> metas(S);
        std::vector<std::vector<mpzch::ProbeResult>> out(S);
        for (std::uint64_t a = start; a < start + count; a += chunk) {
            const std::uint64_t m = std::min(start + count, a + chunk) - a;
#pragma omp parallel for schedule(static)
            for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
                all[i] = stream.at(a + i);
                owner[i] = static_cast<std::uint8_t>(mpzch::shard_of(all[i], layout));
            }
            int failed = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : failed)
            for (std::int64_t s = 0; s < static_cast<std::int64_t>(S); ++s) {
                try {
                    auto& v = ids[s];
                    v.clear();
                    for (std::uint64_t i = 0; i < m; ++i)
                        if (owner[i] == static_cast<std::uint8_t>(s)) v.push_back(all[i]);
                    metas[s].assign(v.size(), meta);
                    out[s].resize(v.size());
                    t->table.process_shard_batch(static_cast<std::uint32_t>(s), v, metas[s], now, policy,
                                                 out[s]);
                } catch (...) {
                    failed = 1;
                }
            }
            if (failed) throw std::runtime_error("prefill failed");
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"
