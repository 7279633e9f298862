// drop_in_parity.cpp -- the SAME C++ test body compiled against the reference API
// (namespace mpzch, /root/reference/proj/include, linked from oracle/_ref) and the B200
// drop-in (namespace mpzch_b200, include/mpzch_b200.hpp over the C-ABI).  It shows the
// drop-in is source-compatible: only the namespace differs.  TEST INFRASTRUCTURE:
// built by oracle/Makefile when /root/reference exists; the binary ships to the GPU box
// and tests/test_gpu_cpp.py runs it.
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "mpzch/batch_engine.hpp"
#include "mpzch/publish.hpp"
#include "mpzch/rng.hpp"
#include "mpzch_b200.hpp"

struct Ref {
    using Table = mpzch::MpzchTable;
    using Config = mpzch::TableConfig;
    using Batch = mpzch::IdBatch;
    using Policy = mpzch::EvictionPolicy;
    using Ttl = mpzch::TtlPolicy;
    static std::vector<std::uint64_t> ident(const Table& t, std::uint32_t s) {
        const auto& a = t.identities(s);
        return std::vector<std::uint64_t>(a.data(), a.data() + a.size());
    }
    static std::vector<std::uint64_t> meta(const Table& t, std::uint32_t s) {
        const auto& a = t.metadata(s);
        std::vector<std::uint64_t> v(a.size());
        for (std::uint64_t i = 0; i < a.size(); ++i) v[i] = a[i];
        return v;
    }
    static auto pb(Table& t, const Batch& b, const Policy& p) { return mpzch::process_batch(t, b, p); }
    using Delta = mpzch::DeltaSource;
    static std::vector<std::uint8_t> snap(const Table& t) { return mpzch::serialize_snapshot(t); }
    static std::uint32_t cks(const std::vector<std::uint8_t>& b) { return mpzch::snapshot_checksum(b); }
    static std::uint32_t shard(std::uint64_t id, const mpzch::TableLayout& l) { return mpzch::shard_of(id, l); }
    static std::uint64_t meta(const Policy& p, std::uint64_t now, std::uint32_t f) {
        return mpzch::make_metadata(p, now, f);
    }
    static auto dd(const std::vector<mpzch::BatchEntry>& e) { return mpzch::dedup(e); }
    using Result = mpzch::ProbeResult;
    using Entry = mpzch::BatchEntry;
    // the row-sharded run: the reference holds every shard in one process
    using Sharded = mpzch::MpzchTable;
    static std::unique_ptr<Sharded> sharded(const Config& c, std::uint32_t) { return std::make_unique<Sharded>(c); }
};

struct Gpu {
    using Table = mpzch_b200::MpzchTable;
    using Config = mpzch_b200::TableConfig;
    using Batch = mpzch_b200::IdBatch;
    using Policy = mpzch_b200::EvictionPolicy;
    using Ttl = mpzch_b200::TtlPolicy;
    static std::vector<std::uint64_t> ident(const Table& t, std::uint32_t s) { return t.identities(s); }
    static std::vector<std::uint64_t> meta(const Table& t, std::uint32_t s) { return t.metadata(s); }
    static auto pb(Table& t, const Batch& b, const Policy& p) { return mpzch_b200::process_batch(t, b, p); }
    using Delta = mpzch_b200::DeltaSource;
    static std::vector<std::uint8_t> snap(const Table& t) { return mpzch_b200::serialize_snapshot(t); }
    static std::uint32_t cks(const std::vector<std::uint8_t>& b) { return mpzch_b200::snapshot_checksum(b); }
    static std::uint32_t shard(std::uint64_t id, const mpzch_b200::TableLayout& l) {
        return mpzch_b200::shard_of(id, l);
    }
    static std::uint64_t meta(const Policy& p, std::uint64_t now, std::uint32_t f) {
        return mpzch_b200::make_metadata(p, now, f);
    }
    static auto dd(const std::vector<mpzch_b200::BatchEntry>& e) { return mpzch_b200::dedup(e); }
    using Result = mpzch_b200::ProbeResult;
    using Entry = mpzch_b200::BatchEntry;
    // the row-sharded run: G ranks (all on GPU 0 here; one per GPU on an NVLink box)
    using Sharded = mpzch_b200::ShardedMpzchTable;
    static std::unique_ptr<Sharded> sharded(const Config& c, std::uint32_t G) {
        return std::make_unique<Sharded>(c, std::vector<int>(G, 0), 4096);
    }
    static std::vector<std::uint64_t> ident(const Sharded& t, std::uint32_t s) { return t.identities(s); }
    static std::vector<std::uint64_t> meta(const Sharded& t, std::uint32_t s) { return t.metadata(s); }
    static auto pb(Sharded& t, const Batch& b, const Policy& p) { return mpzch_b200::process_batch(t, b, p); }
};

struct Trace {
    std::vector<std::uint64_t> out;  // slot, evicted, outcome per position, then state
    std::string error;
    std::vector<std::pair<std::size_t, const char*>> marks;  // section starts, for the report
    void mark(const char* what) { marks.emplace_back(out.size(), what); }
};

// first differing word and the section it falls in (sections are marked on the GPU side)
static void report_diff(const Trace& a, const Trace& b, int shown = 0) {
  for (std::size_t i = 0; i < a.out.size() && i < b.out.size(); ++i) {
    if (a.out[i] == b.out[i]) continue;
    if (++shown > 6) return;
    const char* sec = "start";
    std::size_t sec0 = 0;
    for (const auto& m : b.marks)
        if (m.first <= i) {
            sec = m.second;
            sec0 = m.first;
        }
    std::printf("  first difference at word %zu (section '%s' + %zu): %llu vs %llu\n", i, sec, i - sec0,
                (unsigned long long)(i < a.out.size() ? a.out[i] : 0),
                (unsigned long long)(i < b.out.size() ? b.out[i] : 0));
  }
  for (const auto& m : b.marks)
    if (std::string(m.second) == "failing batch ids")
      for (int k = 0; k < 6; ++k) std::printf("    sid[%d] = %llu\n", k, (unsigned long long)b.out[m.first + k]);
}

// One workload in the style of proj/tests/test_table_batch.cpp:291-328.
template <class NS>
Trace run(std::uint64_t seed, int mode) {
    Trace tr;
    mpzch::SplitMix64 rng(seed);
    typename NS::Config cfg = NS::Config::even(200 + rng.next_below(800), 1 + rng.next_below(6),
                                               1 + rng.next_below(16), rng.next(), 4, rng.next());
    typename NS::Table table(cfg);
    typename NS::Ttl ttl;
    ttl.default_ttl_seconds = 15;
    ttl.per_feature_ttl = {{1, 4}};
    const typename NS::Policy pol = mode == 0   ? NS::Policy::disabled()
                                    : mode == 1 ? NS::Policy::lru()
                                                : NS::Policy::ttl(ttl);
    mpzch::DistinctIdStream ids(rng.next());
    std::uint64_t now = 1;
    std::vector<std::uint64_t> last_rows;
    for (int b = 0; b < 25; ++b) {
        now += rng.next_below(5);
        typename NS::Batch batch;
        batch.now = now;
        const std::uint64_t len = 1 + rng.next_below(400);
        for (std::uint64_t k = 0; k < len; ++k)
            batch.ids.push_back({ids.at(rng.next_below(1500)), static_cast<std::uint32_t>(rng.next_below(3))});
        try {
            last_rows.clear();
            for (const auto& r : NS::pb(table, batch, pol)) {
                last_rows.push_back(r.slot);
                tr.out.push_back(r.slot);
                tr.out.push_back(r.evicted);
                tr.out.push_back(static_cast<std::uint64_t>(r.outcome));
            }
        } catch (const std::exception& e) {
            tr.error = e.what();
            return tr;
        }
    }
    // a training step on the last batch's rows (repeated rows compound in order), its dirty
    // set, and a step that fails on its second row after updating the first
    auto bits = [&tr](float f) {
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        tr.out.push_back(u);
    };
    std::vector<float> grads(last_rows.size() * table.dim());
    for (float& g : grads) g = static_cast<float>(rng.next_unit() - 0.5);
    // publication: the .mpzc image byte for byte, then a delta source cut after the training
    // step (rows, identities, weights of every dirtied row)
    const std::vector<std::uint8_t> img = NS::snap(table);
    tr.out.push_back(img.size());
    for (std::size_t i = 0; i < img.size(); i += 8) {
        std::uint64_t w = 0;
        std::memcpy(&w, img.data() + i, std::min<std::size_t>(8, img.size() - i));
        tr.out.push_back(w);
    }
    typename NS::Delta src(table, NS::cks(img));
    const auto cursor = table.make_cursor();
    table.sgd_step(last_rows, grads, 0.05f, 0.9f);
    {
        const auto log = src.cut();
        tr.out.push_back(log.base_checksum);
        tr.out.push_back(log.sequence);
        tr.out.push_back(log.records.size());
        for (const auto& r : log.records) {
            tr.out.push_back(r.global_row);
            tr.out.push_back(r.identity);
            for (float v : r.weights) bits(v);
        }
    }
    for (float v : table.gather(last_rows)) bits(v);
    for (std::uint64_t r : last_rows) {
        for (float v : table.momentum_row(r)) bits(v);
        tr.out.push_back(table.row_trained(r));
    }
    for (auto r : table.dirty_rows_since(cursor)) tr.out.push_back(r);
    const std::vector<std::uint64_t> bad_rows = {last_rows[0], table.total_rows()};
    try {
        table.sgd_step(bad_rows, std::vector<float>(2 * table.dim(), 0.25f), 0.1f, 0.5f);
    } catch (const std::out_of_range& e) {
        tr.out.push_back(0xE77);
    }
    for (float v : table.gather(std::vector<std::uint64_t>{last_rows[0]})) bits(v);
    for (std::uint32_t s = 0; s < table.num_shards(); ++s) {
        for (auto v : NS::ident(table, s)) tr.out.push_back(v);
        for (auto v : NS::meta(table, s)) tr.out.push_back(v);
    }
    // error path: an invalid id names its batch position, nothing is mutated
    typename NS::Batch bad;
    bad.now = now;
    bad.ids = {{1, 0}, {1ull << 63, 0}};
    try {
        NS::pb(table, bad, pol);
    } catch (const std::invalid_argument& e) {
        tr.error = e.what();
    }
    return tr;
}

// The row-sharded table: the same batches through mpzch_b200::ShardedMpzchTable
// (G ranks, the device-side protocol) must give exactly what the reference's single-process
// process_batch gives -- every position's result, every shard's identities and metadata, and the
// invalid-id error with its global position.
template <class NS>
Trace run_sharded(std::uint64_t seed, int mode) {
    Trace tr;
    mpzch::SplitMix64 rng(seed);
    const std::uint32_t S = 4 << rng.next_below(2);  // 4 or 8 logical shards
    const std::uint32_t G = 2 << rng.next_below(2);  // 2 or 4 ranks
    typename NS::Config cfg = NS::Config::even(S * (150 + rng.next_below(300)), S, 1 + rng.next_below(24),
                                               rng.next(), 0, rng.next());
    auto table = NS::sharded(cfg, G);
    typename NS::Ttl ttl;
    ttl.default_ttl_seconds = 12;
    ttl.per_feature_ttl = {{2, 3}};
    const typename NS::Policy pol = mode == 0   ? NS::Policy::disabled()
                                    : mode == 1 ? NS::Policy::lru()
                                                : NS::Policy::ttl(ttl);
    mpzch::DistinctIdStream ids(rng.next());
    std::uint64_t now = 1;
    tr.mark("sharded batches");
    for (int b = 0; b < 12; ++b) {
        now += rng.next_below(6);
        typename NS::Batch batch;
        batch.now = now;
        const std::uint64_t len = 1 + rng.next_below(900);
        for (std::uint64_t k = 0; k < len; ++k)
            batch.ids.push_back({ids.at(rng.next_below(cfg.shard_capacities[0] * S + 200)),
                                 static_cast<std::uint32_t>(rng.next_below(3))});
        try {
            for (const auto& r : NS::pb(*table, batch, pol)) {
                tr.out.push_back(r.slot);
                tr.out.push_back(r.evicted);
                tr.out.push_back(static_cast<std::uint64_t>(r.outcome));
            }
        } catch (const std::exception& e) {
            tr.error = e.what();
            return tr;
        }
    }
    tr.mark("sharded state");
    for (std::uint32_t s = 0; s < S; ++s) {
        for (auto v : NS::ident(*table, s)) tr.out.push_back(v);
        for (auto v : NS::meta(*table, s)) tr.out.push_back(v);
    }
    typename NS::Batch bad;
    bad.now = now;
    for (int k = 0; k < 40; ++k) bad.ids.push_back({ids.at(5000 + k), 0});
    bad.ids[29].id = 1ull << 63;  // in a later rank's slice: every rank reports position 29
    try {
        NS::pb(*table, bad, pol);
    } catch (const std::invalid_argument& e) {
        tr.error = e.what();
    }
    return tr;
}

// The rest of the kept surface: layout() / shard_config(s), dedup, the per-shard
// entry process_shard_batch (repeated ids probe again; a bad metadata word stops the loop after
// the earlier positions took effect), reset_row, embeddings(), state_equals.
template <class NS>
Trace run_surface(std::uint64_t seed, int mode) {
    Trace tr;
    mpzch::SplitMix64 rng(seed);
    typename NS::Config cfg = NS::Config::even(300 + rng.next_below(700), 1 + rng.next_below(5),
                                               2 + rng.next_below(12), rng.next(), 8, rng.next());
    typename NS::Table table(cfg), twin(cfg);
    typename NS::Ttl ttl;
    ttl.default_ttl_seconds = 9;
    ttl.per_feature_ttl = {{2, 3}};
    const typename NS::Policy pol = mode == 0   ? NS::Policy::disabled()
                                    : mode == 1 ? NS::Policy::lru()
                                                : NS::Policy::ttl(ttl);
    const auto& L = table.layout();
    tr.out.push_back(L.num_shards());
    tr.out.push_back(L.total_rows());
    tr.out.push_back(L.seed);
    for (auto v : L.shard_offsets) tr.out.push_back(v);
    for (std::uint32_t s = 0; s < table.num_shards(); ++s) {
        const auto& sc = table.shard_config(s);
        tr.out.push_back(sc.capacity);
        tr.out.push_back(sc.max_probe);
        tr.out.push_back(sc.shard_id);
        tr.out.push_back(sc.seed);
    }
    try {
        (void)table.shard_config(table.num_shards());
    } catch (const std::out_of_range& e) {
        tr.error += std::string(e.what()) + "|";
    }
    mpzch::DistinctIdStream ids(rng.next());
    tr.mark("dedup");
    // dedup on (id, feature) with its inverse, then its first-bad-position error
    std::vector<typename NS::Entry> entries;
    for (int k = 0; k < 300; ++k)
        entries.push_back({ids.at(rng.next_below(120)), static_cast<std::uint32_t>(rng.next_below(3))});
    const auto d = NS::dd(entries);
    tr.out.push_back(d.uniques.size());
    for (const auto& u : d.uniques) {
        tr.out.push_back(u.id);
        tr.out.push_back(u.feature);
    }
    for (auto i : d.inverse) tr.out.push_back(i);
    entries[17].id = ~0ull;
    entries[41].id = 1ull << 63;
    try {
        (void)NS::dd(entries);
    } catch (const std::invalid_argument& e) {
        tr.error += std::string(e.what()) + "|";
    }
    // per-shard batches in several rounds (ids routed with shard_of, repeats included)
    std::uint64_t now = 1;
    std::vector<std::uint64_t> rows;
    tr.mark("shard batches");
    for (int round = 0; round < 6; ++round) {
        now += 1 + rng.next_below(4);
        for (std::uint32_t s = 0; s < table.num_shards(); ++s) {
            std::vector<std::uint64_t> sid, smeta;
            for (int k = 0; k < 400 && sid.size() < 60; ++k) {
                const std::uint64_t id = ids.at(rng.next_below(900));
                if (NS::shard(id, L) != s) continue;
                sid.push_back(id);
                smeta.push_back(NS::meta(pol, now, static_cast<std::uint32_t>(rng.next_below(3))));
            }
            std::vector<typename NS::Result> out(sid.size());
            table.process_shard_batch(s, sid, smeta, now, pol, out);
            twin.process_shard_batch(s, sid, smeta, now, pol, out);
            for (const auto& r : out) {
                tr.out.push_back(r.slot);
                tr.out.push_back(r.evicted);
                tr.out.push_back(static_cast<std::uint64_t>(r.outcome));
                rows.push_back(r.slot);
            }
        }
    }
    // a metadata word make_metadata could not produce, at position 3 of a shard batch: the
    // first three positions take effect and have results, then invalid_argument
    tr.mark("bad metadata shard batch");
    {
        std::vector<std::uint64_t> sid, smeta;
        for (int k = 0; sid.size() < 6; ++k) {
            const std::uint64_t id = ids.at(5000 + k);
            if (NS::shard(id, L) != 0) continue;
            sid.push_back(id);
            smeta.push_back(NS::meta(pol, now, 0));
        }
        smeta[3] = mode == 2 ? now : now + 1;
        tr.mark("failing batch ids");
        for (auto v : sid) tr.out.push_back(v);
        std::vector<typename NS::Result> out(sid.size(), typename NS::Result{7, true, {}});
        try {
            table.process_shard_batch(0, sid, smeta, now, pol, out);
        } catch (const std::invalid_argument& e) {
            tr.error += std::string(e.what()) + "|";
        }
        for (const auto& r : out) {
            tr.out.push_back(r.slot);
            tr.out.push_back(static_cast<std::uint64_t>(r.outcome));
        }
        sid[1] = 1ull << 63;  // an invalid id stops at position 1
        try {
            twin.process_shard_batch(0, sid, smeta, now, pol, out);
        } catch (const std::invalid_argument& e) {
            tr.error += std::string(e.what()) + "|";
        }
        // an invalid id at position 300 of a 600-position batch: the reference validates each
        // 256-position chunk before probing it, so positions 0..255 take effect, 256.. do not
        {
            std::vector<std::uint64_t> lid, lmeta;
            for (int k = 0; lid.size() < 600; ++k) {
                const std::uint64_t id = ids.at(20000 + rng.next_below(2000));
                if (NS::shard(id, L) != 0) continue;
                lid.push_back(id);
                lmeta.push_back(NS::meta(pol, now, 0));
            }
            lid[300] = ~0ull;
            std::vector<typename NS::Result> lo(lid.size(), typename NS::Result{7, true, {}});
            try {
                twin.process_shard_batch(0, lid, lmeta, now, pol, lo);
            } catch (const std::invalid_argument& e) {
                tr.error += std::string(e.what()) + "|";
            }
            for (const auto& r : lo) {
                tr.out.push_back(r.slot);
                tr.out.push_back(static_cast<std::uint64_t>(r.outcome));
            }
            lid[300] = ids.at(1);
            lmeta[290] = mode == 2 ? now : now + 1;  // a bad metadata word stops at its position
            try {
                twin.process_shard_batch(0, lid, lmeta, now, pol, lo);
            } catch (const std::invalid_argument& e) {
                tr.error += std::string(e.what()) + "|";
            }
            for (const auto& r : lo) tr.out.push_back(r.slot);
        }
        try {
            std::vector<typename NS::Result> o2(1);
            twin.process_shard_batch(table.num_shards(), std::vector<std::uint64_t>{1},
                                     std::vector<std::uint64_t>{now}, now, pol, o2);
        } catch (const std::out_of_range& e) {
            tr.error += std::string(e.what()) + "|";
        }
    }
    // training on some rows, then resets; the view of the embeddings; state_equals
    tr.mark("table identities after the failing shard batches");
    for (std::uint32_t s = 0; s < table.num_shards(); ++s)
        for (auto v : NS::ident(table, s)) tr.out.push_back(v);
    tr.mark("twin identities after the failing shard batches");
    for (std::uint32_t s = 0; s < table.num_shards(); ++s)
        for (auto v : NS::ident(twin, s)) tr.out.push_back(v);
    tr.mark("sgd / reset / state_equals");
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    std::vector<std::uint64_t> some(rows.begin(), rows.begin() + std::min<std::size_t>(rows.size(), 16));
    std::vector<float> g(some.size() * table.dim());
    for (float& x : g) x = static_cast<float>(rng.next_unit() - 0.5);
    table.sgd_step(some, g, 0.1f, 0.5f);
    twin.sgd_step(some, g, 0.1f, 0.5f);
    tr.out.push_back(table.state_equals(twin));
    const std::uint64_t untouched = table.total_rows() - 1 - rng.next_below(table.total_rows() / 2);
    if (!std::binary_search(some.begin(), some.end(), untouched)) {
        table.reset_row(untouched);  // a never-trained row redraws its own initial values
        tr.out.push_back(table.state_equals(twin));
    }
    table.reset_row(some[0]);
    tr.out.push_back(table.state_equals(twin));
    tr.out.push_back(table.row_trained(some[0]));
    tr.out.push_back(table.row_trained(some[1]));
    try {
        table.reset_row(table.total_rows());
    } catch (const std::out_of_range& e) {
        tr.error += std::string(e.what()) + "|";
    }
    auto bits = [&tr](float f) {
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        tr.out.push_back(u);
    };
    tr.mark("embeddings view");
    const auto& emb = table.embeddings();
    tr.out.push_back(emb.rows());
    tr.out.push_back(emb.dim());
    tr.out.push_back(emb.weights_count());
    for (float v : emb.row(some[0])) bits(v);
    for (float v : emb.row(some[1])) bits(v);
    for (float v : emb.momentum_row(some[0])) bits(v);
    for (float v : emb.momentum_row(some[1])) bits(v);
    tr.out.push_back(emb.trained(some[1]));
    tr.mark("gather");
    for (float v : emb.gather(some)) bits(v);
    tr.mark("row_identity / identities / metadata");
    for (std::uint64_t r = 0; r < table.total_rows(); r += 37) tr.out.push_back(table.row_identity(r));
    for (std::uint32_t s = 0; s < table.num_shards(); ++s) {
        for (auto v : NS::ident(table, s)) tr.out.push_back(v);
        for (auto v : NS::meta(table, s)) tr.out.push_back(v);
    }
    return tr;
}

int main(int argc, char** argv) {
    const int cases = argc > 1 ? std::atoi(argv[1]) : 60;
    int bad = 0;
    std::uint64_t checked = 0;
    for (int c = 0; c < cases; ++c) {
        const Trace a = run<Ref>(0x5eed0000 + c, c % 3);
        const Trace b = run<Gpu>(0x5eed0000 + c, c % 3);
        if (a.out != b.out || a.error != b.error) {
            std::printf("MISMATCH case %d (mode %d): %zu vs %zu words, '%s' vs '%s'\n", c, c % 3,
                        a.out.size(), b.out.size(), a.error.c_str(), b.error.c_str());
            report_diff(a, b);
            ++bad;
        }
        checked += a.out.size();
        const Trace sa = run_surface<Ref>(0x5afe0000 + c, c % 3);
        const Trace sb = run_surface<Gpu>(0x5afe0000 + c, c % 3);
        if (sa.out != sb.out || sa.error != sb.error) {
            std::printf("MISMATCH surface case %d (mode %d): %zu vs %zu words, '%s' vs '%s'\n", c, c % 3,
                        sa.out.size(), sb.out.size(), sa.error.c_str(), sb.error.c_str());
            report_diff(sa, sb);
            ++bad;
        }
        checked += sa.out.size();
        if (c < 24) {
            const Trace ha = run_sharded<Ref>(0x5a4d0000 + c, c % 3);
            const Trace hb = run_sharded<Gpu>(0x5a4d0000 + c, c % 3);
            if (ha.out != hb.out || ha.error != hb.error) {
                std::printf("MISMATCH sharded case %d (mode %d): %zu vs %zu words, '%s' vs '%s'\n", c, c % 3,
                            ha.out.size(), hb.out.size(), ha.error.c_str(), hb.error.c_str());
                report_diff(ha, hb);
                ++bad;
            }
            checked += ha.out.size();
        }
    }
    std::printf("%s: %d cases, %llu result/state words compared, %d mismatches\n",
                bad ? "FAIL" : "PASS", cases, (unsigned long long)checked, bad);
    return bad ? 1 : 0;
}
