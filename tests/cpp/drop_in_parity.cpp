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
};

struct Trace {
    std::vector<std::uint64_t> out;  // slot, evicted, outcome per position, then state
    std::string error;
};

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
            ++bad;
        }
        checked += a.out.size();
    }
    std::printf("%s: %d cases, %llu result/state words compared, %d mismatches\n",
                bad ? "FAIL" : "PASS", cases, (unsigned long long)checked, bad);
    return bad ? 1 : 0;
}
