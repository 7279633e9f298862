// table.hpp -- host-side state of one device-resident MPZCH table handle.
//
// Mirrors the reference's MpzchTable members (proj/include/mpzch/table.hpp:115-131)
// with the arrays resident in HBM: one contiguous identity array and one
// metadata array in global-row order (shard s owns [offset[s], offset[s+1])),
// so a global row is a direct index and a probe window never leaves its
// shard's segment except through the explicit wrap at the shard end.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mpzch_b200.h"
#include "common.cuh"

namespace mpzch_b200 {

// Thrown inside the library, mapped to a status + thread-local text at the C boundary.
struct Error {
    mpzch_status code;
    std::string msg;
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what);

#define MPZCH_CUDA(call)                                   \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) ::mpzch_b200::throw_cuda(e_, #call); \
    } while (0)

// Reusable device scratch, grown monotonically (the reference keeps
// thread_local BatchScratch for the same reason, batch_engine.cpp:112-129).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t want);
    template <class T> T* as() const { return static_cast<T*>(p); }
    ~DevBuf();
};

// Small pinned block the host reads once per batch.
struct BatchCounters {
    BatchErr err;
    unsigned int new_count;      // positions appended to the new list by the probe
    unsigned int entry_count;    // distinct new ids (claim participants)
    unsigned int reset_count;    // rows to reset
    unsigned int evicted_count;  // canonical evicted-list length
    unsigned long long found, inserted, evicted, collision;  // per position
    unsigned int overflow_list;  // claim-log overflow (defensive)
    unsigned int pad;
    unsigned int dup_items;      // fast path: new-list items whose id was already in the id table
    unsigned int lru_abort;      // LRU on the fast path: an eviction the claim path cannot place
                                 // exactly -> the batch reverts and takes the rounds path
    unsigned int lru_evict;      // LRU on the fast path: entries whose window is full (evictors)
    unsigned long long bad_id;   // lookups: the id at err.bad_pos (the exception text needs it)
    unsigned long long id_sectors, meta_sectors;  // sectors the probe kernel read
    // rounds path (device-driven): pending count per round parity, new suspects per closure
    // step parity, lowest rank among the unmarked last-step suspects, rounds run, uniques left
    // for the ordered kernel
    unsigned int r_cnt[2], r_newc[3], r_minrank, r_rounds, r_left, r_iters;
    unsigned int r_marked, r_checked;  // closure steps / windows marked / range checks (diagnostics)
    unsigned int deferred;             // TTL probe: walks handed to the resume pass
    unsigned int ldeferred;            // synchronous lookups: walks handed to the resume pass
    unsigned long long n_live;         // positions of the batch when only the device knows them
                                       // (row-sharded owner: the received count); ~0 = kernel arg
    unsigned int path_taken;           // 0: the claim path; 1: the ordered / rounds path ran
                                       // (an LRU claim attempt that aborted, decided on the device)
    unsigned int pad2;
};

// sgd_step scratch counters (train.cu)
struct SgdCounters {
    unsigned long long bad;  // first out-of-range position (~0: none)
    unsigned dup, dup_total, dup_entries, pad;
};

struct Policy {
    int mode = 0;
    uint64_t default_ttl = 0;
    std::vector<uint32_t> keys;
    std::vector<uint64_t> ttls;
    uint64_t ttl_for(uint32_t f) const {
        for (size_t i = 0; i < keys.size(); ++i)
            if (keys[i] == f) return ttls[i];
        return default_ttl;
    }
};

class Table {
public:
    Table(const uint64_t* caps, uint32_t num_shards, uint32_t max_probe, uint64_t seed,
          uint32_t dim, uint64_t init_seed, int device, uint32_t shard_lo = 0,
          uint32_t shard_hi = ~0u);
    ~Table();

    // layout (TableLayout, proj/include/mpzch/shard_router.hpp:13-29)
    std::vector<uint64_t> caps, offsets;
    uint64_t total = 0;
    uint32_t S = 0, P = 0, dim = 0;
    uint64_t seed = 0, init_seed = 0;
    int device = 0;
    // row-sharded mode: this handle holds logical shards [shard_lo, shard_hi), i.e. global
    // rows [row_lo, row_hi); the device pointers in `dev` are offset so that global row
    // numbers index them directly (identity/metadata allocations start 4-row aligned)
    uint32_t shard_lo = 0, shard_hi = 0;
    uint64_t row_lo = 0, row_hi = 0, row_base = 0;
    uint64_t held_rows() const { return row_hi - row_lo; }
    uint64_t gen_clock = 1;  // MpzchTable::generation_clock_
    bool hole_free = true;   // SURVEY A.2 invariant; false after raw imports
    bool resets_pending = false;  // MPZCH_RESET_DEFERRED: a batch may have marked rows pending
    int path_override = MPZCH_PATH_AUTO;
    uint64_t lru_fallbacks = 0;  // LRU batches that needed an eviction (claim attempt reverted)
    uint32_t lru_backoff = 0, lru_skip_left = 0;  // claim-attempt backoff after evictions
    bool lru_recent_abort = false;  // the last decided LRU attempt aborted (gated decision next)
    mpzch_batch_stats last{};
    uint64_t launches = 0;
    bool profiling = false;
    mpzch_profile prof{};
    cudaEvent_t* ev = nullptr;  // the current batch slot's profiling events

    // ---- in-flight batches (mpzch_process_batch_device_async): a ring of counter blocks,
    // each with its completion event; results of completed batches kept by ticket
    static constexpr int kRing = 8, kResults = 64;
    struct Slot {
        bool busy = false, fast = false, overflow_all = false, profiled = false;
        uint32_t path = 0, rounds = 0;
        uint64_t ticket = 0, n = 0;
        cudaEvent_t done = nullptr;
        bool lookup = false;  // a batched read-only lookup (mpzch_lookup_device_async)
        bool lru_try = false; // an LRU claim attempt with the gated rounds path behind it
        cudaEvent_t ev[8] = {};
    };
    struct Result {
        uint64_t ticket = ~0ull;
        mpzch_status status = MPZCH_OK;
        std::string msg;
        mpzch_batch_stats stats{};
        uint64_t evicted_n = 0;
    };
    Slot slots[kRing];
    Result results[kResults];
    uint64_t next_ticket = 1;
    cudaStream_t last_stream = nullptr;
    uint64_t last_ticket = 0;
    BatchCounters* d_ring = nullptr;  // kRing blocks
    BatchCounters* h_ring = nullptr;  // pinned
    BatchCounters* d_aux = nullptr;   // synchronous helpers (lookup, validate, dirty rows)
    BatchCounters* d_alt = nullptr;   // the gated ordered / rounds path's counters (LRU attempts)
    BatchCounters* h_aux = nullptr;

    // resident arrays
    uint64_t* ident = nullptr;
    uint64_t* meta = nullptr;
    uint8_t* tags = nullptr;  // P >= kTagMinProbe: identity tags from tag_base (128-row aligned)
    float* weights = nullptr;
    float* momentum = nullptr;
    uint32_t* trained = nullptr;  // bitmap: one bit per held row
    uint64_t* row_gen = nullptr;
    ShardDev* d_shards = nullptr;
    TableDev dev{};

    cudaStream_t stream = nullptr;
    BatchCounters* h_ctr = nullptr;  // the current batch's counters (pinned / device)
    BatchCounters* d_ctr = nullptr;

    // scratch
    DevBuf s_newpos, s_newid, s_newa, s_newm, s_newent;  // new-list (fast path)
    DevBuf s_dupl;                                   // new-list items whose id an earlier item inserted
    DevBuf s_defer;  // TTL probe: (position, offset, first expired) of walks handed to the resume pass
    // synchronous lookups (mpzch_lookup[_device], lookup_gather): their own hand-over list and
    // a lock, so concurrent const lookups on one handle never share scratch or the error word
    DevBuf s_ldefer, l_ids, l_oslot, l_ooc;
    DevBuf sb_buf;  // process_shard_batch / reset_row / gather staging
    DevBuf pend_map;  // MPZCH_RESET_DEFERRED: reset-pending bit per held row (dev.pend_bits)
    std::mutex lookup_mu;
    DevBuf s_tent;                                   // dense 64-byte entry records (fast path)
    DevBuf s_hkey;                                   // hash index of the new ids: 16-byte keys
    uint64_t tcap = 0;                               // allocated hash-index capacity (pow2)
    uint64_t epoch = 0;                              // id-table batch epoch (0 = never used)
    uint64_t fast_ready = 0;                         // largest n the fast scratch is ready for
    DevBuf s_reset;                                  // rows to reset
    DevBuf s_evflag, s_evslot, s_blk;                // evicted-list compaction
    DevBuf s_ids, s_feats, s_oslot, s_ooc, s_oev;    // staging for host-buffer calls
    DevBuf s_featk, s_featv;                         // per-feature TTL map
    DevBuf s_grads;                                  // staging for host-buffer sgd_step
    // ordered path
    DevBuf o_key, o_min, o_posent, o_flag, o_upos, o_entu, o_ushard, o_umeta, o_uslot, o_uoc, o_todo;
    uint64_t ocap = 0;
    // rounds path: epoch-keyed reservation marks (<= 2^27 words each, aliased)
    DevBuf r_mark_any, r_mark_id, r_mark_win, r_pend, r_next, r_slot, r_oc, r_d, r_susp;
    uint64_t r_mark_mask = 0;  // mark arrays alias slots modulo their size (sound: more suspects)
    uint32_t mark_epoch = 0;
    // sgd_step (train.cu): row hash, occurrence lists
    DevBuf g_key, g_cnt, g_base, g_pe, g_pr, g_list, g_dupent, g_ctr;
    uint64_t g_cap = 0;
    // publish / dirty rows (table.cu, publish.cu)
    DevBuf p_flags, p_rows, p_blk, p_ids, p_w, p_rec;
    // per-feature TTL on the fast path: (id, feature) groups and per-slot last writers
    DevBuf mf_tab, mf_ent, sl_tab, sl_ent;
    uint64_t mf_cap = 0;
    // route (route.cu)
    DevBuf rt_s2p, rt_cnt, rt_tot;
    std::vector<uint8_t> rt_map;
    // the last count-only route (mpzch_route_count_device), which a scatter must match
    const uint64_t* rt_ids = nullptr;
    uint64_t rt_n = 0, rt_nchunks = 0;
    uint32_t rt_parts = 0;

    void ensure_fast_scratch(uint64_t n);
    void ensure_pf_scratch(uint64_t n);  // per-feature TTL last-writer tables
    void ensure_ordered_scratch(uint64_t n);
};

// kernel entry points (each .cu file), all enqueued on t.stream / stream
void launch_init_table(Table& t);
// eager: resets the listed rows; deferred (t.dev.deferred): marks them reset-pending
void launch_reset_rows(Table& t, const uint64_t* rows, const unsigned int* count, cudaStream_t st);
// trained flags (bitmap) <-> the reference's bytes (synchronous on t.stream)
void copy_trained_bytes(Table& t, uint64_t row0, uint64_t n, uint8_t* host_out);
void set_trained_flag(Table& t, uint64_t row, bool v);
// writes every pending reset (deferred mode) before a reader that is not reset-aware
void flush_resets(Table& t, cudaStream_t st);
void launch_write_slots(Table& t, const uint64_t* gslots, const uint64_t* ids, const uint64_t* metas,
                        uint64_t n, cudaStream_t st);
bool run_hole_check(Table& t);
// lookup into a ring counter block (error word + the first bad id), all enqueued on st
void launch_lookup_async(Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots, uint8_t* out_oc,
                         BatchCounters* c, cudaStream_t st);
// ldefer (nullable): scratch for the walk hand-over, reserved only when the hand-over runs
void run_lookup(const Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots,
                uint8_t* out_oc, BatchErr* err, cudaStream_t st, DevBuf* ldefer = nullptr,
                unsigned* dcount = nullptr);
void run_lookup_gather(const Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots,
                       uint8_t* out_oc, float* out_rows, BatchErr* err, cudaStream_t st);
// publish.cu: CRC-32 (raw register from 0; finish() applies the reference's init/final xor)
uint32_t crc32_raw_device(const uint8_t* data, uint64_t n, cudaStream_t st, int device);
uint32_t crc32_raw_host(uint32_t raw, const uint8_t* p, uint64_t n);
uint32_t crc32_shift(uint32_t raw, uint64_t n);
uint32_t crc32_finish(uint32_t raw, uint64_t n);
void launch_pack_delta(Table& t, const uint64_t* rows, const unsigned* count, uint64_t max_n,
                       uint8_t* out, cudaStream_t st);

// returns the first out-of-range position (~0 if none); synchronous on st
uint64_t run_sgd_step(Table& t, const uint64_t* rows, uint64_t n, const float* grads, float lr,
                      float beta, cudaStream_t st);
void run_gather_rows(const Table& t, const uint64_t* rows, uint64_t n, uint64_t* out_ids,
                     float* out_w, cudaStream_t st);

struct BatchArgs {
    const uint64_t* ids;
    const uint32_t* feats;
    uint64_t n;
    uint64_t now;
    uint64_t uniform_meta;      // meta value when every unique shares it
    bool uniform;               // all metadata writes carry the same value
    bool overflow_all;          // uniform TTL expiry overflows: validate, then fail
    const Policy* pol;
    const uint32_t* d_featk;    // per-feature map on device
    const uint64_t* d_featv;
    uint64_t* out_slots;
    uint8_t* out_oc;
    uint64_t* out_ev;
    uint64_t ev_cap;
    uint8_t* out_mark = nullptr;  // optional: 1 at the first position of every Evicted unique
    bool per_feature = false;     // TTL with differing per-feature values on the fast path:
                                  // metadata written by the last-writer pass (remap_fast.cu)
    uint32_t nk = 0;              // per-feature map size
    // row-sharded owner (sharded.cu): n is only an upper bound; the batch's errors and its
    // received count come from this device state (k_sh_adopt replaces validation), and the
    // evicted flags are left set for the return scatter instead of compacted here
    const void* sh_state = nullptr;
    // LRU claim attempt followed on the same stream by the ordered / rounds path, which runs only
    // if the attempt aborted (read from this counter block on the device: no host round trip)
    const BatchCounters* gate_ctr = nullptr;
};

// table.cu: the batch machinery the row-sharded layer (sharded.cu) reuses
Policy parse_policy(const mpzch_policy* p);
uint64_t enqueue_batch(Table& t, const uint64_t* ids, const uint32_t* feats, uint64_t n, uint64_t now,
                       const Policy& pol, uint64_t* out_slots, uint8_t* out_oc, uint64_t* out_ev,
                       uint64_t ev_cap, cudaStream_t st, uint8_t* out_mark = nullptr, bool host_waits = false);
uint64_t wait_batch(Table& t, uint64_t ticket);
// force-load kernels (lazy module loading can wait for running work; see common.cuh)
void preload_remap_kernels();
void preload_ordered_kernels();
void preload_rounds_kernels();
void preload_row_kernels();
void preload_route_kernels();
void preload_all_kernels();
// C-ABI error mapping: runs f, maps Error / bad_alloc / exceptions to a status + mpzch_last_error
mpzch_status run_guarded(const std::function<void()>& f);

// one-metadata-value / per-feature decision and the per-feature map upload of a batch
// (make_metadata, eviction.cpp:20-30); shared by enqueue_batch and the row-sharded owner
void fill_policy_args(Table& t, const Policy& pol, uint64_t now, const uint32_t* feats, BatchArgs& a,
                      cudaStream_t st);
// count-only route (route.cu) without a host sync: per-chunk offsets and per-part totals
// stay on the device (t.rt_cnt, t.rt_tot); the shard -> part map must be uploaded already
// bad (nullable): the validation pass fused in -- atomicMin of the first invalid position
void enqueue_route_count(Table& t, const uint64_t* ids, uint64_t n, uint32_t parts, cudaStream_t st,
                         unsigned long long* bad = nullptr);
void upload_route_map(Table& t, const uint32_t* shard_to_part, uint32_t parts);

// enqueue the whole batch; counters land in t.h_ctr after the stream syncs
void enqueue_fast_batch(Table& t, const BatchArgs& a, cudaStream_t st);
void enqueue_ordered_batch(Table& t, const BatchArgs& a, cudaStream_t st, bool rounds = false);
// after a gated ordered path run on t.d_ctr: its counters replace `attempt`'s if it ran
void adopt_gated_counters(Table& t, BatchCounters* attempt, const BatchCounters* alt, cudaStream_t st);
void enqueue_rounds(Table& t, const BatchArgs& a, cudaStream_t st, uint8_t* todo);
void ensure_rounds_scratch(Table& t, uint64_t n, cudaStream_t st);
// gate (nullable): device word, 0 = no evicted flag can be set (LRU batches without evictors);
// slots (nullable): the slot of flagged index i (the fast path: the batch's out_slots, flags by
// position), else the rounds / ordered paths' per-unique s_evslot
void enqueue_compact_evicted(Table& t, uint64_t n, uint64_t* out_ev, uint64_t ev_cap, cudaStream_t st,
                             const unsigned* gate = nullptr, const uint64_t* slots = nullptr);
void run_route(Table& t, const uint64_t* ids, uint64_t n, const uint32_t* shard_to_part,
               uint32_t parts, uint32_t* perm, uint64_t* counts, cudaStream_t st);
void run_validate(Table& t, const uint64_t* ids, uint64_t n, cudaStream_t st);
// peer-memory routing (route.cu): addresses are device addresses valid in this process (local,
// P2P or IPC-mapped peer memory)
struct PeerScatter {
    const uint64_t* ids_to;     // [parts] u64 id arrays of the owners' receive buffers
    const uint64_t* feats_to;   // [parts] u32 feature arrays (0: no features)
    const uint64_t* src_to;     // [parts] u32 source-position arrays
    const uint64_t* offset;     // [parts] this rank's first index in each owner's buffers
    // row-sharded device protocol: offsets read on the device (overrides `offset`), a gate word
    // (nonzero: the batch failed, store nothing) and a system-scope fence after the stores
    const uint64_t* dev_offset = nullptr;
    const uint64_t* gate = nullptr;
};
void run_route_scatter(Table& t, const uint64_t* ids, const uint32_t* feats, uint64_t n,
                       uint32_t parts, const PeerScatter& d, cudaStream_t st);
void run_return_scatter(uint64_t n_recv, const uint64_t* slots, const uint8_t* oc, const uint8_t* mark,
                        const uint32_t* src, uint32_t parts, const uint64_t* recv_offset,
                        const uint64_t* slots_to, const uint64_t* oc_to, const uint64_t* mark_to,
                        cudaStream_t st);

// surface.cu: process_shard_batch (one warp, positions in order; st = {first failing position,
// kind 1 id / 2 metadata, id}), dedup (returns the unique count; *bad_pos = first invalid
// position or ~0; synchronous), state_equals word compare (synchronous), row gather
void launch_shard_batch(Table& t, uint32_t shard, int mode, const uint64_t* ids, const uint64_t* metas,
                        uint64_t n, uint64_t now, uint64_t* out_slots, uint8_t* out_oc, uint64_t* reset_rows,
                        unsigned* reset_count, unsigned long long* st, cudaStream_t s);
uint64_t run_dedup(const uint64_t* ids, const uint32_t* feats, uint64_t n, uint64_t* uids, uint32_t* ufeats,
                   uint32_t* inverse, uint64_t* bad_pos, cudaStream_t st);
bool run_words_equal(const void* a, const void* b, uint64_t bytes, cudaStream_t st);
void run_gather_weights(const Table& t, const uint64_t* rows, uint64_t n, float* out, cudaStream_t st);

}  // namespace mpzch_b200

// The C-ABI handle (include/mpzch_b200.h): one device-resident table.
struct mpzch_table {
    mpzch_b200::Table* t;
};

namespace mpzch_b200 {

inline unsigned grid_for(uint64_t n, unsigned block, unsigned max_blocks = 148u * 32u) {
    uint64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (unsigned)g;
}

}  // namespace mpzch_b200
