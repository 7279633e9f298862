// table.cu -- the C-ABI (include/mpzch_b200.h) over the device-resident table.
//
// Host-side control flow of the reference calls it replaces:
//   MpzchTable ctor            proj/src/table.cpp:34-56
//   process_batch              proj/src/batch_engine.cpp:141-221 (error order :143-158)
//   MpzchTable::lookup         proj/src/table.cpp:150-156
//   MpzchTable::lookup_or_insert proj/src/table.cpp:98-110
//   make_cursor / dirty_rows_since proj/src/table.cpp:209-225
// Every error is detected before the first mutation and reported with the
// reference's exception category and what() text.
#include <cuda.h>  // CUresult / CUdeviceptr types only (driver entry point, no -lcuda)
#include <cuda_runtime.h>

#include <functional>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/mpzch_b200.h"
#include "common.cuh"
#include "compact.cuh"
#include "table.hpp"

#ifndef MPZCH_BUILD_INFO
#define MPZCH_BUILD_INFO "sm_100a"
#endif

namespace mpzch_b200 {

static thread_local std::string g_last_error;

void throw_cuda(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        throw Error{MPZCH_ENOMEM, std::string("device allocation failed: ") + what};
    throw Error{MPZCH_ECUDA, std::string(cudaGetErrorString(e)) + " in " + what};
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) MPZCH_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Resets the synchronous helpers' error block on the device: a pageable host->device copy
// would first wait for everything already queued on the stream.
__global__ void k_init_err(BatchErr* e) { *e = BatchErr{~0ull, 0, 0, ~0ull}; }
static void init_aux_err(Table& T, cudaStream_t st) {
    k_init_err<<<1, 1, 0, st>>>(&T.d_aux->err);
    ++T.launches;
}

// Grows geometrically (x1.5, 1 MiB granules): scratch sized by batch length must not be
// reallocated -- cudaFree synchronises the device -- every time the length creeps up.
void DevBuf::reserve(size_t want) {
    if (want <= bytes) return;
    size_t grow = std::max(want, bytes + bytes / 2);
    if (grow > (1u << 20)) grow = (grow + (1u << 20) - 1) & ~((size_t)(1u << 20) - 1);
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    MPZCH_CUDA(cudaMalloc(&p, grow));
    bytes = grow;
}

DevBuf::~DevBuf() {
    if (p) cudaFree(p);
}

static uint64_t pow2_at_least(uint64_t x) {
    uint64_t c = 1024;
    while (c < x) c <<= 1;
    return c;
}

Table::Table(const uint64_t* cap_in, uint32_t num_shards, uint32_t max_probe, uint64_t seed_in,
             uint32_t dim_in, uint64_t init_seed_in, int device_in, uint32_t lo, uint32_t hi) {
    // TableLayout::with_capacities shard_router.cpp:8-25, ShardConfig::validate probe_core.cpp:8-15
    if (num_shards == 0) throw Error{MPZCH_EINVAL, "layout needs at least one shard"};
    for (uint32_t s = 0; s < num_shards; ++s)
        if (cap_in[s] == 0) throw Error{MPZCH_EINVAL, "shard capacity must be >= 1"};
    for (uint32_t s = 0; s < num_shards; ++s)
        if (max_probe < 1 || max_probe > cap_in[s])
            throw Error{MPZCH_EINVAL, "max_probe must satisfy 1 <= max_probe <= capacity"};
    S = num_shards;
    P = max_probe;
    seed = seed_in;
    dim = dim_in;
    init_seed = init_seed_in;
    device = device_in;
    caps.assign(cap_in, cap_in + num_shards);
    offsets.assign(num_shards + 1, 0);
    for (uint32_t s = 0; s < S; ++s) offsets[s + 1] = offsets[s] + caps[s];
    total = offsets[S];
    if (hi == ~0u) hi = S;
    if (lo >= hi || hi > S) throw Error{MPZCH_ERANGE, "shard range out of range"};
    shard_lo = lo;
    shard_hi = hi;
    row_lo = offsets[lo];
    row_hi = offsets[hi];
    row_base = row_lo & ~15ull;  // identity/metadata lines are 128-byte aligned in global rows
    const uint64_t held = row_hi - row_lo;

    DeviceGuard g(device);
    MPZCH_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    MPZCH_CUDA(cudaMallocHost((void**)&h_ring, (kRing + 1) * sizeof(BatchCounters)));
    MPZCH_CUDA(cudaMalloc((void**)&d_ring, (kRing + 2) * sizeof(BatchCounters)));
    h_aux = h_ring + kRing;
    d_aux = d_ring + kRing;
    d_alt = d_ring + kRing + 1;
    h_ctr = h_ring;
    d_ctr = d_ring;
    for (auto& sl : slots) MPZCH_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    // identity/metadata start 16-row (128-byte line) aligned and are padded to whole lines, so
    // a line read (line_scan.cuh) at the first or last held slot stays in bounds
    const uint64_t padded = ((row_hi - row_base + 15) & ~15ull) + 16;
    MPZCH_CUDA(cudaMalloc((void**)&ident, padded * sizeof(uint64_t)));
    MPZCH_CUDA(cudaMalloc((void**)&meta, padded * sizeof(uint64_t)));
    MPZCH_CUDA(cudaMalloc((void**)&row_gen, held * sizeof(uint64_t)));
    MPZCH_CUDA(cudaMemsetAsync(ident, 0xff, padded * sizeof(uint64_t), stream));
    MPZCH_CUDA(cudaMemsetAsync(meta, 0, padded * sizeof(uint64_t), stream));
    MPZCH_CUDA(cudaMemsetAsync(row_gen, 0, held * sizeof(uint64_t), stream));
    // identity tags (common.cuh) for long windows: 128-row (one 128-byte tag line) aligned in
    // global rows and padded by a line, so the probe's tag-line reads stay in bounds
    const uint64_t tag_base = row_lo & ~127ull;
    if (P >= kTagMinProbe) {
        const uint64_t tag_rows = ((row_hi - tag_base + 127) & ~127ull) + 128;
        MPZCH_CUDA(cudaMalloc((void**)&tags, tag_rows));
        MPZCH_CUDA(cudaMemsetAsync(tags, 0, tag_rows, stream));
    }
    if (dim > 0) {
        MPZCH_CUDA(cudaMalloc((void**)&weights, held * dim * sizeof(float)));
        MPZCH_CUDA(cudaMalloc((void**)&momentum, held * dim * sizeof(float)));
        MPZCH_CUDA(cudaMalloc((void**)&trained, (held + 31) / 32 * 4));
        MPZCH_CUDA(cudaMemsetAsync(momentum, 0, held * dim * sizeof(float), stream));
        MPZCH_CUDA(cudaMemsetAsync(trained, 0, (held + 31) / 32 * 4, stream));
    }
    std::vector<ShardDev> hs(S);
    for (uint32_t s = 0; s < S; ++s) hs[s] = ShardDev{offsets[s], make_fastmod(caps[s])};
    MPZCH_CUDA(cudaMalloc((void**)&d_shards, S * sizeof(ShardDev)));
    MPZCH_CUDA(cudaMemcpyAsync(d_shards, hs.data(), S * sizeof(ShardDev), cudaMemcpyHostToDevice, stream));
    // global-row-indexed views of the held allocations
    dev.ident = ident - row_base;
    dev.meta = meta - row_base;
    dev.weights = weights ? weights - row_lo * dim : nullptr;
    dev.momentum = momentum ? momentum - row_lo * dim : nullptr;
    dev.trained = trained;  // bit (row - row_lo)
    dev.row_gen = row_gen - row_lo;
    dev.tag = tags ? tags - tag_base : nullptr;
    dev.row_lo = row_lo;
    dev.row_hi = row_hi;
    dev.shard_lo = shard_lo;
    dev.shard_hi = shard_hi;
    dev.shards = d_shards;
    dev.nshards = make_fastmod(S);
    dev.seed = seed;
    dev.init_seed = init_seed;
    dev.total = total;
    // draw_row's bound, embedding_store.cpp:14 (IEEE sqrt and division are exact-rounded on the host)
    dev.bound = dim ? std::ldexp(1.0 / std::sqrt(static_cast<double>(dim)), -52) : 0.0;
    dev.P = P;
    dev.dim = dim;
    launch_init_table(*this);
    // every kernel loaded now, once per device: lazy loading would put a one-off load (18 ms
    // for the LRU rounds path) into some batch's latency instead
    static std::mutex mu;
    static std::vector<int> loaded;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (std::find(loaded.begin(), loaded.end(), device) == loaded.end()) {
            preload_all_kernels();
            loaded.push_back(device);
        }
    }
    MPZCH_CUDA(cudaStreamSynchronize(stream));
}

Table::~Table() {
    DeviceGuard g(device);
    if (stream) cudaStreamSynchronize(stream);
    cudaFree(ident);
    cudaFree(meta);
    cudaFree(tags);
    cudaFree(row_gen);
    cudaFree(weights);
    cudaFree(momentum);
    cudaFree(trained);
    cudaFree(d_shards);
    cudaFree(d_ring);
    if (h_ring) cudaFreeHost(h_ring);
    for (auto& sl : slots) {
        if (sl.done) cudaEventDestroy(sl.done);
        for (auto& e : sl.ev)
            if (e) cudaEventDestroy(e);
    }
    if (stream) cudaStreamDestroy(stream);
}

void Table::ensure_fast_scratch(uint64_t n) {
    s_newpos.reserve(n * 4);
    s_newid.reserve(n * 8);
    s_newa.reserve(n * 4);
    s_newm.reserve(n * 4);
    s_newent.reserve(n * 4);
    s_dupl.reserve(n * 4);
    s_defer.reserve(n * 12);
    const uint64_t want = pow2_at_least(2 * n);
    if (want > tcap) {
        // hash index: epoch-tagged 16-byte keys (epoch 0 = empty); dense 64-byte entry records,
        // one per new-list item (their rank words are epoch-tagged too: zeroed once)
        s_hkey.reserve(want * 16);
        MPZCH_CUDA(cudaMemsetAsync(s_hkey.p, 0, want * 16, stream));
        tcap = want;
    }
    if (s_tent.bytes < std::max<uint64_t>(n, 1) * 64) {
        s_tent.reserve(std::max<uint64_t>(n, 1) * 64);
        MPZCH_CUDA(cudaMemsetAsync(s_tent.p, 0, s_tent.bytes, stream));
    }
    s_reset.reserve(n * 8);
    const size_t fl = ((n + 15) & ~15ull) + 16;
    if (s_evflag.bytes < fl) {  // zero the whole allocation: it may exceed fl
        s_evflag.reserve(fl);
        MPZCH_CUDA(cudaMemsetAsync(s_evflag.p, 0, s_evflag.bytes, stream));
    }
    s_evslot.reserve(n * 8);
    s_blk.reserve(((n + kCompactChunk - 1) / kCompactChunk + 1) * 4);
    if (n > fast_ready) {  // first use at this size: the memsets above must land first
        MPZCH_CUDA(cudaStreamSynchronize(stream));
        fast_ready = n;
    }
}

void Table::ensure_pf_scratch(uint64_t n) {
    mf_ent.reserve(n * 4);
    sl_ent.reserve(n * 4);
    const uint64_t want = pow2_at_least(2 * n);
    if (want > mf_cap) {  // 32-byte epoch-keyed records; epoch 0 = empty (t.epoch starts at 1)
        mf_tab.reserve(want * 32);
        sl_tab.reserve(want * 32);
        MPZCH_CUDA(cudaMemsetAsync(mf_tab.p, 0, mf_tab.bytes, stream));
        MPZCH_CUDA(cudaMemsetAsync(sl_tab.p, 0, sl_tab.bytes, stream));
        MPZCH_CUDA(cudaStreamSynchronize(stream));
        mf_cap = want;
    }
}

void Table::ensure_ordered_scratch(uint64_t n) {
    const uint64_t want = pow2_at_least(2 * n);
    if (want > ocap) {
        o_key.reserve(want * 16);
        o_min.reserve(want * 4);
        o_entu.reserve(want * 4);
        MPZCH_CUDA(cudaMemsetAsync(o_key.p, 0xff, want * 16, stream));
        MPZCH_CUDA(cudaMemsetAsync(o_min.p, 0xff, want * 4, stream));
        ocap = want;
    }
    o_posent.reserve(n * 4);
    const size_t fl = ((n + 15) & ~15ull) + 16;
    if (o_flag.bytes < fl) {
        o_flag.reserve(fl);
        MPZCH_CUDA(cudaMemsetAsync(o_flag.p, 0, o_flag.bytes, stream));
    }
    o_upos.reserve(n * 4);
    o_ushard.reserve(n * 4);
    o_umeta.reserve(n * 8);
    o_uslot.reserve(n * 8);
    o_uoc.reserve(n);
    s_reset.reserve(n * 8);
    if (s_evflag.bytes < fl) {  // zero the whole allocation: it may exceed fl
        s_evflag.reserve(fl);
        MPZCH_CUDA(cudaMemsetAsync(s_evflag.p, 0, s_evflag.bytes, stream));
    }
    s_evslot.reserve(n * 8);
    s_blk.reserve(((n + kCompactChunk - 1) / kCompactChunk + 1) * 4);
    MPZCH_CUDA(cudaStreamSynchronize(stream));
}

namespace {

struct EmitEvicted {
    const uint64_t* evslot;
    uint64_t* out;
    uint64_t cap;
    __device__ void operator()(uint64_t i, unsigned k) const {
        if (out && k < cap) out[k] = evslot[i];
    }
};

__global__ void k_dirty_flags(const uint64_t* __restrict__ row_gen, uint64_t total, uint64_t gen,
                              uint8_t* __restrict__ flags) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < total;
         r += (uint64_t)gridDim.x * blockDim.x)
        flags[r] = row_gen[r] > gen ? 1 : 0;
}

struct EmitIndex {
    uint64_t* out;
    uint64_t cap;
    uint64_t offset;
    __device__ void operator()(uint64_t i, unsigned k) const {
        if (k < cap) out[k] = offset + i;
    }
};

// Rows of this handle dirtied since `gen` (row_generation > gen), ascending, into T.p_rows;
// returns the count.  Persistent scratch: k_dirty_flags writes every held flag, the padding
// past `held` is zeroed once at allocation.
unsigned run_dirty_compact(Table& T, uint64_t gen, cudaStream_t st) {
    const uint64_t held = T.held_rows();
    const size_t fl = ((held + 15) & ~15ull) + 16;
    if (T.p_flags.bytes < fl) {
        T.p_flags.reserve(fl);
        MPZCH_CUDA(cudaMemsetAsync(T.p_flags.p, 0, T.p_flags.bytes, st));
    }
    T.p_rows.reserve(std::max<uint64_t>(held, 1) * 8);
    T.p_blk.reserve(((held + kCompactChunk - 1) / kCompactChunk + 1) * 4);
    k_dirty_flags<<<grid_for(held, 256), 256, 0, st>>>(T.row_gen, held, gen, T.p_flags.as<uint8_t>());
    ++T.launches;
    unsigned* d_n = &T.d_aux->pad;
    EmitIndex em{T.p_rows.as<uint64_t>(), held, T.row_lo};
    compact_flags(T.p_flags.as<uint8_t>(), held, T.p_blk.as<unsigned>(), d_n, false, em, st, T.launches);
    MPZCH_CUDA(cudaMemcpyAsync(&T.h_aux->pad, d_n, 4, cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaStreamSynchronize(st));
    return T.h_aux->pad;
}

}  // namespace

Policy parse_policy(const mpzch_policy* p) {
    Policy pol;
    if (!p) return pol;  // Disabled
    if (p->mode < 0 || p->mode > 2) throw Error{MPZCH_EINVAL, "unknown eviction mode"};
    pol.mode = p->mode;
    if (pol.mode != kModeTtl) return pol;
    // TtlPolicy::validate, eviction.cpp:8-18
    if (p->default_ttl == 0) throw Error{MPZCH_EINVAL, "default TTL must be strictly positive"};
    pol.default_ttl = p->default_ttl;
    for (uint32_t i = 0; i < p->n_feat; ++i) {
        if (p->feat_ttls[i] == 0)
            throw Error{MPZCH_EINVAL, "per-feature TTL must be strictly positive (feature " +
                                          std::to_string(p->feat_keys[i]) + ")"};
        for (uint32_t j = 0; j < i; ++j)
            if (p->feat_keys[j] == p->feat_keys[i])
                throw Error{MPZCH_EINVAL, "duplicate feature in per-feature TTL map"};
        pol.keys.push_back(p->feat_keys[i]);
        pol.ttls.push_back(p->feat_ttls[i]);
    }
    return pol;
}

void require_valid_id(uint64_t id) {  // ids.hpp:25-31
    if ((id >> 63) == 0) return;
    throw Error{MPZCH_EINVAL, id == ~0ull ? "id is the empty-slot sentinel"
                                          : "id exceeds the 63-bit ID space"};
}

// Turn a finished slot's counters into its Result (errors in the reference's order).
void complete_slot(Table& t, int si) {
    Table::Slot& sl = t.slots[si];
    if (!sl.busy) return;
    MPZCH_CUDA(cudaEventSynchronize(sl.done));
    const BatchCounters& c = t.h_ring[si];
    Table::Result r;
    r.ticket = sl.ticket;
    if (sl.lookup && c.err.bad_pos != ~0ull) {  // MpzchTable::lookup -> require_valid_id (ids.hpp:25-31)
        r.status = MPZCH_EINVAL;
        r.msg = c.bad_id == ~0ull ? "id is the empty-slot sentinel" : "id exceeds the 63-bit ID space";
    } else if (c.err.too_many == 2) {
        r.status = MPZCH_ECUDA;
        r.msg = "internal error: claim invariant violated";
    } else if (c.err.bad_pos != ~0ull) {
        r.status = MPZCH_EINVAL;
        r.msg = "invalid id at batch position " + std::to_string(c.err.bad_pos);
    } else if (c.err.foreign_pos != ~0ull) {
        r.status = MPZCH_ERANGE;
        r.msg = "id at batch position " + std::to_string(c.err.foreign_pos) +
                " routes to a shard this handle does not hold";
    } else if (sl.overflow_all || c.err.overflow) {
        r.status = MPZCH_EOVERFLOW;
        r.msg = "TTL expiry overflows the 64-bit timestamp range";
    }
    uint32_t path = sl.path;
    if (sl.lru_try) {  // the claim attempt aborted on the device -> the gated rounds path ran
        path = c.path_taken ? MPZCH_PATH_ROUNDS : MPZCH_PATH_AUTO;
        t.lru_recent_abort = c.path_taken != 0;
        if (c.path_taken) {  // skip the attempt for 1, 3, 7, ... (at most 15) LRU batches
            ++t.lru_fallbacks;
            t.lru_backoff = std::min<uint32_t>(2 * t.lru_backoff + 1, 15);
            t.lru_skip_left = t.lru_backoff;
        } else if (r.status == MPZCH_OK) {
            t.lru_backoff = 0;
        }
    }
    if (r.status == MPZCH_OK) {
        r.evicted_n = c.evicted_count;
        mpzch_batch_stats& s = r.stats;
        s.positions = sl.n;
        s.new_positions = (sl.fast && path == MPZCH_PATH_AUTO) ? c.new_count : 0;
        s.new_ids = c.entry_count;
        s.found = c.found;
        s.inserted = c.inserted;
        s.evicted = c.evicted;
        s.collision = c.collision;
        s.evicted_rows = c.evicted_count;
        s.path = path;
        s.rounds = path == MPZCH_PATH_ROUNDS ? c.r_rounds : 0;
        if (path == MPZCH_PATH_ROUNDS && getenv("MPZCH_DEBUG_ROUNDS"))
            fprintf(stderr, "rounds u=%u rounds=%u iters=%u marked=%u left=%u\n", c.entry_count,
                    c.r_rounds, c.r_iters, c.r_marked, c.r_left);
        if (sl.profiled && sl.fast) {
            float a01 = 0, a12 = 0, a23 = 0, a03 = 0, k70 = 0, k14 = 0, k45 = 0, k52 = 0, k26 = 0;
            MPZCH_CUDA(cudaEventElapsedTime(&a01, sl.ev[0], sl.ev[1]));
            MPZCH_CUDA(cudaEventElapsedTime(&a12, sl.ev[1], sl.ev[2]));
            MPZCH_CUDA(cudaEventElapsedTime(&a23, sl.ev[2], sl.ev[3]));
            MPZCH_CUDA(cudaEventElapsedTime(&a03, sl.ev[0], sl.ev[3]));
            MPZCH_CUDA(cudaEventElapsedTime(&k70, sl.ev[7], sl.ev[0]));
            MPZCH_CUDA(cudaEventElapsedTime(&k14, sl.ev[1], sl.ev[4]));
            MPZCH_CUDA(cudaEventElapsedTime(&k45, sl.ev[4], sl.ev[5]));
            MPZCH_CUDA(cudaEventElapsedTime(&k52, sl.ev[5], sl.ev[2]));
            MPZCH_CUDA(cudaEventElapsedTime(&k26, sl.ev[2], sl.ev[6]));
            mpzch_profile& p = t.prof;
            p.validate_ms += k70;
            p.dedup_ms += k14;
            p.claimk_ms += k45;
            p.commit_ms += k52;
            p.finalize_ms += k26;
            const uint64_t n = sl.n;
            p.batches += 1;
            p.probe_launches += 1;
            p.probe_ms += a01;
            p.claim_ms += a12;
            p.tail_ms += a23;
            p.batch_ms += a03;
            const uint64_t sectors = c.id_sectors + c.meta_sectors;
            const uint64_t n_final = n - c.new_count;
            p.probe_sectors += sectors;
            // probe kernel: sectors read + 8 B id per position + 9 B result and one metadata
            // sector written per final position + 12 B new-list record per new position
            p.probe_bytes += 32 * sectors + 8 * n + (9 + 32) * n_final + 12ull * c.new_count;
            // whole batch (SURVEY 8d terms, counted per position): probe reads, 8 B id in,
            // 9 B result out, one metadata sector written per position, one identity sector +
            // 8 B row_generation per Inserted/Evicted position, 8*dim+1 B per reset row
            p.batch_bytes += 32 * sectors + 8 * n + 9 * n + 32 * n +
                             40ull * (c.inserted + c.evicted) +
                             (uint64_t)c.reset_count * (8ull * t.dim + 1);
        }
    }
    t.results[r.ticket % Table::kResults] = std::move(r);
    sl.busy = false;
}

// one metadata value for the batch, or per-feature values through the fast path's last-writer
// pass (make_metadata, eviction.cpp:20-30); uploads the per-feature map
void fill_policy_args(Table& t, const Policy& pol, uint64_t now, const uint32_t* feats, BatchArgs& a,
                      cudaStream_t st) {
    a.uniform = true;
    uint64_t ttl = 0;
    if (pol.mode == kModeTtl) {
        if (!feats) {
            ttl = pol.ttl_for(0);
        } else {
            ttl = pol.default_ttl;
            for (uint64_t v : pol.ttls)
                if (v != pol.default_ttl) a.uniform = false;
        }
        if (a.uniform) {
            a.overflow_all = ttl > ~0ull - now;
            a.uniform_meta = a.overflow_all ? 0 : now + ttl;
        }
    } else {
        a.uniform_meta = now;
    }
    const uint32_t nk = (uint32_t)pol.keys.size();
    if (nk) {
        t.s_featk.reserve(nk * 4);
        t.s_featv.reserve(nk * 8);
        MPZCH_CUDA(cudaMemcpyAsync(t.s_featk.p, pol.keys.data(), nk * 4, cudaMemcpyHostToDevice, st));
        MPZCH_CUDA(cudaMemcpyAsync(t.s_featv.p, pol.ttls.data(), nk * 8, cudaMemcpyHostToDevice, st));
        a.d_featk = t.s_featk.as<uint32_t>();
        a.d_featv = t.s_featv.as<uint64_t>();
    }
    // per-feature TTL (differing values) takes the fast path too -- its metadata goes through the
    // last-writer pass -- unless some TTL of the map could overflow at this `now` (the ordered
    // path then reports exactly which position does, eviction.cpp:26-28); MPZCH_PF_FAST=0 keeps
    // such batches on the rounds path
    static const bool pf_env = [] {
        const char* e = getenv("MPZCH_PF_FAST");
        return !(e && std::string(e) == "0");
    }();
    a.nk = nk;
    if (pol.mode == kModeTtl && !a.uniform && pf_env) {
        bool ovf = pol.default_ttl > ~0ull - now;
        for (uint64_t v : pol.ttls) ovf = ovf || v > ~0ull - now;
        a.per_feature = !ovf;
        a.uniform_meta = 0;
    }
}

// Enqueue one batch on `st`; returns its ticket.  Host-detectable argument errors throw
// here; device-detected ones (invalid id, ...) are reported by wait_batch.
uint64_t enqueue_batch(Table& t, const uint64_t* ids, const uint32_t* feats, uint64_t n,
                       uint64_t now, const Policy& pol, uint64_t* out_slots, uint8_t* out_oc,
                       uint64_t* out_ev, uint64_t ev_cap, cudaStream_t st,
                       uint8_t* out_mark, bool host_waits) {
    if (n > 0xffffffffull) throw Error{MPZCH_ELENGTH, "batch exceeds 2^32 - 1 positions"};
    const uint64_t ticket = t.next_ticket++;
    const int si = (int)(ticket % Table::kRing);
    if (n == 0) {
        Table::Result r;
        r.ticket = ticket;
        t.results[ticket % Table::kResults] = r;
        return ticket;
    }
    complete_slot(t, si);  // the ring wrapped: retire the batch that used this block
    // batches of one handle share scratch: order a new stream after the previous batch
    if (t.last_ticket && st != t.last_stream) {
        const Table::Slot& prev = t.slots[t.last_ticket % Table::kRing];
        if (prev.busy && prev.ticket == t.last_ticket) MPZCH_CUDA(cudaStreamWaitEvent(st, prev.done, 0));
    }
    Table::Slot& sl = t.slots[si];
    t.d_ctr = t.d_ring + si;
    t.h_ctr = t.h_ring + si;
    if (t.profiling && !sl.ev[0])
        for (auto& e : sl.ev) MPZCH_CUDA(cudaEventCreate(&e));
    t.ev = sl.ev;
    BatchArgs a{};
    a.ids = ids;
    a.feats = feats;
    a.n = n;
    a.now = now;
    a.pol = &pol;
    a.out_slots = out_slots;
    a.out_oc = out_oc;
    a.out_ev = out_ev;
    a.ev_cap = out_ev ? ev_cap : 0;
    a.out_mark = out_mark;
    fill_policy_args(t, pol, now, feats, a, st);
    bool fast = t.path_override == MPZCH_PATH_AUTO && t.hole_free && (a.uniform || a.per_feature) &&
                n <= (1ull << 29);
    const bool profiled = t.profiling;
    // LRU: after attempts that needed an eviction, skip the claim attempt for a growing number
    // of batches (1, 3, 7, 15 ... at most 15), so a stream whose windows are full pays for
    // the rounds path only
    bool lru_try = fast && pol.mode == kModeLru;
    if (lru_try && t.lru_skip_left > 0) {
        --t.lru_skip_left;
        lru_try = false;
        fast = false;
    }
    // LRU differs from Disabled only when a new id finds its window full (it evicts the least
    // recently used slot, which depends on the batch's own refreshes).  The claim path runs with
    // its metadata writes held back; if an eviction cannot be placed exactly it reverts its
    // claims on the device and the batch takes the rounds path.  Who decides:
    //  * gated (asynchronous calls, or after a recent abort): the rounds path is enqueued right
    //    behind the attempt and runs only if the attempt's abort flag is set -- the host never
    //    waits and the rounds path's launches overlap the attempt (LRU pool 1.2 x rows: 142 ->
    //    210 M/s), but an attempt that succeeds still pays the gated launches;
    //  * host (a synchronous call whose recent attempts succeeded): one round trip for the flag,
    //    the rounds path enqueued only if needed (LRU pool 0.8 x rows: 699 vs 498 M/s gated).
    if (lru_try) {  // the rounds path's scratch, sized before any batch may need it
        t.ensure_ordered_scratch(n);
        ensure_rounds_scratch(t, n, t.stream);
        MPZCH_CUDA(cudaStreamSynchronize(t.stream));
    }
    const bool gated = lru_try && (!host_waits || t.lru_recent_abort);
    const bool lru_attempted = lru_try;
    if (lru_try && !gated) {
        t.profiling = false;
        enqueue_fast_batch(t, a, st);
        MPZCH_CUDA(cudaMemcpyAsync(t.h_ctr, t.d_ctr, sizeof(BatchCounters), cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        const BatchErr& e = t.h_ctr->err;
        const bool failed = e.bad_pos != ~0ull || e.overflow || e.too_many || e.foreign_pos != ~0ull;
        fast = failed || !t.h_ctr->lru_abort;
        lru_try = false;  // decided here
        if (!fast) {
            ++t.lru_fallbacks;
            t.lru_recent_abort = true;
            t.lru_backoff = std::min<uint32_t>(2 * t.lru_backoff + 1, 15);
            t.lru_skip_left = t.lru_backoff;
        } else {
            t.lru_backoff = 0;
        }
    } else if (gated) {
        t.profiling = false;
        enqueue_fast_batch(t, a, st);
        BatchArgs g = a;
        g.gate_ctr = t.d_ctr;
        BatchCounters* attempt = t.d_ctr;
        t.d_ctr = t.d_alt;
        enqueue_ordered_batch(t, g, st, /*rounds*/ true);
        t.d_ctr = attempt;
        adopt_gated_counters(t, attempt, t.d_alt, st);
    } else if (fast) {
        enqueue_fast_batch(t, a, st);
    }
    const bool rounds = !fast && t.hole_free && t.path_override != MPZCH_PATH_ORDERED;
    if (!fast) {
        t.profiling = false;  // events are recorded by the fast path only
        enqueue_ordered_batch(t, a, st, rounds);
    }
    t.profiling = profiled;
    MPZCH_CUDA(cudaGetLastError());
    MPZCH_CUDA(cudaMemcpyAsync(t.h_ctr, t.d_ctr, sizeof(BatchCounters), cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaEventRecord(sl.done, st));
    sl.busy = true;
    sl.ticket = ticket;
    sl.n = n;
    sl.fast = fast;
    sl.path = fast ? MPZCH_PATH_AUTO : (rounds ? MPZCH_PATH_ROUNDS : MPZCH_PATH_ORDERED);
    sl.lru_try = lru_try;  // path decided on the device (complete_slot reads it)
    sl.overflow_all = a.overflow_all;
    sl.profiled = profiled && fast && !lru_attempted;  // per-kernel events: plain fast batches only
    sl.lookup = false;
    t.last_stream = st;
    t.last_ticket = ticket;
    return ticket;
}

// Wait for a ticket; rethrow its error; return its evicted-list length.
uint64_t wait_batch(Table& t, uint64_t ticket) {
    const int si = (int)(ticket % Table::kRing);
    if (t.slots[si].busy && t.slots[si].ticket == ticket) complete_slot(t, si);
    const Table::Result& r = t.results[ticket % Table::kResults];
    if (r.ticket != ticket) throw Error{MPZCH_EINVAL, "unknown or expired batch ticket"};
    t.last = r.stats;  // mpzch_last_stats: the batch most recently waited for
    if (r.status != MPZCH_OK) throw Error{r.status, r.msg};
    return r.evicted_n;
}

void run_batch(Table& t, const uint64_t* ids, const uint32_t* feats, uint64_t n, uint64_t now,
               const Policy& pol, uint64_t* out_slots, uint8_t* out_oc, uint64_t* out_ev,
               uint64_t ev_cap, uint64_t* out_ev_n, cudaStream_t st, uint8_t* out_mark = nullptr) {
    if (out_ev_n) *out_ev_n = 0;
    const uint64_t tk = enqueue_batch(t, ids, feats, n, now, pol, out_slots, out_oc, out_ev, ev_cap,
                                      st, out_mark, /*host_waits*/ true);
    const uint64_t nev = wait_batch(t, tk);
    if (out_ev_n) *out_ev_n = nev;
    if (n == 0) t.last = mpzch_batch_stats{};
}

namespace {

template <class F>
mpzch_status guarded(F&& f) {
    try {
        f();
        return MPZCH_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return MPZCH_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MPZCH_EINVAL;
    }
}

}  // namespace

mpzch_status run_guarded(const std::function<void()>& f) { return guarded(f); }

// every kernel a batch can launch, loaded on the current device (lazy loading, common.cuh)
void preload_all_kernels() {
    preload_remap_kernels();
    preload_ordered_kernels();
    preload_rounds_kernels();
    preload_row_kernels();
    preload_route_kernels();
    preload_compact<EmitEvicted>();
    preload_compact<EmitIndex>();
}

void enqueue_compact_evicted(Table& t, uint64_t n, uint64_t* out_ev, uint64_t ev_cap, cudaStream_t st,
                             const unsigned* gate, const uint64_t* slots) {
    EmitEvicted em{slots ? slots : t.s_evslot.as<uint64_t>(), out_ev, ev_cap};
    compact_flags(t.s_evflag.as<uint8_t>(), n, t.s_blk.as<unsigned>(), &t.d_ctr->evicted_count, true,
                  em, st, t.launches, gate);
}

}  // namespace mpzch_b200

using namespace mpzch_b200;


#define CHECK_T(t)                                                     \
    do {                                                               \
        if (!(t) || !(t)->t) {                                         \
            g_last_error = "null table handle";                        \
            return MPZCH_EINVAL;                                       \
        }                                                              \
    } while (0)

extern "C" {

static void order_after_last_batch(Table& T, cudaStream_t st);

// Readers that are not reset-aware (copies, snapshots, deltas, state_equals, raw pointers)
// first materialise the resets a deferred-mode batch left pending (rows.cu); observable state
// is then exactly the eager (reference) state.  Synchronous on the handle's stream.
static void flush_for_read(const Table& Tc) {
    Table& T = const_cast<Table&>(Tc);
    if (!T.resets_pending) return;
    DeviceGuard g(T.device);
    order_after_last_batch(T, T.stream);
    flush_resets(T, T.stream);
    MPZCH_CUDA(cudaStreamSynchronize(T.stream));
}

const char* mpzch_last_error(void) { return g_last_error.c_str(); }

const char* mpzch_build_info(void) { return MPZCH_BUILD_INFO; }

mpzch_status mpzch_table_create(const uint64_t* caps, uint32_t num_shards, uint32_t max_probe,
                                uint64_t seed, uint32_t dim, uint64_t init_seed, int device,
                                mpzch_table** out) {
    if (!out) {
        g_last_error = "null output pointer";
        return MPZCH_EINVAL;
    }
    *out = nullptr;
    return guarded([&] {
        if (num_shards && !caps) throw Error{MPZCH_EINVAL, "null capacities"};
        Table* t = new Table(caps, num_shards, max_probe, seed, dim, init_seed, device);
        *out = new mpzch_table{t};
    });
}

mpzch_status mpzch_table_create_sharded(const uint64_t* caps, uint32_t num_shards,
                                        uint32_t max_probe, uint64_t seed, uint32_t dim,
                                        uint64_t init_seed, int device, uint32_t shard_lo,
                                        uint32_t shard_hi, mpzch_table** out) {
    if (!out) {
        g_last_error = "null output pointer";
        return MPZCH_EINVAL;
    }
    *out = nullptr;
    return guarded([&] {
        if (num_shards && !caps) throw Error{MPZCH_EINVAL, "null capacities"};
        Table* t = new Table(caps, num_shards, max_probe, seed, dim, init_seed, device, shard_lo,
                             shard_hi);
        *out = new mpzch_table{t};
    });
}

mpzch_status mpzch_held_rows(const mpzch_table* t, uint64_t* row_lo, uint64_t* row_hi,
                             uint32_t* shard_lo, uint32_t* shard_hi) {
    CHECK_T(t);
    if (row_lo) *row_lo = t->t->row_lo;
    if (row_hi) *row_hi = t->t->row_hi;
    if (shard_lo) *shard_lo = t->t->shard_lo;
    if (shard_hi) *shard_hi = t->t->shard_hi;
    return MPZCH_OK;
}

mpzch_status mpzch_validate_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                   uint64_t* out_bad_pos, void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        *out_bad_pos = ~0ull;
        if (n == 0) return;
        run_validate(T, ids, n, (cudaStream_t)stream);
        *out_bad_pos = T.h_aux->err.bad_pos;
    });
}

mpzch_status mpzch_route_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                const uint32_t* shard_to_part, uint32_t parts, uint32_t* perm,
                                uint64_t* counts, void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        run_route(T, ids, n, shard_to_part, parts, perm, counts, (cudaStream_t)stream);
    });
}

mpzch_status mpzch_route_count_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                      const uint32_t* shard_to_part, uint32_t parts, uint64_t* counts,
                                      void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        run_route(T, ids, n, shard_to_part, parts, nullptr, counts, (cudaStream_t)stream);
    });
}

mpzch_status mpzch_route_scatter_device(const mpzch_table* t, const uint64_t* ids,
                                        const uint32_t* features, uint64_t n, uint32_t parts,
                                        const uint64_t* ids_to, const uint64_t* features_to,
                                        const uint64_t* src_to, const uint64_t* offset, void* stream) {
    CHECK_T(t);
    return guarded([&] {
        if (!ids_to || !src_to || !offset || (features && !features_to))
            throw Error{MPZCH_EINVAL, "route scatter: null destination table"};
        Table& T = *t->t;
        DeviceGuard g(T.device);
        PeerScatter d{ids_to, features_to, src_to, offset};
        run_route_scatter(T, ids, features, n, parts, d, (cudaStream_t)stream);
    });
}

mpzch_status mpzch_return_scatter_device(int device, uint64_t n_recv, const uint64_t* slots,
                                         const uint8_t* outcomes, const uint8_t* marks,
                                         const uint32_t* src, uint32_t parts, const uint64_t* recv_offset,
                                         const uint64_t* slots_to, const uint64_t* outcomes_to,
                                         const uint64_t* marks_to, void* stream) {
    return guarded([&] {
        if (!recv_offset || !slots_to || !outcomes_to)
            throw Error{MPZCH_EINVAL, "return scatter: null destination table"};
        DeviceGuard g(device);
        run_return_scatter(n_recv, slots, outcomes, marks, src, parts, recv_offset, slots_to, outcomes_to,
                           marks_to, (cudaStream_t)stream);
    });
}

namespace {
// CUDA IPC of buffers that may sit inside a larger allocation (PyTorch's caching allocator):
// the handle names the allocation, the record carries the offset.  Imports are reference
// counted per handle (a process maps an allocation once).
struct IpcRecord {
    cudaIpcMemHandle_t h;
    uint64_t offset;
};
static_assert(sizeof(IpcRecord) == MPZCH_IPC_RECORD_BYTES, "IPC record size");
std::mutex g_ipc_mu;
struct IpcMap {
    void* base;
    int refs;
};
std::map<std::string, IpcMap> g_ipc_open;        // handle bytes -> mapping
std::map<uint64_t, std::string> g_ipc_addr;      // imported address -> handle bytes

CUresult (*get_range_fn())(CUdeviceptr*, size_t*, CUdeviceptr) {
    static CUresult (*fn)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        MPZCH_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error{MPZCH_ECUDA, "cuMemGetAddressRange unavailable"};
        fn = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(p);
    }
    return fn;
}
}  // namespace

mpzch_status mpzch_ipc_export(const void* device_ptr, uint8_t* out) {
    return guarded([&] {
        if (!device_ptr || !out) throw Error{MPZCH_EINVAL, "ipc export: null pointer"};
        CUdeviceptr base = 0;
        size_t size = 0;
        if (get_range_fn()(&base, &size, (CUdeviceptr)device_ptr) != CUDA_SUCCESS)
            throw Error{MPZCH_EINVAL, "ipc export: not a device allocation"};
        IpcRecord r{};
        MPZCH_CUDA(cudaIpcGetMemHandle(&r.h, (void*)base));
        r.offset = (uint64_t)device_ptr - (uint64_t)base;
        std::memcpy(out, &r, sizeof r);
    });
}

mpzch_status mpzch_ipc_import(int device, const uint8_t* in, uint64_t* out_addr) {
    return guarded([&] {
        if (!in || !out_addr) throw Error{MPZCH_EINVAL, "ipc import: null pointer"};
        IpcRecord r;
        std::memcpy(&r, in, sizeof r);
        const std::string key(reinterpret_cast<const char*>(&r.h), sizeof r.h);
        DeviceGuard g(device);
        std::lock_guard<std::mutex> lk(g_ipc_mu);
        auto it = g_ipc_open.find(key);
        if (it == g_ipc_open.end()) {
            void* base = nullptr;
            MPZCH_CUDA(cudaIpcOpenMemHandle(&base, r.h, cudaIpcMemLazyEnablePeerAccess));
            it = g_ipc_open.emplace(key, IpcMap{base, 0}).first;
        }
        ++it->second.refs;
        const uint64_t addr = (uint64_t)it->second.base + r.offset;
        g_ipc_addr[addr] = key;  // (same address imported twice: one entry, refs counts both)
        *out_addr = addr;
    });
}

mpzch_status mpzch_ipc_close(uint64_t addr) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(g_ipc_mu);
        auto a = g_ipc_addr.find(addr);
        if (a == g_ipc_addr.end()) throw Error{MPZCH_EINVAL, "ipc close: address was not imported"};
        const std::string key = a->second;
        auto it = g_ipc_open.find(key);
        if (--it->second.refs == 0) {
            void* base = it->second.base;
            g_ipc_open.erase(it);
            // forget every address of this mapping
            for (auto i = g_ipc_addr.begin(); i != g_ipc_addr.end();)
                i = i->second == key ? g_ipc_addr.erase(i) : std::next(i);
            MPZCH_CUDA(cudaIpcCloseMemHandle(base));
        }
    });
}

mpzch_status mpzch_process_batch_device_marked(mpzch_table* t, const uint64_t* ids,
                                               const uint32_t* feats, uint64_t n, uint64_t now,
                                               const mpzch_policy* policy, uint64_t* out_slots,
                                               uint8_t* out_oc, uint8_t* out_first_evicted,
                                               uint64_t* out_ev_n, void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        const Policy pol = parse_policy(policy);
        run_batch(T, ids, feats, n, now, pol, out_slots, out_oc, nullptr, 0, out_ev_n,
                  (cudaStream_t)stream, out_first_evicted);
    });
}

mpzch_status mpzch_table_destroy(mpzch_table* t) {
    if (!t) return MPZCH_OK;
    delete t->t;
    delete t;
    return MPZCH_OK;
}

uint64_t mpzch_total_rows(const mpzch_table* t) { return t && t->t ? t->t->total : 0; }
uint32_t mpzch_num_shards(const mpzch_table* t) { return t && t->t ? t->t->S : 0; }
uint32_t mpzch_max_probe(const mpzch_table* t) { return t && t->t ? t->t->P : 0; }
uint32_t mpzch_dim(const mpzch_table* t) { return t && t->t ? t->t->dim : 0; }

mpzch_status mpzch_shard_layout(const mpzch_table* t, uint64_t* capacities, uint64_t* offsets) {
    CHECK_T(t);
    if (capacities) std::memcpy(capacities, t->t->caps.data(), t->t->S * 8);
    if (offsets) std::memcpy(offsets, t->t->offsets.data(), (t->t->S + 1) * 8);
    return MPZCH_OK;
}

mpzch_status mpzch_process_batch_device(mpzch_table* t, const uint64_t* ids, const uint32_t* feats,
                                        uint64_t n, uint64_t now, const mpzch_policy* policy,
                                        uint64_t* out_slots, uint8_t* out_oc, uint64_t* out_ev,
                                        uint64_t ev_cap, uint64_t* out_ev_n, void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        const Policy pol = parse_policy(policy);
        // CUDA convention: 0 is the legacy default stream (torch's default stream has
        // handle 0), so the caller's producer kernels are ordered before ours
        run_batch(T, ids, feats, n, now, pol, out_slots, out_oc, out_ev, ev_cap, out_ev_n,
                  (cudaStream_t)stream);
    });
}

mpzch_status mpzch_process_batch_device_async(mpzch_table* t, const uint64_t* ids,
                                              const uint32_t* feats, uint64_t n, uint64_t now,
                                              const mpzch_policy* policy, uint64_t* out_slots,
                                              uint8_t* out_oc, uint64_t* out_ev, uint64_t ev_cap,
                                              void* stream, uint64_t* out_ticket) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        const Policy pol = parse_policy(policy);
        *out_ticket = enqueue_batch(T, ids, feats, n, now, pol, out_slots, out_oc, out_ev, ev_cap,
                                    (cudaStream_t)stream);
    });
}

mpzch_status mpzch_batch_wait(mpzch_table* t, uint64_t ticket, uint64_t* out_ev_n) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        const uint64_t nev = wait_batch(T, ticket);
        if (out_ev_n) *out_ev_n = nev;
    });
}

mpzch_status mpzch_process_batch(mpzch_table* t, const uint64_t* ids, const uint32_t* feats,
                                 uint64_t n, uint64_t now, const mpzch_policy* policy,
                                 uint64_t* out_slots, uint8_t* out_oc, uint64_t* out_ev,
                                 uint64_t ev_cap, uint64_t* out_ev_n) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        const Policy pol = parse_policy(policy);
        if (n > 0xffffffffull) throw Error{MPZCH_ELENGTH, "batch exceeds 2^32 - 1 positions"};
        if (out_ev_n) *out_ev_n = 0;
        if (n == 0) {
            T.last = mpzch_batch_stats{};
            return;
        }
        cudaStream_t st = T.stream;
        T.s_ids.reserve(n * 8);
        T.s_oslot.reserve(n * 8);
        T.s_ooc.reserve(n);
        MPZCH_CUDA(cudaMemcpyAsync(T.s_ids.p, ids, n * 8, cudaMemcpyHostToDevice, st));
        const uint32_t* dfe = nullptr;
        if (feats) {
            T.s_feats.reserve(n * 4);
            MPZCH_CUDA(cudaMemcpyAsync(T.s_feats.p, feats, n * 4, cudaMemcpyHostToDevice, st));
            dfe = T.s_feats.as<uint32_t>();
        }
        uint64_t* dev_ev = nullptr;
        if (out_ev && ev_cap) {
            T.s_oev.reserve(std::min<uint64_t>(ev_cap, n) * 8);
            dev_ev = T.s_oev.as<uint64_t>();
        }
        uint64_t nev = 0;
        run_batch(T, T.s_ids.as<uint64_t>(), dfe, n, now, pol, T.s_oslot.as<uint64_t>(),
                  T.s_ooc.as<uint8_t>(), dev_ev, std::min<uint64_t>(ev_cap, n), &nev, st);
        MPZCH_CUDA(cudaMemcpyAsync(out_slots, T.s_oslot.p, n * 8, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaMemcpyAsync(out_oc, T.s_ooc.p, n, cudaMemcpyDeviceToHost, st));
        if (dev_ev && nev)
            MPZCH_CUDA(cudaMemcpyAsync(out_ev, dev_ev, std::min(nev, ev_cap) * 8,
                                       cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        if (out_ev_n) *out_ev_n = nev;
    });
}

mpzch_status mpzch_lookup_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                 uint64_t* out_slots, uint8_t* out_oc, void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        if (n == 0) return;
        cudaStream_t st = (cudaStream_t)stream;  // 0 = legacy default stream
        std::lock_guard<std::mutex> lk(T.lookup_mu);
        order_after_last_batch(T, st);
        init_aux_err(T, st);
        run_lookup(T, ids, n, out_slots, out_oc, &T.d_aux->err, st, &T.s_ldefer, &T.d_aux->ldeferred);
        ++T.launches;
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(&T.h_aux->err, &T.d_aux->err, sizeof(BatchErr),
                                   cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        if (T.h_aux->err.bad_pos != ~0ull) {
            uint64_t bad = 0;
            MPZCH_CUDA(cudaMemcpy(&bad, ids + T.h_aux->err.bad_pos, 8, cudaMemcpyDeviceToHost));
            require_valid_id(bad);
        }
        if (T.h_aux->err.foreign_pos != ~0ull)
            throw Error{MPZCH_ERANGE, "id at batch position " + std::to_string(T.h_aux->err.foreign_pos) +
                                          " routes to a shard this handle does not hold"};
    });
}

mpzch_status mpzch_lookup_device_async(mpzch_table* t, const uint64_t* ids, uint64_t n,
                                       uint64_t* out_slots, uint8_t* out_oc, void* stream,
                                       uint64_t* out_ticket) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        cudaStream_t st = (cudaStream_t)stream;
        const uint64_t ticket = T.next_ticket++;
        const int si = (int)(ticket % Table::kRing);
        *out_ticket = ticket;
        if (n == 0) {
            Table::Result r;
            r.ticket = ticket;
            T.results[ticket % Table::kResults] = r;
            return;
        }
        complete_slot(T, si);
        if (T.last_ticket && st != T.last_stream) {  // after the handle's pending batches
            const Table::Slot& prev = T.slots[T.last_ticket % Table::kRing];
            if (prev.busy && prev.ticket == T.last_ticket) MPZCH_CUDA(cudaStreamWaitEvent(st, prev.done, 0));
        }
        Table::Slot& sl = T.slots[si];
        BatchCounters* dc = T.d_ring + si;
        launch_lookup_async(T, ids, n, out_slots, out_oc, dc, st);
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(T.h_ring + si, dc, sizeof(BatchCounters), cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaEventRecord(sl.done, st));
        sl.busy = true;
        sl.ticket = ticket;
        sl.n = n;
        sl.fast = false;
        sl.path = MPZCH_PATH_AUTO;
        sl.overflow_all = false;
        sl.profiled = false;
        sl.lookup = true;
        T.last_stream = st;
        T.last_ticket = ticket;
    });
}

mpzch_status mpzch_lookup(const mpzch_table* t, const uint64_t* ids, uint64_t n, uint64_t* out_slots,
                          uint8_t* out_oc) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        if (n == 0) return;
        cudaStream_t st = T.stream;
        std::lock_guard<std::mutex> lk(T.lookup_mu);
        order_after_last_batch(T, st);
        DevBuf &ids_d = T.l_ids, &oslot_d = T.l_oslot, &ooc_d = T.l_ooc;  // lookup-owned staging
        ids_d.reserve(n * 8);
        oslot_d.reserve(n * 8);
        ooc_d.reserve(n);
        MPZCH_CUDA(cudaMemcpyAsync(ids_d.p, ids, n * 8, cudaMemcpyHostToDevice, st));
        init_aux_err(T, st);
        run_lookup(T, ids_d.as<uint64_t>(), n, oslot_d.as<uint64_t>(), ooc_d.as<uint8_t>(),
                   &T.d_aux->err, st, &T.s_ldefer, &T.d_aux->ldeferred);
        ++T.launches;
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(&T.h_aux->err, &T.d_aux->err, sizeof(BatchErr),
                                   cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaMemcpyAsync(out_slots, oslot_d.p, n * 8, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaMemcpyAsync(out_oc, ooc_d.p, n, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        if (T.h_aux->err.bad_pos != ~0ull) require_valid_id(ids[T.h_aux->err.bad_pos]);
        if (T.h_aux->err.foreign_pos != ~0ull)
            throw Error{MPZCH_ERANGE, "id at batch position " + std::to_string(T.h_aux->err.foreign_pos) +
                                          " routes to a shard this handle does not hold"};
    });
}

mpzch_status mpzch_lookup_or_insert(mpzch_table* t, uint64_t id, uint32_t feature, uint64_t now,
                                    const mpzch_policy* policy, uint64_t* out_slot,
                                    uint8_t* out_oc) {
    CHECK_T(t);
    return guarded([&] {
        const Policy pol = parse_policy(policy);
        require_valid_id(id);  // shard_of -> require_valid_id, table.cpp:101
        if (pol.mode == kModeTtl && pol.ttl_for(feature) > ~0ull - now)  // make_metadata :102
            throw Error{MPZCH_EOVERFLOW, "TTL expiry overflows the 64-bit timestamp range"};
        mpzch_policy p2{pol.mode, (uint32_t)pol.keys.size(), pol.default_ttl, pol.keys.data(),
                        pol.ttls.data()};
        uint64_t nev = 0;
        const mpzch_status rc =
            mpzch_process_batch(t, &id, &feature, 1, now, &p2, out_slot, out_oc, nullptr, 0, &nev);
        if (rc != MPZCH_OK) throw Error{rc, g_last_error};
    });
}

mpzch_status mpzch_copy_identities(const mpzch_table* t, uint64_t* out) {
    CHECK_T(t);
    return guarded([&] {
        DeviceGuard g(t->t->device);
        MPZCH_CUDA(cudaStreamSynchronize(t->t->stream));
        const Table& T = *t->t;
        MPZCH_CUDA(cudaMemcpy(out, T.ident + (T.row_lo - T.row_base), T.held_rows() * 8,
                              cudaMemcpyDeviceToHost));
    });
}

mpzch_status mpzch_copy_metadata(const mpzch_table* t, uint64_t* out) {
    CHECK_T(t);
    return guarded([&] {
        DeviceGuard g(t->t->device);
        MPZCH_CUDA(cudaStreamSynchronize(t->t->stream));
        const Table& T = *t->t;
        MPZCH_CUDA(cudaMemcpy(out, T.meta + (T.row_lo - T.row_base), T.held_rows() * 8,
                              cudaMemcpyDeviceToHost));
    });
}

// row0 is a global row; the range must lie inside the rows this handle holds
static void check_rows(const Table& T, uint64_t row0, uint64_t nrows) {
    if (T.dim == 0) throw Error{MPZCH_ELOGIC, "table has no embedding payload (dim = 0)"};
    if (row0 < T.row_lo || row0 > T.row_hi || nrows > T.row_hi - row0)
        throw Error{MPZCH_ERANGE, "embedding row out of range"};
}

mpzch_status mpzch_copy_weights(const mpzch_table* t, uint64_t row0, uint64_t nrows, float* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        flush_for_read(T);
        check_rows(T, row0, nrows);
        DeviceGuard g(T.device);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        MPZCH_CUDA(cudaMemcpy(out, T.dev.weights + row0 * T.dim, nrows * T.dim * 4, cudaMemcpyDeviceToHost));
    });
}

mpzch_status mpzch_copy_momentum(const mpzch_table* t, uint64_t row0, uint64_t nrows, float* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        flush_for_read(T);
        check_rows(T, row0, nrows);
        DeviceGuard g(T.device);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        MPZCH_CUDA(cudaMemcpy(out, T.dev.momentum + row0 * T.dim, nrows * T.dim * 4, cudaMemcpyDeviceToHost));
    });
}

mpzch_status mpzch_copy_trained(const mpzch_table* t, uint8_t* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        flush_for_read(T);
        check_rows(T, T.row_lo, 0);
        DeviceGuard g(T.device);
        copy_trained_bytes(const_cast<Table&>(T), T.row_lo, T.held_rows(), out);
    });
}

mpzch_status mpzch_copy_row_generation(const mpzch_table* t, uint64_t* out) {
    CHECK_T(t);
    return guarded([&] {
        DeviceGuard g(t->t->device);
        MPZCH_CUDA(cudaStreamSynchronize(t->t->stream));
        MPZCH_CUDA(cudaMemcpy(out, t->t->row_gen, t->t->held_rows() * 8, cudaMemcpyDeviceToHost));
    });
}

mpzch_status mpzch_device_arrays(const mpzch_table* t, uint64_t** identities, uint64_t** metadata,
                                 float** weights) {
    CHECK_T(t);
    if (weights) {  // a raw weights pointer: no reset may stay pending behind it
        const mpzch_status st = guarded([&] { flush_for_read(*t->t); });
        if (st != MPZCH_OK) return st;
    }
    if (identities) *identities = t->t->ident;
    if (metadata) *metadata = t->t->meta;
    if (weights) *weights = t->t->weights;
    return MPZCH_OK;
}

mpzch_status mpzch_write_slots(mpzch_table* t, uint32_t shard, const uint64_t* local_slots,
                               const uint64_t* identities, const uint64_t* metadata, uint64_t n) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        if (shard >= T.S) throw Error{MPZCH_ERANGE, "shard index out of range"};
        if (shard < T.shard_lo || shard >= T.shard_hi)
            throw Error{MPZCH_ERANGE, "shard is not held by this handle"};
        std::vector<uint64_t> g(n), m(n);
        for (uint64_t i = 0; i < n; ++i) {
            if (local_slots[i] >= T.caps[shard])
                throw Error{MPZCH_ERANGE, "local slot exceeds shard capacity"};
            g[i] = T.offsets[shard] + local_slots[i];
        }
        if (!n) return;
        DeviceGuard gd(T.device);
        uint64_t* buf = nullptr;
        MPZCH_CUDA(cudaMalloc((void**)&buf, n * 24));
        MPZCH_CUDA(cudaMemcpyAsync(buf, g.data(), n * 8, cudaMemcpyHostToDevice, T.stream));
        MPZCH_CUDA(cudaMemcpyAsync(buf + n, identities, n * 8, cudaMemcpyHostToDevice, T.stream));
        if (metadata) MPZCH_CUDA(cudaMemcpyAsync(buf + 2 * n, metadata, n * 8, cudaMemcpyHostToDevice, T.stream));
        else {
            // keep the existing metadata words
            MPZCH_CUDA(cudaStreamSynchronize(T.stream));
            for (uint64_t i = 0; i < n; ++i)
                MPZCH_CUDA(cudaMemcpy(&m[i], T.dev.meta + g[i], 8, cudaMemcpyDeviceToHost));
            MPZCH_CUDA(cudaMemcpyAsync(buf + 2 * n, m.data(), n * 8, cudaMemcpyHostToDevice, T.stream));
        }
        launch_write_slots(T, buf, buf + n, buf + 2 * n, n, T.stream);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        cudaFree(buf);
        T.hole_free = false;
    });
}

mpzch_status mpzch_check_hole_free(mpzch_table* t, int* out) {
    CHECK_T(t);
    return guarded([&] {
        DeviceGuard g(t->t->device);
        t->t->hole_free = run_hole_check(*t->t);
        if (out) *out = t->t->hole_free ? 1 : 0;
    });
}

mpzch_status mpzch_write_row(mpzch_table* t, uint64_t row, const float* w, const float* m,
                             uint8_t trained) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        check_rows(T, row, 1);
        flush_for_read(T);
        DeviceGuard g(T.device);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        if (w) MPZCH_CUDA(cudaMemcpy(T.dev.weights + row * T.dim, w, T.dim * 4, cudaMemcpyHostToDevice));
        if (m) MPZCH_CUDA(cudaMemcpy(T.dev.momentum + row * T.dim, m, T.dim * 4, cudaMemcpyHostToDevice));
        set_trained_flag(T, row, trained != 0);
        // a training write stamps the row dirty, as sgd_step does (table.cpp:170-176)
        MPZCH_CUDA(cudaMemcpy(T.dev.row_gen + row, &T.gen_clock, 8, cudaMemcpyHostToDevice));
    });
}

// EmbeddingTable::sgd_step argument checks in the reference's order (table.cpp:174-178,
// embedding_store.cpp:70-81); the per-row range check happens on the device
static void check_sgd_args(const Table& T, uint64_t n, uint64_t n_grads, float lr, float beta) {
    if (T.dim == 0) throw Error{MPZCH_ELOGIC, "table has no embedding payload (dim = 0)"};
    if (n_grads != n * T.dim) throw Error{MPZCH_EINVAL, "gradient shape does not match rows * dim"};
    if (!(lr > 0.0f)) throw Error{MPZCH_EINVAL, "learning rate must be positive"};
    if (beta < 0.0f || beta >= 1.0f)
        throw Error{MPZCH_EINVAL, "momentum coefficient must lie in [0, 1)"};
}

// a stream that is not the one the handle's last batch ran on waits for that batch
static void order_after_last_batch(Table& T, cudaStream_t st) {
    if (T.last_ticket && st != T.last_stream) {
        const Table::Slot& prev = T.slots[T.last_ticket % Table::kRing];
        if (prev.busy && prev.ticket == T.last_ticket) MPZCH_CUDA(cudaStreamWaitEvent(st, prev.done, 0));
    }
}

static void sgd_common(Table& T, const uint64_t* d_rows, uint64_t n, const float* d_grads, float lr,
                       float beta, cudaStream_t st) {
    const uint64_t bad = run_sgd_step(T, d_rows, n, d_grads, lr, beta, st);
    if (bad != ~0ull) throw Error{MPZCH_ERANGE, "embedding row out of range"};
}

mpzch_status mpzch_sgd_step(mpzch_table* t, const uint64_t* rows, uint64_t n, const float* grads,
                            uint64_t n_grads, float lr, float beta) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        check_sgd_args(T, n, n_grads, lr, beta);
        if (n == 0) return;
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        T.s_ids.reserve(n * 8);
        T.s_grads.reserve(n_grads * 4);
        MPZCH_CUDA(cudaMemcpyAsync(T.s_ids.p, rows, n * 8, cudaMemcpyHostToDevice, st));
        MPZCH_CUDA(cudaMemcpyAsync(T.s_grads.p, grads, n_grads * 4, cudaMemcpyHostToDevice, st));
        sgd_common(T, T.s_ids.as<uint64_t>(), n, T.s_grads.as<float>(), lr, beta, st);
    });
}

mpzch_status mpzch_sgd_step_device(mpzch_table* t, const uint64_t* rows, uint64_t n,
                                   const float* grads, uint64_t n_grads, float lr, float beta,
                                   void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        check_sgd_args(T, n, n_grads, lr, beta);
        if (n == 0) return;
        DeviceGuard g(T.device);
        cudaStream_t st = (cudaStream_t)stream;
        order_after_last_batch(T, st);
        sgd_common(T, rows, n, grads, lr, beta, st);
    });
}

mpzch_status mpzch_make_cursor(mpzch_table* t, uint64_t* out_generation) {
    CHECK_T(t);
    *out_generation = t->t->gen_clock++;  // MpzchTable::make_cursor, table.cpp:209-214
    return MPZCH_OK;
}

mpzch_status mpzch_dirty_rows_since(const mpzch_table* t, uint64_t gen, uint64_t* out, uint64_t cap,
                                    uint64_t* out_n) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        // table.cpp:216-225
        if (gen == 0 || gen >= T.gen_clock)
            throw Error{MPZCH_EINVAL, "stale or unknown publication cursor"};
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        const unsigned nn = run_dirty_compact(T, gen, st);
        if (cap && out && nn)
            MPZCH_CUDA(cudaMemcpy(out, T.p_rows.p, std::min<uint64_t>(nn, cap) * 8, cudaMemcpyDeviceToHost));
        *out_n = nn;
    });
}

mpzch_status mpzch_set_profiling(mpzch_table* t, int on) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        DeviceGuard g(T.device);
        T.profiling = on != 0;
        T.prof = mpzch_profile{};
    });
}

mpzch_status mpzch_get_profile(const mpzch_table* t, mpzch_profile* out) {
    CHECK_T(t);
    *out = t->t->prof;
    return MPZCH_OK;
}

mpzch_status mpzch_lookup_gather_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                        uint64_t* out_slots, uint8_t* out_oc, float* out_rows,
                                        void* stream) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        if (T.dim == 0) throw Error{MPZCH_ELOGIC, "table has no embedding payload (dim = 0)"};
        DeviceGuard g(T.device);
        if (n == 0) return;
        cudaStream_t st = (cudaStream_t)stream;
        std::lock_guard<std::mutex> lk(T.lookup_mu);
        order_after_last_batch(T, st);
        init_aux_err(T, st);
        run_lookup_gather(T, ids, n, out_slots, out_oc, out_rows, &T.d_aux->err, st);
        ++T.launches;
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(&T.h_aux->err, &T.d_aux->err, sizeof(BatchErr),
                                   cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        if (T.h_aux->err.bad_pos != ~0ull) {
            uint64_t bad = 0;
            MPZCH_CUDA(cudaMemcpy(&bad, ids + T.h_aux->err.bad_pos, 8, cudaMemcpyDeviceToHost));
            require_valid_id(bad);
        }
        if (T.h_aux->err.foreign_pos != ~0ull)
            throw Error{MPZCH_ERANGE, "id at batch position " + std::to_string(T.h_aux->err.foreign_pos) +
                                          " routes to a shard this handle does not hold"};
    });
}

mpzch_status mpzch_delta_cut(mpzch_table* t, uint64_t generation, uint64_t* out_rows,
                             uint64_t* out_identities, float* out_weights, uint64_t cap,
                             uint64_t* out_n, uint64_t* out_next_generation) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        // DeltaSource::cut (publish.cpp:288-305): rows dirtied since the cursor, then a fresh
        // cursor; index-only tables cannot be published (publish.cpp:282-286)
        if (T.dim == 0) throw Error{MPZCH_ELOGIC, "index-only tables (dim = 0) cannot be published"};
        if (generation == 0 || generation >= T.gen_clock)
            throw Error{MPZCH_EINVAL, "stale or unknown publication cursor"};
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        flush_for_read(T);
        const unsigned nn = run_dirty_compact(T, generation, st);
        const uint64_t k = std::min<uint64_t>(nn, cap);
        if (k) {
            T.p_ids.reserve(k * 8);
            T.p_w.reserve(k * T.dim * 4);
            run_gather_rows(T, T.p_rows.as<uint64_t>(), k, T.p_ids.as<uint64_t>(), T.p_w.as<float>(), st);
            T.launches += 2;
            MPZCH_CUDA(cudaGetLastError());
            if (out_rows) MPZCH_CUDA(cudaMemcpyAsync(out_rows, T.p_rows.p, k * 8, cudaMemcpyDeviceToHost, st));
            if (out_identities)
                MPZCH_CUDA(cudaMemcpyAsync(out_identities, T.p_ids.p, k * 8, cudaMemcpyDeviceToHost, st));
            if (out_weights)
                MPZCH_CUDA(cudaMemcpyAsync(out_weights, T.p_w.p, k * T.dim * 4, cudaMemcpyDeviceToHost, st));
            MPZCH_CUDA(cudaStreamSynchronize(st));
        }
        *out_n = nn;
        if (nn <= cap && out_next_generation) *out_next_generation = T.gen_clock++;  // new cursor
    });
}

// ---- publish: .mpzc / .mpzd images (proj/src/publish.cpp; csrc/publish.cu)

namespace {
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back((uint8_t)(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back((uint8_t)(v >> (8 * i)));
}
void put_magic(std::vector<uint8_t>& b, const char* m) { b.insert(b.end(), m, m + 4); }
}  // namespace

mpzch_status mpzch_crc32_device(const void* bytes, uint64_t n, uint32_t* out_crc, void* stream) {
    return guarded([&] {
        int dev = 0;
        MPZCH_CUDA(cudaGetDevice(&dev));
        const uint32_t raw = crc32_raw_device((const uint8_t*)bytes, n, (cudaStream_t)stream, dev);
        *out_crc = crc32_finish(raw, n);
    });
}

mpzch_status mpzch_serialize_snapshot(const mpzch_table* t, uint8_t* out, uint64_t cap,
                                      uint64_t* out_len) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        // serialize_snapshot, publish.cpp:126-155
        if (T.dim == 0) throw Error{MPZCH_ELOGIC, "index-only tables (dim = 0) cannot be published"};
        if (T.row_lo != 0 || T.row_hi != T.total)
            throw Error{MPZCH_EINVAL, "a snapshot needs every shard (this handle is row-sharded)"};
        const uint64_t id_bytes = T.total * 8, w_bytes = T.total * T.dim * 4ull;
        const uint64_t need = 48 + 8ull * T.S + id_bytes + w_bytes;
        *out_len = need;
        if (!out) return;  // size query
        if (cap < need) throw Error{MPZCH_ELENGTH, "output buffer too small"};
        std::vector<uint8_t> h;
        put_magic(h, "MPZC");
        put_u32(h, 1);  // kFormatVersion
        put_u64(h, T.seed);
        put_u32(h, T.P);
        put_u32(h, T.dim);
        put_u32(h, T.S);
        for (uint64_t c : T.caps) put_u64(h, c);
        put_u64(h, T.total);
        std::vector<uint8_t> cnt;
        put_u64(cnt, T.total * T.dim);
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        flush_for_read(T);
        // CRC over header | identities | weight count | weights (device sections on the GPU)
        uint32_t raw = crc32_raw_host(0, h.data(), h.size());
        raw = crc32_shift(raw, id_bytes) ^ crc32_raw_device((const uint8_t*)T.dev.ident, id_bytes, st, T.device);
        raw = crc32_raw_host(raw, cnt.data(), 8);
        raw = crc32_shift(raw, w_bytes) ^ crc32_raw_device((const uint8_t*)T.dev.weights, w_bytes, st, T.device);
        const uint32_t crc = crc32_finish(raw, need - 4);
        uint8_t* o = out;
        std::memcpy(o, h.data(), h.size());
        o += h.size();
        MPZCH_CUDA(cudaMemcpyAsync(o, T.dev.ident, id_bytes, cudaMemcpyDeviceToHost, st));
        o += id_bytes;
        std::memcpy(o, cnt.data(), 8);
        o += 8;
        MPZCH_CUDA(cudaMemcpyAsync(o, T.dev.weights, w_bytes, cudaMemcpyDeviceToHost, st));
        o += w_bytes;
        for (int i = 0; i < 4; ++i) o[i] = (uint8_t)(crc >> (8 * i));
        MPZCH_CUDA(cudaStreamSynchronize(st));
    });
}

mpzch_status mpzch_serialize_delta(mpzch_table* t, uint64_t generation, uint32_t base_checksum,
                                   uint64_t sequence, uint8_t* out, uint64_t cap, uint64_t* out_len,
                                   uint64_t* out_next_generation) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        if (T.dim == 0) throw Error{MPZCH_ELOGIC, "index-only tables (dim = 0) cannot be published"};
        if (generation == 0 || generation >= T.gen_clock)
            throw Error{MPZCH_EINVAL, "stale or unknown publication cursor"};
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        flush_for_read(T);
        const unsigned k = run_dirty_compact(T, generation, st);
        const uint64_t rec = 16 + 4ull * T.dim, body = k * rec;
        const uint64_t need = 32 + body + 4;
        *out_len = need;
        if (!out) return;  // size query: the cursor does not move
        if (cap < need) throw Error{MPZCH_ELENGTH, "output buffer too small"};
        std::vector<uint8_t> h;  // serialize_delta, publish.cpp:212-230
        put_magic(h, "MPZD");
        put_u32(h, 1);
        put_u32(h, base_checksum);
        put_u64(h, sequence);
        put_u32(h, T.dim);
        put_u64(h, k);
        uint32_t raw = crc32_raw_host(0, h.data(), h.size());
        if (k) {
            T.p_rec.reserve(body);
            launch_pack_delta(T, T.p_rows.as<uint64_t>(), &T.d_aux->pad, k, T.p_rec.as<uint8_t>(), st);
            MPZCH_CUDA(cudaGetLastError());
            raw = crc32_shift(raw, body) ^ crc32_raw_device(T.p_rec.as<uint8_t>(), body, st, T.device);
            MPZCH_CUDA(cudaMemcpyAsync(out + 32, T.p_rec.p, body, cudaMemcpyDeviceToHost, st));
        }
        const uint32_t crc = crc32_finish(raw, 32 + body);
        std::memcpy(out, h.data(), 32);
        for (int i = 0; i < 4; ++i) out[32 + body + i] = (uint8_t)(crc >> (8 * i));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        *out_next_generation = T.gen_clock++;  // DeltaSource::cut: cursor_ = make_cursor()
    });
}

mpzch_status mpzch_set_reset_mode(mpzch_table* t, int mode) {
    CHECK_T(t);
    if (mode != MPZCH_RESET_EAGER && mode != MPZCH_RESET_DEFERRED) {
        g_last_error = "unknown reset mode";
        return MPZCH_EINVAL;
    }
    return guarded([&] {
        Table& T = *t->t;
        if (mode == MPZCH_RESET_EAGER) {
            flush_for_read(T);
            T.dev.pend_bits = nullptr;
        } else if (T.dim > 0 && !T.dev.pend_bits) {
            DeviceGuard g(T.device);
            const uint64_t bytes = (T.held_rows() + 31) / 32 * 4;
            T.pend_map.reserve(bytes);
            MPZCH_CUDA(cudaMemsetAsync(T.pend_map.p, 0, bytes, T.stream));
            MPZCH_CUDA(cudaStreamSynchronize(T.stream));
            T.dev.pend_bits = T.pend_map.as<uint32_t>();
        }
    });
}

mpzch_status mpzch_flush_resets(mpzch_table* t) {
    CHECK_T(t);
    return guarded([&] { flush_for_read(*t->t); });
}

mpzch_status mpzch_set_path(mpzch_table* t, int path) {
    CHECK_T(t);
    if (path != MPZCH_PATH_AUTO && path != MPZCH_PATH_ORDERED && path != MPZCH_PATH_ROUNDS) {
        g_last_error = "unknown execution path";
        return MPZCH_EINVAL;
    }
    t->t->path_override = path;
    return MPZCH_OK;
}

mpzch_status mpzch_last_stats(const mpzch_table* t, mpzch_batch_stats* out) {
    CHECK_T(t);
    *out = t->t->last;
    return MPZCH_OK;
}

uint64_t mpzch_kernel_launches(const mpzch_table* t) { return t && t->t ? t->t->launches : 0; }


// ---- the rest of the kept MpzchTable / batch_engine surface (csrc/surface.cu)

mpzch_status mpzch_process_shard_batch(mpzch_table* t, uint32_t shard, const uint64_t* ids,
                                       const uint64_t* metas, uint64_t n, uint64_t now,
                                       const mpzch_policy* policy, uint64_t* out_slots, uint8_t* out_oc) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        const Policy pol = parse_policy(policy);
        // table.cpp:116-119
        if (shard >= T.S) throw Error{MPZCH_ERANGE, "shard index out of range"};
        if (shard < T.shard_lo || shard >= T.shard_hi)
            throw Error{MPZCH_ERANGE, "shard is not held by this handle"};
        if (n == 0) return;
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        T.sb_buf.reserve(n * 33 + 64);
        uint8_t* b = T.sb_buf.as<uint8_t>();
        uint64_t* d_ids = (uint64_t*)b;
        uint64_t* d_metas = d_ids + n;
        uint64_t* d_slots = d_metas + n;
        uint64_t* d_reset = d_slots + n;
        unsigned long long* d_st = (unsigned long long*)(d_reset + n);
        unsigned* d_rc = (unsigned*)(d_st + 3);
        uint8_t* d_oc = (uint8_t*)(d_st + 4);
        MPZCH_CUDA(cudaMemcpyAsync(d_ids, ids, n * 8, cudaMemcpyHostToDevice, st));
        MPZCH_CUDA(cudaMemcpyAsync(d_metas, metas, n * 8, cudaMemcpyHostToDevice, st));
        MPZCH_CUDA(cudaMemsetAsync(d_st, 0xff, 8, st));
        launch_shard_batch(T, shard, pol.mode, d_ids, d_metas, n, now, d_slots, d_oc, d_reset, d_rc, d_st, st);
        if (T.dim) launch_reset_rows(T, d_reset, d_rc, st);
        MPZCH_CUDA(cudaGetLastError());
        unsigned long long h_st[3] = {0, 0, 0};
        MPZCH_CUDA(cudaMemcpyAsync(h_st, d_st, 24, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        // the positions before a failing one took effect and have their results (out[k] is
        // written inside the reference's loop before the next lookup_or_insert can throw)
        const uint64_t done = h_st[0] == ~0ull ? n : h_st[0];
        if (done) {
            MPZCH_CUDA(cudaMemcpyAsync(out_slots, d_slots, done * 8, cudaMemcpyDeviceToHost, st));
            MPZCH_CUDA(cudaMemcpyAsync(out_oc, d_oc, done, cudaMemcpyDeviceToHost, st));
            MPZCH_CUDA(cudaStreamSynchronize(st));
        }
        if (h_st[0] != ~0ull) {
            if (h_st[1] == 1) require_valid_id(h_st[2]);
            throw Error{MPZCH_EINVAL, pol.mode == kModeTtl ? "TTL metadata must be an expiry in the future"
                                                           : "non-TTL metadata must equal the current timestamp"};
        }
    });
}

static void dedup_common(const uint64_t* d_ids, const uint32_t* d_feats, uint64_t n, uint64_t* d_uids,
                         uint32_t* d_ufeats, uint32_t* d_inverse, uint64_t* out_u, cudaStream_t st) {
    uint64_t bad = ~0ull;
    const uint64_t u = run_dedup(d_ids, d_feats, n, d_uids, d_ufeats, d_inverse, &bad, st);
    if (bad != ~0ull) throw Error{MPZCH_EINVAL, "invalid id at batch position " + std::to_string(bad)};
    *out_u = u;
}

mpzch_status mpzch_dedup(int device, const uint64_t* ids, const uint32_t* features, uint64_t n,
                         uint64_t* out_unique_ids, uint32_t* out_unique_features, uint32_t* out_inverse,
                         uint64_t* out_u) {
    return guarded([&] {
        if (n > 0xffffffffull) throw Error{MPZCH_ELENGTH, "batch exceeds 2^32 - 1 positions"};
        *out_u = 0;
        if (n == 0) return;
        DeviceGuard g(device);
        cudaStream_t st = nullptr;
        MPZCH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{st};
        uint8_t* b = nullptr;
        MPZCH_CUDA(cudaMallocAsync((void**)&b, n * 28, st));
        struct FreeGuard {
            uint8_t* p;
            cudaStream_t s;
            ~FreeGuard() { cudaFreeAsync(p, s); cudaStreamSynchronize(s); }
        } fg{b, st};
        uint64_t* d_ids = (uint64_t*)b;
        uint64_t* d_uids = d_ids + n;
        uint32_t* d_feats = (uint32_t*)(d_uids + n);
        uint32_t* d_ufeats = d_feats + n;
        uint32_t* d_inv = d_ufeats + n;
        MPZCH_CUDA(cudaMemcpyAsync(d_ids, ids, n * 8, cudaMemcpyHostToDevice, st));
        if (features) MPZCH_CUDA(cudaMemcpyAsync(d_feats, features, n * 4, cudaMemcpyHostToDevice, st));
        uint64_t u = 0;
        dedup_common(d_ids, features ? d_feats : nullptr, n, d_uids, d_ufeats, d_inv, &u, st);
        MPZCH_CUDA(cudaMemcpyAsync(out_unique_ids, d_uids, u * 8, cudaMemcpyDeviceToHost, st));
        if (out_unique_features)
            MPZCH_CUDA(cudaMemcpyAsync(out_unique_features, d_ufeats, u * 4, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaMemcpyAsync(out_inverse, d_inv, n * 4, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        *out_u = u;
    });
}

mpzch_status mpzch_dedup_device(int device, const uint64_t* ids, const uint32_t* features, uint64_t n,
                                uint64_t* unique_ids, uint32_t* unique_features, uint32_t* inverse,
                                uint64_t* out_u, void* stream) {
    return guarded([&] {
        if (n > 0xffffffffull) throw Error{MPZCH_ELENGTH, "batch exceeds 2^32 - 1 positions"};
        *out_u = 0;
        if (n == 0) return;
        DeviceGuard g(device);
        dedup_common(ids, features, n, unique_ids, unique_features, inverse, out_u, (cudaStream_t)stream);
    });
}

mpzch_status mpzch_reset_row(mpzch_table* t, uint64_t row) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        check_rows(T, row, 1);  // check_embeddings, then check_row (table.cpp:181-186)
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        T.sb_buf.reserve(64);
        uint64_t* d = T.sb_buf.as<uint64_t>();
        const uint64_t h[2] = {row, 1};  // the row, then the list length (as a u32 in word 1)
        MPZCH_CUDA(cudaMemcpyAsync(d, h, 16, cudaMemcpyHostToDevice, st));
        launch_reset_rows(T, d, (const unsigned*)(d + 1), st);
        MPZCH_CUDA(cudaMemcpyAsync(T.dev.row_gen + row, &T.gen_clock, 8, cudaMemcpyHostToDevice, st));  // touch_row
        MPZCH_CUDA(cudaStreamSynchronize(st));
    });
}

mpzch_status mpzch_state_equals(const mpzch_table* a, const mpzch_table* b, int* out_equal) {
    if (!a || !a->t || !b || !b->t) {
        g_last_error = "null table handle";
        return MPZCH_EINVAL;
    }
    return guarded([&] {
        const Table& A = *a->t;
        const Table& B = *b->t;
        flush_for_read(A);
        flush_for_read(B);
        *out_equal = 0;
        // table.cpp:249-260: capacities, dim, identities of every shard, weights (bitwise)
        if (A.caps != B.caps || A.dim != B.dim) return;
        if (A.held_rows() != A.total || B.held_rows() != B.total)
            throw Error{MPZCH_EINVAL, "state_equals needs handles that hold every shard"};
        auto same = [&](const void* pa, const void* pb, uint64_t bytes) {
            if (!bytes) return true;
            DeviceGuard g(A.device);
            MPZCH_CUDA(cudaStreamSynchronize(A.stream));
            if (A.device == B.device) return run_words_equal(pa, pb, bytes, A.stream);
            {
                DeviceGuard gb(B.device);
                MPZCH_CUDA(cudaStreamSynchronize(B.stream));
            }
            const uint64_t chunk = 256ull << 20;  // B's bytes staged on A's device
            void* tmp = nullptr;
            MPZCH_CUDA(cudaMalloc(&tmp, std::min(chunk, bytes)));
            bool eq = true;
            for (uint64_t o = 0; o < bytes && eq; o += chunk) {
                const uint64_t c = std::min(chunk, bytes - o);
                MPZCH_CUDA(cudaMemcpyPeer(tmp, A.device, (const uint8_t*)pb + o, B.device, c));
                eq = run_words_equal((const uint8_t*)pa + o, tmp, c, A.stream);
            }
            cudaFree(tmp);
            return eq;
        };
        if (!same(A.ident + (A.row_lo - A.row_base), B.ident + (B.row_lo - B.row_base), A.total * 8)) return;
        if (A.dim && !same(A.dev.weights, B.dev.weights, A.total * A.dim * 4)) return;
        *out_equal = 1;
    });
}

mpzch_status mpzch_read_identity(const mpzch_table* t, uint64_t row, uint64_t* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        if (row >= T.total) throw Error{MPZCH_ERANGE, "global row out of range"};  // from_global
        if (row < T.row_lo || row >= T.row_hi) throw Error{MPZCH_ERANGE, "row is not held by this handle"};
        DeviceGuard g(T.device);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        MPZCH_CUDA(cudaMemcpy(out, T.dev.ident + row, 8, cudaMemcpyDeviceToHost));
    });
}

static void check_held_range(const Table& T, uint64_t row0, uint64_t nrows) {
    if (row0 < T.row_lo || row0 > T.row_hi || nrows > T.row_hi - row0)
        throw Error{MPZCH_ERANGE, "row range is not held by this handle"};
}

mpzch_status mpzch_copy_identities_range(const mpzch_table* t, uint64_t row0, uint64_t nrows, uint64_t* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        check_held_range(T, row0, nrows);
        DeviceGuard g(T.device);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        if (nrows) MPZCH_CUDA(cudaMemcpy(out, T.dev.ident + row0, nrows * 8, cudaMemcpyDeviceToHost));
    });
}

mpzch_status mpzch_copy_metadata_range(const mpzch_table* t, uint64_t row0, uint64_t nrows, uint64_t* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        check_held_range(T, row0, nrows);
        DeviceGuard g(T.device);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
        if (nrows) MPZCH_CUDA(cudaMemcpy(out, T.dev.meta + row0, nrows * 8, cudaMemcpyDeviceToHost));
    });
}

mpzch_status mpzch_copy_trained_range(const mpzch_table* t, uint64_t row0, uint64_t nrows, uint8_t* out) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        flush_for_read(T);
        check_rows(T, row0, nrows);
        DeviceGuard g(T.device);
        if (nrows) copy_trained_bytes(const_cast<Table&>(T), row0, nrows, out);
    });
}

mpzch_status mpzch_gather(const mpzch_table* t, const uint64_t* rows, uint64_t n, float* out) {
    CHECK_T(t);
    return guarded([&] {
        Table& T = *t->t;
        check_rows(T, T.row_lo, 0);
        for (uint64_t i = 0; i < n; ++i)  // embedding_store.cpp:97-98, first bad row
            if (rows[i] < T.row_lo || rows[i] >= T.row_hi) throw Error{MPZCH_ERANGE, "embedding row out of range"};
        if (n == 0) return;
        DeviceGuard g(T.device);
        cudaStream_t st = T.stream;
        order_after_last_batch(T, st);
        const uint64_t rows_bytes = (n * 8 + 255) & ~255ull;  // the rows stay 16-byte aligned (float4 stores)
        T.sb_buf.reserve(rows_bytes + n * T.dim * 4);
        uint64_t* d_rows = T.sb_buf.as<uint64_t>();
        float* d_out = (float*)(T.sb_buf.as<char>() + rows_bytes);
        MPZCH_CUDA(cudaMemcpyAsync(d_rows, rows, n * 8, cudaMemcpyHostToDevice, st));
        run_gather_weights(T, d_rows, n, d_out, st);
        ++T.launches;
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(out, d_out, n * T.dim * 4, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
    });
}

mpzch_status mpzch_shard_config(const mpzch_table* t, uint32_t shard, uint64_t* capacity, uint32_t* max_probe,
                                uint64_t* seed) {
    CHECK_T(t);
    return guarded([&] {
        const Table& T = *t->t;
        if (shard >= T.S) throw Error{MPZCH_ERANGE, "shard index out of range"};  // table.cpp:241-244
        if (capacity) *capacity = T.caps[shard];
        if (max_probe) *max_probe = T.P;
        if (seed) *seed = T.seed;
    });
}

}  // extern "C"
