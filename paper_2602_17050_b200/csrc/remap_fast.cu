// remap_fast.cu -- the B200 fast path of process_batch (proj/src/batch_engine.cpp:141-221)
// for hole-free tables under Disabled, TTL (one metadata value per batch, or per-feature values
// through the last-writer pass M1-M3 below) and LRU (evictions placed by K3a/K3b below, or the
// batch reverts to the rounds path).
//
// Exactness argument: within a batch the set of slots a new id may
// take only shrinks (EMPTY -> id, expired -> live), every unique probes its own window,
// and the sequential reference gives each new id the first available slot of its
// window not taken by a lower-rank unique.  The kernels below reach exactly that
// assignment without any ordering pass:
//
//   K0 validate   streaming pass over the ids: first invalid position (and, on a
//                 row-sharded handle, ids of shards it does not hold).  Nothing below
//                 mutates a batch that failed here.
//   K1 probe      one thread per POSITION, 32-byte sector loads from the home slot up to
//                 the first match or EMPTY (hole-free early exit); long
//                 windows and small batches: one quad per position, 128-byte lines (long
//                 Disabled windows past their first line: 128-slot tag lines).  TTL:
//                 walks still pending after 8 sector rounds resume in a quad-line launch.
//                 Hits on live slots and full windows are final here and write their
//                 metadata word; everything else goes to the new list.
//   K2 dedup      new positions -> one 64-byte entry per distinct id (128-bit atomicCAS on
//                 an epoch-tagged key), rank = first position (atomicMax of ~position).
//                 (id, feature) secondaries are resolved from the id's first position in K5.
//   K3 claim      every entry claims slots in its window by a 64-bit atomicMin (EMPTY slots,
//                 claim words) or atomicCAS (TTL: expired ids) of a rank-stamped claim word
//                 into the identity array itself.  A claim
//                 with a lower rank replaces a higher one; the thread that displaces a
//                 claim continues the displaced entry's scan ("takeover"), so the
//                 fixpoint -- each entry on the first slot no lower rank holds -- is
//                 reached in one launch with no grid barrier.
//   K4 commit     claim words -> ids, outcomes (Inserted/Evicted/Found-owner), the entry's
//                 metadata word, touch_row, reset list, evicted flags by rank, and the
//                 result of the entry's own (first) position.
//   K5 finalize   results of the later positions of repeated new ids (+ secondary (id, f')
//                 rule); a no-op when the dedup saw no repeated id.
// One metadata value per batch makes every metadata write order-free.
#include <cuda_runtime.h>

#include "common.cuh"
#include "line_scan.cuh"
#include "tag_scan.cuh"
#include "table.hpp"

#include <cstdlib>
#include <string>

namespace mpzch_b200 {

namespace {

constexpr uint64_t kClaimBit = 1ull << 63;
constexpr uint64_t kFlagEmpty = 1ull << 30;  // the claimed slot was EMPTY before the batch
constexpr uint64_t kEntryMask = (1ull << 30) - 1;
constexpr uint8_t kStateCollided = 1;
constexpr uint8_t kStateEvict = 2;     // LRU: the entry evicts the slot at offset `held` (K3b)
constexpr uint8_t kPendingOc = 0xFF;   // LRU: out_oc of a position on the new list until K4/K5
// TTL: newa's flag for "the first available slot was EMPTY when probed" (not expired): K3 tries
// it with a blind atomicMin; K2 moves the flag into the entry record (IdEntry::aempty)
constexpr uint32_t kAEmpty = 1u << 31;

// Distinct new ids: a hash index of 16-byte keys (id | (epoch32 << 32 | e) << 64 -- a key whose
// epoch is not the current batch's is empty, so no cleanup pass is needed) and DENSE entry
// records, entry e = the new-list index of the item that inserted the id.  Most ids occur
// once, so item k's entry is te[k]: the claim / commit / finalize passes over the new list read
// their records coalesced instead of at random hash slots (C3: a 256 MB hash-addressed record
// table for 1.5 M new ids, read at random by every pass).  The rank word (epoch << 32 |
// ~first position) is updated with atomicMax, which keeps the current epoch and the smallest
// first position without an initialising write.
typedef unsigned __int128 u128;

__device__ __forceinline__ u128 make_key(uint32_t epoch32, uint32_t e, uint64_t id) {
    return ((u128)(((uint64_t)epoch32 << 32) | e) << 64) | (u128)id;
}
__device__ __forceinline__ uint64_t key_id(u128 k) { return (uint64_t)k; }
__device__ __forceinline__ uint32_t key_epoch(u128 k) { return (uint32_t)(k >> 96); }
__device__ __forceinline__ uint32_t key_entry(u128 k) { return (uint32_t)(k >> 64); }
__device__ __forceinline__ uint32_t rank_of(uint64_t tr) { return ~(uint32_t)tr; }

// One entry in one 64-byte record, so every kernel's accesses to an entry (rank, claim
// bookkeeping, result) land in the same DRAM burst.
struct __align__(64) IdEntry {
    uint64_t id;
    uint64_t pad2;
    unsigned long long rank;  // epoch << 32 | ~first position   (atomicMax)
    uint32_t a;               // first available offset (taker start)
    uint32_t m;               // owner: offset of the expired own slot, else kNone32
    uint32_t held;            // last taker claim offset          (atomicMax)
    uint8_t state;            // kStateCollided when the window is exhausted
    uint8_t oc;               // committed outcome
    uint8_t aempty;           // TTL: slot a was EMPTY when probed (newa's kAEmpty)
    uint8_t pad0;
    uint64_t slot;            // committed global slot
    uint64_t pad1[2];
};
static_assert(sizeof(IdEntry) == 64, "IdEntry must be one 64-byte record");

__device__ __forceinline__ bool is_claim(uint64_t v) { return (v >> 63) != 0 && v != kEmpty; }
__device__ __forceinline__ uint32_t claim_rank(uint64_t v) { return (uint32_t)(v >> 31); }
__device__ __forceinline__ uint32_t claim_entry(uint64_t v) { return (uint32_t)(v & kEntryMask); }

__device__ __forceinline__ uint64_t wrap_add(uint64_t h, uint64_t off, uint64_t cap) {
    uint64_t x = h + off;
    return x >= cap ? x - cap : x;
}

// Id-table sizing: power of two >= 2 * count, at least 1024, at most the allocation.
// (Sizing by positions instead, so the probe could prefetch records, measured slower.)
__device__ __forceinline__ uint64_t table_mask(unsigned count, uint64_t cap_alloc) {
    uint64_t c = 1024;
    while (c < 2ull * count && c < cap_alloc) c <<= 1;
    return c - 1;
}

__device__ __forceinline__ uint64_t te_home(uint64_t id, uint64_t mask) {
    return mix64(id, 0x2545F4914F6CDD1Dull) & mask;
}

__device__ __forceinline__ u128 ld_cg_u128(const u128* p) {
    uint64_t lo, hi;
    asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p));
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ uint64_t pick4(uint32_t j, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return j == 0 ? a : (j == 1 ? b : (j == 2 ? c : d));
}


__global__ void k_init_counters(BatchCounters* c) {
    if (threadIdx.x == 0) {
        BatchCounters z{};
        z.err.bad_pos = ~0ull;
        z.err.foreign_pos = ~0ull;
        z.n_live = ~0ull;
        *c = z;
    }
}

// row-sharded owner (sharded.cu): the batch's fate was decided by the ranks together -- on any
// error every kernel below skips (the host reports it from the shared state); otherwise the
// received count bounds every position loop (n_live)
__global__ void k_sh_adopt(BatchCounters* c, const ShStateView* st) {
    pdl_wait();
    if (threadIdx.x == 0) {  // the counters' initialisation and the ranks' decision, one launch
        BatchCounters z{};
        z.err.bad_pos = ~0ull;
        z.err.foreign_pos = ~0ull;
        z.n_live = ~0ull;
        if (st->failed) z.err.overflow = 1;
        else z.n_live = st->R;
        *c = z;
    }
}

// K0: streaming validation of the batch (batch_engine.cpp:90-94): min invalid position.
// Runs before anything mutates, so the probe can write metadata for final positions.
__global__ void __launch_bounds__(256) k_validate(TableDev t, const uint64_t* __restrict__ ids,
                                                  uint64_t n, BatchCounters* ctr) {
    pdl_wait();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long bad = ~0ull;
    if ((reinterpret_cast<uintptr_t>(ids) & 15) == 0) {
        const uint64_t n2 = n / 2;
        const ulonglong2* v2 = reinterpret_cast<const ulonglong2*>(ids);
        uint64_t q = tid;
        for (; q + 3 * stride < n2; q += 4 * stride) {  // four 16-byte loads in flight
            ulonglong2 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] = __ldcs(v2 + q + r * stride);
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if ((v[r].x | v[r].y) >> 63) {
                    const uint64_t qq = q + r * stride;
                    bad = min(bad, (unsigned long long)(v[r].x >> 63 ? 2 * qq : 2 * qq + 1));
                }
        }
        for (; q < n2; q += stride) {
            const ulonglong2 v = __ldcs(v2 + q);
            if ((v.x | v.y) >> 63) bad = min(bad, (unsigned long long)(v.x >> 63 ? 2 * q : 2 * q + 1));
        }
        if (tid == 0 && (n & 1) && (ids[n - 1] >> 63)) bad = min(bad, (unsigned long long)(n - 1));
    } else {
        for (uint64_t i = tid; i < n; i += stride)
            if (ids[i] >> 63) bad = min(bad, (unsigned long long)i);
    }
    if (bad != ~0ull) atomicMin(&ctr->err.bad_pos, bad);
    // row-sharded handle: every id must route to a shard it holds
    if (t.shard_lo != 0 || t.shard_hi != t.nshards.d) {
        unsigned long long foreign = ~0ull;
        for (uint64_t i = tid; i < n; i += stride) {
            const uint64_t id = ids[i];
            if (!(id >> 63) && !holds_shard(t, shard_of(id, t))) foreign = min(foreign, (unsigned long long)i);
        }
        if (foreign != ~0ull) atomicMin(&ctr->err.foreign_pos, foreign);
    }
}

// K1: probe; each thread keeps U positions in flight (independent sector loads), all
// positions of a round are issued before any is scanned.
// TTL walks of new ids run to the first EMPTY through windows full of live and expired ids (C2:
// a few % of the positions, but most warps hold one, and the warp waits for it).  With
// defer > 0 a walk still pending after `defer` rounds is handed over -- (position, offset, first
// expired offset) -- to a RESUME launch of the same kernel, whose warps hold long walks only.
// Exact: K1 writes no identity and only refreshes live slots (they stay live), so a resumed
// walk reads what it would have read.
template <int MODE, int U, int MINB, bool PF = false, bool RESUME = false, bool DEFER = false>
__global__ void __launch_bounds__(256, MINB) k_probe(TableDev t, const uint64_t* __restrict__ ids,
                                               uint64_t n, uint64_t now, uint64_t meta_value,
                                               BatchCounters* ctr,
                                               uint64_t* __restrict__ out_slots,
                                               uint8_t* __restrict__ out_oc,
                                               uint32_t* __restrict__ newpos,
                                               uint64_t* __restrict__ newid,
                                               uint32_t* __restrict__ newa,
                                               uint32_t* __restrict__ newm,
                                               uint32_t* __restrict__ dlist = nullptr,
                                               unsigned defer = 0) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    constexpr uint8_t kPending = 0, kHit = 1, kEmptyHit = 2, kExhausted = 3, kIdle = 4, kDeferred = 5;
    const unsigned lane = lane_id();
    const uint64_t tile = (uint64_t)blockDim.x * U;
    unsigned long long my_found = 0, my_coll = 0, my_isec = 0, my_msec = 0;
    const uint64_t total = RESUME ? (uint64_t)*(volatile unsigned*)&ctr->deferred : min(n, (uint64_t)ctr->n_live);
    for (uint64_t t0 = (uint64_t)blockIdx.x * tile; t0 < total; t0 += (uint64_t)gridDim.x * tile) {
        uint64_t id[U], g[U], base[U], cap[U], h[U];
        uint32_t pos[RESUME ? U : 1];  // RESUME: the handed-over positions
        uint32_t off[U];
        uint32_t fe[U];  // TTL: offset of the first expired slot walked before the stop
        bool hexp[U];    // TTL: the matched slot itself is expired
        uint64_t hmv[MODE == kModeTtl ? U : 1];  // TTL: the matched slot's metadata word
        bool mld[U];     // TTL: this round's metadata sector was loaded
        uint8_t st[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = t0 + (uint64_t)u * blockDim.x + threadIdx.x;
            st[u] = kIdle;
            off[u] = 0;
            fe[u] = kNone32;
            hexp[u] = false;
            mld[u] = false;
            if (i < total) {
                uint64_t p = i;
                if (RESUME) {
                    pos[u] = dlist[3 * i];
                    off[u] = dlist[3 * i + 1];
                    fe[u] = dlist[3 * i + 2];
                    p = pos[u];
                }
                id[u] = ids[p];
                const ShardDev sd = t.shards[shard_of(id[u], t)];
                cap[u] = sd.cap.d;
                base[u] = sd.offset;
                h[u] = home_of(id[u], sd, t.seed);
                g[u] = base[u] + (RESUME ? wrap_add(h[u], off[u], cap[u]) : h[u]);
                st[u] = kPending;
            }
        }
        unsigned rounds = 0;  // (DEFER)
        // scan rounds: issue every pending position's next sector, then scan them.  (Handing
        // long runs to a warp-cooperative kernel, or staging sectors in shared memory with
        // cp.async behind block barriers, both measured slower on C5 and C3.)
        for (;;) {
            uint64_t w[U][4];
            uint64_t mw[MODE == kModeTtl ? U : 1][4];  // TTL: the metadata sector, same round
            bool any = false;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (st[u] == kPending) {
                    ld_sector(t.ident + (g[u] & ~3ull), w[u][0], w[u][1], w[u][2], w[u][3]);
                    ++my_isec;
                    // TTL: the metadata sector comes in the same round until the walk has
                    // seen an expired slot (after that only a hit's own word is needed)
                    if (MODE == kModeTtl) {
                        mld[u] = fe[u] == kNone32;
                        if (mld[u]) {
                            ld_sector(t.meta + (g[u] & ~3ull), mw[u][0], mw[u][1], mw[u][2], mw[u][3]);
                            ++my_msec;
                        }
                    }
                }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (st[u] != kPending) continue;
                const uint64_t a4 = g[u] & ~3ull, end = base[u] + cap[u];
                do {
                    const uint32_t jj = (uint32_t)(g[u] - a4);
                    const uint64_t v = pick4(jj, w[u][0], w[u][1], w[u][2], w[u][3]);
                    if (v == id[u]) {
                        st[u] = kHit;
                        if (MODE == kModeTtl) {
                            hmv[MODE == kModeTtl ? u : 0] =
                                mld[u] ? pick4(jj, mw[u][0], mw[u][1], mw[u][2], mw[u][3]) : __ldg(t.meta + g[u]);
                            hexp[u] = hmv[MODE == kModeTtl ? u : 0] < now;
                        }
                        break;
                    }
                    if (v == kEmpty) { st[u] = kEmptyHit; break; }
                    if (MODE == kModeTtl && mld[u] && fe[u] == kNone32 &&
                        pick4(jj, mw[u][0], mw[u][1], mw[u][2], mw[u][3]) < now)
                        fe[u] = off[u];
                    ++off[u];
                    if (++g[u] == end) g[u] = base[u];
                } while (off[u] < t.P && (g[u] >> 2) == (a4 >> 2));
                if (st[u] == kPending) {
                    if (off[u] >= t.P) st[u] = kExhausted;
                    else any = true;
                }
            }
            if (DEFER && any && ++rounds >= defer) {  // hand the long walks over (below)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (st[u] == kPending) st[u] = kDeferred;
                any = false;
            }
            if (!any) break;
        }
        if (DEFER) {  // append the handed-over walks (the new-list ballot below
                                 // carries the warp's other appends)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (st[u] != kDeferred) continue;
                // one counter update per group of deferring lanes
                const unsigned am = __activemask();
                const unsigned leader = __ffs(am) - 1;
                unsigned b0 = 0;
                if (lane == leader) b0 = atomicAdd(&ctr->deferred, (unsigned)__popc(am));
                b0 = __shfl_sync(am, b0, leader);
                const unsigned k = b0 + __popc(am & ((1u << lane) - 1));
                dlist[3 * k] = (uint32_t)(t0 + (uint64_t)u * blockDim.x + threadIdx.x);
                dlist[3 * k + 1] = off[u];
                dlist[3 * k + 2] = fe[u];
            }
        }
        // decisions, final writes (result + metadata word) and the new list
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = RESUME ? (uint64_t)pos[RESUME ? u : 0] : t0 + (uint64_t)u * blockDim.x + threadIdx.x;
            bool is_new = false;
            uint32_t a_off = 0, m_off = kNone32;
            if (st[u] != kIdle && st[u] != kDeferred) {
                uint64_t fslot = kEmpty;
                uint8_t foc = kFound;
                if (MODE != kModeTtl) {
                    if (st[u] == kHit) fslot = g[u];
                    else if (st[u] == kEmptyHit) {
                        is_new = true;
                        a_off = off[u];
                        // Disabled: the likely result -- Inserted at the walk's EMPTY -- written
                        // with this warp's other results; K4 rewrites only positions it differs for
                        if (MODE == kModeDisabled) { out_slots[i] = g[u]; out_oc[i] = kInserted; }
                    }
                    // LRU full window: an evictor -- its claim finds nothing (a = P) and K3b
                    // picks the least recently used slot
                    else if (MODE == kModeLru) { is_new = true; a_off = t.P; }
                    else { fslot = base[u] + h[u]; foc = kCollision; }
                } else {  // TTL with one metadata value per batch (expiry read with the walk)
                    if (st[u] == kHit) {
                        if (!hexp[u]) {
                            fslot = g[u];  // live: nobody can take it in this batch
                        } else {           // expired own slot: lower-rank new ids contest it
                            is_new = true;
                            m_off = off[u];
                            a_off = fe[u] != kNone32 ? fe[u] : off[u];
                        }
                    } else {
                        const uint32_t lim = st[u] == kEmptyHit ? off[u] : t.P;
                        const uint32_t x = fe[u] != kNone32 ? fe[u] : lim;
                        if (x < lim || st[u] == kEmptyHit) {
                            is_new = true;
                            a_off = x | (x == lim ? kAEmpty : 0u);  // (x == lim: the walk's EMPTY)
                            if (x == lim) { out_slots[i] = g[u]; out_oc[i] = kInserted; }  // likely result
                        }
                        else { fslot = base[u] + h[u]; foc = kCollision; }
                    }
                }
                if (fslot != kEmpty) {
                    out_slots[i] = fslot;
                    out_oc[i] = foc;
                    // Found refresh / Collision at home (LRU: deferred to k_lru_meta, the
                    // batch may still turn out to need an eviction)
                    // (per-feature TTL: the last-writer pass after K5 writes it)
                    // (TTL: a live hit whose word already holds the batch's value -- a hot id's
                    // later positions under skewed traffic -- skips the store: thousands of
                    // stores to one word serialise in the L2)
                    if (MODE != kModeLru && !PF &&
                        !(MODE == kModeTtl && foc == kFound && hmv[MODE == kModeTtl ? u : 0] == meta_value))
                        t.meta[fslot] = meta_value;
                    if (foc == kFound) ++my_found; else ++my_coll;
                } else if (MODE == kModeLru) {
                    out_oc[i] = kPendingOc;  // K3a tells Found positions apart by this byte
                }
            }
            // warp-aggregated append of the new positions (a block barrier here would make
            // every warp wait for the slowest probe of the tile: measured slower)
            const unsigned mask = __ballot_sync(0xffffffffu, is_new);
            if (mask) {
                unsigned basek = 0;
                if (lane == 0) basek = atomicAdd(&ctr->new_count, (unsigned)__popc(mask));
                basek = __shfl_sync(0xffffffffu, basek, 0);
                if (is_new) {
                    const unsigned k = basek + __popc(mask & ((1u << lane) - 1));
                    newpos[k] = (uint32_t)i;
                    newid[k] = id[u];
                    newa[k] = a_off;
                    newm[k] = m_off;
                }
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        my_found += __shfl_xor_sync(0xffffffffu, my_found, o);
        my_coll += __shfl_xor_sync(0xffffffffu, my_coll, o);
        my_isec += __shfl_xor_sync(0xffffffffu, my_isec, o);
        my_msec += __shfl_xor_sync(0xffffffffu, my_msec, o);
    }
    if (lane == 0) {
        if (my_found) atomicAdd(&ctr->found, my_found);
        if (my_coll) atomicAdd(&ctr->collision, my_coll);
        if (my_isec) atomicAdd(&ctr->id_sectors, my_isec);
        if (my_msec) atomicAdd(&ctr->meta_sectors, my_msec);
    }
}

// K1 (line variant): one QUAD of lanes per position, U positions in flight per quad.  Each
// scan round reads the whole 128-byte identity line of every pending position with one warp
// instruction (lane j: sector j) -- the same cost per access as a single sector on B200
// (line_scan.cuh) -- and finds the first match / EMPTY of the window part in that line with
// one 16-bit mask.  Decisions, writes and the new-list append are made by lane 0 of the quad.
// RESUME: the walks k_probe<..., DEFER> handed over, continued a 128-byte line per round trip
// (a long walk is a chain of dependent loads: 4x fewer round trips than sector by sector).
template <int MODE, int U, int MINB, bool PF = false, bool RESUME = false>
__global__ void __launch_bounds__(256, MINB) k_probe_line(TableDev t, const uint64_t* __restrict__ ids,
                                                          uint64_t n, uint64_t now, uint64_t meta_value,
                                                          BatchCounters* ctr,
                                                          uint64_t* __restrict__ out_slots,
                                                          uint8_t* __restrict__ out_oc,
                                                          uint32_t* __restrict__ newpos,
                                                          uint64_t* __restrict__ newid,
                                                          uint32_t* __restrict__ newa,
                                                          uint32_t* __restrict__ newm,
                                                          const uint32_t* __restrict__ dlist = nullptr) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    constexpr uint8_t kPending = 0, kHit = 1, kEmptyHit = 2, kExhausted = 3, kIdle = 4;
    const unsigned lane = lane_id();
    const unsigned j = quad_lane(), qm = quad_mask();
    const uint64_t qpb = blockDim.x >> 2;  // quads per block
    const uint64_t qib = threadIdx.x >> 2;
    const uint64_t tile = qpb * U;
    unsigned long long my_found = 0, my_coll = 0, my_isec = 0, my_msec = 0;
    const uint64_t total = RESUME ? (uint64_t)*(volatile unsigned*)&ctr->deferred : min(n, (uint64_t)ctr->n_live);
    for (uint64_t t0 = (uint64_t)blockIdx.x * tile; t0 < total; t0 += (uint64_t)gridDim.x * tile) {
        uint64_t id[U], g[U];
        uint32_t pos[RESUME ? U : 1];
        uint32_t off[U], sh[U];
        uint32_t fe[U];  // TTL: offset of the first expired slot walked before the stop
        bool hexp[U];    // TTL: the matched slot itself is expired
        bool mld[U];     // TTL: this round's metadata line was loaded
        uint8_t st[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = t0 + (uint64_t)u * qpb + qib;
            st[u] = kIdle;
            off[u] = 0;
            fe[u] = kNone32;
            hexp[u] = false;
            mld[u] = false;
            if (i < total) {
                uint64_t p = i;
                if (RESUME) {
                    pos[u] = dlist[3 * i];
                    off[u] = dlist[3 * i + 1];
                    fe[u] = dlist[3 * i + 2];
                    p = pos[u];
                }
                id[u] = ids[p];
                sh[u] = shard_of(id[u], t);
                const ShardDev sd = t.shards[sh[u]];
                const uint64_t hh = home_of(id[u], sd, t.seed);
                g[u] = sd.offset + (RESUME ? wrap_add(hh, off[u], sd.cap.d) : hh);
                st[u] = kPending;
            }
        }
        for (;;) {
            uint64_t w[U][4];
            uint64_t mw[MODE == kModeTtl ? U : 1][4];  // TTL: the metadata line, same round
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (st[u] == kPending) {
                    ld_line_part(t.ident, g[u], j, w[u]);
                    if (MODE == kModeTtl) {  // until the walk has seen an expired slot
                        mld[u] = fe[u] == kNone32;
                        if (mld[u]) ld_line_part(t.meta, g[u], j, mw[u]);
                    }
                }
            bool any = false;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (st[u] != kPending) continue;
                unsigned m = 0, e = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    m |= (unsigned)(w[u][k] == id[u]) << k;
                    e |= (unsigned)(w[u][k] == kEmpty) << k;
                }
                const unsigned x = quad_gather(m, e, j, qm);
                unsigned xe = 0;
                if (MODE == kModeTtl && mld[u]) {
                    unsigned x4 = 0;
#pragma unroll
                    for (int k2 = 0; k2 < 4; ++k2) x4 |= (unsigned)(mw[u][k2] < now) << k2;
                    xe = quad_gather(x4, 0, j, qm) & 0xFFFFu;
                }
                const ShardDev sd = t.shards[sh[u]];
                const uint64_t base = sd.offset, end = base + sd.cap.d;
                const LineSpan sp = line_span(g[u], end, off[u], t.P);
                const unsigned hit = (x | (x >> 16)) & sp.range();
                if (hit) {
                    const unsigned p = __ffs(hit) - 1;
                    st[u] = (x >> p) & 1u ? kHit : kEmptyHit;
                    if (MODE == kModeTtl) {
                        const unsigned before = xe & sp.range() & ((1u << p) - 1u);
                        if (fe[u] == kNone32 && before) fe[u] = off[u] + (__ffs(before) - 1 - sp.s);
                        hexp[u] = mld[u] ? (xe >> p) & 1u : __ldg(t.meta + g[u] + (p - sp.s)) < now;
                        if (mld[u]) my_msec += sp.sectors_to(p);
                    }
                    off[u] += p - sp.s;
                    g[u] += p - sp.s;
                    my_isec += sp.sectors_to(p);
                } else {
                    if (MODE == kModeTtl && mld[u]) {
                        const unsigned ex = xe & sp.range();
                        if (fe[u] == kNone32 && ex) fe[u] = off[u] + (__ffs(ex) - 1 - sp.s);
                        my_msec += sp.sectors_to(sp.s + sp.c - 1);
                    }
                    my_isec += sp.sectors_to(sp.s + sp.c - 1);
                    off[u] += sp.c;
                    g[u] += sp.c;
                    if (g[u] == end) g[u] = base;
                    if (off[u] >= t.P) st[u] = kExhausted;
                    else any = true;
                }
            }
            if (!any) break;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = RESUME ? (uint64_t)pos[RESUME ? u : 0] : t0 + (uint64_t)u * qpb + qib;
            bool is_new = false;
            uint32_t a_off = 0, m_off = kNone32;
            if (st[u] != kIdle) {
                const ShardDev sd = t.shards[sh[u]];
                const uint64_t base = sd.offset;
                const uint64_t h = home_of(id[u], sd, t.seed);
                uint64_t fslot = kEmpty;
                uint8_t foc = kFound;
                if (MODE != kModeTtl) {
                    if (st[u] == kHit) fslot = g[u];
                    else if (st[u] == kEmptyHit) {
                        is_new = true;
                        a_off = off[u];
                        if (MODE == kModeDisabled && j == 0) { out_slots[i] = g[u]; out_oc[i] = kInserted; }  // (as k_probe)
                    }
                    else if (MODE == kModeLru) { is_new = true; a_off = t.P; }  // evictor (K3b)
                    else { fslot = base + h; foc = kCollision; }
                } else {  // TTL with one metadata value per batch (expiry read with the walk)
                    if (st[u] == kHit) {
                        if (!hexp[u]) {
                            fslot = g[u];  // live: nobody can take it in this batch
                        } else {           // expired own slot: lower-rank new ids contest it
                            is_new = true;
                            m_off = off[u];
                            a_off = fe[u] != kNone32 ? fe[u] : off[u];
                        }
                    } else {
                        const uint32_t lim = st[u] == kEmptyHit ? off[u] : t.P;
                        const uint32_t xo = fe[u] != kNone32 ? fe[u] : lim;
                        if (xo < lim || st[u] == kEmptyHit) {
                            is_new = true;
                            a_off = xo | (xo == lim ? kAEmpty : 0u);  // (xo == lim: the walk's EMPTY)
                            if (xo == lim && j == 0) { out_slots[i] = g[u]; out_oc[i] = kInserted; }  // likely result
                        }
                        else { fslot = base + h; foc = kCollision; }
                    }
                }
                if (fslot != kEmpty && j == 0) {
                    out_slots[i] = fslot;
                    out_oc[i] = foc;
                    if (MODE != kModeLru && !PF) t.meta[fslot] = meta_value;  // (LRU: k_lru_meta)
                    if (foc == kFound) ++my_found; else ++my_coll;
                } else if (MODE == kModeLru && st[u] != kIdle && j == 0) {
                    out_oc[i] = kPendingOc;
                }
            }
            is_new = is_new && j == 0;
            const unsigned mask = __ballot_sync(0xffffffffu, is_new);
            if (mask) {
                unsigned basek = 0;
                if (lane == 0) basek = atomicAdd(&ctr->new_count, (unsigned)__popc(mask));
                basek = __shfl_sync(0xffffffffu, basek, 0);
                if (is_new) {
                    const unsigned k = basek + __popc(mask & ((1u << lane) - 1));
                    newpos[k] = (uint32_t)i;
                    newid[k] = id[u];
                    newa[k] = a_off;
                    newm[k] = m_off;
                }
            }
        }
    }
    if (j != 0) my_isec = my_msec = 0;  // every lane of a quad counted the same sectors
    for (int o = 16; o; o >>= 1) {
        my_found += __shfl_xor_sync(0xffffffffu, my_found, o);
        my_coll += __shfl_xor_sync(0xffffffffu, my_coll, o);
        my_isec += __shfl_xor_sync(0xffffffffu, my_isec, o);
        my_msec += __shfl_xor_sync(0xffffffffu, my_msec, o);
    }
    if (lane == 0) {
        if (my_found) atomicAdd(&ctr->found, my_found);
        if (my_coll) atomicAdd(&ctr->collision, my_coll);
        if (my_isec) atomicAdd(&ctr->id_sectors, my_isec);
        if (my_msec) atomicAdd(&ctr->meta_sectors, my_msec);
    }
}

// K1 (long windows, Disabled): the quad line walk with a one-line lookahead.  At 0.95 load a
// miss walks ~6 lines of its 256-slot window one dependent 128-byte load after another; here
// every round loads the current line AND the next line of the window (independent loads, so a
// long walk takes half the round trips).  Decisions and the sector count are those of
// k_probe_line: the second line is consulted only when the first holds neither the id nor an
// EMPTY, so the extra load of a walk that stops in its first line is pure prefetch.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_probe_line_la(TableDev t, const uint64_t* __restrict__ ids,
                                                             uint64_t n, uint64_t now, uint64_t meta_value,
                                                             BatchCounters* ctr,
                                                             uint64_t* __restrict__ out_slots,
                                                             uint8_t* __restrict__ out_oc,
                                                             uint32_t* __restrict__ newpos,
                                                             uint64_t* __restrict__ newid,
                                                             uint32_t* __restrict__ newa,
                                                             uint32_t* __restrict__ newm,
                                                             const uint32_t* __restrict__ dlist = nullptr) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    constexpr uint8_t kPending = 0, kHit = 1, kEmptyHit = 2, kExhausted = 3, kIdle = 4;
    const unsigned lane = lane_id();
    const unsigned j = quad_lane(), qm = quad_mask();
    const uint64_t qpb = blockDim.x >> 2;
    const uint64_t qib = threadIdx.x >> 2;
    unsigned long long my_found = 0, my_coll = 0, my_isec = 0;
    const uint64_t total = min(n, (uint64_t)ctr->n_live);
    // (t0 is block-uniform, so every warp runs every iteration: the ballot below is full-warp)
    for (uint64_t t0 = (uint64_t)blockIdx.x * qpb; t0 < total; t0 += (uint64_t)gridDim.x * qpb) {
        const uint64_t i = t0 + qib;
        uint8_t st = kIdle;
        uint64_t id = 0, g = 0, base = 0, end = 0, h = 0;
        uint32_t off = 0;
        if (i < total) {
            id = ids[i];
            const ShardDev sd = t.shards[shard_of(id, t)];
            base = sd.offset;
            end = base + sd.cap.d;
            h = home_of(id, sd, t.seed);
            g = base + h;
            st = kPending;
        }
        while (st == kPending) {
            const LineSpan sp = line_span(g, end, off, t.P);
            uint64_t g2 = g + sp.c;
            if (g2 == end) g2 = base;
            const uint32_t off2 = off + sp.c;
            uint64_t w[4], w2[4];
            ld_line_part(t.ident, g, j, w);
            const bool second = off2 < t.P;
            if (second) ld_line_part(t.ident, g2, j, w2);
            unsigned m = 0, e = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                m |= (unsigned)(w[k] == id) << k;
                e |= (unsigned)(w[k] == kEmpty) << k;
            }
            unsigned x = quad_gather(m, e, j, qm);
            unsigned hit = (x | (x >> 16)) & sp.range();
            if (hit) {
                const unsigned q = __ffs(hit) - 1;
                st = (x >> q) & 1u ? kHit : kEmptyHit;
                off += q - sp.s;
                g += q - sp.s;
                my_isec += sp.sectors_to(q);
                break;
            }
            my_isec += sp.sectors_to(sp.s + sp.c - 1);
            if (!second) {
                st = kExhausted;
                break;
            }
            const LineSpan sp2 = line_span(g2, end, off2, t.P);
            m = e = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                m |= (unsigned)(w2[k] == id) << k;
                e |= (unsigned)(w2[k] == kEmpty) << k;
            }
            x = quad_gather(m, e, j, qm);
            hit = (x | (x >> 16)) & sp2.range();
            if (hit) {
                const unsigned q = __ffs(hit) - 1;
                st = (x >> q) & 1u ? kHit : kEmptyHit;
                off = off2 + q - sp2.s;
                g = g2 + q - sp2.s;
                my_isec += sp2.sectors_to(q);
                break;
            }
            my_isec += sp2.sectors_to(sp2.s + sp2.c - 1);
            off = off2 + sp2.c;
            g = g2 + sp2.c;
            if (g == end) g = base;
            if (off >= t.P) st = kExhausted;
        }
        bool is_new = false;
        uint32_t a_off = 0;
        if (st != kIdle && j == 0) {
            uint64_t fslot = kEmpty;
            uint8_t foc = kFound;
            if (st == kHit) fslot = g;
            else if (st == kEmptyHit) {
                is_new = true;
                a_off = off;
                out_slots[i] = g;  // the likely result (as k_probe)
                out_oc[i] = kInserted;
            }
            else { fslot = base + h; foc = kCollision; }
            if (fslot != kEmpty) {
                out_slots[i] = fslot;
                out_oc[i] = foc;
                t.meta[fslot] = meta_value;
                if (foc == kFound) ++my_found; else ++my_coll;
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, is_new);
        if (mask) {
            unsigned basek = 0;
            if (lane == 0) basek = atomicAdd(&ctr->new_count, (unsigned)__popc(mask));
            basek = __shfl_sync(0xffffffffu, basek, 0);
            if (is_new) {
                const unsigned k = basek + __popc(mask & ((1u << lane) - 1));
                newpos[k] = (uint32_t)i;
                newid[k] = id;
                newa[k] = a_off;
                newm[k] = kNone32;
            }
        }
    }
    if (j != 0) my_isec = 0;  // every lane of a quad counted the same sectors
    for (int o = 16; o; o >>= 1) {
        my_found += __shfl_xor_sync(0xffffffffu, my_found, o);
        my_coll += __shfl_xor_sync(0xffffffffu, my_coll, o);
        my_isec += __shfl_xor_sync(0xffffffffu, my_isec, o);
    }
    if (lane == 0) {
        if (my_found) atomicAdd(&ctr->found, my_found);
        if (my_coll) atomicAdd(&ctr->collision, my_coll);
        if (my_isec) atomicAdd(&ctr->id_sectors, my_isec);
    }
}

// K1 (long windows, Disabled, tables that keep identity tags): the first identity line of the
// window as in k_probe_line_la -- most hits end there -- then the rest of the window 128 slots
// per round from the TAG lines (common.cuh: one byte per slot, 0 = EMPTY): lane j of the quad
// loads tag bytes [32j, 32j + 32) of the line, and the quad finds the first EMPTY of the window
// part and the slots before it whose tag equals the id's.  Only those candidates are read from
// the identity array (1/255 of the occupied slots), in order, until one holds the id.  At 0.95
// load an absent id's walk to its first EMPTY (~200 slots) costs one identity line and two tag
// lines instead of ~13 identity lines.  Decisions are k_probe_line_la's: the walk stops at the
// same slot (the first holding the id, or the first EMPTY, in window order).
// C3 insert-heavy (ncu): DRAM sectors read 88.6 M -> 38.2 M per batch, probe 0.90 -> 0.73 ms; what
// remains is issue-bound (62% issue-active, half of it the tag byte masks).  Swept: loading 1 or
// 2 tag lines with the identity line (0.76 / 0.71 ms, 48 / 64 registers), 6 or 8 blocks/SM (0.72 /
// 0.80 ms): none clearly better than this plain variant at 5 blocks/SM.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_probe_tag(TableDev t, const uint64_t* __restrict__ ids,
                                                         uint64_t n, uint64_t now, uint64_t meta_value,
                                                         BatchCounters* ctr,
                                                         uint64_t* __restrict__ out_slots,
                                                         uint8_t* __restrict__ out_oc,
                                                         uint32_t* __restrict__ newpos,
                                                         uint64_t* __restrict__ newid,
                                                         uint32_t* __restrict__ newa,
                                                         uint32_t* __restrict__ newm,
                                                         const uint32_t* __restrict__ dlist = nullptr) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    constexpr uint8_t kPending = 0, kHit = 1, kEmptyHit = 2, kExhausted = 3, kIdle = 4;
    const unsigned lane = lane_id();
    const unsigned j = quad_lane(), qm = quad_mask();
    const int jb = 32 * (int)j;  // this lane's first slot of a tag line
    const uint64_t qpb = blockDim.x >> 2;
    const uint64_t qib = threadIdx.x >> 2;
    unsigned long long my_found = 0, my_coll = 0, my_isec = 0, my_tsec = 0;
    const uint64_t total = min(n, (uint64_t)ctr->n_live);
    for (uint64_t t0 = (uint64_t)blockIdx.x * qpb; t0 < total; t0 += (uint64_t)gridDim.x * qpb) {
        const uint64_t i = t0 + qib;
        uint8_t st = kIdle;
        uint64_t id = 0, g = 0, base = 0, end = 0, h = 0;
        uint32_t off = 0;
        if (i < total) {
            id = ids[i];
            const ShardDev sd = t.shards[shard_of(id, t)];
            base = sd.offset;
            end = base + sd.cap.d;
            h = home_of(id, sd, t.seed);
            g = base + h;
            st = kPending;
        }
        const uint32_t pat = (uint32_t)tag_of(id) * 0x01010101u;
        if (st == kPending) {  // round 0: the home slot's identity line
            const LineSpan sp = line_span(g, end, off, t.P);
            uint64_t w[4];
            ld_line_part(t.ident, g, j, w);
            unsigned m = 0, e = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                m |= (unsigned)(w[k] == id) << k;
                e |= (unsigned)(w[k] == kEmpty) << k;
            }
            const unsigned x = quad_gather(m, e, j, qm);
            const unsigned hit = (x | (x >> 16)) & sp.range();
            if (hit) {
                const unsigned q = __ffs(hit) - 1;
                st = (x >> q) & 1u ? kHit : kEmptyHit;
                off += q - sp.s;
                g += q - sp.s;
                my_isec += sp.sectors_to(q);
            } else {
                my_isec += sp.sectors_to(sp.s + sp.c - 1);
                off += sp.c;
                g += sp.c;
                if (g == end) g = base;
                if (off >= t.P) st = kExhausted;
            }
        }
        // the rest of the window on the tag lines, 128 slots per round
        while (st == kPending) {
            const uint64_t tl = g & ~127ull;
            const int s0 = (int)(g & 127u);
            const int c0 = (int)tag_seg_len(g, end, off, t.P);
            uint64_t v[4];
            ld_tag_part(t, tl, j, v);
            ++my_tsec;
            unsigned fe;
            const unsigned q = tag_segment(t, v, pat, id, tl, s0, c0, jb, j, qm, fe, my_isec);
            if (q != 128u) {
                st = kHit;
                off += q - (unsigned)s0;
                g = tl + q;
            } else if (fe != 128u) {
                st = kEmptyHit;
                off += fe - (unsigned)s0;
                g = tl + fe;
            } else {
                off += (uint32_t)c0;
                g += (uint64_t)c0;
                if (g == end) g = base;
                if (off >= t.P) st = kExhausted;
            }
        }
        bool is_new = false;
        uint32_t a_off = 0;
        if (st != kIdle && j == 0) {
            uint64_t fslot = kEmpty;
            uint8_t foc = kFound;
            if (st == kHit) fslot = g;
            else if (st == kEmptyHit) {
                is_new = true;
                a_off = off;
                out_slots[i] = g;  // the likely result (as k_probe)
                out_oc[i] = kInserted;
            }
            else { fslot = base + h; foc = kCollision; }
            if (fslot != kEmpty) {
                out_slots[i] = fslot;
                out_oc[i] = foc;
                t.meta[fslot] = meta_value;
                if (foc == kFound) ++my_found; else ++my_coll;
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, is_new);
        if (mask) {
            unsigned basek = 0;
            if (lane == 0) basek = atomicAdd(&ctr->new_count, (unsigned)__popc(mask));
            basek = __shfl_sync(0xffffffffu, basek, 0);
            if (is_new) {
                const unsigned k = basek + __popc(mask & ((1u << lane) - 1));
                newpos[k] = (uint32_t)i;
                newid[k] = id;
                newa[k] = a_off;
                newm[k] = kNone32;
            }
        }
    }
    // every lane of a quad counted the same identity sectors; each read its own tag sector
    if (j != 0) my_isec = 0;
    for (int o = 16; o; o >>= 1) {
        my_found += __shfl_xor_sync(0xffffffffu, my_found, o);
        my_coll += __shfl_xor_sync(0xffffffffu, my_coll, o);
        my_isec += __shfl_xor_sync(0xffffffffu, my_isec, o);
        my_tsec += __shfl_xor_sync(0xffffffffu, my_tsec, o);
    }
    if (lane == 0) {
        if (my_found) atomicAdd(&ctr->found, my_found);
        if (my_coll) atomicAdd(&ctr->collision, my_coll);
        if (my_isec) atomicAdd(&ctr->id_sectors, my_isec);
        if (my_tsec) atomicAdd(&ctr->meta_sectors, my_tsec);  // (Disabled reads no metadata)
    }
}

// K2: distinct ids over the new positions: a 128-bit CAS inserts (id, epoch, e = this item's
// new-list index) into the hash index; the inserter initialises te[e]; every item (inserter or
// repeat) takes the id's first position into te[e].rank (atomicMax of epoch << 32 | ~position)
// and records its entry.
__global__ void __launch_bounds__(256) k_dedup(BatchCounters* ctr, uint64_t tcap, uint64_t epoch,
                                               const uint32_t* __restrict__ newpos,
                                               const uint64_t* __restrict__ newid,
                                               const uint32_t* __restrict__ newa,
                                               const uint32_t* __restrict__ newm,
                                               uint32_t* __restrict__ newent, u128* hk, IdEntry* te,
                                               uint32_t* __restrict__ dupl) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    const unsigned cnt = ctr->new_count;
    const uint64_t mask = table_mask(cnt, tcap);
    const uint32_t ep32 = (uint32_t)epoch;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
        const uint64_t id = newid[k];
        const u128 mine = make_key(ep32, k, id);
        const unsigned long long myrank = (epoch << 32) | (uint32_t)~newpos[k];
        uint64_t h = te_home(id, mask);
        uint32_t e;
        bool inserted = false;
        for (;;) {
            // a plain 16-byte L2 load first (one round trip less than an atomic read on the
            // common path, a stale key of an older epoch).  It is not single-copy atomic: a
            // torn value can only fail the CAS below, or -- if it shows the current epoch --
            // is re-read atomically before it is trusted.
            u128 cur = ld_cg_u128(&hk[h]);
            if (key_epoch(cur) == ep32) cur = atomicCAS(&hk[h], (u128)0, (u128)0);
            if (key_epoch(cur) != ep32) {  // empty for this batch: try to take it
                const u128 old = atomicCAS(&hk[h], cur, mine);
                if (old == cur) {  // inserted: this item's record is the id's entry
                    e = k;
                    inserted = true;
                    break;
                }
                cur = old;
                if (key_epoch(cur) != ep32) continue;  // raced with a stale value: retry
            }
            if (key_id(cur) == id) {
                e = key_entry(cur);
                break;
            }
            h = (h + 1) & mask;
        }
        if (inserted) {
            // the inserter fills its record (read only by later kernels); the rank word takes
            // every item's rank by atomicMax -- inserter and repeats alike, in any order, no
            // fence: a word left by an older batch holds an older epoch, so it is smaller
            te[k].id = id;
            uint64_t* w = reinterpret_cast<uint64_t*>(&te[k].a);
            const uint32_t na = newa[k];
            w[0] = (uint64_t)(na & ~kAEmpty) | ((uint64_t)newm[k] << 32);
            w[1] = (na & kAEmpty) ? (1ull << 48) : 0ull;  // held = state = oc = 0, aempty
            atomicMax(&te[k].rank, myrank);
        } else if (__ldcg(&te[e].rank) < myrank) {  // (a hot id's later positions skip the atomic)
            atomicMax(&te[e].rank, myrank);
        }
        newent[k] = e;
        if (!inserted) {  // a repeat item (not the inserter): listed for K5, one counter update
                          // per group of converged repeat lanes
            const unsigned am = __activemask();
            const unsigned lane = lane_id(), leader = __ffs(am) - 1;
            unsigned b0 = 0;
            if (lane == leader) b0 = atomicAdd(&ctr->dup_items, (unsigned)__popc(am));
            b0 = __shfl_sync(am, b0, leader);
            dupl[b0 + __popc(am & ((1u << lane) - 1))] = k;
        }
    }
}

// The entry's bookkeeping words in two 16-byte loads: (rank, a | m << 32) and
// (held | state << 32 | oc << 40, slot).
struct EntryView {
    unsigned long long rank;
    uint32_t a, m, held;
    uint8_t state;
    bool aempty;
};
__device__ __forceinline__ EntryView load_entry(const IdEntry* te, uint32_t e) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(&te[e].rank);
    const ulonglong2 w1 = p[0], w2 = p[1];
    EntryView v;
    v.rank = w1.x;
    v.a = (uint32_t)w1.y;
    v.m = (uint32_t)(w1.y >> 32);
    v.held = (uint32_t)w2.x;
    v.state = (uint8_t)(w2.x >> 32);
    v.aempty = ((w2.x >> 48) & 0xFF) != 0;
    return v;
}

// The primary item of an entry (the new-list item at the id's first position) does the
// entry's work in K3/K4; every other item of the same id only reads the result in K5.
__device__ __forceinline__ bool is_primary(const IdEntry* te, uint32_t e, uint32_t pos) {
    return rank_of(te[e].rank) == pos;
}

// K3: rank-priority claims with takeover.
template <int MODE>
__global__ void __launch_bounds__(256) k_claim(TableDev t, uint64_t now, BatchCounters* ctr,
                                               const uint32_t* __restrict__ newpos,
                                               const uint32_t* __restrict__ newent,
                                               IdEntry* te, uint32_t* __restrict__ evl) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    const unsigned cnt = ctr->new_count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
        uint32_t e = newent[k];
        EntryView ev = load_entry(te, e);
        if (rank_of(ev.rank) != newpos[k]) continue;  // not the primary item
        bool fresh = true;
        uint32_t resume = 0;
        for (;;) {
            if (!fresh) ev = load_entry(te, e);  // a taken-over entry
            const uint64_t id = te[e].id;
            const uint32_t rank = rank_of(ev.rank);
            const uint32_t s = shard_of(id, t);
            const ShardDev sd = t.shards[s];
            const uint64_t cap = sd.cap.d, base = sd.offset;
            const uint64_t h = home_of(id, sd, t.seed);
            const uint64_t cv = kClaimBit | ((uint64_t)rank << 31) | (uint64_t)e;
            uint32_t next = kNone32;
            uint64_t gnext = 0;
            bool held = false;
            uint32_t off;
            if (MODE == kModeTtl && fresh && ev.m != kNone32) {
                // owner: try to keep (refresh) the expired slot holding our own id
                const uint32_t m = ev.m;
                const uint64_t gm = base + wrap_add(h, m, cap);
                uint64_t v = ld_cg(t.ident + gm);
                for (;;) {
                    uint64_t nv;
                    if (v == id) nv = cv;
                    else if (is_claim(v) && claim_rank(v) > rank) nv = cv | (v & kFlagEmpty);
                    else break;  // a lower rank evicted our id first
                    const uint64_t old = atomicCAS((unsigned long long*)(t.ident + gm),
                                                   (unsigned long long)v, (unsigned long long)nv);
                    if (old == v) {
                        held = true;
                        if (is_claim(v)) { next = claim_entry(v); gnext = gm; }
                        break;
                    }
                    v = old;
                }
                off = ev.a;
            } else {
                off = fresh ? ev.a : resume;
            }
            if (!held && MODE != kModeTtl && t.tag) {
                // Disabled / LRU on a table that keeps identity tags: the claimable slots (EMPTY or
                // claim words) are exactly the slots EMPTY at the batch start -- tag 0 (no identity
                // changes before K4) -- so the scan reads 32 tags per load instead of 4
                // identities, and tries atomicMin on each tag-0 slot in order (a lower-rank claim
                // word stays: atomicMin leaves a smaller word).  A fresh entry's first available
                // slot was EMPTY when probed: its first attempt reads nothing.
                const uint64_t end = base + cap;
                const uint64_t nv = cv | kFlagEmpty;
                if (fresh && off < t.P) {
                    const uint64_t g = base + wrap_add(h, off, cap);
                    const uint64_t old = atomicMin((unsigned long long*)(t.ident + g), (unsigned long long)nv);
                    if (old >= nv) {
                        atomicMax(&te[e].held, off);
                        held = true;
                        if (old != kEmpty) { next = claim_entry(old); gnext = g; }
                    } else {
                        ++off;
                    }
                }
                while (!held && off < t.P) {
                    const uint64_t g = base + wrap_add(h, off, cap);
                    const uint64_t c32 = g & ~31ull;
                    const uint32_t j0 = (uint32_t)(g - c32);
                    uint32_t lim = 32 - j0;
                    if (t.P - off < lim) lim = t.P - off;
                    if (end - g < lim) lim = (uint32_t)(end - g);
                    uint64_t v[4];
                    ld_sector(reinterpret_cast<const uint64_t*>(t.tag + c32), v[0], v[1], v[2], v[3]);
                    unsigned z = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        z |= msb_bits4(zero_bytes((uint32_t)(v[k >> 1] >> (32 * (k & 1))))) << (4 * k);
                    z &= bit_range((int)j0, (int)(j0 + lim));
                    while (z) {
                        const unsigned k = __ffs(z) - 1;
                        z &= z - 1;
                        const uint64_t gk = c32 + k;
                        const uint64_t old = atomicMin((unsigned long long*)(t.ident + gk), (unsigned long long)nv);
                        if (old < nv) continue;  // a lower rank holds it
                        atomicMax(&te[e].held, off + (k - j0));
                        held = true;
                        if (old != kEmpty) { next = claim_entry(old); gnext = gk; }
                        break;
                    }
                    if (!held) off += lim;
                }
                if (!held) {
                    te[e].state = kStateCollided;
                    if (MODE == kModeLru) {  // (as below)
                        const unsigned am = __activemask();
                        const unsigned leader = __ffs(am) - 1;
                        unsigned b0 = 0;
                        if (lane_id() == leader) b0 = atomicAdd(&ctr->lru_evict, (unsigned)__popc(am));
                        b0 = __shfl_sync(am, b0, leader);
                        evl[b0 + __popc(am & ((1u << lane_id()) - 1))] = e;
                    }
                }
            } else if (!held && MODE != kModeTtl) {
                // Disabled / LRU: only EMPTY slots and claim words of a higher rank are
                // claimable.  Sector by sector: one L2 read, a 4-bit mask of the claimable slots
                // in the window part of the sector, then atomicMin on them in order -- the
                // occupied slots (95% of a window at C3's load) cost no per-slot iteration.
                // A fresh entry's first available slot was EMPTY when probed (claim words only
                // ever land on such slots, all flagged kFlagEmpty): its first attempt is a blind
                // atomicMin, no read before it.
                const uint64_t end = base + cap;
                if (fresh && off < t.P) {
                    const uint64_t g = base + wrap_add(h, off, cap);
                    const uint64_t nv = cv | kFlagEmpty;
                    const uint64_t old = atomicMin((unsigned long long*)(t.ident + g), (unsigned long long)nv);
                    if (old >= nv) {
                        atomicMax(&te[e].held, off);
                        held = true;
                        if (old != kEmpty) { next = claim_entry(old); gnext = g; }
                    } else {
                        ++off;
                    }
                }
                while (!held && off < t.P) {
                    const uint64_t g = base + wrap_add(h, off, cap);
                    const uint64_t a4 = g & ~3ull;
                    const uint32_t j0 = (uint32_t)(g - a4);
                    uint32_t lim = 4 - j0;  // slots of this sector inside the window and the shard
                    if (t.P - off < lim) lim = t.P - off;
                    if (end - g < lim) lim = (uint32_t)(end - g);
                    uint64_t w[4];
                    ld_sector_cg(t.ident + a4, w[0], w[1], w[2], w[3]);
                    unsigned cand = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t v = w[k];
                        cand |= (unsigned)((v >> 63) && (v == kEmpty || claim_rank(v) >= rank)) << k;
                    }
                    cand &= ((1u << lim) - 1u) << j0;
                    while (cand) {
                        const unsigned k = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const uint64_t v = pick4(k, w[0], w[1], w[2], w[3]);
                        const uint64_t gk = a4 + k;
                        const uint64_t nv = cv | (v == kEmpty ? kFlagEmpty : (v & kFlagEmpty));
                        const uint64_t old = atomicMin((unsigned long long*)(t.ident + gk), (unsigned long long)nv);
                        if (old < nv) continue;  // an id, or a lower rank got here first
                        atomicMax(&te[e].held, off + (k - j0));
                        held = true;
                        if (old != kEmpty) { next = claim_entry(old); gnext = gk; }
                        break;
                    }
                    if (held) break;
                    off += lim;
                }
                if (!held) {
                    te[e].state = kStateCollided;
                    // LRU: a full window evicts its least recently used slot: K3b picks it
                    // (a collided entry holds nothing, so it is never taken over again)
                    if (MODE == kModeLru) {  // one counter update per warp (Zipf: ~166 K evictors)
                        const unsigned am = __activemask();
                        const unsigned leader = __ffs(am) - 1;
                        unsigned b0 = 0;
                        if (lane_id() == leader) b0 = atomicAdd(&ctr->lru_evict, (unsigned)__popc(am));
                        b0 = __shfl_sync(am, b0, leader);
                        evl[b0 + __popc(am & ((1u << lane_id()) - 1))] = e;
                    }
                }
            } else if (!held) {
                // TTL, a fresh taker whose first available slot was EMPTY when probed: a blind
                // atomicMin first (EMPTY slots only ever become claim words, all flagged EMPTY)
                if (MODE == kModeTtl && fresh && ev.aempty && off < t.P) {
                    const uint64_t g = base + wrap_add(h, off, cap);
                    const uint64_t nv = cv | kFlagEmpty;
                    const uint64_t old = atomicMin((unsigned long long*)(t.ident + g), (unsigned long long)nv);
                    if (old >= nv) {
                        atomicMax(&te[e].held, off);
                        held = true;
                        if (old != kEmpty) { next = claim_entry(old); gnext = g; }
                    } else {
                        ++off;
                    }
                }
            }
            if (!held && MODE == kModeTtl) {
                // TTL: the same sector mask with the metadata sector in the same round --
                // claimable: EMPTY or a higher-rank claim word (atomicMin, as above), or an
                // expired id (CAS, re-evaluated on failure) -- so the scan takes no dependent
                // metadata load per occupied slot
                const uint64_t end = base + cap;
                while (off < t.P) {
                    const uint64_t g = base + wrap_add(h, off, cap);
                    const uint64_t a4 = g & ~3ull;
                    const uint32_t j0 = (uint32_t)(g - a4);
                    uint32_t lim = 4 - j0;
                    if (t.P - off < lim) lim = t.P - off;
                    if (end - g < lim) lim = (uint32_t)(end - g);
                    uint64_t w[4], mt[4];
                    ld_sector_cg(t.ident + a4, w[0], w[1], w[2], w[3]);
                    ld_sector_cg(t.meta + a4, mt[0], mt[1], mt[2], mt[3]);
                    unsigned cand = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t v = w[k];
                        const bool c = (v >> 63) ? (v == kEmpty || claim_rank(v) >= rank) : (mt[k] < now);
                        cand |= (unsigned)c << k;
                    }
                    cand &= ((1u << lim) - 1u) << j0;
                    while (cand) {
                        const unsigned k = __ffs(cand) - 1;
                        cand &= cand - 1;
                        uint64_t v = pick4(k, w[0], w[1], w[2], w[3]);
                        const uint64_t gk = a4 + k;
                        const uint32_t offk = off + (k - j0);
                        if (v >> 63) {
                            const uint64_t nv = cv | (v == kEmpty ? kFlagEmpty : (v & kFlagEmpty));
                            const uint64_t old = atomicMin((unsigned long long*)(t.ident + gk), (unsigned long long)nv);
                            if (old < nv) continue;  // an id, or a lower rank got here first
                            atomicMax(&te[e].held, offk);
                            held = true;
                            if (old != kEmpty) { next = claim_entry(old); gnext = gk; }
                            break;
                        }
                        for (;;) {  // an expired foreign id
                            uint64_t nv;
                            if (v == kEmpty) {
                                nv = cv | kFlagEmpty;
                            } else if (v >> 63) {
                                if (claim_rank(v) < rank) break;  // a lower rank holds it for good
                                nv = cv | (v & kFlagEmpty);
                            } else {
                                if (!(ld_cg(t.meta + gk) < now)) break;  // live
                                nv = cv;
                            }
                            const uint64_t old = atomicCAS((unsigned long long*)(t.ident + gk),
                                                           (unsigned long long)v, (unsigned long long)nv);
                            if (old == v) {
                                // taker claims of one entry move strictly forward, so the max is the
                                // slot it holds last (a late max from a displaced claim is harmless)
                                atomicMax(&te[e].held, offk);
                                held = true;
                                if (is_claim(v)) { next = claim_entry(v); gnext = gk; }
                                break;
                            }
                            v = old;
                        }
                        if (held) break;
                    }
                    if (held) break;
                    off += lim;
                }
                if (!held) {
                    te[e].state = kStateCollided;
                    // LRU: a full window evicts its least recently used slot: K3b picks it
                    // (a collided entry holds nothing, so it is never taken over again)
                    if (MODE == kModeLru) {  // one counter update per warp (Zipf: ~166 K evictors)
                        const unsigned am = __activemask();
                        const unsigned leader = __ffs(am) - 1;
                        unsigned b0 = 0;
                        if (lane_id() == leader) b0 = atomicAdd(&ctr->lru_evict, (unsigned)__popc(am));
                        b0 = __shfl_sync(am, b0, leader);
                        evl[b0 + __popc(am & ((1u << lane_id()) - 1))] = e;
                    }
                }
            }
            if (next == kNone32) break;
            // take over the displaced entry: it resumes right after the slot it lost,
            // or -- if it was an owner losing its own id's slot -- as a taker from its
            // first available offset.
            {
                const uint64_t id2 = te[next].id;
                const uint64_t h2 = home_of(id2, sd, t.seed);  // same shard as the slot
                const uint64_t loc = gnext - base;
                const uint32_t off2 = (uint32_t)(loc >= h2 ? loc - h2 : loc + cap - h2);
                if (MODE == kModeTtl && te[next].m != kNone32 && off2 == te[next].m)
                    resume = te[next].a;
                else
                    resume = off2 + 1;
                e = next;
                fresh = false;
            }
        }
    }
}

// K4: commit claims: claim word -> id, outcome, the entry's metadata word (one value per
// batch, so duplicates / (id, f') secondaries of the entry need no write of their own),
// touch_row, reset list and rank-indexed evicted flags.
template <int MODE, bool PF = false>
__global__ void __launch_bounds__(256) k_commit(TableDev t, BatchCounters* ctr,
                                                const uint32_t* __restrict__ newpos,
                                                const uint64_t* __restrict__ newid,
                                                const uint32_t* __restrict__ newent,
                                                IdEntry* te, uint64_t gen_clock,
                                                uint64_t meta_value,
                                                uint64_t* __restrict__ reset_rows,
                                                uint8_t* __restrict__ evflag,
                                                uint64_t* __restrict__ evslot,
                                                uint64_t* __restrict__ out_slots,
                                                uint8_t* __restrict__ out_oc) {
    pdl_wait();
    if (batch_failed(&ctr->err) || (MODE == kModeLru && ctr->lru_abort)) return;
    const unsigned cnt = ctr->new_count;
    const bool dups = ctr->dup_items != 0;
    unsigned long long c[4] = {0, 0, 0, 0};
    unsigned np = 0;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
        const uint32_t e = newent[k];
        const uint32_t rank = newpos[k];
        const EntryView ev = load_entry(te, e);
        if (rank_of(ev.rank) != rank) continue;  // not the primary item
        const uint64_t id = newid[k];
        const uint32_t s = shard_of(id, t);
        const ShardDev sd = t.shards[s];
        const uint64_t cap = sd.cap.d, base = sd.offset;
        const uint64_t h = home_of(id, sd, t.seed);
        const uint64_t mine = kClaimBit | ((uint64_t)rank << 31) | (uint64_t)e;
        uint8_t oc = kCollision;
        uint64_t g = base + h;
        uint64_t v = 0;
        bool ok = true;
        if (MODE == kModeTtl && ev.m != kNone32 &&
            ((v = t.ident[base + wrap_add(h, ev.m, cap)]) & ~kFlagEmpty) == mine) {
            g = base + wrap_add(h, ev.m, cap);  // the owner kept (refreshed) its own slot
            oc = kFound;
        } else if (MODE == kModeLru && ev.state == kStateEvict) {
            g = base + wrap_add(h, ev.held, cap);  // K3b's victim (still its pre-batch id)
            oc = kEvicted;
        } else if (ev.state != kStateCollided) {
            g = base + wrap_add(h, ev.held, cap);
            v = t.ident[g];
            ok = (v & ~kFlagEmpty) == mine;
            oc = (v & kFlagEmpty) ? kInserted : kEvicted;
        }
        if (!ok) {
            atomicExch(&ctr->err.too_many, 2u);  // internal invariant violated
            continue;
        }
        if (oc != kCollision) {
            t.ident[g] = id;
            store_tag(t, g, id);
        }
        if (!PF) t.meta[g] = meta_value;  // per-feature TTL: the last-writer pass
        if (oc == kInserted || oc == kEvicted) t.row_gen[g] = gen_clock;
        {   // reset list: one warp-aggregated append (a per-row atomic on one counter word
            // serialises at the L2 -- C4 evicts ~0.8 M rows per 1 M-position batch); the
            // evicted-list length is the rank-ordered compaction's count (TTL; no evictions
            // otherwise on this path)
            const unsigned am = __activemask();
            const unsigned em = __ballot_sync(am, oc == kEvicted);
            if (oc == kEvicted) {
                const unsigned leader = __ffs(em) - 1;
                unsigned r0 = 0;
                if (lane_id() == leader) r0 = atomicAdd(&ctr->reset_count, (unsigned)__popc(em));
                r0 = __shfl_sync(em, r0, leader);
                reset_rows[r0 + __popc(em & ((1u << lane_id()) - 1))] = g;
                evflag[rank] = 1;  // (the compaction reads the slot from out_slots[rank])
            }
        }
        if (dups) {  // K5 reads the entry's result for the later positions of its id
            te[e].slot = g;
            te[e].oc = oc;
        }
        // the primary item's own position (its feature is the entry's): result written
        // here, so K5 only has items of repeated ids left.  Disabled, and TTL takers whose first
        // available slot was EMPTY: the probe already wrote Inserted at that slot -- rewritten
        // only where the claims moved it (a random write pair per new id saved)
        if (!((MODE == kModeDisabled || (MODE == kModeTtl && ev.aempty)) && oc == kInserted && ev.held == ev.a)) {
            out_slots[rank] = g;
            out_oc[rank] = oc;
        }
        ++c[oc];
        ++np;
    }
    for (int j = 0; j < 4; ++j)
        for (int o = 16; o; o >>= 1) c[j] += __shfl_xor_sync(0xffffffffu, c[j], o);
    for (int o = 16; o; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
    if (lane_id() == 0) {
        if (c[0]) atomicAdd(&ctr->found, c[0]);
        if (c[1]) atomicAdd(&ctr->inserted, c[1]);
        if (c[2]) atomicAdd(&ctr->evicted, c[2]);
        if (c[3]) atomicAdd(&ctr->collision, c[3]);
        if (np) atomicAdd(&ctr->entry_count, np);
    }
}

// ---- per-feature TTL on the fast path.  With differing per-feature TTLs the uniques of one
// batch write different metadata values, so a slot's final word is the value of the LAST
// unique writing it in the reference's order (batch_engine.cpp:160-221: uniques in first-
// occurrence order), i.e. of the (id, feature) unique with the largest first position among
// those whose result slot it is.  Every decision is the same as with one value per batch (each
// value is now + ttl > now: expiry does not change inside the batch), so K1..K5 run unchanged
// with their metadata writes held back, then:
//   M1 k_pf_group  every position -> its (id, feature) group, first position by atomicMax of
//                  epoch << 32 | ~position (the dedup trick);
//   M2 k_pf_slot   every group's first position -> its result slot's record, the largest first
//                  position by atomicMax of epoch << 32 | position;
//   M3 k_pf_write  the winning group writes now + ttl(feature) (eviction.cpp:20-30).
struct __align__(32) PfEntry {
    u128 key;                 // (id | feature << 64 | epoch << 96) or (slot | epoch << 96)
    unsigned long long rank;  // epoch << 32 | ~first position (groups) / | position (slots)
    unsigned long long pad;
};

__device__ __forceinline__ uint64_t pf_ttl(uint32_t f, uint64_t def, const uint32_t* keys,
                                           const uint64_t* vals, uint32_t nk) {
    for (uint32_t i = 0; i < nk; ++i)
        if (keys[i] == f) return vals[i];
    return def;
}

// insert-or-find an epoch-tagged 128-bit key (epoch in the top 32 bits); returns the record
__device__ __forceinline__ uint32_t pf_find(PfEntry* tab, uint64_t mask, u128 mine, uint64_t h) {
    const uint32_t ep = (uint32_t)(mine >> 96);
    for (;;) {
        // a plain L2 load first: under skewed traffic thousands of positions look up one hot
        // record, and atomic reads of one address serialise.  A torn read equal to `mine` can only
        // come from a record that holds `mine` (the halves of any other value differ from it)
        u128 cur = ld_cg_u128(&tab[h].key);
        if (cur == mine) return (uint32_t)h;
        cur = atomicCAS(&tab[h].key, (u128)0, (u128)0);
        if ((uint32_t)(cur >> 96) != ep) {
            const u128 old = atomicCAS(&tab[h].key, cur, mine);
            if (old == cur) return (uint32_t)h;
            cur = old;
            if ((uint32_t)(cur >> 96) != ep) continue;
        }
        if (cur == mine) return (uint32_t)h;
        h = (h + 1) & mask;
    }
}

__global__ void __launch_bounds__(256) k_pf_group(const BatchCounters* ctr, const uint64_t* __restrict__ ids,
                                                  const uint32_t* __restrict__ feats, uint64_t n, uint32_t ep,
                                                  PfEntry* tab, uint64_t mask, uint32_t* __restrict__ ent) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    n = min(n, (uint64_t)ctr->n_live);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t id = ids[i];
        const uint32_t f = feats[i];
        const u128 mine = (u128)id | ((u128)f << 64) | ((u128)ep << 96);
        const uint32_t e = pf_find(tab, mask, mine, mix64(id ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull), 0x51ED27ull) & mask);
        const unsigned long long r = ((unsigned long long)ep << 32) | (uint32_t)~(uint32_t)i;
        if (__ldcg(&tab[e].rank) < r) atomicMax(&tab[e].rank, r);  // (skip the hot records' no-op atomics)
        ent[i] = e;
    }
}

__global__ void __launch_bounds__(256) k_pf_slot(const BatchCounters* ctr, uint64_t n, uint32_t ep,
                                                 const PfEntry* gtab, const uint32_t* __restrict__ gent,
                                                 const uint64_t* __restrict__ out_slots, PfEntry* stab,
                                                 uint64_t mask, uint32_t* __restrict__ sent) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    n = min(n, (uint64_t)ctr->n_live);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (~(uint32_t)__ldcg(&gtab[gent[i]].rank) != (uint32_t)i) continue;  // not its group's first
        const uint64_t g = out_slots[i];
        const u128 mine = (u128)g | ((u128)ep << 96);
        const uint32_t e = pf_find(stab, mask, mine, mix64(g, 0x5107ull) & mask);
        atomicMax(&stab[e].rank, ((unsigned long long)ep << 32) | (uint32_t)i);
        sent[i] = e;
    }
}

__global__ void __launch_bounds__(256) k_pf_write(TableDev t, const BatchCounters* ctr,
                                                  const uint32_t* __restrict__ feats, uint64_t n,
                                                  const PfEntry* gtab, const uint32_t* __restrict__ gent,
                                                  const PfEntry* stab, const uint32_t* __restrict__ sent,
                                                  const uint64_t* __restrict__ out_slots, uint64_t now,
                                                  uint64_t def_ttl, const uint32_t* keys, const uint64_t* vals,
                                                  uint32_t nk) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    n = min(n, (uint64_t)ctr->n_live);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (~(uint32_t)__ldcg(&gtab[gent[i]].rank) != (uint32_t)i) continue;
        if ((uint32_t)__ldcg(&stab[sent[i]].rank) != (uint32_t)i) continue;  // a later group wrote last
        t.meta[out_slots[i]] = now + pf_ttl(feats[i], def_ttl, keys, vals, nk);
    }
}

// ---- LRU evictions on the claim path.  A new id whose window is full evicts the window's least
// recently used slot: the first slot of smallest metadata (strict <, probe_core.cpp:97-101 and
// 125-129) in the table as the sequential reference has it at that id's turn.  At that turn
// every slot touched earlier in the batch (Found refresh, insert, eviction) holds metadata
// `now`; every other slot its pre-batch value.  K3a maps every Found slot to its first Found
// position; K3b decides every evictor in parallel on K3's end state, counting claimed slots and
// slots Found before the evictor's position as `now`.  Its pick v is the reference's whenever
//   * v holds a pre-batch id whose metadata is older than `now` -- then no slot touched before
//     the evictor's turn (metadata `now`) can beat or tie it, and a slot touched only after it
//     still had its pre-batch value, which K3b compared;
//   * no other evictor picked v -- an earlier eviction elsewhere in the window only raises
//     that slot to `now` (the first point again);
//   * no position Found v's id (after the evictor's turn, since one before would have made v
//     `now`) -- else that position would miss the evicted id: a cascade.
// Any other case sets lru_abort: the claims revert and the batch takes the rounds path.
__device__ __forceinline__ uint32_t found_first(const PfEntry* tab, uint64_t mask, uint64_t g, uint32_t ep) {
    for (uint64_t h = mix64(g, 0xF0D5ull) & mask;; h = (h + 1) & mask) {
        const u128 key = ld_cg_u128(&tab[h].key);
        if ((uint32_t)(key >> 96) != ep) return kNone32;  // no position Found this slot
        if ((uint64_t)key == g) return ~(uint32_t)__ldcg(&tab[h].rank);
    }
}

// K3a (LRU, evictors only): Found slot -> its first Found position
__global__ void __launch_bounds__(256) k_lru_found(BatchCounters* ctr, uint64_t n,
                                                   const uint64_t* __restrict__ out_slots,
                                                   const uint8_t* __restrict__ out_oc,
                                                   PfEntry* ftab, uint64_t mask, uint32_t ep) {
    pdl_wait();
    if (batch_failed(&ctr->err) || ctr->lru_evict == 0) return;
    n = min(n, (uint64_t)ctr->n_live);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (out_oc[i] != kFound) continue;
        const uint64_t g = out_slots[i];
        const uint32_t r = pf_find(ftab, mask, (u128)g | ((u128)ep << 96), mix64(g, 0xF0D5ull) & mask);
        const unsigned long long v = ((unsigned long long)ep << 32) | (uint32_t)~(uint32_t)i;
        if (__ldcg(&ftab[r].rank) < v) atomicMax(&ftab[r].rank, v);  // (hot slots: skip no-op atomics)
    }
}

// K3b
__global__ void __launch_bounds__(256) k_lru_victim(TableDev t, uint64_t now, BatchCounters* ctr,
                                                    const uint32_t* __restrict__ evl, IdEntry* te,
                                                    PfEntry* vtab, uint64_t cap_alloc, const PfEntry* ftab,
                                                    uint64_t fmask, uint32_t ep) {
    pdl_wait();
    if (batch_failed(&ctr->err)) return;
    const unsigned cnt = ctr->lru_evict;
    if (cnt == 0) return;
    const uint64_t mask = table_mask(cnt, cap_alloc);
    const unsigned lane = lane_id();
    const unsigned warps = gridDim.x * (blockDim.x >> 5);
    for (unsigned k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < cnt; k += warps) {
        const uint32_t e = evl[k];
        const uint64_t id = te[e].id;
        const uint32_t rank = rank_of(te[e].rank);
        const ShardDev sd = t.shards[shard_of(id, t)];
        const uint64_t cap = sd.cap.d, base = sd.offset, h = home_of(id, sd, t.seed);
        // lane j scans offsets j, j + 32, ...: first smallest per lane, then across the warp
        uint64_t best = ~0ull;
        uint32_t boff = kNone32;
        for (uint32_t off = lane; off < t.P; off += 32) {
            const uint64_t g = base + wrap_add(h, off, cap);
            const uint64_t v = t.ident[g];
            uint64_t m = now;  // claimed in this batch
            if (!(v >> 63)) {
                m = t.meta[g];
                if (m < now && found_first(ftab, fmask, g, ep) < rank) m = now;  // refreshed before
            }
            if (m < best) { best = m; boff = off; }
        }
        uint64_t wb = best;
        for (int o = 16; o; o >>= 1) {
            const uint64_t x = __shfl_xor_sync(0xffffffffu, wb, o);
            wb = x < wb ? x : wb;
        }
        uint32_t wo = best == wb ? boff : kNone32;
        for (int o = 16; o; o >>= 1) wo = min(wo, __shfl_xor_sync(0xffffffffu, wo, o));
        if (lane == 0) {
            bool ok = wb < now && wo != kNone32;  // < now: a pre-batch id, untouched before the turn
            const uint64_t g = base + wrap_add(h, ok ? wo : 0, cap);
            if (ok) ok = found_first(ftab, fmask, g, ep) == kNone32;  // else a later position Found it
            if (ok) {
                const uint32_t r = pf_find(vtab, mask, (u128)g | ((u128)ep << 96), mix64(g, 0x5107ull) & mask);
                const unsigned long long tag = ((unsigned long long)ep << 32) | 1ull;
                ok = atomicExch(&vtab[r].rank, tag) != tag;  // else two evictors picked one slot
            }
            if (ok) {
                te[e].held = wo;
                te[e].state = kStateEvict;
            } else {
                atomicExch(&ctr->lru_abort, 1u);
            }
        }
    }
}

// LRU attempt aborted after K3: put every claimed slot back to EMPTY (only EMPTY slots are
// claimable outside TTL, and every claimed slot ends held by exactly one entry -- the one
// whose last claim offset points at it), so the rounds path starts from the pre-batch state.
__global__ void __launch_bounds__(256) k_lru_revert(TableDev t, BatchCounters* ctr,
                                                    const uint32_t* __restrict__ newpos,
                                                    const uint32_t* __restrict__ newent,
                                                    const IdEntry* te) {
    pdl_wait();
    if (batch_failed(&ctr->err) || !ctr->lru_abort) return;
    const unsigned cnt = ctr->new_count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
        const uint32_t e = newent[k];
        if (!is_primary(te, e, newpos[k]) || te[e].state == kStateCollided) continue;
        const uint64_t id = te[e].id;
        const ShardDev sd = t.shards[shard_of(id, t)];
        const uint64_t g = sd.offset + wrap_add(home_of(id, sd, t.seed), te[e].held, sd.cap.d);
        const uint64_t v = t.ident[g];
        if (is_claim(v) && claim_entry(v) == e) t.ident[g] = kEmpty;
    }
}

// LRU batch that needed no eviction: it is a Disabled batch whose metadata writes were held
// back; every position's final slot gets the batch's metadata value (Found refresh; new ids'
// slots were written in K4 already -- the same word).
__global__ void __launch_bounds__(256) k_lru_meta(TableDev t, const BatchCounters* ctr, uint64_t n,
                                                  const uint64_t* __restrict__ out_slots,
                                                  uint64_t meta_value) {
    pdl_wait();
    if (batch_failed(&ctr->err) || ctr->lru_abort) return;
    n = min(n, (uint64_t)ctr->n_live);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        t.meta[out_slots[i]] = meta_value;
}

// K5: results of the non-primary items -- later positions of a repeated new id: the
// primary's slot and outcome, or, for an (id, f') secondary (same id, other feature, later
// first position), Found on the primary's slot / Collision if the primary collided.  Primary
// items got their result in K4.  Only the repeat items K2 listed are visited: a repeat that is
// not its entry's primary writes its own position; a repeat that IS the primary (an earlier
// position than the inserting item) writes the inserter's position instead, which is then the
// entry's one non-primary item not on the list.
__global__ void __launch_bounds__(256) k_finalize(BatchCounters* ctr,
                                                  const uint32_t* __restrict__ feats,
                                                  const uint32_t* __restrict__ newpos,
                                                  const uint32_t* __restrict__ newent,
                                                  const uint32_t* __restrict__ dupl,
                                                  const IdEntry* te,
                                                  uint64_t* __restrict__ out_slots,
                                                  uint8_t* __restrict__ out_oc) {
    pdl_wait();
    if (batch_failed(&ctr->err) || ctr->dup_items == 0 || ctr->lru_abort) return;
    const unsigned cnt = ctr->dup_items;
    unsigned long long c[4] = {0, 0, 0, 0};
    for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += gridDim.x * blockDim.x) {
        const uint32_t k = dupl[q];
        const uint32_t e = newent[k];
        const uint32_t first = rank_of(te[e].rank);
        uint32_t pos = newpos[k];
        if (first == pos) pos = newpos[e];  // k is the primary: the inserter's position is the later one
        uint8_t oc = te[e].oc;
        if (feats && feats[pos] != feats[first]) oc = oc == kCollision ? kCollision : kFound;
        out_slots[pos] = te[e].slot;
        out_oc[pos] = oc;
        ++c[oc];
    }
    for (int j = 0; j < 4; ++j)
        for (int o = 16; o; o >>= 1) c[j] += __shfl_xor_sync(0xffffffffu, c[j], o);
    if (lane_id() == 0) {
        if (c[0]) atomicAdd(&ctr->found, c[0]);
        if (c[1]) atomicAdd(&ctr->inserted, c[1]);
        if (c[2]) atomicAdd(&ctr->evicted, c[2]);
        if (c[3]) atomicAdd(&ctr->collision, c[3]);
    }
}

}  // namespace

void preload_remap_kernels() {
#define PL(k) preload_kernel((const void*)(k))
    PL(k_init_counters); PL(k_sh_adopt); PL(k_validate);
    PL((k_probe_line<kModeTtl, 2, 3, true>)); PL((k_probe_line<kModeTtl, 2, 3>));
    PL((k_probe_line<kModeLru, 2, 4>)); PL((k_probe_line<kModeDisabled, 1, 8>)); PL(k_probe_line_la<8>); PL((k_probe_tag<5>));
    PL((k_probe_line<kModeDisabled, 2, 4>)); PL((k_probe_line<kModeTtl, 1, 4, true, true>));
    PL((k_probe_line<kModeTtl, 1, 4, false, true>));
    PL((k_probe<kModeTtl, 2, 3, true, false, true>)); PL((k_probe<kModeTtl, 2, 3, true>));
    PL((k_probe<kModeTtl, 2, 3, false, false, true>)); PL((k_probe<kModeTtl, 2, 3>));
    PL((k_probe<kModeLru, 1, 6>)); PL((k_probe<kModeDisabled, 1, 6>));
    PL(k_dedup); PL(k_claim<kModeDisabled>); PL(k_claim<kModeTtl>); PL(k_claim<kModeLru>);
    PL((k_commit<kModeDisabled>)); PL((k_commit<kModeTtl>)); PL((k_commit<kModeTtl, true>));
    PL((k_commit<kModeLru>)); PL(k_lru_found); PL(k_lru_victim); PL(k_lru_revert); PL(k_lru_meta);
    PL(k_finalize); PL(k_pf_group); PL(k_pf_slot); PL(k_pf_write);
#undef PL
}

void run_validate(Table& t, const uint64_t* ids, uint64_t n, cudaStream_t st) {
    k_init_counters<<<1, 32, 0, st>>>(t.d_aux);
    k_validate<<<grid_for(n / 2 + 1, 256, 148u * 8u), 256, 0, st>>>(t.dev, ids, n, t.d_aux);
    t.launches += 2;
    MPZCH_CUDA(cudaGetLastError());
    MPZCH_CUDA(cudaMemcpyAsync(&t.h_aux->err, &t.d_aux->err, sizeof(BatchErr), cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaStreamSynchronize(st));
}

void enqueue_fast_batch(Table& t, const BatchArgs& a, cudaStream_t st) {
    constexpr int kU = 1;  // positions per probe thread (more threads beat more positions per
                           // thread: C5 probe 0.46 -> 0.39 ms going from 2 x 4 blocks/SM to 1 x 6)
    const uint64_t n = a.n;
    t.ensure_fast_scratch(n);
    if (a.pol->mode == kModeLru) t.ensure_pf_scratch(n);  // the found map and victim set (K3a/K3b)
    uint64_t epoch = ++t.epoch;
    if ((uint32_t)epoch == 0) {  // the keys' 32-bit epoch wrapped: start the index and records over
        MPZCH_CUDA(cudaMemsetAsync(t.s_hkey.p, 0, t.s_hkey.bytes, st));
        MPZCH_CUDA(cudaMemsetAsync(t.s_tent.p, 0, t.s_tent.bytes, st));
        if (t.mf_tab.p) MPZCH_CUDA(cudaMemsetAsync(t.mf_tab.p, 0, t.mf_tab.bytes, st));
        if (t.sl_tab.p) MPZCH_CUDA(cudaMemsetAsync(t.sl_tab.p, 0, t.sl_tab.bytes, st));
        t.epoch = epoch = 1;
    }
    const unsigned B = 256;
    const unsigned gW = grid_for(n, B, 148u * 8u);  // count-driven kernels (4/16/32 x 148: same)
    // 24 blocks per SM of grid (4 waves at 6 resident): 18 / 30 / 36 / 48 measured slower
    const unsigned gP = grid_for((n + kU - 1) / kU, B, 148u * 24u);
    const bool ttl = a.pol->mode == kModeTtl;
    const bool lru = a.pol->mode == kModeLru;
    uint32_t* newpos = t.s_newpos.as<uint32_t>();
    uint64_t* newid = t.s_newid.as<uint64_t>();
    uint32_t* newa = t.s_newa.as<uint32_t>();
    uint32_t* newm = t.s_newm.as<uint32_t>();
    uint32_t* newent = t.s_newent.as<uint32_t>();
    if (t.profiling) cudaEventRecord(t.ev[7], st);
    if (a.sh_state) {  // row-sharded owner: the sources validated; adopt the ranks' decision
        launch_pdl(k_sh_adopt, 1, 32, st, t.d_ctr, (const ShStateView*)a.sh_state);
        t.launches += 1;
    } else {
        k_init_counters<<<1, 32, 0, st>>>(t.d_ctr);
        launch_pdl(k_validate, grid_for(n / 2 + 1, B, 148u * 8u), B, st, t.dev, a.ids, n, t.d_ctr);
        t.launches += 2;
    }
    if (a.overflow_all) return;  // validation only; the host reports the error
    if (t.profiling) cudaEventRecord(t.ev[0], st);
    // probe kernel: the quad line walk when windows run long (max_probe >= 256: at 0.95 load
    // 16% of misses walk all 256 slots) or the batch is small, else the per-thread sector walk (DESIGN.md section 4
    // has the measurements behind the rule); MPZCH_PROBE=sector|line overrides it
    static const int forced = [] {
        const char* e = std::getenv("MPZCH_PROBE");
        return !e ? -1 : (std::string(e) == "line" ? 1 : 0);
    }();
    // small batches (C1: 64K positions) cannot fill the GPU with one thread per position: the
    // quad kernel runs 4x the threads and a quarter of the rounds per walk
    const bool line = forced >= 0 ? forced == 1 : (t.P >= 256 || n <= (1ull << 18));
    static const bool la_env = [] {  // the one-line lookahead for long Disabled walks (MPZCH_LOOKAHEAD=0: off)
        const char* e = std::getenv("MPZCH_LOOKAHEAD");
        return !(e && std::string(e) == "0");
    }();
    static const bool tag_env = [] {  // the tag walk for long Disabled windows (MPZCH_TAGS=0: off)
        const char* e = std::getenv("MPZCH_TAGS");
        return !(e && std::string(e) == "0");
    }();
#define MPZCH_PROBE_ARGS t.dev, a.ids, n, a.now, a.uniform_meta, t.d_ctr, a.out_slots, a.out_oc, newpos, newid, newa, newm
    if (line) {
        constexpr int kUL = 2;
        const unsigned gl = grid_for(4 * ((n + kUL - 1) / kUL), B, 148u * 16u);
        const uint32_t* nol = nullptr;
        if (ttl && a.per_feature) launch_pdl(k_probe_line<kModeTtl, kUL, 3, true>, gl, B, st, MPZCH_PROBE_ARGS, nol);
        else if (ttl) launch_pdl(k_probe_line<kModeTtl, kUL, 3>, gl, B, st, MPZCH_PROBE_ARGS, nol);
        else if (lru) launch_pdl(k_probe_line<kModeLru, kUL, 4>, gl, B, st, MPZCH_PROBE_ARGS, nol);
        // long windows: one position per quad at 8 blocks/SM (C3 insert-heavy 1.88 -> 2.07 G/s);
        // small batches keep 2 per quad (C1 1.10 vs 1.04 G/s pipelined)
        else if (t.P >= 256 && t.dev.tag && tag_env)
            launch_pdl(k_probe_tag<5>, grid_for(4 * n, B, 148u * 32u), B, st, MPZCH_PROBE_ARGS, nol);
        else if (t.P >= 256 && la_env)
            launch_pdl(k_probe_line_la<8>, grid_for(4 * n, B, 148u * 32u), B, st, MPZCH_PROBE_ARGS, nol);
        else if (t.P >= 256)
            launch_pdl(k_probe_line<kModeDisabled, 1, 8>, grid_for(4 * n, B, 148u * 32u), B, st, MPZCH_PROBE_ARGS, nol);
        else launch_pdl(k_probe_line<kModeDisabled, kUL, 4>, gl, B, st, MPZCH_PROBE_ARGS, nol);
    } else {
        // TTL walks carry a metadata sector per round too: 2 positions per thread at 3 blocks/SM
        // (C2: 2.78 vs 2.40 G/s for 1 x 4; C4 1.04 vs 1.09)
        // (C2 swept: 1 or 4 positions per thread, 3-32 blocks/SM of grid: all slower)
        // TTL: walks still pending after `defer` sector rounds finish in a resume launch of the
        // quad line walk, whose warps hold long walks only (MPZCH_DEFER=0 disables)
        static const unsigned defer = [] {
            const char* e = std::getenv("MPZCH_DEFER");
            return e ? (unsigned)std::atoi(e) : 8u;  // C2 2.75 -> 3.05-3.09, C4 1.03 -> 1.09 G/s
        }();
        uint32_t* dl = t.s_defer.as<uint32_t>();
        const unsigned gT = grid_for((n + 1) / 2, B, 148u * 16u), gR = 148u * 4u;
        if (ttl && a.per_feature) {
            if (defer) {
                launch_pdl(k_probe<kModeTtl, 2, 3, true, false, true>, gT, B, st, MPZCH_PROBE_ARGS, dl, defer);
                launch_pdl(k_probe_line<kModeTtl, 1, 4, true, true>, gR, B, st, MPZCH_PROBE_ARGS,
                           (const uint32_t*)dl);
            } else {
                launch_pdl(k_probe<kModeTtl, 2, 3, true>, gT, B, st, MPZCH_PROBE_ARGS, dl, 0u);
            }
        } else if (ttl) {
            if (defer) {
                launch_pdl(k_probe<kModeTtl, 2, 3, false, false, true>, gT, B, st, MPZCH_PROBE_ARGS, dl, defer);
                launch_pdl(k_probe_line<kModeTtl, 1, 4, false, true>, gR, B, st, MPZCH_PROBE_ARGS,
                           (const uint32_t*)dl);
            } else {
                launch_pdl(k_probe<kModeTtl, 2, 3>, gT, B, st, MPZCH_PROBE_ARGS, dl, 0u);
            }
        } else if (lru) {
            launch_pdl(k_probe<kModeLru, 1, 6>, gP, B, st, MPZCH_PROBE_ARGS, (uint32_t*)nullptr, 0u);
        } else {
            launch_pdl(k_probe<kModeDisabled, 1, 6>, gP, B, st, MPZCH_PROBE_ARGS, (uint32_t*)nullptr, 0u);
        }
        if (ttl && defer) ++t.launches;
    }
#undef MPZCH_PROBE_ARGS
    ++t.launches;
    if (t.profiling) cudaEventRecord(t.ev[1], st);
    IdEntry* te = t.s_tent.as<IdEntry>();
    launch_pdl(k_dedup, gW, B, st, t.d_ctr, t.tcap, epoch, (const uint32_t*)newpos, (const uint64_t*)newid,
               (const uint32_t*)newa, (const uint32_t*)newm, newent, t.s_hkey.as<u128>(), te, t.s_dupl.as<uint32_t>());
    if (t.profiling) cudaEventRecord(t.ev[4], st);
#define MPZCH_CLAIM_COMMIT(MODE)                                                                   \
    launch_pdl(k_claim<MODE>, gW, B, st, t.dev, a.now, t.d_ctr, newpos, newent, te, nullptr);     \
    if (t.profiling) cudaEventRecord(t.ev[5], st);                                               \
    launch_pdl(k_commit<MODE>, gW, B, st, t.dev, t.d_ctr, newpos, newid, newent, te, t.gen_clock, \
                                     a.uniform_meta, t.s_reset.as<uint64_t>(),                     \
                                     t.s_evflag.as<uint8_t>(), t.s_evslot.as<uint64_t>(),         \
                                     a.out_slots, a.out_oc)
    if (ttl && a.per_feature) {
        launch_pdl(k_claim<kModeTtl>, gW, B, st, t.dev, a.now, t.d_ctr, newpos, newent, te, nullptr);
        if (t.profiling) cudaEventRecord(t.ev[5], st);
        launch_pdl(k_commit<kModeTtl, true>, gW, B, st, t.dev, t.d_ctr, newpos, newid, newent, te, t.gen_clock,
                   a.uniform_meta, t.s_reset.as<uint64_t>(), t.s_evflag.as<uint8_t>(), t.s_evslot.as<uint64_t>(),
                   a.out_slots, a.out_oc);
    }
    else if (ttl) { MPZCH_CLAIM_COMMIT(kModeTtl); }
    else if (lru) {
        // evictors listed in newa's storage (dead after K2)
        launch_pdl(k_claim<kModeLru>, gW, B, st, t.dev, a.now, t.d_ctr, newpos, newent, te, newa);
        if (t.profiling) cudaEventRecord(t.ev[5], st);
        PfEntry* vtab = t.sl_tab.as<PfEntry>();
        const uint32_t ep = (uint32_t)epoch;
        PfEntry* ftab = t.mf_tab.as<PfEntry>();
        launch_pdl(k_lru_found, grid_for(n, B, 148u * 8u), B, st, t.d_ctr, n, (const uint64_t*)a.out_slots,
                   (const uint8_t*)a.out_oc, ftab, t.mf_cap - 1, ep);
        launch_pdl(k_lru_victim, 148u * 4u, B, st, t.dev, a.now, t.d_ctr, (const uint32_t*)newa, te, vtab,
                   t.mf_cap, (const PfEntry*)ftab, t.mf_cap - 1, ep);
        launch_pdl(k_lru_revert, gW, B, st, t.dev, t.d_ctr, newpos, newent, te);
        launch_pdl(k_commit<kModeLru>, gW, B, st, t.dev, t.d_ctr, newpos, newid, newent, te, t.gen_clock,
                                             a.uniform_meta, t.s_reset.as<uint64_t>(),
                                             t.s_evflag.as<uint8_t>(), t.s_evslot.as<uint64_t>(),
                                             a.out_slots, a.out_oc);
        t.launches += 3;
    }
    else { MPZCH_CLAIM_COMMIT(kModeDisabled); }
#undef MPZCH_CLAIM_COMMIT
    t.launches += 3;
    if (t.profiling) cudaEventRecord(t.ev[2], st);
    launch_pdl(k_finalize, gW, B, st, t.d_ctr, a.feats, (const uint32_t*)newpos, (const uint32_t*)newent,
               (const uint32_t*)t.s_dupl.as<uint32_t>(), (const IdEntry*)te, a.out_slots, a.out_oc);
    if (t.profiling) cudaEventRecord(t.ev[6], st);
    ++t.launches;
    if (lru) {
        launch_pdl(k_lru_meta, grid_for(n, B, 148u * 8u), B, st, t.dev, t.d_ctr, n, a.out_slots, a.uniform_meta);
        ++t.launches;
    }
    if (ttl && a.per_feature) {  // the metadata words, by last writer (M1..M3 above)
        t.ensure_pf_scratch(n);
        uint64_t cap = 1024;
        while (cap < 2 * n) cap <<= 1;
        const uint32_t ep = (uint32_t)t.epoch;
        const unsigned gN = grid_for(n, B, 148u * 8u);
        PfEntry* gtab = t.mf_tab.as<PfEntry>();
        PfEntry* stab = t.sl_tab.as<PfEntry>();
        launch_pdl(k_pf_group, gN, B, st, (const BatchCounters*)t.d_ctr, a.ids, a.feats, n, ep, gtab, cap - 1,
                   t.mf_ent.as<uint32_t>());
        launch_pdl(k_pf_slot, gN, B, st, (const BatchCounters*)t.d_ctr, n, ep, (const PfEntry*)gtab,
                   (const uint32_t*)t.mf_ent.as<uint32_t>(), (const uint64_t*)a.out_slots, stab, cap - 1,
                   t.sl_ent.as<uint32_t>());
        launch_pdl(k_pf_write, gN, B, st, t.dev, (const BatchCounters*)t.d_ctr, a.feats, n, (const PfEntry*)gtab,
                   (const uint32_t*)t.mf_ent.as<uint32_t>(), (const PfEntry*)stab,
                   (const uint32_t*)t.sl_ent.as<uint32_t>(), (const uint64_t*)a.out_slots, a.now,
                   a.pol->default_ttl, a.d_featk, a.d_featv, a.nk);
        t.launches += 3;
    }
    if (t.dim > 0) launch_reset_rows(t, t.s_reset.as<uint64_t>(), &t.d_ctr->reset_count, st);
    if (a.out_mark) {  // first positions of Evicted uniques (row-sharded evicted list)
        if (ttl || lru) MPZCH_CUDA(cudaMemcpyAsync(a.out_mark, t.s_evflag.p, n, cudaMemcpyDeviceToDevice, st));
        else MPZCH_CUDA(cudaMemsetAsync(a.out_mark, 0, n, st));
    }
    // (row-sharded owner: the return scatter reads and clears the evicted flags)
    if ((ttl || lru) && !a.sh_state)
        enqueue_compact_evicted(t, n, a.out_ev, a.ev_cap, st, lru ? &t.d_ctr->lru_evict : nullptr, a.out_slots);
    if (t.profiling) cudaEventRecord(t.ev[3], st);
}

}  // namespace mpzch_b200
