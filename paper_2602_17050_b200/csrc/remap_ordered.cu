// remap_ordered.cu -- the general, always-exact path of process_batch
// (proj/src/batch_engine.cpp:141-221) for the cases the fast claim path does not
// cover: LRU, TTL with several per-feature TTLs in one batch (last-writer
// metadata order), and tables whose raw-imported state may hold probe-window
// holes (proj/tests/test_probe_core.cpp:113-121).
//
//   G1  validate + (id, feature) dedup: 128-bit atomicCAS key, rank = first
//       position (atomicMin)                                   batch_engine.cpp:79-108
//   G2  first occurrences -> uniques in dedup order (ordered compaction)
//   G3  per-unique shard + metadata (make_metadata)           eviction.cpp:20-30
//   G4  one warp per shard walks the uniques in rank order and runs the two-pass
//       probe of probe_core.cpp:69-134 with 32-slot coalesced window loads and
//       __ballot_sync/__ffs decisions; shards run concurrently (the OpenMP
//       parallel-for of batch_engine.cpp:203-208)
//   G5  scatter to positions                                   batch_engine.cpp:213-220
#include <cuda_runtime.h>

#include "common.cuh"
#include "compact.cuh"
#include "ordered_probe.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

typedef unsigned __int128 u128;
constexpr u128 kKeyEmpty = ~(u128)0;

__device__ __forceinline__ uint64_t ttl_lookup(uint32_t f, uint64_t def, const uint32_t* keys,
                                               const uint64_t* vals, uint32_t nk) {
    for (uint32_t i = 0; i < nk; ++i)
        if (keys[i] == f) return vals[i];
    return def;
}

__global__ void k_init_counters_o(BatchCounters* c) {
    if (threadIdx.x == 0) {
        BatchCounters z{};
        z.err.bad_pos = ~0ull;
        z.err.foreign_pos = ~0ull;
        z.n_live = ~0ull;
        z.path_taken = 1;
        *c = z;
    }
}

// gated start (behind an LRU claim attempt): the path runs only if the attempt aborted; else
// its counter block is marked failed, and every kernel below returns at once
__global__ void k_init_counters_gated(BatchCounters* c, const BatchCounters* attempt) {
    if (threadIdx.x == 0) {
        BatchCounters z{};
        z.err.bad_pos = ~0ull;
        z.err.foreign_pos = ~0ull;
        z.n_live = ~0ull;
        z.path_taken = 1;
        if (!(attempt->lru_abort && !batch_failed(&attempt->err))) z.err.too_many = 3;  // skip
        *c = z;
    }
}

// after the gated path: its counters become the batch's if it ran
__global__ void k_adopt_counters(BatchCounters* attempt, const BatchCounters* alt) {
    if (threadIdx.x == 0 && alt->err.too_many != 3) *attempt = *alt;
}

__global__ void k_zero_marks(const BatchCounters* ctr, uint64_t n, uint8_t* __restrict__ mark) {
    if (batch_failed(&ctr->err)) return;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        mark[i] = 0;
}

__global__ void __launch_bounds__(256) k_validate_dedup(TableDev t, const uint64_t* __restrict__ ids,
                                                        const uint32_t* __restrict__ feats, uint64_t n,
                                                        uint64_t now, int mode, uint64_t def_ttl,
                                                        const uint32_t* fk, const uint64_t* fv,
                                                        uint32_t nk, BatchCounters* ctr, u128* key,
                                                        unsigned* kmin, uint32_t* posent,
                                                        uint64_t mask) {
    if (ctr->err.too_many == 3) return;  // gated off
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t id = ids[i];
        const uint32_t f = feats ? feats[i] : 0u;
        if (id >> 63) {
            atomicMin(&ctr->err.bad_pos, (unsigned long long)i);
            posent[i] = kNone32;
            continue;
        }
        if (!holds_shard(t, shard_of(id, t))) {
            atomicMin(&ctr->err.foreign_pos, (unsigned long long)i);
            posent[i] = kNone32;
            continue;
        }
        if (mode == kModeTtl) {
            const uint64_t ttl = ttl_lookup(f, def_ttl, fk, fv, nk);
            if (ttl > ~0ull - now) atomicExch(&ctr->err.overflow, 1u);
        }
        const u128 k = ((u128)f << 64) | (u128)id;
        uint64_t h = mix64(id ^ ((uint64_t)f << 32), 0) & mask;
        for (;;) {
            u128 cur = key[h];
            if (cur == kKeyEmpty) {
                cur = atomicCAS(key + h, kKeyEmpty, k);
                if (cur == kKeyEmpty) break;
            }
            if (cur == k) break;
            h = (h + 1) & mask;
        }
        // (a plain read first: a hot id's thousands of positions would serialise on no-op atomics)
        if (__ldcg(kmin + h) > (unsigned)i) atomicMin(kmin + h, (unsigned)i);
        posent[i] = (uint32_t)h;
    }
}

__global__ void __launch_bounds__(256) k_first_flags(const BatchCounters* ctr, uint64_t n,
                                                     const uint32_t* __restrict__ posent,
                                                     const unsigned* __restrict__ kmin,
                                                     uint8_t* __restrict__ flag) {
    if (ctr->err.too_many == 3) return;  // gated off (the flags stay all zero)
    const bool failed = batch_failed(&ctr->err);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = posent[i];
        flag[i] = (!failed && e != kNone32 && kmin[e] == (unsigned)i) ? 1 : 0;
    }
}

struct EmitUnique {
    uint32_t* upos;
    uint32_t* entu;
    const uint32_t* posent;
    __device__ void operator()(uint64_t i, unsigned k) const {
        upos[k] = (uint32_t)i;
        entu[posent[i]] = k;
    }
};

__global__ void __launch_bounds__(256) k_prep(TableDev t, const BatchCounters* ctr,
                                              const uint64_t* __restrict__ ids,
                                              const uint32_t* __restrict__ feats,
                                              const uint32_t* __restrict__ upos, uint64_t now,
                                              int mode, uint64_t def_ttl, const uint32_t* fk,
                                              const uint64_t* fv, uint32_t nk,
                                              uint32_t* __restrict__ ushard,
                                              uint64_t* __restrict__ umeta) {
    if (ctr->err.too_many == 3) return;  // gated off
    const unsigned u = ctr->entry_count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < u; k += gridDim.x * blockDim.x) {
        const uint32_t pos = upos[k];
        const uint64_t id = ids[pos];
        ushard[k] = shard_of(id, t);
        umeta[k] = mode == kModeTtl
                       ? now + ttl_lookup(feats ? feats[pos] : 0u, def_ttl, fk, fv, nk)
                       : now;
    }
}

// G4: one warp per shard, uniques in rank order, reference two-pass probe.
template <int MODE>
__global__ void __launch_bounds__(256) k_ordered(TableDev t, BatchCounters* ctr,
                                                 const uint64_t* __restrict__ ids,
                                                 const uint32_t* __restrict__ upos,
                                                 const uint32_t* __restrict__ ushard,
                                                 const uint64_t* __restrict__ umeta, uint64_t now,
                                                 uint64_t gen_clock, uint64_t* __restrict__ uslot,
                                                 uint8_t* __restrict__ uoc,
                                                 uint64_t* __restrict__ reset_rows,
                                                 uint8_t* __restrict__ evflag,
                                                 uint64_t* __restrict__ evslot,
                                                 const uint8_t* __restrict__ todo) {
    if (batch_failed(&ctr->err) || (todo && !ctr->r_left)) return;  // rounds left nothing
    const uint32_t shard = t.shard_lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (shard >= t.shard_hi) return;
    const unsigned lane = lane_id();
    const unsigned u = ctr->entry_count;
    const ShardDev sd = t.shards[shard];
    const uint64_t cap = sd.cap.d, base = sd.offset;
    for (unsigned k0 = 0; k0 < u; k0 += 32) {
        const unsigned kk = k0 + lane;
        unsigned mine = __ballot_sync(0xffffffffu, kk < u && ushard[kk] == shard && (!todo || todo[kk]));
        while (mine) {
            const unsigned k = k0 + __ffs(mine) - 1;
            mine &= mine - 1;
            const uint64_t id = ids[upos[k]];
            const uint64_t meta_in = umeta[k];
            const uint64_t h = home_of(id, sd, t.seed);
            uint64_t gslot;
            uint8_t oc;
            two_pass_probe<MODE>(t, base, cap, h, id, now, lane, gslot, oc);
            if (lane == 0) {
                if (oc == kInserted || oc == kEvicted) {
                    t.ident[gslot] = id;
                    store_tag(t, gslot, id);
                }
                t.meta[gslot] = meta_in;  // Found refresh / insert / evict / Collision at home
                if (oc == kInserted || oc == kEvicted) t.row_gen[gslot] = gen_clock;
                if (oc == kEvicted) {
                    if (t.dim) reset_rows[atomicAdd(&ctr->reset_count, 1u)] = gslot;
                    evflag[k] = 1;
                    evslot[k] = gslot;
                    atomicAdd(&ctr->evicted_count, 1u);
                }
                uslot[k] = gslot;
                uoc[k] = oc;
            }
            __syncwarp();
        }
    }
}

// G4' (hole-free tables): the same per-shard rank-order walk, but one pass per unique that
// stops at the first match or EMPTY.  With no hole in any window "exists"
// (pass 1, probe_core.cpp:78-86) is "a match before the first EMPTY", so pass 2's decision
// (probe_core.cpp:89-133) can be taken on the fly: match -> Found; EMPTY -> the first expired
// slot before it (TTL) else Inserted; neither in the window -> first expired (TTL), the first
// strict LRU minimum (LRU), else Collision.  The first 32-slot chunk of the NEXT unique of
// the shard is loaded while the current one is decided and patched with the current one's
// writes, so consecutive uniques overlap their latency.
template <int MODE>
__global__ void __launch_bounds__(256) k_ordered_hf(TableDev t, BatchCounters* ctr,
                                                    const uint64_t* __restrict__ ids,
                                                    const uint32_t* __restrict__ upos,
                                                    const uint32_t* __restrict__ ushard,
                                                    const uint64_t* __restrict__ umeta, uint64_t now,
                                                    uint64_t gen_clock, uint64_t* __restrict__ uslot,
                                                    uint8_t* __restrict__ uoc,
                                                    uint64_t* __restrict__ reset_rows,
                                                    uint8_t* __restrict__ evflag,
                                                    uint64_t* __restrict__ evslot,
                                                    const uint8_t* __restrict__ todo) {
    if (batch_failed(&ctr->err) || (todo && !ctr->r_left)) return;  // rounds left nothing
    const uint32_t shard = t.shard_lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (shard >= t.shard_hi) return;
    const unsigned lane = lane_id();
    const unsigned u = ctr->entry_count;
    const ShardDev sd = t.shards[shard];
    const uint64_t cap = sd.cap.d, base = sd.offset;
    const uint32_t P = t.P;
    auto slot_at = [&](uint64_t h, uint32_t off) {
        uint64_t x = h + off;
        return base + (x >= cap ? x - cap : x);
    };
    // prefetched first chunk of the next unique of this shard
    unsigned pf_k = kNone32;
    uint64_t pf_v = 0, pf_m = 0;
    for (unsigned k0 = 0; k0 < u; k0 += 32) {
        const unsigned kk = k0 + lane;
        unsigned mine = __ballot_sync(0xffffffffu, kk < u && ushard[kk] == shard && (!todo || todo[kk]));
        while (mine) {
            const unsigned k = k0 + __ffs(mine) - 1;
            mine &= mine - 1;
            const uint64_t id = ids[upos[k]];
            const uint64_t meta_in = umeta[k];
            const uint64_t h = home_of(id, sd, t.seed);
            // issue the next unique's first chunk now
            const unsigned nk = mine ? k0 + __ffs(mine) - 1 : kNone32;
            uint64_t n_v = 0, n_m = 0, n_g = kEmpty;
            if (nk != kNone32 && lane < P) {
                const uint64_t nid = ids[upos[nk]];
                n_g = slot_at(home_of(nid, sd, t.seed), lane);
                n_v = ld_cg(t.ident + n_g);
                if (MODE != kModeDisabled) n_m = ld_cg(t.meta + n_g);
            }
            uint8_t oc = kCollision;
            uint64_t gslot = base + h;
            bool decided = false;
            uint32_t exp_off = kNone32;
            uint64_t exp_g = 0, best_m = 0, best_g = 0;
            uint32_t best_off = kNone32;
            for (uint32_t c = 0; c < P; c += 32) {
                const uint32_t off = c + lane;
                const bool valid = off < P;
                uint64_t g = 0, v = 0, m = 0;
                if (valid) {
                    g = slot_at(h, off);
                    if (c == 0 && pf_k == k) {
                        v = pf_v;
                        m = pf_m;
                    } else {
                        v = ld_cg(t.ident + g);
                        if (MODE != kModeDisabled) m = ld_cg(t.meta + g);
                    }
                }
                const bool is_match = valid && v == id;
                const bool is_empty = valid && v == kEmpty;
                const unsigned stop = __ballot_sync(0xffffffffu, is_match || is_empty);
                const int sl = stop ? __ffs(stop) - 1 : 32;
                const unsigned before = sl == 32 ? 0xffffffffu : ((1u << sl) - 1);
                if (MODE == kModeTtl && exp_off == kNone32) {
                    const unsigned em = __ballot_sync(0xffffffffu, valid && !is_match && !is_empty &&
                                                                       m < now) & before;
                    if (em) {
                        const int src = __ffs(em) - 1;
                        exp_off = c + src;
                        exp_g = __shfl_sync(0xffffffffu, g, src);
                    }
                }
                if (MODE == kModeLru && !stop) {
                    // first strict minimum over the window, ties -> lowest offset
                    uint64_t bm = valid ? m : ~0ull;
                    uint32_t bo = valid ? off : kNone32;
                    uint64_t bg = g;
                    for (int o = 16; o; o >>= 1) {
                        const uint64_t om = __shfl_xor_sync(0xffffffffu, bm, o);
                        const uint32_t oo = __shfl_xor_sync(0xffffffffu, bo, o);
                        const uint64_t og = __shfl_xor_sync(0xffffffffu, bg, o);
                        if (om < bm || (om == bm && oo < bo)) { bm = om; bo = oo; bg = og; }
                    }
                    if (bo != kNone32 && (best_off == kNone32 || bm < best_m)) {
                        best_m = bm;
                        best_off = bo;
                        best_g = bg;
                    }
                }
                if (stop) {
                    const bool match = __shfl_sync(0xffffffffu, is_match, sl);
                    const uint64_t gs = __shfl_sync(0xffffffffu, g, sl);
                    if (match) {
                        gslot = gs;
                        oc = kFound;
                    } else if (MODE == kModeTtl && exp_off != kNone32) {
                        gslot = exp_g;
                        oc = kEvicted;
                    } else {
                        gslot = gs;
                        oc = kInserted;
                    }
                    decided = true;
                    break;
                }
            }
            if (!decided) {
                if (MODE == kModeTtl && exp_off != kNone32) {
                    gslot = exp_g;
                    oc = kEvicted;
                } else if (MODE == kModeLru && best_off != kNone32) {
                    gslot = best_g;
                    oc = kEvicted;  // LRU fallback, probe_core.cpp:125-129
                }
            }
            if (lane == 0) {
                if (oc == kInserted || oc == kEvicted) {
                    t.ident[gslot] = id;
                    store_tag(t, gslot, id);
                }
                t.meta[gslot] = meta_in;
                if (oc == kInserted || oc == kEvicted) t.row_gen[gslot] = gen_clock;
                if (oc == kEvicted) {
                    if (t.dim) reset_rows[atomicAdd(&ctr->reset_count, 1u)] = gslot;
                    evflag[k] = 1;
                    evslot[k] = gslot;
                    atomicAdd(&ctr->evicted_count, 1u);
                }
                uslot[k] = gslot;
                uoc[k] = oc;
            }
            // patch the prefetched chunk with this unique's writes
            if (n_g == gslot) {
                if (oc == kInserted || oc == kEvicted) n_v = id;
                n_m = meta_in;
            }
            pf_k = nk;
            pf_v = n_v;
            pf_m = n_m;
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(256) k_scatter(BatchCounters* ctr, uint64_t n,
                                                 const uint32_t* __restrict__ posent,
                                                 const uint32_t* __restrict__ entu,
                                                 const uint64_t* __restrict__ uslot,
                                                 const uint8_t* __restrict__ uoc,
                                                 uint64_t* __restrict__ out_slots,
                                                 uint8_t* __restrict__ out_oc) {
    if (batch_failed(&ctr->err)) return;
    unsigned long long c[4] = {0, 0, 0, 0};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = entu[posent[i]];
        out_slots[i] = uslot[k];
        const uint8_t oc = uoc[k];
        out_oc[i] = oc;
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

__global__ void __launch_bounds__(256) k_mark_first(const BatchCounters* ctr,
                                                    const uint32_t* __restrict__ upos,
                                                    const uint8_t* __restrict__ evflag,
                                                    uint8_t* __restrict__ mark) {
    if (batch_failed(&ctr->err)) return;
    const unsigned u = ctr->entry_count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < u; k += gridDim.x * blockDim.x)
        if (evflag[k]) mark[upos[k]] = 1;
}

__global__ void __launch_bounds__(256) k_cleanup_o(const BatchCounters* ctr, uint64_t n,
                                                   const uint32_t* __restrict__ posent,
                                                   u128* key, unsigned* kmin) {
    if (ctr->err.too_many == 3) return;  // gated off: validate_dedup wrote nothing
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = posent[i];
        // only the unique's first position clears its entry: a hot id's thousands of positions
        // would otherwise store to one record
        if (e == kNone32 || __ldcg(kmin + e) != (unsigned)i) continue;
        key[e] = kKeyEmpty;
        kmin[e] = kNone32;
    }
}

}  // namespace

void preload_ordered_kernels() {
#define PL(k) preload_kernel((const void*)(k))
    PL(k_init_counters_o); PL(k_init_counters_gated); PL(k_adopt_counters); PL(k_zero_marks);
    PL(k_validate_dedup); PL(k_first_flags); PL(k_prep);
    PL(k_ordered<kModeDisabled>); PL(k_ordered<kModeTtl>); PL(k_ordered<kModeLru>);
    PL(k_ordered_hf<kModeDisabled>); PL(k_ordered_hf<kModeTtl>); PL(k_ordered_hf<kModeLru>);
    PL(k_scatter); PL(k_mark_first); PL(k_cleanup_o);
#undef PL
    preload_compact<EmitUnique>();
}

void adopt_gated_counters(Table& t, BatchCounters* attempt, const BatchCounters* alt, cudaStream_t st) {
    k_adopt_counters<<<1, 32, 0, st>>>(attempt, alt);
    ++t.launches;
}

void enqueue_ordered_batch(Table& t, const BatchArgs& a, cudaStream_t st, bool rounds) {
    const uint64_t n = a.n;
    t.ensure_ordered_scratch(n);
    const unsigned B = 256;
    const unsigned gN = grid_for(n, B);
    const Policy& p = *a.pol;
    const uint32_t nk = (uint32_t)p.keys.size();
    if (a.gate_ctr) k_init_counters_gated<<<1, 32, 0, st>>>(t.d_ctr, a.gate_ctr);
    else k_init_counters_o<<<1, 32, 0, st>>>(t.d_ctr);
    uint64_t mask = 1024;
    while (mask < 2 * n) mask <<= 1;
    mask -= 1;
    u128* key = t.o_key.as<u128>();
    unsigned* kmin = t.o_min.as<unsigned>();
    uint32_t* posent = t.o_posent.as<uint32_t>();
    k_validate_dedup<<<gN, B, 0, st>>>(t.dev, a.ids, a.feats, n, a.now, p.mode, p.default_ttl, a.d_featk,
                                       a.d_featv, nk, t.d_ctr, key, kmin, posent, mask);
    k_first_flags<<<gN, B, 0, st>>>(t.d_ctr, n, posent, kmin, t.o_flag.as<uint8_t>());
    t.launches += 3;
    EmitUnique em{t.o_upos.as<uint32_t>(), t.o_entu.as<uint32_t>(), posent};
    compact_flags(t.o_flag.as<uint8_t>(), n, t.s_blk.as<unsigned>(), &t.d_ctr->entry_count, true, em,
                  st, t.launches);
    k_prep<<<gN, B, 0, st>>>(t.dev, t.d_ctr, a.ids, a.feats, t.o_upos.as<uint32_t>(), a.now, p.mode,
                             p.default_ttl, a.d_featk, a.d_featv, nk, t.o_ushard.as<uint32_t>(),
                             t.o_umeta.as<uint64_t>());
    const unsigned gS = (unsigned)(((uint64_t)(t.shard_hi - t.shard_lo) * 32 + B - 1) / B);
    // rounds path (hole-free tables): parallel A.4 rounds, then the remainder (if any) in order
    const uint8_t* todo = nullptr;
    if (rounds) {
        t.o_todo.reserve(n);
        enqueue_rounds(t, a, st, t.o_todo.as<uint8_t>());
        todo = t.o_todo.as<uint8_t>();
    }
#define MPZCH_ORDERED(MODE)                                                                       \
    (t.hole_free ? k_ordered_hf<MODE> : k_ordered<MODE>)<<<gS, B, 0, st>>>(                      \
        t.dev, t.d_ctr, a.ids, t.o_upos.as<uint32_t>(), t.o_ushard.as<uint32_t>(),                \
        t.o_umeta.as<uint64_t>(), a.now, t.gen_clock, t.o_uslot.as<uint64_t>(),                   \
        t.o_uoc.as<uint8_t>(), t.s_reset.as<uint64_t>(), t.s_evflag.as<uint8_t>(),                 \
        t.s_evslot.as<uint64_t>(), todo)
    if (p.mode == kModeTtl) MPZCH_ORDERED(kModeTtl);
    else if (p.mode == kModeLru) MPZCH_ORDERED(kModeLru);
    else MPZCH_ORDERED(kModeDisabled);
    ++t.launches;
#undef MPZCH_ORDERED
    k_scatter<<<gN, B, 0, st>>>(t.d_ctr, n, posent, t.o_entu.as<uint32_t>(), t.o_uslot.as<uint64_t>(),
                                t.o_uoc.as<uint8_t>(), a.out_slots, a.out_oc);
    t.launches += 2;
    if (t.dim > 0) launch_reset_rows(t, t.s_reset.as<uint64_t>(), &t.d_ctr->reset_count, st);
    if (a.out_mark) {  // unique k's first position is upos[k]
        k_zero_marks<<<grid_for(n, B, 148u * 8u), B, 0, st>>>(t.d_ctr, n, a.out_mark);
        k_mark_first<<<gN, B, 0, st>>>(t.d_ctr, t.o_upos.as<uint32_t>(), t.s_evflag.as<uint8_t>(),
                                       a.out_mark);
        ++t.launches;
    }
    if (p.mode != kModeDisabled) enqueue_compact_evicted(t, n, a.out_ev, a.ev_cap, st);
    k_cleanup_o<<<gN, B, 0, st>>>(t.d_ctr, n, posent, key, kmin);
    ++t.launches;
}

}  // namespace mpzch_b200
