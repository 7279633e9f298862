// lookup.cu -- batched read-only lookup: one MpzchTable::lookup per position
// (proj/src/table.cpp:150-156 -> lookup_readonly proj/src/probe_core.cpp:32-43).
//
// lookup_readonly scans the whole P-slot window for the first match.  On a
// hole-free table an id never sits behind an EMPTY slot of its own
// window, so the scan stops at the first match or EMPTY and touches ~1.5
// sectors per hit at 0.8 load instead of P/4.  Tables with raw-imported state
// keep the full-window scan.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "line_scan.cuh"
#include "tag_scan.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

__device__ __forceinline__ uint64_t pick4(uint32_t j, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return j == 0 ? a : (j == 1 ? b : (j == 2 ? c : d));
}

template <bool kHoleFree>
__global__ void __launch_bounds__(256) k_lookup(TableDev t, const uint64_t* __restrict__ ids, uint64_t n,
                                                uint64_t* __restrict__ out_slots,
                                                uint8_t* __restrict__ out_oc, BatchErr* err) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t id = ids[i];
        if (id >> 63) {
            atomicMin(&err->bad_pos, (unsigned long long)i);
            continue;
        }
        const uint32_t s = shard_of(id, t);
        if (!holds_shard(t, s)) {
            atomicMin(&err->foreign_pos, (unsigned long long)i);
            continue;
        }
        const ShardDev sd = t.shards[s];
        const uint64_t cap = sd.cap.d, base = sd.offset, end = base + cap;
        const uint64_t h = home_of(id, sd, t.seed);
        uint32_t off = 0;
        uint64_t g = base + h, gf = kEmpty;
        bool stop = false;
        while (off < t.P && !stop) {
            const uint64_t a4 = g & ~3ull;
            uint64_t w0, w1, w2, w3;
            ld_sector(t.ident + a4, w0, w1, w2, w3);
            do {
                const uint64_t v = pick4((uint32_t)(g - a4), w0, w1, w2, w3);
                if (v == id) { gf = g; stop = true; break; }
                if (kHoleFree && v == kEmpty) { stop = true; break; }
                ++off;
                if (++g == end) g = base;
            } while (off < t.P && (g >> 2) == (a4 >> 2));
        }
        if (gf != kEmpty) {
            out_slots[i] = gf;
            out_oc[i] = kFound;
        } else {
            out_slots[i] = base + h;
            out_oc[i] = kCollision;
        }
    }
}

// Quad line walk (line_scan.cuh): one quad per position, U positions in flight per quad,
// 16 slots per round.  Used when windows run long (max_probe >= 256 or a full-window scan).
// DEFER: walks still pending after `defer` line rounds are handed over -- (position, offset) in
// dlist, counted in *dcount -- to a RESUME launch whose warps hold long walks only (a warp
// otherwise waits for its longest walk; the table is read-only here, so a resumed walk reads
// what it would have read).
template <bool kHoleFree, int U, bool RESUME = false, bool DEFER = false>
__global__ void __launch_bounds__(256, U == 1 ? 6 : 4) k_lookup_line(TableDev t, const uint64_t* __restrict__ ids,
                                                        uint64_t n, uint64_t* __restrict__ out_slots,
                                                        uint8_t* __restrict__ out_oc, BatchErr* err,
                                                        uint32_t* __restrict__ dlist = nullptr,
                                                        unsigned* dcount = nullptr, unsigned defer = 0) {
    constexpr uint8_t kPending = 0, kHit = 1, kStop = 2, kIdle = 3, kDeferred = 4;
    if (RESUME) pdl_wait();
    const unsigned j = quad_lane(), qm = quad_mask();
    const uint64_t qpb = blockDim.x >> 2, qib = threadIdx.x >> 2, tile = qpb * U;
    const uint64_t total = RESUME ? (uint64_t)*(volatile unsigned*)dcount : n;
    for (uint64_t t0 = (uint64_t)blockIdx.x * tile; t0 < total; t0 += (uint64_t)gridDim.x * tile) {
        uint64_t id[U], g[U], home[U];
        uint32_t off[U], sh[U];
        uint32_t pos[RESUME ? U : 1];
        uint8_t st[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = t0 + (uint64_t)u * qpb + qib;
            st[u] = kIdle;
            off[u] = 0;
            if (RESUME && i < total) {
                pos[u] = dlist[2 * i];
                off[u] = dlist[2 * i + 1];
                id[u] = ids[pos[u]];
                sh[u] = shard_of(id[u], t);
                const ShardDev sd = t.shards[sh[u]];
                const uint64_t hh = home_of(id[u], sd, t.seed);
                home[u] = sd.offset + hh;
                uint64_t x = hh + off[u];
                if (x >= sd.cap.d) x -= sd.cap.d;
                g[u] = sd.offset + x;
                st[u] = kPending;
            } else if (!RESUME && i < n) {
                id[u] = ids[i];
                if (id[u] >> 63) {
                    if (j == 0) atomicMin(&err->bad_pos, (unsigned long long)i);
                    continue;
                }
                sh[u] = shard_of(id[u], t);
                if (!holds_shard(t, sh[u])) {
                    if (j == 0) atomicMin(&err->foreign_pos, (unsigned long long)i);
                    continue;
                }
                const ShardDev sd = t.shards[sh[u]];
                home[u] = sd.offset + home_of(id[u], sd, t.seed);
                g[u] = home[u];
                st[u] = kPending;
            }
        }
        unsigned rounds = 0;  // (DEFER)
        for (;;) {
            uint64_t w[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (st[u] == kPending) ld_line_part(t.ident, g[u], j, w[u]);
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
                const unsigned x = quad_gather(m, kHoleFree ? e : 0u, j, qm);
                const ShardDev sd = t.shards[sh[u]];
                const uint64_t base = sd.offset, end = base + sd.cap.d;
                const LineSpan sp = line_span(g[u], end, off[u], t.P);
                const unsigned hit = (x | (x >> 16)) & sp.range();
                if (hit) {
                    const unsigned p = __ffs(hit) - 1;
                    st[u] = (x >> p) & 1u ? kHit : kStop;
                    g[u] += p - sp.s;
                } else {
                    off[u] += sp.c;
                    g[u] += sp.c;
                    if (g[u] == end) g[u] = base;
                    if (off[u] >= t.P) st[u] = kStop;
                    else any = true;
                }
            }
            if (DEFER && any && ++rounds >= defer) {
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (st[u] == kPending) st[u] = kDeferred;
                any = false;
            }
            if (!any) break;
        }
        if (j == 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = RESUME ? (uint64_t)pos[RESUME ? u : 0] : t0 + (uint64_t)u * qpb + qib;
                if (DEFER && st[u] == kDeferred) {
                    const unsigned k = atomicAdd(dcount, 1u);
                    dlist[2 * (uint64_t)k] = (uint32_t)i;
                    dlist[2 * (uint64_t)k + 1] = off[u];
                } else if (st[u] == kHit) {
                    out_slots[i] = g[u];
                    out_oc[i] = kFound;
                } else if (st[u] == kStop) {
                    out_slots[i] = home[u];
                    out_oc[i] = kCollision;
                }
            }
        }
    }
}

// Long-window lookups on hole-free tables that keep identity tags: the first identity line of
// the window, then 128-slot tag lines (tag_scan.cuh) -- k_probe_tag's walk without its writes.
// An absent id at 0.95 load reads one identity line and ~2 tag lines instead of ~13 identity
// lines to reach its first EMPTY.
__global__ void __launch_bounds__(256, 5) k_lookup_tag(TableDev t, const uint64_t* __restrict__ ids, uint64_t n,
                                                       uint64_t* __restrict__ out_slots,
                                                       uint8_t* __restrict__ out_oc, BatchErr* err) {
    constexpr uint8_t kPending = 0, kHit = 1, kStop = 2, kIdle = 3;
    const unsigned j = quad_lane(), qm = quad_mask();
    const int jb = 32 * (int)j;
    const uint64_t qpb = blockDim.x >> 2, qib = threadIdx.x >> 2;
    unsigned long long isec = 0;  // (not reported by lookups)
    for (uint64_t t0 = (uint64_t)blockIdx.x * qpb; t0 < n; t0 += (uint64_t)gridDim.x * qpb) {
        const uint64_t i = t0 + qib;
        uint8_t st = kIdle;
        uint64_t id = 0, g = 0, home = 0, base = 0, end = 0;
        uint32_t off = 0;
        if (i < n) {
            id = ids[i];
            if (id >> 63) {
                if (j == 0) atomicMin(&err->bad_pos, (unsigned long long)i);
            } else {
                const uint32_t sh = shard_of(id, t);
                if (!holds_shard(t, sh)) {
                    if (j == 0) atomicMin(&err->foreign_pos, (unsigned long long)i);
                } else {
                    const ShardDev sd = t.shards[sh];
                    base = sd.offset;
                    end = base + sd.cap.d;
                    home = base + home_of(id, sd, t.seed);
                    g = home;
                    st = kPending;
                }
            }
        }
        if (st == kPending) {  // the home slot's identity line
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
                st = (x >> q) & 1u ? kHit : kStop;
                g += q - sp.s;
            } else {
                off += sp.c;
                g += sp.c;
                if (g == end) g = base;
                if (off >= t.P) st = kStop;
            }
        }
        const uint32_t pat = (uint32_t)tag_of(id) * 0x01010101u;
        while (st == kPending) {  // then 128 slots of tags per round
            const uint64_t tl = g & ~127ull;
            const int s0 = (int)(g & 127u);
            const int c0 = (int)tag_seg_len(g, end, off, t.P);
            uint64_t v[4];
            ld_tag_part(t, tl, j, v);
            unsigned fe;
            const unsigned q = tag_segment(t, v, pat, id, tl, s0, c0, jb, j, qm, fe, isec);
            if (q != 128u) {
                st = kHit;
                g = tl + q;
            } else if (fe != 128u) {
                st = kStop;
            } else {
                off += (uint32_t)c0;
                g += (uint64_t)c0;
                if (g == end) g = base;
                if (off >= t.P) st = kStop;
            }
        }
        if (j == 0) {
            if (st == kHit) {
                out_slots[i] = g;
                out_oc[i] = kFound;
            } else if (st == kStop) {
                out_slots[i] = home;
                out_oc[i] = kCollision;
            }
        }
    }
}

// Fused lookup + gather (the frozen-replica read path, MpzchTable::lookup
// table.cpp:150-156 then MpzchTable::gather table.cpp:158-163 / EmbeddingTable::gather
// embedding_store.cpp:95-103): each lane of a warp probes one position, then the warp copies
// the 32 resolved rows with 16-byte loads/stores (one row per step, dim/4 lanes busy).
template <bool kHoleFree>
__global__ void __launch_bounds__(256) k_lookup_gather(TableDev t, const uint64_t* __restrict__ ids,
                                                       uint64_t n, uint64_t* __restrict__ out_slots,
                                                       uint8_t* __restrict__ out_oc,
                                                       float* __restrict__ out_rows, BatchErr* err) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32 < n; w += warps) {
        const uint64_t i = w * 32 + lane;
        uint64_t slot = kEmpty;
        if (i < n) {
            const uint64_t id = ids[i];
            if (id >> 63) {
                atomicMin(&err->bad_pos, (unsigned long long)i);
            } else if (!holds_shard(t, shard_of(id, t))) {
                atomicMin(&err->foreign_pos, (unsigned long long)i);
            } else {
                const ShardDev sd = t.shards[shard_of(id, t)];
                const uint64_t cap = sd.cap.d, base = sd.offset, end = base + cap;
                const uint64_t h = home_of(id, sd, t.seed);
                uint32_t off = 0;
                uint64_t g = base + h, gf = kEmpty;
                bool stop = false;
                while (off < t.P && !stop) {
                    const uint64_t a4 = g & ~3ull;
                    uint64_t w0, w1, w2, w3;
                    ld_sector(t.ident + a4, w0, w1, w2, w3);
                    do {
                        const uint64_t v = pick4((uint32_t)(g - a4), w0, w1, w2, w3);
                        if (v == id) { gf = g; stop = true; break; }
                        if (kHoleFree && v == kEmpty) { stop = true; break; }
                        ++off;
                        if (++g == end) g = base;
                    } while (off < t.P && (g >> 2) == (a4 >> 2));
                }
                slot = gf != kEmpty ? gf : base + h;
                out_slots[i] = slot;
                out_oc[i] = gf != kEmpty ? kFound : kCollision;
            }
        }
        // cooperative row copy
        for (int r = 0; r < 32; ++r) {
            const uint64_t sr = __shfl_sync(0xffffffffu, slot, r);
            const uint64_t ir = w * 32 + r;
            if (ir >= n || sr == kEmpty) continue;
            copy_row_or_draw(t, sr, out_rows + ir * t.dim, lane);
        }
    }
}

__global__ void k_lookup_init(BatchCounters* c) {
    if (threadIdx.x == 0) {
        BatchCounters z{};
        z.err.bad_pos = ~0ull;
        z.err.foreign_pos = ~0ull;
        *c = z;
    }
}

// the id at the first invalid position (the exception text distinguishes EMPTY from > 2^63)
__global__ void k_lookup_bad_id(const uint64_t* __restrict__ ids, BatchCounters* c) {
    pdl_wait();
    if (threadIdx.x == 0 && c->err.bad_pos != ~0ull) c->bad_id = ids[c->err.bad_pos];
}

}  // namespace

void launch_lookup_async(Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots, uint8_t* out_oc,
                         BatchCounters* c, cudaStream_t st) {
    k_lookup_init<<<1, 32, 0, st>>>(c);
    run_lookup(t, ids, n, out_slots, out_oc, &c->err, st);
    launch_pdl(k_lookup_bad_id, 1, 32, st, ids, c);
    t.launches += 3;
}

void run_lookup_gather(const Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots,
                       uint8_t* out_oc, float* out_rows, BatchErr* err, cudaStream_t st) {
    const unsigned grid = grid_for((n + 31) / 32 * 32, 256, 148u * 16u);
    if (t.hole_free)
        k_lookup_gather<true><<<grid, 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, out_rows, err);
    else
        k_lookup_gather<false><<<grid, 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, out_rows, err);
}

void run_lookup(const Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots, uint8_t* out_oc,
                BatchErr* err, cudaStream_t st, DevBuf* ldefer, unsigned* dcount) {
    // long windows (max_probe >= 256, or the full-window scan of a table with holes): quad
    // line walk; else the per-thread sector walk (remap_fast.cu has the same rule)
    static const bool tag_env = [] {  // the tag walk for long windows (MPZCH_TAGS=0: off)
        const char* e = getenv("MPZCH_TAGS");
        return !(e && e[0] == '0' && e[1] == 0);
    }();
    if (t.P >= 256 && t.hole_free && t.dev.tag && tag_env) {
        k_lookup_tag<<<grid_for(4 * n, 256, 148u * 32u), 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
    } else if (t.P >= 256 || !t.hole_free) {
        const unsigned gl = grid_for(4 * ((n + 1) / 2), 256, 148u * 16u);
        // one position per quad, 6 blocks/SM (C3 lookups 7.15 -> 8.68 G/s vs 2 per quad)
        static const unsigned defer = [] {
            const char* e = getenv("MPZCH_LOOKUP_DEFER");
            return e ? (unsigned)atoi(e) : 4u;  // C3 synchronous lookups 9.7 -> 10.4 G/s (2: slower)
        }();
        // the list stores 32-bit positions: batches beyond 2^32 - 1 positions walk in one pass
        if (t.hole_free && ldefer && defer && n >= (1ull << 18) && n <= 0xffffffffull) {
            ldefer->reserve(n * 8);  // (position, offset) per handed-over walk
            uint32_t* dlist = ldefer->as<uint32_t>();
            MPZCH_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned), st));
            k_lookup_line<true, 1, false, true><<<grid_for(4 * n, 256, 148u * 24u), 256, 0, st>>>(
                t.dev, ids, n, out_slots, out_oc, err, dlist, dcount, defer);
            launch_pdl(k_lookup_line<true, 1, true, false>, 148u * 12u, 256u, st, t.dev, ids, n, out_slots, out_oc,
                       err, dlist, dcount, 0u);
        } else if (t.hole_free)
            k_lookup_line<true, 1><<<grid_for(4 * n, 256, 148u * 24u), 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
        else
            k_lookup_line<false, 2><<<gl, 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
    } else if (t.hole_free) {
        k_lookup<true><<<grid_for(n, 256), 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
    } else {
        k_lookup<false><<<grid_for(n, 256), 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
    }
}

}  // namespace mpzch_b200
