// remap_rounds.cu -- exact parallel remap for the policies the claim path does not cover
// (LRU, TTL with several per-feature TTLs in one batch) on hole-free tables: the optimistic
// round algorithm of SURVEY Appendix A.4, run over the (id, feature) uniques that the ordered
// path's dedup produced (rank = unique index, first-occurrence order).
//
// One round, over the pending uniques, against the committed state C:
//   R1 k_tentative  each unique k decides against C exactly as probe_core.cpp:69-134 would
//                   (single pass to the first match/EMPTY: hole-free), recording its
//                   read range R_k = [h, h+d] and its write slot w_k in R_k, and marks w_k with
//                   its rank: ident-changing writes (Inserted/Evicted) in mark_id, metadata-only
//                   writes (Found refresh, Collision's home touch) in mark_any (64-bit atomicMin
//                   of epoch-keyed words, so marks never need clearing).
//   R2 k_check      k is SUSPECT if a lower rank left a mark (either array) on w_k, or -- LRU
//                   victim whose metadata is not older than `now` -- any lower-rank mark in R_k.
//                   A lower-rank write at x != w_k changes no decision of k against C:
//                   * a unique with k's own id decides exactly as k does against the same C, so
//                     it writes w_k (or, as a suspect, marks a window holding w_k);
//                   * any other id written at x is not k's, so k's discovery pass is unchanged,
//                     and no write empties a slot;
//                   * Found and Inserted-at-EMPTY read no metadata; under TTL a write only makes
//                     x live (refresh, or an expired x replaced -- then x lies past k's first
//                     expired slot w_k, or k found its id first); an LRU victim with metadata
//                     older than `now` is not beaten or tied by x raised to `now`.
//   R3 mark_window  a suspect may end up writing anywhere in its window: a new suspect marks its
//                   whole window at once (so cascades spread inside a pass) in mark_win, one
//                   word per 16-slot block (9 atomics for a 128-slot window, not 128), and R2
//                   repeats until a pass finds no new suspect (the fixpoint).  After kClosureMax
//                   passes the last pass's suspects are left unmarked; with m = the lowest of
//                   their ranks, every non-suspect of rank < m is final (every suspect below it
//                   was marked before that pass).
//   R4 k_commit     non-suspects of rank < m are final (induction on rank, A.4) and have pairwise
//                   distinct write slots (own-slot rule), so they commit in any order; the rest
//                   is the next round's pending set.  A committed k never lies in the window of a
//                   lower-rank unique that stays pending (those are marked suspects), so later
//                   rounds never read what k wrote out of order.
// The lowest-rank pending unique is never suspect, so every round commits at least one.
//
// All rounds run in ONE persistent cooperative kernel (grid-wide barriers between the phases,
// the closure iterated to its fixpoint), so the path needs no host round trip: after kMaxRounds
// the remaining uniques are flagged for the per-shard ordered kernel (always exact), which the
// host enqueues unconditionally and which returns at once when nothing is left.  Data other
// blocks wrote inside the kernel is read through L2 (ld.cg), never the .nc/L1 path.  The mark
// arrays alias slots modulo their size: an alias only adds suspicion.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace cg = cooperative_groups;

namespace {

constexpr int kMaxRounds = 32;
constexpr int kClosureMax = 16;  // R2/R3 passes before the closure falls back to the rank bound

__device__ __forceinline__ uint64_t mark_key(uint32_t epoch, uint32_t rank) {
    return ((uint64_t)(0xffffffffu - epoch) << 32) | rank;
}
// rank of this epoch's mark, or ~0 when the word holds an older epoch's mark
__device__ __forceinline__ uint32_t mark_rank(uint64_t mk, uint32_t epoch) {
    return (uint32_t)(mk >> 32) == 0xffffffffu - epoch ? (uint32_t)mk : kNone32;
}

__device__ __forceinline__ uint64_t pick4r(uint32_t j, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return j == 0 ? a : (j == 1 ? b : (j == 2 ? c : d));
}

__device__ __forceinline__ uint64_t slot_of(const ShardDev& sd, uint64_t h, uint32_t off) {
    uint64_t x = h + off;
    if (x >= sd.cap.d) x -= sd.cap.d;
    return sd.offset + x;
}

__device__ __forceinline__ unsigned ldcg_u32(const unsigned* p) { return __ldcg(p); }
__device__ __forceinline__ uint8_t ldcg_u8(const uint8_t* p) {
    return (uint8_t)__ldcg(reinterpret_cast<const unsigned char*>(p));
}
__device__ __forceinline__ void stcg_u8(uint8_t* p, uint8_t v) {
    __stcg(reinterpret_cast<unsigned char*>(p), (unsigned char)v);
}

struct RoundsArgs {
    TableDev t;
    BatchCounters* ctr;
    const uint64_t* ids;
    const uint32_t* upos;
    const uint32_t* ushard;
    const uint64_t* umeta;
    uint64_t now, gen_clock;
    uint32_t epoch0;
    uint32_t* pend[2];
    uint64_t* td_slot;
    uint8_t* td_oc;
    uint32_t* td_d;
    uint64_t* pc;   // per pending entry x (same thread every pass): k | mark_win word << 32 |
                    // wide << 62 | suspect << 63, written by the round's first closure pass
    uint8_t* todo;
    unsigned long long* mark_any;  // metadata-only writes
    unsigned long long* mark_id;   // ident-changing writes
    unsigned long long* mark_win;  // suspect windows, one word per 16-slot block of mark_id
    uint64_t mark_base, mark_mask;
    int closure_max;
    uint64_t* uslot;
    uint8_t* uoc;
    uint64_t* reset_rows;
    uint8_t* evflag;
    uint64_t* evslot;
    __device__ __forceinline__ uint64_t mi(uint64_t g) const { return (g - mark_base) & mark_mask; }
};

// R1.  The walk reads a whole 128-byte line (16 slots) of identities -- and of metadata
// words outside Disabled -- per round trip: four independent 32-byte loads issued together.
// LRU windows are full by the time this path runs, so a miss walks all P slots: 8 round trips
// at P = 128 instead of 32 sector by sector.
template <int MODE>
__device__ __forceinline__ void tentative(const RoundsArgs& r, uint32_t k, uint32_t epoch) {
    const TableDev& t = r.t;
    const uint64_t id = r.ids[r.upos[k]];
    const ShardDev sd = t.shards[r.ushard[k]];
    const uint64_t cap = sd.cap.d, base = sd.offset, end = base + cap;
    const uint64_t h = home_of(id, sd, t.seed);
    uint64_t g = base + h;
    uint32_t off = 0;
    int kind = 0;  // 1 match, 2 empty
    uint32_t exp_off = kNone32;
    uint64_t exp_g = 0, best_m = 0, best_g = 0;
    bool have_best = false;
    while (off < t.P && !kind) {
        const uint64_t L = g & ~15ull;
        const unsigned s0 = (unsigned)(g - L);
        uint64_t c = 16 - s0;
        if (end - g < c) c = end - g;
        if (t.P - off < c) c = t.P - off;
        uint64_t iw[16], mw[MODE != kModeDisabled ? 16 : 1];
#pragma unroll
        for (int q = 0; q < 4; ++q) ld_sector_cg(t.ident + L + 4 * q, iw[4 * q], iw[4 * q + 1], iw[4 * q + 2], iw[4 * q + 3]);
        if (MODE != kModeDisabled) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ld_sector_cg(t.meta + L + 4 * q, mw[4 * q], mw[4 * q + 1], mw[4 * q + 2], mw[4 * q + 3]);
        }
        unsigned stop = 16;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            if (stop != 16 || q < (int)s0 || q >= (int)(s0 + c)) continue;
            const uint64_t v = iw[q];
            if (v == id) { kind = 1; stop = q; continue; }
            if (v == kEmpty) { kind = 2; stop = q; continue; }
            if (MODE != kModeDisabled) {
                const uint64_t m = mw[q];
                if (MODE == kModeTtl && exp_off == kNone32 && m < r.now) { exp_off = off + (q - s0); exp_g = L + q; }
                if (MODE == kModeLru && (!have_best || m < best_m)) { have_best = true; best_m = m; best_g = L + q; }
            }
        }
        if (stop != 16) {
            off += stop - s0;
            g = L + stop;
        } else {
            off += (uint32_t)c;
            g += c;
            if (g == end) g = base;
        }
    }
    uint8_t oc = kCollision;
    uint64_t ws = base + h;
    if (kind == 1) { oc = kFound; ws = g; }
    else if (kind == 2) {
        if (MODE == kModeTtl && exp_off != kNone32) { oc = kEvicted; ws = exp_g; }
        else { oc = kInserted; ws = g; }
    } else if (MODE == kModeTtl && exp_off != kNone32) { oc = kEvicted; ws = exp_g; }
    else if (MODE == kModeLru && have_best) { oc = kEvicted; ws = best_g; }
    __stcg(r.td_slot + k, ws);
    stcg_u8(r.td_oc + k, oc);
    // read range [h, h + d]; bit 31: the decision reads every metadata word of the range (an
    // LRU victim whose metadata is not older than `now` -- slots raised to `now` by lower ranks
    // would tie it)
    const bool wide = MODE == kModeLru && oc == kEvicted && best_m >= r.now;
    __stcg(r.td_d + k, (kind ? off : t.P - 1) | (wide ? 1u << 31 : 0u));
    const bool ident_write = oc == kInserted || oc == kEvicted;
    atomicMin((ident_write ? r.mark_id : r.mark_any) + r.mi(ws), (unsigned long long)mark_key(epoch, k));
}

// R2 (rule in the header).  The read range's mark words are read 16 at a time (four
// 32-byte loads of one 128-byte block of the mark array per round trip).
template <int MODE>
__device__ __forceinline__ bool suspect(const RoundsArgs& r, uint32_t k, uint32_t epoch, uint32_t& win,
                                        bool& wide) {
    const uint32_t dw = __ldcg(r.td_d + k);
    const uint64_t w = __ldcg(r.td_slot + k);
    wide = dw >> 31;
    if (!wide) {  // the write slot decides (header): one word in each mark array
        const uint64_t i = r.mi(w);
        win = (uint32_t)(i >> 4);
        return mark_rank(__ldcg(r.mark_id + i), epoch) < k || mark_rank(__ldcg(r.mark_any + i), epoch) < k ||
               mark_rank(__ldcg(r.mark_win + (i >> 4)), epoch) < k;
    }
    win = 0;
    const uint64_t id = r.ids[r.upos[k]];
    const ShardDev sd = r.t.shards[r.ushard[k]];
    const uint64_t h = home_of(id, sd, r.t.seed);
    const uint32_t d = dw & 0x7fffffffu;
    const bool meta_dep = true;  // LRU victim tied with `now`: any mark in the range
    const uint64_t end = sd.offset + sd.cap.d;
    uint64_t g = slot_of(sd, h, 0);
    uint32_t off = 0;
    while (off <= d) {
        const uint64_t i = r.mi(g), I = i & ~15ull;
        const unsigned s0 = (unsigned)(i - I);
        uint64_t c = 16 - s0;
        if (end - g < c) c = end - g;
        if ((uint64_t)(d + 1 - off) < c) c = d + 1 - off;
        if (mark_rank(__ldcg(r.mark_win + (I >> 4)), epoch) < k) return true;  // a suspect's window
        uint64_t mid[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) ld_sector_cg((const uint64_t*)(r.mark_id + I + 4 * q), mid[4 * q], mid[4 * q + 1], mid[4 * q + 2], mid[4 * q + 3]);
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (q >= (int)s0 && q < (int)(s0 + c) && mark_rank(mid[q], epoch) < k) return true;
        if (meta_dep) {
            uint64_t man[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) ld_sector_cg((const uint64_t*)(r.mark_any + I + 4 * q), man[4 * q], man[4 * q + 1], man[4 * q + 2], man[4 * q + 3]);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (q >= (int)s0 && q < (int)(s0 + c) && mark_rank(man[q], epoch) < k) return true;
        } else if (w >= g && w < g + c) {  // the write slot lies in this block
            if (mark_rank(__ldcg(r.mark_any + i + (w - g)), epoch) < k) return true;
        }
        off += (uint32_t)c;
        g += c;
        if (g == end) g = sd.offset;
    }
    return false;
}

// R3
__device__ __forceinline__ void mark_window(const RoundsArgs& r, uint32_t k, uint32_t epoch) {
    const uint64_t id = r.ids[r.upos[k]];
    const ShardDev sd = r.t.shards[r.ushard[k]];
    const uint64_t h = home_of(id, sd, r.t.seed);
    const uint64_t end = sd.offset + sd.cap.d;
    for (uint32_t off = 0; off < r.t.P;) {  // one atomic per 16-slot block the window touches
        const uint64_t g = slot_of(sd, h, off);
        const uint64_t i = r.mi(g);
        atomicMin(r.mark_win + (i >> 4), (unsigned long long)mark_key(epoch, k));
        uint64_t step = 16 - (i & 15);
        if (end - g < step) step = end - g;  // the window wraps inside the shard
        off += (uint32_t)step;
    }
}

// R4
__device__ __forceinline__ void commit(const RoundsArgs& r, uint32_t k) {
    const TableDev& t = r.t;
    const uint64_t g = __ldcg(r.td_slot + k);
    const uint8_t oc = ldcg_u8(r.td_oc + k);
    if (oc == kInserted || oc == kEvicted) {
        __stcg(t.ident + g, r.ids[r.upos[k]]);
        store_tag(t, g, r.ids[r.upos[k]]);
        t.row_gen[g] = r.gen_clock;
    }
    __stcg(t.meta + g, r.umeta[k]);
    // the evicted uniques of the warp's active lanes: one counter update per warp (a Zipf LRU
    // batch evicts ~166 K rows; same-address atomics serialise)
    const unsigned am = __activemask();
    const unsigned em = __ballot_sync(am, oc == kEvicted);
    if (em) {
        const unsigned leader = __ffs(em) - 1;
        const unsigned below = __popc(em & ((1u << lane_id()) - 1));
        unsigned r0 = 0;
        if (lane_id() == leader) {
            if (t.dim) r0 = atomicAdd(&r.ctr->reset_count, (unsigned)__popc(em));
            atomicAdd(&r.ctr->evicted_count, (unsigned)__popc(em));
        }
        r0 = __shfl_sync(am, r0, leader);
        if (oc == kEvicted) {
            if (t.dim) r.reset_rows[r0 + below] = g;
            r.evflag[k] = 1;
            r.evslot[k] = g;
        }
    }
    r.uslot[k] = g;
    r.uoc[k] = oc;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_rounds(RoundsArgs r) {
    cg::grid_group grid = cg::this_grid();
    BatchCounters* ctr = r.ctr;
    if (batch_failed(&ctr->err)) return;  // uniform: the error words are final before this kernel
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const unsigned u = ctr->entry_count;
    for (unsigned x = tid; x < u; x += nth) {
        __stcg(r.pend[0] + x, x);
        r.todo[x] = 0;
    }
    if (tid == 0) {
        ctr->r_cnt[0] = u;
        ctr->r_cnt[1] = 0;
    }
    grid.sync();
    int round = 0;
    unsigned npend = u;
    for (; round < kMaxRounds; ++round) {
        const int par = round & 1;
        npend = ldcg_u32(&ctr->r_cnt[par]);
        if (!npend) break;
        const uint32_t epoch = r.epoch0 + round;
        const uint32_t* pend = r.pend[par];
        if (tid == 0) {  // closure pass c uses slot c % 3 (reset two passes ahead: see below)
            ctr->r_newc[0] = ctr->r_newc[1] = 0;
            ctr->r_minrank = kNone32;
        }
        for (unsigned x = tid; x < npend; x += nth) tentative<MODE>(r, __ldcg(pend + x), epoch);
        grid.sync();
        if (tid == 0) ctr->r_cnt[par ^ 1] = 0;
        for (int c = 0;; ++c) {  // suspicion closure: check and mark in one pass
            const bool last = c == r.closure_max;
            // slot (c + 1) % 3 was last read (the break test) right after pass c - 2's barrier,
            // which every thread has passed, so pass c may reset it for pass c + 1 (resetting it
            // after this pass's barrier would race with pass c + 1's first updates)
            if (tid == 0 && c > 0) ctr->r_newc[(c + 1) % 3] = 0;
            for (unsigned x = tid; x < npend; x += nth) {
                uint32_t k;
                if (c == 0) {  // the full check (R2), its outcome and mark word cached for later passes
                    k = __ldcg(pend + x);
                    uint32_t win;
                    bool wide;
                    const bool s = suspect<MODE>(r, k, epoch, win, wide);
                    __stcg(r.pc + x, (uint64_t)k | ((uint64_t)win << 32) | ((uint64_t)wide << 62) |
                                         ((uint64_t)s << 63));
                    if (!s) continue;
                } else {
                    // later passes: only suspects' window marks were added since the first pass,
                    // so a non-wide unique re-reads the one window word over its write slot
                    const uint64_t cw = __ldcg(r.pc + x);
                    if (cw >> 63) continue;
                    k = (uint32_t)cw;
                    bool s;
                    if ((cw >> 62) & 1) {
                        uint32_t win;
                        bool wide;
                        s = suspect<MODE>(r, k, epoch, win, wide);
                    } else {
                        s = mark_rank(__ldcg(r.mark_win + ((cw >> 32) & 0x3fffffffu)), epoch) < k;
                    }
                    if (!s) continue;
                    __stcg(r.pc + x, cw | (1ull << 63));
                }
                if (last) {
                    atomicMin(&ctr->r_minrank, k);
                } else {
                    mark_window(r, k, epoch);
                    // (hundreds of thousands of new suspects per batch under Zipf LRU: one
                    // counter update per warp, not per suspect -- same-address atomics serialise)
                    const unsigned am = __activemask();
                    if (lane_id() == __ffs(am) - 1) {
                        atomicAdd(&ctr->r_newc[c % 3], (unsigned)__popc(am));
                        atomicAdd(&ctr->r_marked, (unsigned)__popc(am));
                    }
                }
            }
            grid.sync();
            if (tid == 0) ++ctr->r_iters;
            if (last || !ldcg_u32(&ctr->r_newc[c % 3])) break;
        }
        const uint32_t bound = ldcg_u32(&ctr->r_minrank);
        uint32_t* next = r.pend[par ^ 1];
        for (unsigned x = tid; x < npend; x += nth) {
            const uint64_t cw = __ldcg(r.pc + x);
            const uint32_t k = (uint32_t)cw;
            if ((cw >> 63) || k > bound) {
                // warp-aggregated append to the next round's pending list (its order is free)
                const unsigned am = __activemask();
                const unsigned leader = __ffs(am) - 1;
                unsigned b0 = 0;
                if (lane_id() == leader) b0 = atomicAdd(&ctr->r_cnt[par ^ 1], (unsigned)__popc(am));
                b0 = __shfl_sync(am, b0, leader);
                __stcg(next + b0 + __popc(am & ((1u << lane_id()) - 1)), k);
            } else {
                commit(r, k);
            }
        }
        grid.sync();
    }
    if (round == kMaxRounds) npend = ldcg_u32(&ctr->r_cnt[round & 1]);
    else npend = 0;
    const uint32_t* left = r.pend[round & 1];
    for (unsigned x = tid; x < npend; x += nth) r.todo[__ldcg(left + x)] = 1;
    if (tid == 0) {
        ctr->r_left = npend;
        ctr->r_rounds = round + (npend ? 1 : 0);
    }
}

template <int MODE>
int rounds_grid(uint64_t n) {
    static int max_blocks = 0;
    if (!max_blocks) {
        int dev = 0, sms = 0, per = 0;
        MPZCH_CUDA(cudaGetDevice(&dev));
        MPZCH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MPZCH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rounds<MODE>, 256, 0));
        max_blocks = sms * std::max(per, 1);
    }
    const uint64_t want = std::max<uint64_t>(148, (n + 255) / 256);
    return (int)std::min<uint64_t>(want, (uint64_t)max_blocks);
}

}  // namespace

void preload_rounds_kernels() {
    preload_kernel((const void*)k_rounds<kModeDisabled>);
    preload_kernel((const void*)k_rounds<kModeTtl>);
    preload_kernel((const void*)k_rounds<kModeLru>);
}

// The rounds path's scratch: epoch-keyed mark arrays over the held rows (<= 2^27 words each)
// and per-unique lists for n uniques.
void ensure_rounds_scratch(Table& t, uint64_t n, cudaStream_t st) {
    const uint64_t held = t.held_rows();
    uint64_t msize = 1024;
    while (msize < held && msize < (1ull << 27)) msize <<= 1;
    if (t.r_mark_mask != msize - 1 || t.mark_epoch > 0xffff0000u) {
        t.r_mark_any.reserve(msize * 8);
        t.r_mark_id.reserve(msize * 8);
        t.r_mark_win.reserve(msize / 2);
        MPZCH_CUDA(cudaMemsetAsync(t.r_mark_win.p, 0xff, msize / 2, st));
        MPZCH_CUDA(cudaMemsetAsync(t.r_mark_any.p, 0xff, msize * 8, st));
        MPZCH_CUDA(cudaMemsetAsync(t.r_mark_id.p, 0xff, msize * 8, st));
        t.r_mark_mask = msize - 1;
        t.mark_epoch = 0;
    }
    t.r_pend.reserve(n * 4);
    t.r_next.reserve(n * 4);
    t.r_slot.reserve(n * 8);
    t.r_oc.reserve(n);
    t.r_d.reserve(n * 4);
    t.r_susp.reserve(n * 8);
    t.o_todo.reserve(n);
}

// Enqueues the rounds kernel for the uniques prepared by enqueue_ordered_batch (no host sync).
// The uniques it leaves (if any) are flagged in `todo` and counted in BatchCounters::r_left.
void enqueue_rounds(Table& t, const BatchArgs& a, cudaStream_t st, uint8_t* todo) {
    const Policy& p = *a.pol;
    const uint64_t n = a.n;
    ensure_rounds_scratch(t, n, st);
    RoundsArgs r;
    r.t = t.dev;
    r.ctr = t.d_ctr;
    r.ids = a.ids;
    r.upos = t.o_upos.as<uint32_t>();
    r.ushard = t.o_ushard.as<uint32_t>();
    r.umeta = t.o_umeta.as<uint64_t>();
    r.now = a.now;
    r.gen_clock = t.gen_clock;
    r.epoch0 = t.mark_epoch + 1;
    t.mark_epoch += kMaxRounds;
    r.pend[0] = t.r_pend.as<uint32_t>();
    r.pend[1] = t.r_next.as<uint32_t>();
    r.td_slot = t.r_slot.as<uint64_t>();
    r.td_oc = t.r_oc.as<uint8_t>();
    r.td_d = t.r_d.as<uint32_t>();
    r.pc = t.r_susp.as<uint64_t>();
    r.todo = todo;
    r.mark_any = t.r_mark_any.as<unsigned long long>();
    r.mark_id = t.r_mark_id.as<unsigned long long>();
    r.mark_win = t.r_mark_win.as<unsigned long long>();
    static const int closure_max = [] {
        const char* e = getenv("MPZCH_CLOSURE_MAX");
        return e ? atoi(e) : kClosureMax;
    }();
    r.closure_max = closure_max;
    r.mark_base = t.row_lo;
    r.mark_mask = t.r_mark_mask;
    r.uslot = t.o_uslot.as<uint64_t>();
    r.uoc = t.o_uoc.as<uint8_t>();
    r.reset_rows = t.s_reset.as<uint64_t>();
    r.evflag = t.s_evflag.as<uint8_t>();
    r.evslot = t.s_evslot.as<uint64_t>();
    void* args[] = {&r};
    const dim3 block(256);
#define MPZCH_ROUNDS(MODE) \
    MPZCH_CUDA(cudaLaunchCooperativeKernel((void*)k_rounds<MODE>, dim3(rounds_grid<MODE>(n)), block, args, 0, st))
    if (p.mode == kModeTtl) MPZCH_ROUNDS(kModeTtl);
    else if (p.mode == kModeLru) MPZCH_ROUNDS(kModeLru);
    else MPZCH_ROUNDS(kModeDisabled);
#undef MPZCH_ROUNDS
    ++t.launches;
}

}  // namespace mpzch_b200
