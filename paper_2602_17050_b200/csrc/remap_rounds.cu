// remap_rounds.cu -- exact parallel remap for the policies the claim path does not cover
// (LRU, TTL with several per-feature TTLs in one batch) on hole-free tables: the optimistic
// round algorithm of SURVEY Appendix A.4, run over the (id, feature) uniques that the ordered
// path's dedup produced (rank = unique index, first-occurrence order).
//
// One round, over the pending uniques, against the committed state C:
//   R1 k_tentative  each unique decides against C exactly as probe_core.cpp:69-134 would
//                   (single pass to the first match/EMPTY: hole-free), recording
//                   its read range [h, h+d] (identity and metadata words it looked at) and
//                   its write slot, and marks the write slot with its rank (64-bit atomicMin
//                   of an epoch-keyed word, so marks never need clearing).
//   R2 k_check      a unique is SUSPECT if a lower-rank pending unique marked a slot inside
//                   its read range (first order) ...
//   R3 k_mark_win   ... or a lower-rank suspect's whole window overlaps it (transitive):
//                   new suspects mark their windows and R2 runs again until no new suspect.
//   R4 k_commit     non-suspects are final (by induction on rank, A.4) and have pairwise
//                   disjoint write slots (every write slot lies in its writer's read range),
//                   so they commit in any order; the suspects are the next round's pending set.
// The lowest-rank pending unique is never suspect, so every round commits at least one; after
// kMaxRounds the remaining uniques go to the per-shard ordered kernel (always exact).
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

constexpr int kMaxRounds = 24;

__device__ __forceinline__ uint64_t mark_key(uint32_t epoch, uint32_t rank) {
    return ((uint64_t)(0xffffffffu - epoch) << 32) | rank;
}
__device__ __forceinline__ bool mark_is(uint64_t mk, uint32_t epoch) {
    return (uint32_t)(mk >> 32) == 0xffffffffu - epoch;
}

__device__ __forceinline__ uint64_t pick4r(uint32_t j, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    return j == 0 ? a : (j == 1 ? b : (j == 2 ? c : d));
}

template <int MODE>
__global__ void __launch_bounds__(256) k_tentative(TableDev t, const BatchCounters* ctr,
                                                   const uint64_t* __restrict__ ids,
                                                   const uint32_t* __restrict__ upos,
                                                   const uint32_t* __restrict__ ushard,
                                                   const uint32_t* __restrict__ pend, unsigned npend,
                                                   uint64_t now, uint32_t epoch,
                                                   uint64_t* __restrict__ td_slot,
                                                   uint8_t* __restrict__ td_oc,
                                                   uint32_t* __restrict__ td_d,
                                                   unsigned long long* mark, uint64_t mark_base) {
    if (batch_failed(&ctr->err)) return;
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < npend; x += gridDim.x * blockDim.x) {
        const uint32_t k = pend[x];
        const uint64_t id = ids[upos[k]];
        const ShardDev sd = t.shards[ushard[k]];
        const uint64_t cap = sd.cap.d, base = sd.offset, end = base + cap;
        const uint64_t h = home_of(id, sd, t.seed);
        uint64_t g = base + h;
        uint32_t off = 0;
        int kind = 0;  // 1 match, 2 empty
        uint32_t exp_off = kNone32;
        uint64_t exp_g = 0, best_m = 0, best_g = 0;
        bool have_best = false;
        while (off < t.P && !kind) {
            const uint64_t a4 = g & ~3ull;
            uint64_t i0, i1, i2, i3, m0 = 0, m1 = 0, m2 = 0, m3 = 0;
            ld_sector(t.ident + a4, i0, i1, i2, i3);
            if (MODE != kModeDisabled) ld_sector(t.meta + a4, m0, m1, m2, m3);
            do {
                const uint32_t j = (uint32_t)(g - a4);
                const uint64_t v = pick4r(j, i0, i1, i2, i3);
                if (v == id) { kind = 1; break; }
                if (v == kEmpty) { kind = 2; break; }
                if (MODE != kModeDisabled) {
                    const uint64_t m = pick4r(j, m0, m1, m2, m3);
                    if (MODE == kModeTtl && exp_off == kNone32 && m < now) { exp_off = off; exp_g = g; }
                    if (MODE == kModeLru && (!have_best || m < best_m)) { have_best = true; best_m = m; best_g = g; }
                }
                ++off;
                if (++g == end) g = base;
            } while (off < t.P && (g >> 2) == (a4 >> 2));
        }
        uint8_t oc = kCollision;
        uint64_t ws = base + h;
        if (kind == 1) { oc = kFound; ws = g; }
        else if (kind == 2) {
            if (MODE == kModeTtl && exp_off != kNone32) { oc = kEvicted; ws = exp_g; }
            else { oc = kInserted; ws = g; }
        } else if (MODE == kModeTtl && exp_off != kNone32) { oc = kEvicted; ws = exp_g; }
        else if (MODE == kModeLru && have_best) { oc = kEvicted; ws = best_g; }
        td_slot[k] = ws;
        td_oc[k] = oc;
        td_d[k] = kind ? off : t.P - 1;  // read range [h, h + d]
        atomicMin(mark + (ws - mark_base), (unsigned long long)mark_key(epoch, k));
    }
}

__device__ __forceinline__ uint64_t slot_of(const ShardDev& sd, uint64_t h, uint32_t off) {
    uint64_t x = h + off;
    if (x >= sd.cap.d) x -= sd.cap.d;
    return sd.offset + x;
}

// R2: first-order and transitive suspicion (marks of lower ranks inside my read range)
__global__ void __launch_bounds__(256) k_check(TableDev t, BatchCounters* ctr,
                                               const uint64_t* __restrict__ ids,
                                               const uint32_t* __restrict__ upos,
                                               const uint32_t* __restrict__ ushard,
                                               const uint32_t* __restrict__ pend, unsigned npend,
                                               uint32_t epoch, const uint32_t* __restrict__ td_d,
                                               uint8_t* susp, const unsigned long long* mark,
                                               uint64_t mark_base, uint32_t* newsusp) {
    if (batch_failed(&ctr->err)) return;
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < npend; x += gridDim.x * blockDim.x) {
        const uint32_t k = pend[x];
        if (susp[k]) continue;
        const uint64_t id = ids[upos[k]];
        const ShardDev sd = t.shards[ushard[k]];
        const uint64_t h = home_of(id, sd, t.seed);
        const uint32_t d = td_d[k];
        bool s = false;
        for (uint32_t off = 0; off <= d && !s; ++off) {
            const uint64_t mk = __ldcg(mark + (slot_of(sd, h, off) - mark_base));
            s = mark_is(mk, epoch) && (uint32_t)mk < k;
        }
        if (s) {
            susp[k] = 1;
            newsusp[atomicAdd(&ctr->r_new, 1u)] = k;
        }
    }
}

// R3: a suspect may end up writing anywhere in its window
__global__ void __launch_bounds__(256) k_mark_windows(TableDev t, const BatchCounters* ctr,
                                                      const uint64_t* __restrict__ ids,
                                                      const uint32_t* __restrict__ upos,
                                                      const uint32_t* __restrict__ ushard,
                                                      const uint32_t* __restrict__ list, unsigned cnt,
                                                      uint32_t epoch, unsigned long long* mark,
                                                      uint64_t mark_base) {
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < cnt; x += gridDim.x * blockDim.x) {
        const uint32_t k = list[x];
        const uint64_t id = ids[upos[k]];
        const ShardDev sd = t.shards[ushard[k]];
        const uint64_t h = home_of(id, sd, t.seed);
        for (uint32_t off = 0; off < t.P; ++off)
            atomicMin(mark + (slot_of(sd, h, off) - mark_base), (unsigned long long)mark_key(epoch, k));
    }
}

// R4: commit the non-suspects; collect the suspects as the next pending set
__global__ void __launch_bounds__(256) k_commit_round(TableDev t, BatchCounters* ctr,
                                                      const uint64_t* __restrict__ ids,
                                                      const uint32_t* __restrict__ upos,
                                                      const uint64_t* __restrict__ umeta,
                                                      const uint32_t* __restrict__ pend, unsigned npend,
                                                      uint8_t* susp, const uint64_t* __restrict__ td_slot,
                                                      const uint8_t* __restrict__ td_oc,
                                                      uint64_t gen_clock, uint64_t* __restrict__ uslot,
                                                      uint8_t* __restrict__ uoc,
                                                      uint64_t* __restrict__ reset_rows,
                                                      uint8_t* __restrict__ evflag,
                                                      uint64_t* __restrict__ evslot, uint32_t* next) {
    if (batch_failed(&ctr->err)) return;
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < npend; x += gridDim.x * blockDim.x) {
        const uint32_t k = pend[x];
        if (susp[k]) {
            susp[k] = 0;
            next[atomicAdd(&ctr->r_next, 1u)] = k;
            continue;
        }
        const uint64_t g = td_slot[k];
        const uint8_t oc = td_oc[k];
        if (oc == kInserted || oc == kEvicted) {
            t.ident[g] = ids[upos[k]];
            t.row_gen[g] = gen_clock;
        }
        t.meta[g] = umeta[k];
        if (oc == kEvicted) {
            if (t.dim) reset_rows[atomicAdd(&ctr->reset_count, 1u)] = g;
            evflag[k] = 1;
            evslot[k] = g;
            atomicAdd(&ctr->evicted_count, 1u);
        }
        uslot[k] = g;
        uoc[k] = oc;
    }
}

__global__ void k_iota(uint32_t* p, const BatchCounters* ctr) {
    const unsigned u = ctr->entry_count;
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < u; x += gridDim.x * blockDim.x) p[x] = x;
}

__global__ void k_flag_list(const uint32_t* list, unsigned cnt, uint8_t* flag) {
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < cnt; x += gridDim.x * blockDim.x)
        flag[list[x]] = 1;
}

__global__ void k_reset_round_ctr(BatchCounters* c) {
    c->r_new = 0;
    c->r_next = 0;
}

}  // namespace

// Runs the rounds for the uniques prepared by enqueue_ordered_batch (host-synchronous: the
// pending counts steer the loop).  Returns the number of uniques left for the ordered kernel,
// flagged in `todo`.
unsigned run_rounds(Table& t, const BatchArgs& a, cudaStream_t st, uint8_t* todo) {
    const Policy& p = *a.pol;
    MPZCH_CUDA(cudaMemcpyAsync(t.h_ctr, t.d_ctr, sizeof(BatchCounters), cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaStreamSynchronize(st));
    if (t.h_ctr->err.bad_pos != ~0ull || t.h_ctr->err.overflow || t.h_ctr->err.foreign_pos != ~0ull)
        return 0;  // invalid batch: nothing runs, the host reports the error
    const unsigned u = t.h_ctr->entry_count;
    if (!u) return 0;
    const uint64_t held = t.held_rows();
    if (t.r_mark.bytes < held * 8) {
        t.r_mark.reserve(held * 8);
        MPZCH_CUDA(cudaMemsetAsync(t.r_mark.p, 0xff, held * 8, st));
    }
    t.r_pend.reserve(u * 4ull);
    t.r_next.reserve(u * 4ull);
    t.r_new.reserve(u * 4ull);
    t.r_slot.reserve(u * 8ull);
    t.r_oc.reserve(u);
    t.r_d.reserve(u * 4ull);
    t.r_susp.reserve(u);
    MPZCH_CUDA(cudaMemsetAsync(t.r_susp.p, 0, u, st));
    unsigned long long* mark = t.r_mark.as<unsigned long long>();
    const uint64_t mb = t.row_lo;
    uint32_t* pend = t.r_pend.as<uint32_t>();
    uint32_t* next = t.r_next.as<uint32_t>();
    const unsigned B = 256;
    k_iota<<<grid_for(u, B), B, 0, st>>>(pend, t.d_ctr);
    ++t.launches;
    unsigned npend = u;
    const uint64_t* ids = a.ids;
    const uint32_t* upos = t.o_upos.as<uint32_t>();
    const uint32_t* ushard = t.o_ushard.as<uint32_t>();
    const uint64_t* umeta = t.o_umeta.as<uint64_t>();
    for (int round = 0; round < kMaxRounds && npend; ++round) {
        const uint32_t epoch = ++t.mark_epoch;
        const unsigned g = grid_for(npend, B);
        k_reset_round_ctr<<<1, 1, 0, st>>>(t.d_ctr);
#define MPZCH_TENT(MODE)                                                                           \
    k_tentative<MODE><<<g, B, 0, st>>>(t.dev, t.d_ctr, ids, upos, ushard, pend, npend, a.now, epoch, \
                                       t.r_slot.as<uint64_t>(), t.r_oc.as<uint8_t>(),              \
                                       t.r_d.as<uint32_t>(), mark, mb)
        if (p.mode == kModeTtl) MPZCH_TENT(kModeTtl);
        else if (p.mode == kModeLru) MPZCH_TENT(kModeLru);
        else MPZCH_TENT(kModeDisabled);
#undef MPZCH_TENT
        t.launches += 2;
        for (;;) {  // suspicion closure
            MPZCH_CUDA(cudaMemsetAsync(&t.d_ctr->r_new, 0, sizeof(unsigned), st));
            k_check<<<g, B, 0, st>>>(t.dev, t.d_ctr, ids, upos, ushard, pend, npend, epoch,
                                     t.r_d.as<uint32_t>(), t.r_susp.as<uint8_t>(), mark, mb,
                                     t.r_new.as<uint32_t>());
            ++t.launches;
            unsigned nn = 0;
            MPZCH_CUDA(cudaMemcpyAsync(&nn, &t.d_ctr->r_new, 4, cudaMemcpyDeviceToHost, st));
            MPZCH_CUDA(cudaStreamSynchronize(st));
            if (!nn) break;
            k_mark_windows<<<grid_for(nn, B), B, 0, st>>>(t.dev, t.d_ctr, ids, upos, ushard,
                                                          t.r_new.as<uint32_t>(), nn, epoch, mark, mb);
            ++t.launches;
        }
        k_commit_round<<<g, B, 0, st>>>(t.dev, t.d_ctr, ids, upos, umeta, pend, npend,
                                        t.r_susp.as<uint8_t>(), t.r_slot.as<uint64_t>(),
                                        t.r_oc.as<uint8_t>(), t.gen_clock, t.o_uslot.as<uint64_t>(),
                                        t.o_uoc.as<uint8_t>(), t.s_reset.as<uint64_t>(),
                                        t.s_evflag.as<uint8_t>(), t.s_evslot.as<uint64_t>(), next);
        ++t.launches;
        MPZCH_CUDA(cudaMemcpyAsync(&npend, &t.d_ctr->r_next, 4, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        std::swap(pend, next);
        ++t.last_rounds;
    }
    if (npend) {  // the remainder goes to the per-shard ordered kernel
        MPZCH_CUDA(cudaMemsetAsync(todo, 0, u, st));
        k_flag_list<<<grid_for(npend, B), B, 0, st>>>(pend, npend, todo);
        ++t.launches;
    }
    return npend;
}

}  // namespace mpzch_b200
