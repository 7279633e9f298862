// ordered_probe.cuh -- the reference's two-pass probe (proj/src/probe_core.cpp:69-134) as a
// warp-cooperative decision: 32 consecutive window slots per warp load (ld.global.cg, so the
// warp's own earlier writes are seen), __ballot_sync/__ffs for the first match / EMPTY /
// expired slot, a warp argmin (first strict minimum) for the LRU victim.  Works on tables with
// probe-window holes (pass 1 scans the whole window).  Used by the ordered path (one warp per
// shard, uniques in rank order) and by process_shard_batch (one warp, positions in order).
#pragma once

#include "common.cuh"

namespace mpzch_b200 {

// Decides (warp-uniform) the slot and outcome of `id` with home `h` (local) in the shard whose
// rows are [base, base + cap), against the current table state; writes nothing.
template <int MODE>
__device__ __forceinline__ void two_pass_probe(const TableDev& t, uint64_t base, uint64_t cap, uint64_t h,
                                               uint64_t id, uint64_t now, unsigned lane, uint64_t& gslot,
                                               uint8_t& oc) {
    const uint32_t P = t.P;
    // Pass 1: discovery (probe_core.cpp:78-86)
    bool exists = false;
    for (uint32_t c = 0; c < P; c += 32) {
        const uint32_t off = c + lane;
        bool hit = false;
        if (off < P) {
            uint64_t x = h + off;
            x = x >= cap ? x - cap : x;
            hit = ld_cg(t.ident + base + x) == id;
        }
        if (__ballot_sync(0xffffffffu, hit)) { exists = true; break; }
    }
    // Pass 2: update / insert / evict (probe_core.cpp:89-121)
    oc = kCollision;
    gslot = base + h;
    bool decided = false;
    uint64_t best_m = 0;
    uint32_t best_off = kNone32;
    for (uint32_t c = 0; c < P && !decided; c += 32) {
        const uint32_t off = c + lane;
        const bool valid = off < P;
        uint64_t g = 0, v = 0, m = 0;
        if (valid) {
            uint64_t x = h + off;
            x = x >= cap ? x - cap : x;
            g = base + x;
            v = ld_cg(t.ident + g);
            if (MODE != kModeDisabled) m = ld_cg(t.meta + g);
        }
        const bool is_match = valid && v == id;
        const bool is_empty = valid && v == kEmpty;
        const bool is_exp = valid && MODE == kModeTtl && !exists && !is_match && !is_empty &&
                            m < now;
        const unsigned stop = __ballot_sync(0xffffffffu, is_match || is_empty || is_exp);
        if (stop) {
            const int src = __ffs(stop) - 1;
            const uint64_t gs = __shfl_sync(0xffffffffu, g, src);
            const int kind = __shfl_sync(0xffffffffu, is_match ? 0 : (is_empty ? 1 : 2), src);
            gslot = gs;
            oc = kind == 0 ? kFound : (kind == 1 ? kInserted : kEvicted);
            decided = true;
        } else if (MODE == kModeLru && !exists) {
            // first strict minimum over the window, ties -> lowest offset
            uint64_t bm = valid ? m : ~0ull;
            uint32_t bo = valid ? off : kNone32;
            for (int o = 16; o; o >>= 1) {
                const uint64_t om = __shfl_xor_sync(0xffffffffu, bm, o);
                const uint32_t oo = __shfl_xor_sync(0xffffffffu, bo, o);
                if (om < bm || (om == bm && oo < bo)) { bm = om; bo = oo; }
            }
            if (bo != kNone32 && (best_off == kNone32 || bm < best_m)) {
                best_m = bm;
                best_off = bo;
            }
        }
    }
    if (!decided && MODE == kModeLru && best_off != kNone32) {
        uint64_t x = h + best_off;
        x = x >= cap ? x - cap : x;
        gslot = base + x;
        oc = kEvicted;  // LRU fallback, probe_core.cpp:125-129
    }
}

}  // namespace mpzch_b200
