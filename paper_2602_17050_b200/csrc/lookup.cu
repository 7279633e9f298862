// lookup.cu -- batched read-only lookup: one MpzchTable::lookup per position
// (proj/src/table.cpp:150-156 -> lookup_readonly proj/src/probe_core.cpp:32-43).
//
// lookup_readonly scans the whole P-slot window for the first match.  On a
// hole-free table an id never sits behind an EMPTY slot of its own
// window, so the scan stops at the first match or EMPTY and touches ~1.5
// sectors per hit at 0.8 load instead of P/4.  Tables with raw-imported state
// keep the full-window scan.
#include <cuda_runtime.h>

#include "common.cuh"
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

}  // namespace

void run_lookup(const Table& t, const uint64_t* ids, uint64_t n, uint64_t* out_slots, uint8_t* out_oc,
                BatchErr* err, cudaStream_t st) {
    if (t.hole_free)
        k_lookup<true><<<grid_for(n, 256), 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
    else
        k_lookup<false><<<grid_for(n, 256), 256, 0, st>>>(t.dev, ids, n, out_slots, out_oc, err);
}

}  // namespace mpzch_b200
