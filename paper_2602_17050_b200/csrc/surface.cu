// surface.cu -- the rest of the reference's MpzchTable / batch_engine surface (SURVEY 8b
// "Surface kept"), each on the device:
//
//   process_shard_batch   MpzchTable::process_shard_batch   proj/src/table.cpp:112-148
//   dedup                 mpzch::dedup                       proj/src/batch_engine.cpp:79-108,133-139
//   reset_row             MpzchTable::reset_row              proj/src/table.cpp:181-186
//   state_equals          MpzchTable::state_equals           proj/src/table.cpp:249-260
//   gather / row reads    MpzchTable::gather, row_identity   proj/src/table.cpp:158-163,188-191
#include <cuda_runtime.h>

#include "common.cuh"
#include "compact.cuh"
#include "ordered_probe.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

typedef unsigned __int128 u128;
constexpr u128 kKeyEmpty = ~(u128)0;

// ---- process_shard_batch: one warp runs the reference's per-shard loop (table.cpp:126-147) in
// position order -- no dedup, each position probes with its own metadata word.  Errors stop the
// loop where the reference's would: the reference hoists home_slot (which runs require_valid_id,
// probe_core.cpp:27-30) over each 256-position chunk before probing it (table.cpp:129-133), so an
// invalid id stops the batch at the START of its chunk; a bad metadata word stops it at its own
// position (check_metadata_input inside lookup_or_insert, probe_core.cpp:76-77), after the
// earlier positions took effect.  st[0] = positions that took effect (~0: all), st[1] = 1 invalid
// id / 2 metadata word, st[2] = the offending id.
constexpr uint64_t kShardChunk = 256;  // table.cpp:129

template <int MODE>
__global__ void __launch_bounds__(32) k_shard_batch(TableDev t, uint32_t shard, const uint64_t* __restrict__ ids,
                                                    const uint64_t* __restrict__ metas, uint64_t n,
                                                    uint64_t now, uint64_t gen_clock,
                                                    uint64_t* __restrict__ out_slots,
                                                    uint8_t* __restrict__ out_oc,
                                                    uint64_t* __restrict__ reset_rows,
                                                    unsigned* __restrict__ reset_count,
                                                    unsigned long long* __restrict__ st) {
    const unsigned lane = lane_id();
    const ShardDev sd = t.shards[shard];
    const uint64_t cap = sd.cap.d, base = sd.offset;
    // first invalid id (warp scan) -> the chunk the reference's home hoisting throws in
    uint64_t kb = n;
    for (uint64_t c = 0; c < n && kb == n; c += 32) {
        const bool bad_id = c + lane < n && (ids[c + lane] >> 63);
        const unsigned m = __ballot_sync(0xffffffffu, bad_id);
        if (m) kb = c + (uint64_t)(__ffs(m) - 1);
    }
    const uint64_t stop = kb == n ? n : kb / kShardChunk * kShardChunk;
    unsigned nreset = 0;
    bool failed = false;
    for (uint64_t k = 0; k < stop; ++k) {
        const uint64_t id = ids[k];
        const uint64_t meta_in = metas[k];
        if (MODE == kModeTtl ? meta_in <= now : meta_in != now) {  // check_metadata_input
            if (lane == 0) {
                st[0] = k;
                st[1] = 2ull;
                st[2] = id;
            }
            failed = true;
            break;
        }
        uint64_t gslot;
        uint8_t oc;
        two_pass_probe<MODE>(t, base, cap, home_of(id, sd, t.seed), id, now, lane, gslot, oc);
        if (lane == 0) {
            if (oc == kInserted || oc == kEvicted) {
                t.ident[gslot] = id;
                store_tag(t, gslot, id);
                t.row_gen[gslot] = gen_clock;  // touch_row, table.cpp:143-144
            }
            t.meta[gslot] = meta_in;
            if (oc == kEvicted && t.dim) reset_rows[nreset] = gslot;  // table.cpp:142
            out_slots[k] = gslot;
            out_oc[k] = oc;
        }
        nreset += (oc == kEvicted && t.dim) ? 1u : 0u;
        __syncwarp();
    }
    if (lane == 0) {
        if (!failed && kb < n) {
            st[0] = stop;
            st[1] = 1ull;
            st[2] = ids[kb];
        }
        *reset_count = nreset;
    }
}

// ---- dedup (batch_engine.cpp:79-108): first-occurrence uniques keyed on (id, feature) and the
// inverse map.  D1 validates and inserts 128-bit keys (first position by atomicMin), D2 flags
// first occurrences, the ordered compaction numbers them, D3 writes the inverse.
__global__ void __launch_bounds__(256) k_dd_hash(const uint64_t* __restrict__ ids, const uint32_t* __restrict__ feats,
                                                 uint64_t n, u128* key, unsigned* kmin,
                                                 uint32_t* __restrict__ posent, uint64_t mask,
                                                 unsigned long long* bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t id = ids[i];
        const uint32_t f = feats ? feats[i] : 0u;
        if (id >> 63) {
            atomicMin(bad, (unsigned long long)i);
            posent[i] = kNone32;
            continue;
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
        atomicMin(kmin + h, (unsigned)i);
        posent[i] = (uint32_t)h;
    }
}

__global__ void __launch_bounds__(256) k_dd_flags(uint64_t n, const uint32_t* __restrict__ posent,
                                                  const unsigned* __restrict__ kmin, const unsigned long long* bad,
                                                  uint8_t* __restrict__ flag) {
    const bool failed = *bad != ~0ull;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = posent[i];
        flag[i] = (!failed && e != kNone32 && kmin[e] == (unsigned)i) ? 1 : 0;
    }
}

struct EmitDedup {
    const uint64_t* ids;
    const uint32_t* feats;
    const uint32_t* posent;
    uint64_t* uids;
    uint32_t* ufeats;
    uint32_t* entu;
    __device__ void operator()(uint64_t i, unsigned k) const {
        uids[k] = ids[i];
        ufeats[k] = feats ? feats[i] : 0u;
        entu[posent[i]] = k;
    }
};

__global__ void __launch_bounds__(256) k_dd_inverse(uint64_t n, const uint32_t* __restrict__ posent,
                                                    const uint32_t* __restrict__ entu,
                                                    const unsigned long long* bad, uint32_t* __restrict__ inverse) {
    if (*bad != ~0ull) return;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        inverse[i] = entu[posent[i]];
}

// ---- state_equals (table.cpp:249-260): compare of two device arrays of 32-bit words
__global__ void __launch_bounds__(256) k_words_differ(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                      uint64_t n, unsigned* differ) {
    bool d = false;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        d |= __ldcs(a + i) != __ldcs(b + i);
    if (__any_sync(0xffffffffu, d) && lane_id() == 0) atomicExch(differ, 1u);
}

// ---- gather (embedding_store.cpp:95-103): one warp per requested row, 16-byte copies
__global__ void __launch_bounds__(256) k_gather_weights(TableDev t, const uint64_t* __restrict__ rows, uint64_t n,
                                                        float* __restrict__ out) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        copy_row_or_draw(t, rows[r], out + r * t.dim, lane);
    }
}

}  // namespace

void launch_shard_batch(Table& t, uint32_t shard, int mode, const uint64_t* ids, const uint64_t* metas,
                        uint64_t n, uint64_t now, uint64_t* out_slots, uint8_t* out_oc, uint64_t* reset_rows,
                        unsigned* reset_count, unsigned long long* st, cudaStream_t s) {
#define MPZCH_SB(M) \
    k_shard_batch<M><<<1, 32, 0, s>>>(t.dev, shard, ids, metas, n, now, t.gen_clock, out_slots, out_oc, reset_rows, \
                                      reset_count, st)
    if (mode == kModeTtl) MPZCH_SB(kModeTtl);
    else if (mode == kModeLru) MPZCH_SB(kModeLru);
    else MPZCH_SB(kModeDisabled);
#undef MPZCH_SB
    ++t.launches;
}

uint64_t run_dedup(const uint64_t* ids, const uint32_t* feats, uint64_t n, uint64_t* uids, uint32_t* ufeats,
                   uint32_t* inverse, uint64_t* bad_pos, cudaStream_t st) {
    uint64_t mask = 1024;
    while (mask < 2 * n) mask <<= 1;
    // scratch: keys (16 B) + kmin (4 B) per table entry; posent (4), flag (1) per position;
    // entu (4) per table entry; block counts; the bad word and the unique count
    const uint64_t nblk = (n + kCompactChunk - 1) / kCompactChunk + 1;
    const size_t bytes = mask * 16 + mask * 4 + mask * 4 + n * 4 + ((n + 31) & ~15ull) + nblk * 4 + 64;
    uint8_t* s = nullptr;
    MPZCH_CUDA(cudaMallocAsync((void**)&s, bytes, st));
    u128* key = reinterpret_cast<u128*>(s);
    unsigned* kmin = reinterpret_cast<unsigned*>(s + mask * 16);
    uint32_t* entu = reinterpret_cast<uint32_t*>(s + mask * 20);
    uint32_t* posent = reinterpret_cast<uint32_t*>(s + mask * 24);
    uint8_t* flag = s + mask * 24 + n * 4;
    unsigned* blk = reinterpret_cast<unsigned*>(flag + ((n + 31) & ~15ull));
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(blk + nblk + (nblk & 1));
    unsigned* count = reinterpret_cast<unsigned*>(bad + 1);
    MPZCH_CUDA(cudaMemsetAsync(key, 0xff, mask * 16, st));
    MPZCH_CUDA(cudaMemsetAsync(kmin, 0xff, mask * 4, st));
    MPZCH_CUDA(cudaMemsetAsync(flag, 0, (n + 31) & ~15ull, st));
    MPZCH_CUDA(cudaMemsetAsync(bad, 0xff, 8, st));
    MPZCH_CUDA(cudaMemsetAsync(count, 0, 4, st));
    const unsigned g = grid_for(n, 256);
    k_dd_hash<<<g, 256, 0, st>>>(ids, feats, n, key, kmin, posent, mask - 1, bad);
    k_dd_flags<<<g, 256, 0, st>>>(n, posent, kmin, bad, flag);
    uint64_t launches = 0;
    compact_flags(flag, n, blk, count, false, EmitDedup{ids, feats, posent, uids, ufeats, entu}, st, launches);
    k_dd_inverse<<<g, 256, 0, st>>>(n, posent, entu, bad, inverse);
    MPZCH_CUDA(cudaGetLastError());
    unsigned long long h_bad = 0;
    unsigned h_count = 0;
    MPZCH_CUDA(cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaMemcpyAsync(&h_count, count, 4, cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaFreeAsync(s, st));
    MPZCH_CUDA(cudaStreamSynchronize(st));
    *bad_pos = h_bad;
    return h_bad == ~0ull ? h_count : 0;
}

bool run_words_equal(const void* a, const void* b, uint64_t bytes, cudaStream_t st) {
    unsigned* d = nullptr;
    MPZCH_CUDA(cudaMallocAsync((void**)&d, 4, st));
    MPZCH_CUDA(cudaMemsetAsync(d, 0, 4, st));
    // bytes is a multiple of 4 (identity words, fp32 weights)
    k_words_differ<<<grid_for(bytes / 4, 256, 148u * 8u), 256, 0, st>>>((const uint32_t*)a, (const uint32_t*)b,
                                                                         bytes / 4, d);
    MPZCH_CUDA(cudaGetLastError());
    unsigned h = 0;
    MPZCH_CUDA(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaFreeAsync(d, st));
    MPZCH_CUDA(cudaStreamSynchronize(st));
    return h == 0;
}

void run_gather_weights(const Table& t, const uint64_t* rows, uint64_t n, float* out, cudaStream_t st) {
    if (!n) return;
    k_gather_weights<<<grid_for(n * 32, 256, 148u * 16u), 256, 0, st>>>(t.dev, rows, n, out);
}

}  // namespace mpzch_b200
