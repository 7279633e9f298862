// route.cu -- routing of a rank's positions to the ranks that own their logical shards
// (row-sharded mode).  shard_of (proj/src/shard_router.cpp:42-46) decides the
// shard; a host table maps shards to parts (ranks).  The permutation is STABLE: within a
// part, positions keep their input order, so after the all-to-all the owner sees every
// source's positions in global first-occurrence order (the reference's dedup order,
// proj/src/batch_engine.cpp:100-106) without any sort.
//
//   k_route_count  one warp per 1024-position chunk: per-part counts (ballot + popc)
//   k_route_scan   one block: part-major exclusive scan of the chunk counts
//   k_route_write  one warp per chunk: ballot ranks -> perm[offset + rank] = position
//
// Peer-memory transport (replaces the NCCL all-to-all pair of the row-sharded mode):
//   k_route_scatter  the write phase of the same partition, but every position's id, feature
//                    and source index are stored straight into the OWNER's receive buffer
//                    (P2P / IPC-mapped peer memory over NVLink) at this rank's offset there --
//                    partition and transfer in one kernel, no staging copy, no collective;
//   k_return_scatter the owner stores every received position's (slot, outcome, first-evicted
//                    mark) straight into the SOURCE rank's result buffers at the source
//                    position -- the reverse transfer and the inverse permutation in one kernel.
#include <cuda_runtime.h>

#include "common.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

constexpr unsigned kChunk = 1024;
constexpr unsigned kMaxParts = 64;

__device__ __forceinline__ uint32_t part_of(uint64_t id, const TableDev& t, const uint8_t* s2p) {
    return s2p[shard_of(id, t)];
}

__global__ void __launch_bounds__(256) k_route_count(TableDev t, const uint64_t* __restrict__ ids,
                                                     uint64_t n, const uint8_t* __restrict__ s2p,
                                                     uint32_t parts, unsigned* __restrict__ cnt,
                                                     uint64_t nchunks, unsigned long long* bad) {
    pdl_wait();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = lane_id();
    if (warp >= nchunks) return;
    unsigned c = 0;  // lane p accumulates part p (parts <= 32 per lane slot, see below)
    unsigned c2 = 0; // parts 32..63
    unsigned long long first_bad = ~0ull;  // (bad != null: the validation pass, fused)
    for (uint64_t i0 = warp * kChunk; i0 < (warp + 1) * kChunk && i0 < n; i0 += 32) {
        const uint64_t i = i0 + lane;
        const uint64_t id = i < n ? ids[i] : 0;
        if (bad && (id >> 63) && first_bad == ~0ull) first_bad = i;
        const uint32_t p = i < n ? part_of(id, t, s2p) : kNone32;
        for (uint32_t q = 0; q < parts; ++q) {
            const unsigned m = __ballot_sync(0xffffffffu, p == q);
            if (lane == (q & 31)) (q < 32 ? c : c2) += __popc(m);
        }
    }
    if (lane < parts) cnt[(uint64_t)lane * nchunks + warp] = c;
    if (lane + 32 < parts) cnt[(uint64_t)(lane + 32) * nchunks + warp] = c2;
    if (bad) {
        for (int o = 16; o; o >>= 1) first_bad = min(first_bad, __shfl_xor_sync(0xffffffffu, first_bad, o));
        if (lane == 0 && first_bad != ~0ull) atomicMin(bad, first_bad);
    }
}

__global__ void __launch_bounds__(256) k_route_write(TableDev t, const uint64_t* __restrict__ ids,
                                                     uint64_t n, const uint8_t* __restrict__ s2p,
                                                     uint32_t parts, const unsigned* __restrict__ off,
                                                     uint64_t nchunks, uint32_t* __restrict__ perm) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = lane_id();
    if (warp >= nchunks) return;
    unsigned base = lane < parts ? off[(uint64_t)lane * nchunks + warp] : 0;
    unsigned base2 = lane + 32 < parts ? off[(uint64_t)(lane + 32) * nchunks + warp] : 0;
    for (uint64_t i0 = warp * kChunk; i0 < (warp + 1) * kChunk && i0 < n; i0 += 32) {
        const uint64_t i = i0 + lane;
        const uint32_t p = i < n ? part_of(ids[i], t, s2p) : kNone32;
        for (uint32_t q = 0; q < parts; ++q) {
            const unsigned m = __ballot_sync(0xffffffffu, p == q);
            if (!m) continue;
            const unsigned b = __shfl_sync(0xffffffffu, q < 32 ? base : base2, q & 31);
            if (p == q) perm[b + __popc(m & ((1u << lane) - 1))] = (uint32_t)i;
            if (lane == (q & 31)) (q < 32 ? base : base2) += __popc(m);
        }
    }
}

// Destinations by value (kernel parameters): one entry per part.
struct PeerDst {
    uint64_t ids[kMaxParts], feats[kMaxParts], src[kMaxParts], off[kMaxParts];
    const uint64_t* dev_off;  // row-sharded device protocol: offsets on the device (or null)
    const uint64_t* gate;     // nonzero word: the batch failed, store nothing (or null)
};

__global__ void __launch_bounds__(256) k_route_scatter(TableDev t, const uint64_t* __restrict__ ids,
                                                       const uint32_t* __restrict__ feats, uint64_t n,
                                                       const uint8_t* __restrict__ s2p, uint32_t parts,
                                                       const unsigned* __restrict__ off, uint64_t nchunks,
                                                       const PeerDst d) {
    pdl_wait();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = lane_id();
    if (warp >= nchunks) return;
    if (d.gate && *(volatile const uint64_t*)d.gate) return;
    // index inside the owner's buffer: this rank's offset there + the position's rank among
    // this rank's positions of that part (the part-major scan minus the part's start)
    uint64_t base = 0, base2 = 0;
    if (lane < parts)
        base = (d.dev_off ? d.dev_off[lane] : d.off[lane]) + off[(uint64_t)lane * nchunks + warp] -
               off[(uint64_t)lane * nchunks];
    if (lane + 32 < parts)
        base2 = (d.dev_off ? d.dev_off[lane + 32] : d.off[lane + 32]) +
                off[(uint64_t)(lane + 32) * nchunks + warp] - off[(uint64_t)(lane + 32) * nchunks];
    for (uint64_t i0 = warp * kChunk; i0 < (warp + 1) * kChunk && i0 < n; i0 += 32) {
        const uint64_t i = i0 + lane;
        const uint64_t id = i < n ? ids[i] : 0;
        const uint32_t p = i < n ? part_of(id, t, s2p) : kNone32;
        for (uint32_t q = 0; q < parts; ++q) {
            const unsigned m = __ballot_sync(0xffffffffu, p == q);
            if (!m) continue;
            const uint64_t b = __shfl_sync(0xffffffffu, q < 32 ? base : base2, q & 31);
            if (p == q) {
                const uint64_t k = b + __popc(m & ((1u << lane) - 1));
                reinterpret_cast<uint64_t*>(d.ids[q])[k] = id;
                if (d.feats[q]) reinterpret_cast<uint32_t*>(d.feats[q])[k] = feats[i];
                reinterpret_cast<uint32_t*>(d.src[q])[k] = (uint32_t)i;
            }
            if (lane == (q & 31)) (q < 32 ? base : base2) += __popc(m);
        }
    }
    // device protocol: the stores reach the owners (NVLink / IPC) before the ready flag, which
    // a later kernel on this stream releases at system scope
    if (d.dev_off) __threadfence_system();
}

struct PeerBack {
    uint64_t slots[kMaxParts], oc[kMaxParts], mark[kMaxParts], roff[kMaxParts + 1];
};

__global__ void __launch_bounds__(256) k_return_scatter(uint64_t n_recv, const uint64_t* __restrict__ slots,
                                                        const uint8_t* __restrict__ oc,
                                                        const uint8_t* __restrict__ mark,
                                                        const uint32_t* __restrict__ src, uint32_t parts,
                                                        const PeerBack b) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_recv; j += (uint64_t)gridDim.x * blockDim.x) {
        // source rank: the part whose received range holds j (sources arrive rank-ordered)
        uint32_t lo = 0, hi = parts;  // roff[lo] <= j < roff[hi]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (b.roff[mid] <= j) lo = mid; else hi = mid;
        }
        const uint32_t p = src[j];
        reinterpret_cast<uint64_t*>(b.slots[lo])[p] = slots[j];
        reinterpret_cast<uint8_t*>(b.oc[lo])[p] = oc[j];
        if (b.mark[lo]) reinterpret_cast<uint8_t*>(b.mark[lo])[p] = mark ? mark[j] : 0;
    }
}

}  // namespace

// exclusive scan over cnt (part-major), declared in compact.cuh's style
__global__ void k_route_scan(unsigned* cnt, uint64_t total, unsigned* part_totals, uint32_t parts,
                             uint64_t nchunks);

__global__ void __launch_bounds__(1024) k_route_scan(unsigned* cnt, uint64_t total,
                                                     unsigned* part_totals, uint32_t parts,
                                                     uint64_t nchunks) {
    pdl_wait();
    __shared__ unsigned wsum[32];
    __shared__ unsigned carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < total; b0 += 1024) {
        const uint64_t i = b0 + threadIdx.x;
        const unsigned v = i < total ? cnt[i] : 0;
        unsigned x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= (unsigned)o) x += y;
        }
        if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned w = wsum[threadIdx.x];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= (unsigned)o) w += y;
            }
            wsum[threadIdx.x] = w;
        }
        __syncthreads();
        const unsigned incl = x + ((threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0);
        if (i < total) cnt[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += incl;
        __syncthreads();
    }
    // per-part totals: difference of consecutive part starts
    if (threadIdx.x < parts) {
        const uint64_t s = (uint64_t)threadIdx.x * nchunks;
        const unsigned start = cnt[s];
        const unsigned end = threadIdx.x + 1 < parts ? cnt[s + nchunks] : carry;
        part_totals[threadIdx.x] = end - start;
    }
}

void preload_route_kernels() {
    preload_kernel((const void*)k_route_count);
    preload_kernel((const void*)k_route_scan);
    preload_kernel((const void*)k_route_write);
    preload_kernel((const void*)k_route_scatter);
}

void upload_route_map(Table& t, const uint32_t* shard_to_part, uint32_t parts) {
    if (parts == 0 || parts > kMaxParts) throw Error{MPZCH_EINVAL, "route: 1..64 parts"};
    std::vector<uint8_t> h(t.S);
    for (uint32_t s = 0; s < t.S; ++s) {
        if (shard_to_part[s] >= parts) throw Error{MPZCH_EINVAL, "route: shard mapped to no part"};
        h[s] = (uint8_t)shard_to_part[s];
    }
    t.rt_s2p.reserve(t.S);
    t.rt_tot.reserve(parts * 4);
    if (h != t.rt_map) {
        MPZCH_CUDA(cudaMemcpyAsync(t.rt_s2p.p, h.data(), t.S, cudaMemcpyHostToDevice, t.stream));
        MPZCH_CUDA(cudaStreamSynchronize(t.stream));  // h is pageable and about to go out of scope
        t.rt_map = h;
    }
}

void enqueue_route_count(Table& t, const uint64_t* ids, uint64_t n, uint32_t parts, cudaStream_t st,
                         unsigned long long* bad) {
    const uint64_t nchunks = (n + kChunk - 1) / kChunk;
    t.rt_cnt.reserve(std::max<uint64_t>(1, nchunks * parts) * 4);
    t.rt_tot.reserve(parts * 4);
    if (n) {
        const unsigned blocks = (unsigned)((nchunks * 32 + 255) / 256);
        launch_pdl(k_route_count, blocks, 256, st, t.dev, ids, n, (const uint8_t*)t.rt_s2p.as<uint8_t>(), parts,
                   t.rt_cnt.as<unsigned>(), nchunks, bad);
        launch_pdl(k_route_scan, 1, 1024, st, t.rt_cnt.as<unsigned>(), (uint64_t)(nchunks * parts),
                   t.rt_tot.as<unsigned>(), parts, nchunks);
        t.launches += 2;
        MPZCH_CUDA(cudaGetLastError());
    }
    t.rt_ids = ids;  // arms run_route_scatter
    t.rt_n = n;
    t.rt_nchunks = nchunks;
    t.rt_parts = parts;
}

void run_route(Table& t, const uint64_t* ids, uint64_t n, const uint32_t* shard_to_part,
               uint32_t parts, uint32_t* perm, uint64_t* counts, cudaStream_t st) {
    if (parts == 0 || parts > kMaxParts) throw Error{MPZCH_EINVAL, "route: 1..64 parts"};
    for (uint32_t s = 0; s < t.S; ++s)
        if (shard_to_part[s] >= parts) throw Error{MPZCH_EINVAL, "route: shard mapped to no part"};
    const uint64_t nchunks = (n + kChunk - 1) / kChunk;
    // per-handle scratch (a temporary allocation would cudaFree -- a device sync -- per call);
    // the shard->part map is uploaded only when it changes
    DevBuf& s2p = t.rt_s2p;
    DevBuf& cnt = t.rt_cnt;
    DevBuf& tot = t.rt_tot;
    s2p.reserve(t.S);
    cnt.reserve(std::max<uint64_t>(1, nchunks * parts) * 4);
    tot.reserve(parts * 4);
    std::vector<uint8_t> h(t.S);
    for (uint32_t s = 0; s < t.S; ++s) h[s] = (uint8_t)shard_to_part[s];
    if (h != t.rt_map) {
        MPZCH_CUDA(cudaMemcpyAsync(s2p.p, h.data(), t.S, cudaMemcpyHostToDevice, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));  // h is pageable and about to go out of scope
        t.rt_map = h;
    }
    std::vector<unsigned> ht(parts, 0);
    if (n) {
        const unsigned blocks = (unsigned)((nchunks * 32 + 255) / 256);
        k_route_count<<<blocks, 256, 0, st>>>(t.dev, ids, n, s2p.as<uint8_t>(), parts,
                                              cnt.as<unsigned>(), nchunks, nullptr);
        k_route_scan<<<1, 1024, 0, st>>>(cnt.as<unsigned>(), nchunks * parts, tot.as<unsigned>(), parts,
                                         nchunks);
        if (perm) {
            k_route_write<<<blocks, 256, 0, st>>>(t.dev, ids, n, s2p.as<uint8_t>(), parts,
                                                  cnt.as<unsigned>(), nchunks, perm);
            ++t.launches;
        }
        t.launches += 2;
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(ht.data(), tot.p, parts * 4, cudaMemcpyDeviceToHost, st));
    }
    MPZCH_CUDA(cudaStreamSynchronize(st));
    for (uint32_t p = 0; p < parts; ++p) counts[p] = ht[p];
    t.rt_ids = perm ? nullptr : ids;  // a count-only route arms run_route_scatter
    t.rt_n = n;
    t.rt_nchunks = nchunks;
    t.rt_parts = parts;
}

void run_route_scatter(Table& t, const uint64_t* ids, const uint32_t* feats, uint64_t n,
                       uint32_t parts, const PeerScatter& d, cudaStream_t st) {
    if (!t.rt_ids || t.rt_ids != ids || t.rt_n != n || t.rt_parts != parts)
        throw Error{MPZCH_EINVAL, "route scatter: call mpzch_route_count_device on the same ids first"};
    PeerDst pd{};
    for (uint32_t q = 0; q < parts; ++q) {
        if (!d.ids_to[q] || !d.src_to[q]) throw Error{MPZCH_EINVAL, "route scatter: null destination"};
        if (feats && !d.feats_to[q]) throw Error{MPZCH_EINVAL, "route scatter: null feature destination"};
        pd.ids[q] = d.ids_to[q];
        pd.feats[q] = feats ? d.feats_to[q] : 0;
        pd.src[q] = d.src_to[q];
        pd.off[q] = d.offset ? d.offset[q] : 0;
    }
    pd.dev_off = d.dev_offset;
    pd.gate = d.gate;
    t.rt_ids = nullptr;
    if (n == 0) return;
    const uint64_t nchunks = t.rt_nchunks;
    const unsigned blocks = (unsigned)((nchunks * 32 + 255) / 256);
    launch_pdl(k_route_scatter, blocks, 256, st, t.dev, ids, feats, n, (const uint8_t*)t.rt_s2p.as<uint8_t>(),
               parts, (const unsigned*)t.rt_cnt.as<unsigned>(), nchunks, pd);
    ++t.launches;
    MPZCH_CUDA(cudaGetLastError());
}

void run_return_scatter(uint64_t n_recv, const uint64_t* slots, const uint8_t* oc, const uint8_t* mark,
                        const uint32_t* src, uint32_t parts, const uint64_t* recv_offset,
                        const uint64_t* slots_to, const uint64_t* oc_to, const uint64_t* mark_to,
                        cudaStream_t st) {
    if (parts == 0 || parts > kMaxParts) throw Error{MPZCH_EINVAL, "return scatter: 1..64 parts"};
    PeerBack b{};
    for (uint32_t r = 0; r <= parts; ++r) b.roff[r] = recv_offset[r];
    if (b.roff[0] != 0 || b.roff[parts] != n_recv)
        throw Error{MPZCH_EINVAL, "return scatter: received offsets must run from 0 to n_recv"};
    for (uint32_t r = 0; r < parts; ++r) {
        if (b.roff[r + 1] < b.roff[r]) throw Error{MPZCH_EINVAL, "return scatter: offsets decrease"};
        if (b.roff[r + 1] > b.roff[r] && (!slots_to[r] || !oc_to[r]))
            throw Error{MPZCH_EINVAL, "return scatter: null destination"};
        b.slots[r] = slots_to[r];
        b.oc[r] = oc_to[r];
        b.mark[r] = mark_to ? mark_to[r] : 0;
    }
    if (n_recv == 0) return;
    k_return_scatter<<<grid_for(n_recv, 256, 148u * 8u), 256, 0, st>>>(n_recv, slots, oc, mark, src, parts, b);
    MPZCH_CUDA(cudaGetLastError());
}

}  // namespace mpzch_b200
