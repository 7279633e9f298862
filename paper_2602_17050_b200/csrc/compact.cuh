// compact.cuh -- order-preserving stream compaction over a u8 flag array.
//
// Used where the reference walks a sequence in order and keeps a subset:
// first occurrences in dedup order (proj/src/batch_engine.cpp:100-106) and the
// canonical evicted list in unique-rank order.  Three launches: per-chunk
// counts, one-block exclusive scan of the chunk counts, ordered write.
#pragma once

#include "common.cuh"

namespace mpzch_b200 {

constexpr unsigned kCompactThreads = 256;
constexpr unsigned kCompactPerThread = 16;
constexpr unsigned kCompactChunk = kCompactThreads * kCompactPerThread;  // 4096 flags per block

__device__ __forceinline__ unsigned count16(const uint8_t* f, uint64_t i0, uint64_t n) {
    unsigned c = 0;
    if (i0 + 16 <= n) {
        const uint4 w = *reinterpret_cast<const uint4*>(f + i0);
        c = __popc(w.x & 0x01010101u) + __popc(w.y & 0x01010101u) + __popc(w.z & 0x01010101u) +
            __popc(w.w & 0x01010101u);
    } else {
        for (uint64_t i = i0; i < n; ++i) c += f[i] & 1u;
    }
    return c;
}

// flags must be 0/1 bytes; the flag array is padded to a multiple of 16 bytes.
// gate (nullable): a device word that is 0 when no flag can be set (the three kernels then only
// write a zero total)
static __global__ void __launch_bounds__(kCompactThreads) k_compact_count(const uint8_t* __restrict__ flags,
                                                                   uint64_t n,
                                                                   unsigned* __restrict__ blk,
                                                                   const unsigned* gate) {
    pdl_wait();
    if (gate && *gate == 0) return;
    __shared__ unsigned red[kCompactThreads / 32];
    const uint64_t i0 = (uint64_t)blockIdx.x * kCompactChunk + threadIdx.x * kCompactPerThread;
    unsigned c = i0 < n ? count16(flags, i0, n) : 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s = 0;
        for (unsigned w = 0; w < kCompactThreads / 32; ++w) s += red[w];
        blk[blockIdx.x] = s;
    }
}

// exclusive scan in place; total -> *total
static __global__ void __launch_bounds__(1024) k_compact_scan(unsigned* blk, unsigned nblk, unsigned* total,
                                                             const unsigned* gate) {
    pdl_wait();
    if (gate && *gate == 0) {
        if (threadIdx.x == 0 && total) *total = 0;
        return;
    }
    __shared__ unsigned carry;
    __shared__ unsigned wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (unsigned base = 0; base < nblk; base += 1024) {
        const unsigned i = base + threadIdx.x;
        const unsigned v = i < nblk ? blk[i] : 0;
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
        if (i < nblk) blk[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

// Ordered write: emit(i, k) is called for every flagged index i with its rank k.
template <class Emit>
__global__ void __launch_bounds__(kCompactThreads) k_compact_write(uint8_t* __restrict__ flags, uint64_t n,
                                                                   const unsigned* __restrict__ blk,
                                                                   bool clear, Emit emit, const unsigned* gate) {
    pdl_wait();
    if (gate && *gate == 0) return;
    __shared__ unsigned wsum[kCompactThreads / 32];
    const uint64_t i0 = (uint64_t)blockIdx.x * kCompactChunk + threadIdx.x * kCompactPerThread;
    const unsigned c = i0 < n ? count16(flags, i0, n) : 0;
    unsigned x = c;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= (unsigned)o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s = 0;
        for (unsigned w = 0; w < kCompactThreads / 32; ++w) {
            const unsigned t = wsum[w];
            wsum[w] = s;
            s += t;
        }
    }
    __syncthreads();
    unsigned k = blk[blockIdx.x] + wsum[threadIdx.x >> 5] + x - c;
    if (c) {
        const uint64_t iend = i0 + 16 < n ? i0 + 16 : n;
        for (uint64_t i = i0; i < iend; ++i) {
            if (flags[i] & 1u) {
                emit(i, k);
                ++k;
                if (clear) flags[i] = 0;
            }
        }
    }
}

template <class Emit>
inline void compact_flags(uint8_t* flags, uint64_t n, unsigned* blk, unsigned* total, bool clear,
                          Emit emit, cudaStream_t st, uint64_t& launches, const unsigned* gate = nullptr) {
    const unsigned nblk = (unsigned)((n + kCompactChunk - 1) / kCompactChunk);
    if (nblk == 0) return;
    launch_pdl(k_compact_count, nblk, kCompactThreads, st, (const uint8_t*)flags, n, blk, gate);
    launch_pdl(k_compact_scan, 1, 1024, st, blk, nblk, total, gate);
    launch_pdl(k_compact_write<Emit>, nblk, kCompactThreads, st, flags, n, (const unsigned*)blk, clear, emit, gate);
    launches += 3;
}

// force-load this translation unit's compaction kernels for Emit (see preload_all_kernels)
template <class Emit>
inline void preload_compact() {
    preload_kernel((const void*)k_compact_count);
    preload_kernel((const void*)k_compact_scan);
    preload_kernel((const void*)k_compact_write<Emit>);
}

}  // namespace mpzch_b200
