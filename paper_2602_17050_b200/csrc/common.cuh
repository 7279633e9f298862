// common.cuh -- device-side primitives shared by every MPZCH sm_100a kernel.
//
// Every constant below is pinned to the reference so hashes, homes, shards
// and reset rows are bit-identical (paths relative to /root/reference/):
//   kEmptySlot / salts / mix64   proj/include/mpzch/ids.hpp:16-43
//   SplitMix64                    proj/include/mpzch/rng.hpp:10-30
//   home_slot                     proj/src/probe_core.cpp:27-30
//   shard_of                      proj/src/shard_router.cpp:42-46
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>

namespace mpzch_b200 {

constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kHomeSalt = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kShardSalt = 0xD1B54A32D192ED03ull;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint32_t kNone32 = 0xffffffffu;

enum : uint8_t { kFound = 0, kInserted = 1, kEvicted = 2, kCollision = 3 };
enum : int { kModeDisabled = 0, kModeTtl = 1, kModeLru = 2 };

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t id, uint64_t seed) {
    uint64_t x = id ^ seed;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// SplitMix64 output for an explicit state value (the generator's state after
// k increments is s0 + k*golden, so element j of a stream is independent).
__host__ __device__ __forceinline__ uint64_t splitmix_out(uint64_t state) {
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Exact 64-bit x mod d without the ~100-instruction software division:
// m = floor((2^64-1)/d), q = umulhi(x, m) is floor(x/d) or at most 2 below it.
struct FastMod {
    uint64_t d;
    uint64_t m;
};

inline FastMod make_fastmod(uint64_t d) { return FastMod{d, ~0ull / d}; }

__device__ __forceinline__ uint64_t fastmod(uint64_t x, FastMod f) {
    const uint64_t q = __umul64hi(x, f.m);
    uint64_t r = x - q * f.d;
    while (r >= f.d) r -= f.d;
    return r;
}

// One logical shard: its global row range [offset, offset + cap).
struct ShardDev {
    uint64_t offset;
    FastMod cap;
};

// The resident table, passed by value to every kernel.
struct TableDev {
    uint64_t* ident;     // identity per global row (EMPTY = ~0)
    uint64_t* meta;      // metadata per global row
    float* weights;      // rows x dim (dim > 0)
    float* momentum;     // rows x dim
    uint32_t* trained;   // one bit per held row (row - row_lo): EmbeddingTable::trained_
                         // (embedding_store.hpp, a byte per row there); bits keep the flag words
                         // L2-resident, so resets and steps pay no DRAM fill for a 1-byte store
    uint64_t* row_gen;   // rows
    const ShardDev* shards;
    FastMod nshards;
    uint64_t seed;
    uint64_t init_seed;
    uint64_t total;      // rows of the whole layout (global row numbering)
    uint64_t row_lo;     // rows this handle holds: [row_lo, row_hi) (all rows unless sharded)
    uint64_t row_hi;
    uint32_t shard_lo;   // logical shards this handle holds: [shard_lo, shard_hi)
    uint32_t shard_hi;
    double bound;        // 1/sqrt(dim) * 2^-52 (draw_row's bound, computed on the host exactly as
                         // the reference does, then scaled by a power of two: see draw_at)
    uint32_t P;          // max_probe
    uint32_t dim;
    uint8_t* tag;        // max_probe >= kTagMinProbe: one byte per global row, 0 for EMPTY, else
                         // tag_of(identity) -- a 1/128-size image of the identity array that the
                         // long-window probe scans (128 slots per 128-byte line) instead of the
                         // identities (16 slots per line); null for shorter windows
    uint32_t* pend_bits; // MPZCH_RESET_DEFERRED: one bit per held row (row - row_lo), set while
                         // the row's reset (draw_row, momentum 0, trained 0) is not yet written;
                         // null in eager mode.  1 bit per row keeps the map L2-resident (16 MiB
                         // at 2^27 rows), so reset-aware readers pay an L2 hit, not a DRAM access
};

// draw_row (proj/src/embedding_store.cpp:12-18), element with SplitMix64 state `state`
// (= mix64(row, init_seed) + (j+1) * golden for element j); see rows.cu
__device__ __forceinline__ float draw_at(uint64_t state, double bound_s) {
    const uint64_t z = splitmix_out(state);
    // (2u - 1) * bound with u = (z >> 11) * 2^-53: 2u - 1 = k * 2^-52 exactly, k = (z >> 11) - 2^52
    // an integer, so the product is k * (bound * 2^-52) -- bound_s, scaled on the host by a power
    // of two (exact) -- rounded once: the reference's single FP64 rounding with one FP64 multiply
    // instead of two (the FP64 pipe bounds the reset kernel), bit for bit the same value
    const double k = (double)((int64_t)(z >> 11) - (1ll << 52));
    return __double2float_rn(__dmul_rn(k, bound_s));
}

__device__ __forceinline__ float draw_elem(uint64_t s0, uint64_t j, double bound) {
    return draw_at(s0 + (j + 1) * kGolden, bound);
}

// elements 4q .. 4q+3 of draw_row(row): one multiply, then golden increments
__device__ __forceinline__ float4 draw_quad(uint64_t s0, uint32_t q, double bound) {
    const uint64_t s1 = s0 + ((uint64_t)q * 4 + 1) * kGolden;
    float4 v;
    v.x = draw_at(s1, bound);
    v.y = draw_at(s1 + kGolden, bound);
    v.z = draw_at(s1 + 2 * kGolden, bound);
    v.w = draw_at(s1 + 3 * kGolden, bound);
    return v;
}

__device__ __forceinline__ void set_trained(const TableDev& t, uint64_t row) {
    const uint64_t r = row - t.row_lo;
    atomicOr(t.trained + (r >> 5), 1u << (r & 31));
}
__device__ __forceinline__ void clear_trained(const TableDev& t, uint64_t row) {
    const uint64_t r = row - t.row_lo;
    atomicAnd(t.trained + (r >> 5), ~(1u << (r & 31)));
}

// is the row's reset pending (deferred mode only)
__device__ __forceinline__ bool reset_pending(const TableDev& t, uint64_t row) {
    if (!t.pend_bits) return false;
    const uint64_t r = row - t.row_lo;
    return (__ldcg(t.pend_bits + (r >> 5)) >> (r & 31)) & 1u;
}

__device__ __forceinline__ void clear_pending(const TableDev& t, uint64_t row) {
    const uint64_t r = row - t.row_lo;
    atomicAnd(t.pend_bits + (r >> 5), ~(1u << (r & 31)));
}

// a warp copies one row's weights to dst (16-byte accesses when dim % 4 == 0); a row whose
// reset is pending is drawn in closed form instead (EmbeddingTable::gather after reset_row)
__device__ __forceinline__ void copy_row_or_draw(const TableDev& t, uint64_t row, float* dst, unsigned lane) {
    const float* src = t.weights + row * t.dim;
    const bool pend = reset_pending(t, row);
    const uint64_t s0 = pend ? mix64(row, t.init_seed) : 0;
    if ((t.dim & 3u) == 0) {
        for (uint32_t q = lane; q < t.dim / 4; q += 32)
            reinterpret_cast<float4*>(dst)[q] =
                pend ? draw_quad(s0, q, t.bound) : __ldg(reinterpret_cast<const float4*>(src) + q);
    } else {
        for (uint32_t j = lane; j < t.dim; j += 32) dst[j] = pend ? draw_elem(s0, j, t.bound) : __ldg(src + j);
    }
}

__device__ __forceinline__ uint32_t shard_of(uint64_t id, const TableDev& t) {
    return (uint32_t)fastmod(mix64(id ^ kShardSalt, t.seed), t.nshards);
}

__device__ __forceinline__ bool holds_shard(const TableDev& t, uint32_t s) {
    return s >= t.shard_lo && s < t.shard_hi;
}

__device__ __forceinline__ uint64_t home_of(uint64_t id, const ShardDev& s, uint64_t seed) {
    return fastmod(mix64(id ^ kHomeSalt, seed), s.cap);
}

// Identity tags (TableDev::tag): kept for tables whose windows run long (C3: P = 256 at 0.95
// load, where an absent id walks ~13 identity lines to its first EMPTY but ~2 tag lines).
constexpr uint32_t kTagMinProbe = 256;
constexpr uint64_t kTagSalt = 0x6A09E667F3BCC909ull;

__host__ __device__ __forceinline__ uint8_t tag_of(uint64_t id) {
    const uint8_t x = (uint8_t)(mix64(id ^ kTagSalt, 0) >> 56);
    return x ? x : 1;  // 0 marks an EMPTY slot
}

// every identity store goes through here (or pairs its store with this), so the tags of a
// table that keeps them always describe its identity array
__device__ __forceinline__ void store_tag(const TableDev& t, uint64_t g, uint64_t id) {
    if (t.tag) t.tag[g] = id == kEmpty ? 0 : tag_of(id);
}

// Error word shared by all kernels of one batch.  Mutating kernels return
// immediately when any field is set, so an invalid batch mutates nothing.
struct BatchErr {
    unsigned long long bad_pos;      // min invalid position, ~0 if none
    unsigned int overflow;           // TTL expiry overflow seen
    unsigned int too_many;           // internal invariant violated
    unsigned long long foreign_pos;  // min position whose shard this handle does not hold
};

// The part of a row-sharded rank's per-batch device state the owner's remap reads
// (sharded.cu keeps the full record; this is its prefix).
struct ShStateView {
    unsigned long long failed;  // some rank's slice failed validation (or a peer timed out)
    unsigned long long R;       // positions received by this owner in this batch
};

__device__ __forceinline__ bool batch_failed(const BatchErr* e) {
    return e->bad_pos != ~0ull || e->overflow != 0 || e->too_many != 0 || e->foreign_pos != ~0ull;
}

// L2-coherent loads/stores for state that other threads mutate in the same kernel.
__device__ __forceinline__ uint64_t ld_cg(const uint64_t* p) { return __ldcg(p); }

// 32-byte (one sector) load of four consecutive slots: LDG.E.256 on sm_100.
__device__ __forceinline__ void ld_sector(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                          uint64_t& d) {
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}

// L2-coherent (L1-bypassing) sector load, for state other threads mutate in this kernel
__device__ __forceinline__ void ld_sector_cg(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                             uint64_t& d) {
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: a kernel launched with the PDL attribute may start while its
// predecessor in the stream drains; it waits here (before touching anything the predecessor
// wrote) for the predecessor's completion and memory flush.  A no-op without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Lazy module loading (the CUDA 12 default) loads a kernel at its first launch, and a load can
// wait for the device's running work.  The row-sharded protocol has kernels that spin until a
// peer's kernels run, so every kernel a batch can launch is loaded up front (cudaFuncGetAttributes
// forces the load); see preload_all_kernels.
inline void preload_kernel(const void* k) {
    cudaFuncAttributes a;
    const cudaError_t e = cudaFuncGetAttributes(&a, k);
    if (e != cudaSuccess) (void)cudaGetLastError();
}

template <class T>
struct same_type { using type = T; };

// Launch `k` as a programmatic dependent of the previous kernel in `st` (it starts while that
// kernel drains and waits in pdl_wait()): a chain of kernels pays one launch latency, not one
// per kernel.  MPZCH_PDL=0 launches plainly.  Launch errors surface through cudaGetLastError.
template <typename... KArgs>
inline cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t st,
                              typename same_type<KArgs>::type... args) {
    static const bool enabled = [] {
        const char* e = std::getenv("MPZCH_PDL");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = enabled ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

}  // namespace mpzch_b200
