// publish.cu -- snapshot / delta serialisation from HBM with the CRC-32 on the device
// (formats: proj/README.md:129-145, proj/src/publish.cpp).
//
// CRC-32 here is the reference's (publish.cpp:110-124: reflected, polynomial 0xEDB88320, init
// and final xor ~0).  It is linear over GF(2), so with raw(M) = the register after M from 0:
//   raw(A || B) = shift(raw(A), |B|) ^ raw(B),   shift(c, L) = c * x^(8L) mod P,
//   crc(M) = raw(M) ^ shift(~0, |M|) ^ ~0.
// Device kernel: a block takes a contiguous run of 16 KB iterations; in an iteration each warp
// owns 2 KB, each lane four 16-byte pieces (coalesced 512-byte rows).  A piece's raw CRC is a
// slicing-by-16 lookup; pieces, lanes, warps and iterations are folded with constant-length
// shifts, each a linear map applied as four byte-indexed lookups.  All tables (56 KB) sit in
// shared memory.  Block results are combined on the host with x^(8L) powers (zlib's
// multmodp / x2nmodp construction).  Bytes that do not fill a 16 KB iteration are folded on
// the host (at most 16 KB per section).
//
// The images themselves are mostly raw copies: the identity array (u64 little-endian, global
// row order = shards in order) and the weights (f32 row-major) are exactly the snapshot's
// sections; a delta's records (row u64 | identity u64 | dim f32) are packed on the device from
// the dirty-row compaction.  Only headers are built on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr uint64_t kIter = 16384;  // bytes per block iteration (256 threads x 64 B)
// shift tables: by 16, 32, 64, 128, 256 B (lane tree), 512 B (piece rows), 2, 4, 8 KB (warp
// tree), 16 KB (iterations)
constexpr int kShifts = 10;
constexpr uint64_t kShiftLen[kShifts] = {16, 32, 64, 128, 256, 512, 2048, 4096, 8192, 16384};
constexpr int kTableWords = 16 * 256 + kShifts * 4 * 256;
constexpr int kTableBytes = kTableWords * 4;

// ---- host GF(2) arithmetic (zlib's construction, reflected: bit 31 = x^0)
uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = b & 1 ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

const uint32_t* x2n_table() {  // x^(2^k) mod P
    static uint32_t t[64];
    static std::once_flag once;
    std::call_once(once, [] {
        uint32_t p = 1u << 30;  // x^1
        t[0] = p;
        for (int k = 1; k < 64; ++k) t[k] = p = multmodp(p, p);
    });
    return t;
}

uint32_t x8nmodp(uint64_t n) {  // x^(8n) mod P
    const uint32_t* t = x2n_table();
    uint32_t p = 1u << 31;  // x^0
    unsigned k = 3;
    while (n) {
        if (n & 1) p = multmodp(t[k & 63], p);
        n >>= 1;
        ++k;
    }
    return p;
}

uint32_t shift_host(uint32_t c, uint64_t len) { return len ? multmodp(x8nmodp(len), c) : c; }

const uint32_t* byte_table() {
    static uint32_t t[256];
    static std::once_flag once;
    std::call_once(once, [] {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
            t[i] = c;
        }
    });
    return t;
}

uint32_t raw_host(uint32_t c, const uint8_t* p, uint64_t n) {
    const uint32_t* t = byte_table();
    for (uint64_t i = 0; i < n; ++i) c = t[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    return c;
}

std::vector<uint32_t> build_tables() {
    std::vector<uint32_t> w(kTableWords);
    const uint32_t* bt = byte_table();
    // slice[k][b]: raw CRC of byte b followed by k zero bytes
    for (int b = 0; b < 256; ++b) {
        uint32_t c = bt[b];
        for (int k = 0; k < 16; ++k) {
            w[k * 256 + b] = c;
            c = bt[c & 0xFFu] ^ (c >> 8);
        }
    }
    // shift tables: shift(c, L) = XOR_i S_L[i][(c >> 8i) & 0xFF]
    for (int s = 0; s < kShifts; ++s) {
        const uint32_t xp = x8nmodp(kShiftLen[s]);
        for (int i = 0; i < 4; ++i)
            for (int b = 0; b < 256; ++b)
                w[16 * 256 + (s * 4 + i) * 256 + b] = multmodp(xp, (uint32_t)b << (8 * i));
    }
    return w;
}

// ---- device
__device__ __forceinline__ uint32_t dshift(const uint32_t* __restrict__ s, uint32_t c) {
    return s[c & 0xFFu] ^ s[256 + ((c >> 8) & 0xFFu)] ^ s[512 + ((c >> 16) & 0xFFu)] ^
           s[768 + (c >> 24)];
}

__device__ __forceinline__ uint32_t slice_word(const uint32_t* __restrict__ sl, uint32_t w, int k0) {
    // bytes of w (little-endian) sit at distances k0+3, k0+2, k0+1, k0 from the piece end
    return sl[(k0 + 3) * 256 + (w & 0xFFu)] ^ sl[(k0 + 2) * 256 + ((w >> 8) & 0xFFu)] ^
           sl[(k0 + 1) * 256 + ((w >> 16) & 0xFFu)] ^ sl[k0 * 256 + (w >> 24)];
}

__device__ __forceinline__ uint32_t slice16(const uint32_t* __restrict__ sl, uint4 v) {
    return slice_word(sl, v.x, 12) ^ slice_word(sl, v.y, 8) ^ slice_word(sl, v.z, 4) ^
           slice_word(sl, v.w, 0);
}

// blocks [0, nb): block b folds iterations [it0(b), it1(b)) of `data` into out[b] (raw CRC)
__global__ void __launch_bounds__(256) k_crc_blocks(const uint4* __restrict__ data, uint64_t iters,
                                                    const uint32_t* __restrict__ tables,
                                                    uint32_t* __restrict__ out) {
    extern __shared__ uint32_t sm[];
    for (int i = threadIdx.x; i < kTableWords; i += blockDim.x) sm[i] = tables[i];
    __syncthreads();
    const uint32_t* sl = sm;
    const uint32_t* sh = sm + 16 * 256;  // shift table s at sh + s * 1024
    const uint64_t q = iters / gridDim.x, r = iters % gridDim.x;
    const uint64_t b = blockIdx.x;
    const uint64_t it0 = b * q + (b < r ? b : r);
    const uint64_t it1 = it0 + q + (b < r ? 1 : 0);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t wcrc[8];
    uint32_t acc = 0;
    for (uint64_t it = it0; it < it1; ++it) {
        // warp region: 2 KB = 4 rows of 512 B; lane piece j at 512 j + 16 lane
        const uint4* p = data + it * (kIter / 16) + warp * 128 + lane;
        const uint4 v0 = __ldcs(p), v1 = __ldcs(p + 32), v2 = __ldcs(p + 64), v3 = __ldcs(p + 96);
        uint32_t c = slice16(sl, v0);
        c = dshift(sh + 5 * 1024, c) ^ slice16(sl, v1);
        c = dshift(sh + 5 * 1024, c) ^ slice16(sl, v2);
        c = dshift(sh + 5 * 1024, c) ^ slice16(sl, v3);
        // lanes: lane l's value must end up shifted by 16 (31 - l)
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint32_t o = __shfl_down_sync(0xffffffffu, c, 1u << k);
            if ((lane & ((2u << k) - 1)) == 0) c = dshift(sh + k * 1024, c) ^ o;
        }
        if (lane == 0) wcrc[warp] = c;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < 8 ? wcrc[lane] : 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const uint32_t o = __shfl_down_sync(0xffffffffu, w, 1u << k);
                if ((lane & ((2u << k) - 1)) == 0) w = dshift(sh + (6 + k) * 1024, w) ^ o;
            }
            if (lane == 0) acc = dshift(sh + 9 * 1024, acc) ^ w;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

struct CrcDevice {
    uint32_t* tables = nullptr;
    uint32_t* out = nullptr;
    uint32_t* h_out = nullptr;
    int blocks = 0;
};

CrcDevice& crc_device(int device) {
    static std::mutex mu;
    static std::vector<CrcDevice> per;
    std::lock_guard<std::mutex> g(mu);
    if ((int)per.size() <= device) per.resize(device + 1);
    CrcDevice& d = per[device];
    if (!d.tables) {
        const std::vector<uint32_t> w = build_tables();
        MPZCH_CUDA(cudaMalloc(&d.tables, kTableBytes));
        MPZCH_CUDA(cudaMemcpy(d.tables, w.data(), kTableBytes, cudaMemcpyHostToDevice));
        MPZCH_CUDA(cudaFuncSetAttribute(k_crc_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kTableBytes));
        int sms = 0, per_sm = 0;
        MPZCH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        MPZCH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_crc_blocks, 256, kTableBytes));
        d.blocks = sms * std::max(per_sm, 1);
        MPZCH_CUDA(cudaMalloc(&d.out, d.blocks * 4));
        MPZCH_CUDA(cudaMallocHost(&d.h_out, d.blocks * 4));
    }
    return d;
}

}  // namespace

// raw CRC (register from 0, no final xor) of n device bytes; synchronous on st
uint32_t crc32_raw_device(const uint8_t* data, uint64_t n, cudaStream_t st, int device) {
    if (n == 0) return 0;
    uint32_t raw = 0;
    // unaligned head (host)
    const uint64_t mis = (uint64_t)(uintptr_t)data & 15u;
    uint64_t head = mis ? std::min<uint64_t>(n, 16 - mis) : 0;
    std::vector<uint8_t> hb;
    if (head) {
        hb.resize(head);
        MPZCH_CUDA(cudaMemcpyAsync(hb.data(), data, head, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        raw = raw_host(0, hb.data(), head);
    }
    const uint8_t* body = data + head;
    const uint64_t rest = n - head;
    const uint64_t iters = rest / kIter;
    if (iters) {
        CrcDevice& d = crc_device(device);
        const int nb = (int)std::min<uint64_t>(iters, (uint64_t)d.blocks);
        k_crc_blocks<<<nb, 256, kTableBytes, st>>>(reinterpret_cast<const uint4*>(body), iters, d.tables,
                                                   d.out);
        MPZCH_CUDA(cudaGetLastError());
        MPZCH_CUDA(cudaMemcpyAsync(d.h_out, d.out, nb * 4, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        const uint64_t q = iters / nb, r = iters % nb;
        const uint32_t xq = x8nmodp(q * kIter), xq1 = x8nmodp((q + 1) * kIter);
        for (int b = 0; b < nb; ++b) raw = multmodp((uint64_t)b < r ? xq1 : xq, raw) ^ d.h_out[b];
    }
    const uint64_t tail = rest - iters * kIter;
    if (tail) {
        std::vector<uint8_t> tb(tail);
        MPZCH_CUDA(cudaMemcpyAsync(tb.data(), body + iters * kIter, tail, cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        raw = raw_host(raw, tb.data(), tail);
    }
    return raw;
}

uint32_t crc32_finish(uint32_t raw, uint64_t n) { return raw ^ shift_host(0xFFFFFFFFu, n) ^ 0xFFFFFFFFu; }

uint32_t crc32_raw_host(uint32_t raw, const uint8_t* p, uint64_t n) { return raw_host(raw, p, n); }

uint32_t crc32_shift(uint32_t raw, uint64_t n) { return shift_host(raw, n); }

namespace {

// delta records: row u64 | identity u64 | dim f32, written as 32-bit words (a record is
// 8-byte aligned only for even dim); one warp per record
__global__ void __launch_bounds__(256) k_pack_delta(TableDev t, const uint64_t* __restrict__ rows,
                                                    const unsigned* __restrict__ count,
                                                    uint32_t* __restrict__ out) {
    const unsigned n = *count;
    const unsigned lane = lane_id();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t words = 4 + t.dim;
    for (uint64_t k = warp; k < n; k += nwarps) {
        const uint64_t row = rows[k];
        uint32_t* rec = out + k * words;
        if (lane < 4) {
            const uint64_t v = lane < 2 ? row : t.ident[row];
            rec[lane] = (uint32_t)(lane & 1 ? v >> 32 : v);
        }
        const uint32_t* w = reinterpret_cast<const uint32_t*>(t.weights + row * t.dim);
        for (uint32_t j = lane; j < t.dim; j += 32) rec[4 + j] = __ldg(w + j);
    }
}

}  // namespace

void launch_pack_delta(Table& t, const uint64_t* rows, const unsigned* count, uint64_t max_n,
                       uint8_t* out, cudaStream_t st) {
    if (!max_n) return;
    const unsigned blocks = (unsigned)std::min<uint64_t>((max_n * 32 + 255) / 256, 148 * 16);
    k_pack_delta<<<blocks, 256, 0, st>>>(t.dev, rows, count, reinterpret_cast<uint32_t*>(out));
    ++t.launches;
}

}  // namespace mpzch_b200
