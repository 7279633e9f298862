// line_scan.cuh -- quad-cooperative 128-byte line scans of the identity / metadata arrays.
//
// Measured on B200 (tools/sector_probe.cu, profiles/line_ceiling_r01.json): a uniformly random
// 32-byte read and a uniformly random 128-byte line read issued as ONE warp instruction (4
// lanes x 32 B) cost the same, ~36 G accesses/s over a 16 GiB array -- the L2 promotes every
// random miss to a full 128-byte DRAM fetch anyway.  One thread walking sector by sector pays
// one access per sector; a quad (4 lanes) reading the whole line pays one per line.  A hit at
// 0.8 load needs ~1.5 sectors but only ~1.13 lines, so every window scan below
// walks lines: lane j of the quad loads sector j of the line, the quad ORs its 4-bit slot
// masks together with two shuffles and picks the first qualifying slot of the window with
// __ffs.  The window is [g, g + c) inside the line: it stops at the line end, the shard end
// (wrap to the shard base) and the remaining max_probe budget.
//
// Requirements: the array is 128-byte aligned in GLOBAL-row numbering (Table allocates from a
// 16-row-aligned base and pads to whole lines), and all 4 lanes of a quad call these helpers
// with identical arguments (quad-uniform control flow; shuffles use the quad's lane mask).
#pragma once

#include "common.cuh"

namespace mpzch_b200 {

constexpr unsigned kLineSlots = 16;  // 128 B of u64 slots

__device__ __forceinline__ unsigned quad_lane() { return threadIdx.x & 3u; }
__device__ __forceinline__ unsigned quad_mask() { return 0xFu << (lane_id() & ~3u); }

// lane j of the quad: the 4 slots [line*16 + 4j, +4) of the line holding slot g
__device__ __forceinline__ void ld_line_part(const uint64_t* arr, uint64_t g, unsigned j, uint64_t (&w)[4]) {
    ld_sector(arr + (g & ~15ull) + 4 * j, w[0], w[1], w[2], w[3]);
}

// OR the quad's 4-bit lane codes into one 16-bit line mask (bit k = slot k of the line);
// `hi` carries a second 4-bit code into bits 16..31
__device__ __forceinline__ unsigned quad_gather(unsigned lo4, unsigned hi4, unsigned j, unsigned qm) {
    unsigned x = (lo4 | (hi4 << 16)) << (4 * j);
    x |= __shfl_xor_sync(qm, x, 1);
    x |= __shfl_xor_sync(qm, x, 2);
    return x;
}

// The part of the window that lies in g's line: slots [s, s + c) of the line.
struct LineSpan {
    unsigned s, c;
    __device__ __forceinline__ unsigned range() const { return ((1u << c) - 1u) << s; }
    // sectors covering slots [s, last] of the line (the algorithmic-bytes count)
    __device__ __forceinline__ unsigned sectors_to(unsigned last) const { return (last >> 2) - (s >> 2) + 1; }
};

__device__ __forceinline__ LineSpan line_span(uint64_t g, uint64_t end, uint32_t off, uint32_t limit) {
    LineSpan sp;
    sp.s = (unsigned)(g & 15u);
    uint64_t c = kLineSlots - sp.s;
    if (end - g < c) c = end - g;
    if (limit - off < c) c = limit - off;
    sp.c = (unsigned)c;
    return sp;
}

}  // namespace mpzch_b200
