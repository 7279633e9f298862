// tag_scan.cuh -- quad scans of the identity TAG lines (common.cuh: TableDev::tag, one byte per
// slot, 0 = EMPTY, else tag_of(identity); kept for tables with max_probe >= kTagMinProbe).  A
// 128-byte tag line describes 128 slots, 8x the reach of a 128-byte identity line: a quad loads
// it with one warp instruction (lane j: bytes [32j, 32j + 32)), finds the window part's first
// EMPTY and the slots before it whose tag equals the id's, and verifies only those against the
// identity array.  Used by the long-window probe (remap_fast.cu k_probe_tag) and lookups
// (lookup.cu k_lookup_tag).  Requirements as line_scan.cuh: quad-uniform arguments; tag lines
// 128-byte aligned in global rows (Table allocates them from a 128-row aligned base).
#pragma once

#include "common.cuh"
#include "line_scan.cuh"

namespace mpzch_b200 {

// 0x80 in every zero byte of x, 0 elsewhere (exact: no borrow between bytes)
__device__ __forceinline__ uint32_t zero_bytes(uint32_t x) {
    const uint32_t t = (x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return ~(t | x | 0x7F7F7F7Fu);
}
// 0x80-per-byte flags -> 4 bits (byte k -> bit k): the multiply moves bit 8k+7 to bit 28+k, and
// its partial products land on distinct bits, so nothing carries
__device__ __forceinline__ uint32_t msb_bits4(uint32_t y) { return (y * 0x00204081u) >> 28; }

__device__ __forceinline__ unsigned quad_min(unsigned x, unsigned qm) {
    x = min(x, __shfl_xor_sync(qm, x, 1));
    return min(x, __shfl_xor_sync(qm, x, 2));
}

// bits [a, b) of a 32-bit word (0 <= a, b <= 32)
__device__ __forceinline__ unsigned bit_range(int a, int b) {
    if (b <= a) return 0u;
    const unsigned w = (unsigned)(b - a);
    return (w >= 32 ? 0xffffffffu : ((1u << w) - 1u)) << a;
}

// One window segment of tag line `tl`: slots [s, s + c) of the line.  Returns the line slot
// of the first one holding the id (its candidates -- tag matches before the segment's first
// EMPTY -- verified against the identity array in slot order) or 128, and in `fe` the
// segment's first EMPTY (or 128).  Quad-uniform arguments; lane j holds tag bytes [32j, +32).
__device__ __forceinline__ unsigned tag_segment(const TableDev& t, const uint64_t (&v)[4], uint32_t pat, uint64_t id,
                                                uint64_t tl, int s, int c, int jb, unsigned j, unsigned qm,
                                                unsigned& fe, unsigned long long& isec) {
    unsigned mm = 0, ee = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t x = (uint32_t)(v[k >> 1] >> (32 * (k & 1)));
        mm |= msb_bits4(zero_bytes(x ^ pat)) << (4 * k);
        ee |= msb_bits4(zero_bytes(x)) << (4 * k);
    }
    const unsigned r = bit_range(max(s, jb) - jb, min(s + c, jb + 32) - jb);
    mm &= r;
    ee &= r;
    fe = quad_min(ee ? (unsigned)jb + __ffs(ee) - 1 : 128u, qm);
    mm &= bit_range(0, min(max((int)fe - jb, 0), 32));
    for (;;) {  // every lane verifies its lowest candidate; the lowest verified match wins
                // unless a lower lane still holds an unverified candidate (rare: ~0.5 per line)
        const bool have = mm != 0;
        const unsigned cq = have ? (unsigned)jb + __ffs(mm) - 1 : 128u;
        const bool match = have && t.ident[tl + cq] == id;
        isec += have;
        const unsigned qmatch = quad_min(match ? cq : 128u, qm);
        if (have && !match) mm &= mm - 1;
        // lowest candidate still unverified after this step
        const unsigned rest = quad_min(mm && !match ? (unsigned)jb + __ffs(mm) - 1 : 128u, qm);
        if (qmatch < rest || rest == 128u) return qmatch;
    }
}

// the window part inside g's tag line: [g, g + c), c bounded by the line, the shard end and the
// remaining max_probe budget
__device__ __forceinline__ uint32_t tag_seg_len(uint64_t g, uint64_t end, uint32_t off, uint32_t P) {
    uint64_t c = 128 - (g & 127u);
    if (end - g < c) c = end - g;
    const uint32_t left = off < P ? P - off : 0u;
    if (left < c) c = left;
    return (uint32_t)c;
}


// lane j's 32 bytes of the tag line holding global row tl (128-row aligned)
__device__ __forceinline__ void ld_tag_part(const TableDev& t, uint64_t tl, unsigned j, uint64_t (&v)[4]) {
    ld_sector(reinterpret_cast<const uint64_t*>(t.tag + tl) + 4 * j, v[0], v[1], v[2], v[3]);
}

}  // namespace mpzch_b200
