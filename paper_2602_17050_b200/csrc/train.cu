// train.cu -- MpzchTable::sgd_step (proj/src/table.cpp:174-179) over EmbeddingTable::sgd_step
// (proj/src/embedding_store.cpp:70-93), SURVEY 8f row 3.
//
// Reference semantics, in position order i = 0..n-1:
//   check_row(rows[i]); m := beta*m + g_i; w := w - lr*m (fp32, mul and add rounded
//   separately: the reference is built for baseline x86-64, no FMA); trained[row] := 1;
// then touch_row(row) for every position.  A row out of range throws out_of_range after the
// rows before it were updated and before any touch.  Duplicate rows compound in order.
//
// Device plan (HBM-bound: per position 4*dim B of gradient read + 2 x 4*dim B read-modify-write
// of weights and momentum):
//   G1 k_sgd_prep     range check (first bad position by atomicMin) and a hash of the rows
//                     (64-bit CAS keys): entry, per-entry occurrence count, arrival slot;
//   G2 k_sgd_dup_base entries with more than one occurrence get a contiguous segment
//   G3 k_sgd_dup_fill (both skip at once when no row repeats);
//   G4 k_sgd_apply    positions whose row occurs once: a group of L lanes per position
//                     (L = dim/4 rounded up to a power of two, <= 32), float4 traffic;
//   G5 k_sgd_dups     one warp per repeated row: lane 0 orders the row's positions, then the
//                     warp applies them one after another (the reference's order);
//   G6 k_sgd_clean    clears the used hash entries.
// Positions at or after the first bad one are not applied, and no row is touched then.
// Deferred resets (MPZCH_RESET_DEFERRED, rows.cu): a row the batch evicted is still marked
// pending; its update starts from the closed-form draw_row and momentum 0 instead of reading
// the row -- the reset and the step share one write of the row.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

__device__ __forceinline__ void sgd_quad(float4& w, float4& m, const float4 g, float lr, float beta) {
    m.x = __fadd_rn(__fmul_rn(beta, m.x), g.x);
    m.y = __fadd_rn(__fmul_rn(beta, m.y), g.y);
    m.z = __fadd_rn(__fmul_rn(beta, m.z), g.z);
    m.w = __fadd_rn(__fmul_rn(beta, m.w), g.w);
    w.x = __fsub_rn(w.x, __fmul_rn(lr, m.x));
    w.y = __fsub_rn(w.y, __fmul_rn(lr, m.y));
    w.z = __fsub_rn(w.z, __fmul_rn(lr, m.z));
    w.w = __fsub_rn(w.w, __fmul_rn(lr, m.w));
}

// one position's update by `width` cooperating lanes (lane index `sub`).  pend: the row's
// eviction reset is deferred (rows.cu) -- the old row is the closed-form draw_row and momentum
// 0, exactly what the reset would have written, so nothing is read and the row is written once
__device__ __forceinline__ void apply_row(const TableDev& t, uint64_t row, const float* g,
                                          float lr, float beta, bool vec, unsigned sub,
                                          unsigned width, bool pend) {
    float* w = t.weights + row * t.dim;
    float* m = t.momentum + row * t.dim;
    const uint64_t s0 = pend ? mix64(row, t.init_seed) : 0;
    if (vec) {
        float4* w4 = reinterpret_cast<float4*>(w);
        float4* m4 = reinterpret_cast<float4*>(m);
        const float4* g4 = reinterpret_cast<const float4*>(g);
        for (uint32_t q = sub; q < t.dim / 4; q += width) {
            float4 wv, mv;
            if (pend) {
                wv = draw_quad(s0, q, t.bound);
                mv = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                wv = w4[q];
                mv = m4[q];
            }
            sgd_quad(wv, mv, __ldg(g4 + q), lr, beta);
            m4[q] = mv;
            w4[q] = wv;
        }
    } else {
        for (uint32_t j = sub; j < t.dim; j += width) {
            const float m0 = pend ? 0.f : m[j];
            const float w0 = pend ? draw_elem(s0, j, t.bound) : w[j];
            const float mv = __fadd_rn(__fmul_rn(beta, m0), __ldg(g + j));
            m[j] = mv;
            w[j] = __fsub_rn(w0, __fmul_rn(lr, mv));
        }
    }
}

__global__ void k_sgd_init(SgdCounters* c) {
    *c = SgdCounters{~0ull, 0, 0, 0, 0};
}

__global__ void __launch_bounds__(256) k_sgd_prep(TableDev t, const uint64_t* __restrict__ rows,
                                                  uint64_t n, unsigned long long* key,
                                                  unsigned* cnt, uint32_t* pe, uint32_t* pr,
                                                  uint64_t mask, SgdCounters* c) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = rows[i];
        if (row < t.row_lo || row >= t.row_hi) {  // embedding_store.cpp:50-54
            atomicMin(&c->bad, (unsigned long long)i);
            pe[i] = kNone32;
            continue;
        }
        uint64_t h = mix64(row, 0x7367645f73746570ull) & mask;
        for (;;) {
            const unsigned long long k = __ldcg(key + h);
            if (k == row) break;
            if (k == kEmpty) {
                const unsigned long long prev = atomicCAS(key + h, kEmpty, row);
                if (prev == kEmpty || prev == row) break;
            }
            h = (h + 1) & mask;
        }
        const unsigned r = atomicAdd(cnt + h, 1u);
        pe[i] = (uint32_t)h;
        pr[i] = r;
        if (r == 1) c->dup = 1;
    }
}

__global__ void __launch_bounds__(256) k_sgd_dup_base(const unsigned* __restrict__ cnt, uint64_t m,
                                                      unsigned* base, uint32_t* dupent, SgdCounters* c) {
    if (!c->dup) return;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned k = cnt[e];
        if (k < 2) continue;
        base[e] = atomicAdd(&c->dup_total, k);
        dupent[atomicAdd(&c->dup_entries, 1u)] = (uint32_t)e;
    }
}

__global__ void __launch_bounds__(256) k_sgd_dup_fill(const uint32_t* __restrict__ pe,
                                                      const uint32_t* __restrict__ pr, uint64_t n,
                                                      const unsigned* __restrict__ cnt,
                                                      const unsigned* __restrict__ base,
                                                      uint32_t* list, const SgdCounters* c) {
    if (!c->dup) return;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = pe[i];
        if (e != kNone32 && cnt[e] > 1) list[base[e] + pr[i]] = (uint32_t)i;
    }
}

__global__ void __launch_bounds__(256) k_sgd_apply(TableDev t, const uint64_t* __restrict__ rows,
                                                   const float* __restrict__ grads, uint64_t n,
                                                   const uint32_t* __restrict__ pe,
                                                   const unsigned* __restrict__ cnt, float lr,
                                                   float beta, bool vec, unsigned width,
                                                   uint64_t gen_clock, const SgdCounters* c) {
    const uint64_t bad = c->bad;
    const uint64_t lim = bad < n ? bad : n;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned sub = (unsigned)(gtid % width);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x / width;
    for (uint64_t i = gtid / width; i < lim; i += stride) {
        const uint32_t e = pe[i];
        const uint64_t row = rows[i];
        // the pending bit (an L2 hit) is loaded in the same round as the occurrence count, so
        // the deferred reset adds no dependent round trip (only this group touches the bit)
        const bool pend = reset_pending(t, row);
        if (cnt[e] != 1) continue;  // repeated rows: k_sgd_dups
        apply_row(t, row, grads + i * t.dim, lr, beta, vec, sub, width, pend);
        if (sub == 0) {
            if (pend) clear_pending(t, row);
            set_trained(t, row);
            if (bad == kEmpty) t.row_gen[row] = gen_clock;  // table.cpp:179
        }
    }
}

__global__ void __launch_bounds__(256) k_sgd_dups(TableDev t, const uint64_t* __restrict__ rows,
                                                  const float* __restrict__ grads,
                                                  const unsigned* __restrict__ cnt,
                                                  const unsigned* __restrict__ base,
                                                  const uint32_t* __restrict__ dupent, uint32_t* list,
                                                  float lr, float beta, bool vec, uint64_t gen_clock,
                                                  const SgdCounters* c) {
    if (!c->dup) return;
    const uint64_t bad = c->bad;
    const unsigned lane = lane_id();
    const unsigned nent = c->dup_entries;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t d = warp; d < nent; d += nwarps) {
        const uint32_t e = dupent[d];
        const unsigned k = cnt[e];
        uint32_t* seg = list + base[e];
        if (lane == 0) {  // arrival order -> position order (insertion sort; rows repeat rarely)
            for (unsigned a = 1; a < k; ++a) {
                const uint32_t v = seg[a];
                unsigned b = a;
                for (; b > 0 && seg[b - 1] > v; --b) seg[b] = seg[b - 1];
                seg[b] = v;
            }
        }
        __syncwarp();
        const uint64_t row = rows[seg[0]];
        bool any = false;
        const bool pend0 = reset_pending(t, row);
        bool pend = pend0;
        for (unsigned a = 0; a < k; ++a) {
            const uint64_t i = seg[a];
            if (i >= bad) break;
            apply_row(t, row, grads + i * t.dim, lr, beta, vec, lane, 32, pend);
            __syncwarp();
            pend = false;  // later occurrences read what the first one wrote
            any = true;
        }
        if (lane == 0 && any) {
            if (pend0) clear_pending(t, row);
            set_trained(t, row);
            if (bad == kEmpty) t.row_gen[row] = gen_clock;
        }
    }
}

__global__ void __launch_bounds__(256) k_sgd_clean(const uint32_t* __restrict__ pe, uint64_t n,
                                                   unsigned long long* key, unsigned* cnt) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = pe[i];
        if (e == kNone32) continue;
        key[e] = kEmpty;
        cnt[e] = 0;
    }
}

}  // namespace

uint64_t run_sgd_step(Table& t, const uint64_t* rows, uint64_t n, const float* grads, float lr,
                      float beta, cudaStream_t st) {
    uint64_t m = 1024;
    while (m < 2 * n) m <<= 1;
    if (t.g_cap < m) {
        t.g_key.reserve(m * 8);
        t.g_cnt.reserve(m * 4);
        t.g_base.reserve(m * 4);
        MPZCH_CUDA(cudaMemsetAsync(t.g_key.p, 0xff, m * 8, st));
        MPZCH_CUDA(cudaMemsetAsync(t.g_cnt.p, 0, m * 4, st));
        t.g_cap = m;
    }
    m = t.g_cap;
    t.g_pe.reserve(n * 4);
    t.g_pr.reserve(n * 4);
    t.g_list.reserve(n * 4);
    t.g_dupent.reserve(n * 4);
    t.g_ctr.reserve(sizeof(SgdCounters));
    SgdCounters* c = t.g_ctr.as<SgdCounters>();
    k_sgd_init<<<1, 1, 0, st>>>(c);  // (a pageable H2D copy would stall the host on the stream)
    unsigned long long* key = t.g_key.as<unsigned long long>();
    unsigned* cnt = t.g_cnt.as<unsigned>();
    unsigned* base = t.g_base.as<unsigned>();
    uint32_t* pe = t.g_pe.as<uint32_t>();
    uint32_t* pr = t.g_pr.as<uint32_t>();
    const unsigned B = 256;
    const unsigned gN = grid_for(n, B);
    k_sgd_prep<<<gN, B, 0, st>>>(t.dev, rows, n, key, cnt, pe, pr, m - 1, c);
    k_sgd_dup_base<<<grid_for(m, B), B, 0, st>>>(cnt, m, base, t.g_dupent.as<uint32_t>(), c);
    k_sgd_dup_fill<<<gN, B, 0, st>>>(pe, pr, n, cnt, base, t.g_list.as<uint32_t>(), c);
    const bool vec = (t.dim & 3u) == 0 && ((uintptr_t)grads & 15u) == 0;
    const uint32_t lanes_needed = vec ? t.dim / 4 : t.dim;
    unsigned width = 1;
    while (width < lanes_needed && width < 32) width <<= 1;
    k_sgd_apply<<<std::min<unsigned>(grid_for(n * width, B), 148 * 32), B, 0, st>>>(t.dev, rows, grads, n, pe, cnt, lr, beta, vec,
                                                      width, t.gen_clock, c);
    k_sgd_dups<<<std::min<unsigned>(grid_for(n * 32, B), 148 * 16), B, 0, st>>>(t.dev, rows, grads, cnt, base,
                                                  t.g_dupent.as<uint32_t>(), t.g_list.as<uint32_t>(),
                                                  lr, beta, vec, t.gen_clock, c);
    k_sgd_clean<<<gN, B, 0, st>>>(pe, n, key, cnt);
    t.launches += 7;
    MPZCH_CUDA(cudaGetLastError());
    uint64_t bad = ~0ull;
    MPZCH_CUDA(cudaMemcpyAsync(&bad, &c->bad, 8, cudaMemcpyDeviceToHost, st));
    MPZCH_CUDA(cudaStreamSynchronize(st));
    return bad;
}

}  // namespace mpzch_b200
