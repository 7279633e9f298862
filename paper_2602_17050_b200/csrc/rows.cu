// rows.cu -- embedding-row payload kernels: table init and eviction reset.
//
// draw_row (proj/src/embedding_store.cpp:12-18) seeds SplitMix64 with
// mix64(row, init_seed) and draws w[j] = float((2*u_j - 1) * (1/sqrt(dim))),
// u_j = (next() >> 11) * 2^-53 (proj/include/mpzch/rng.hpp:23).  The stream
// state after j+1 steps is s0 + (j+1)*golden, so every element is computed
// independently and stored as 16-byte vectors.  2*u-1 is exact; the product
// is one FP64 rounding (__dmul_rn: no contraction), then __double2float_rn,
// exactly the reference's static_cast<float> sequence.
// reset_row (embedding_store.cpp:62-68): redraw + momentum 0 + trained 0 -- written by the batch
// (MPZCH_RESET_EAGER, the reference's order) or marked pending and fused into the next
// sgd_step / gather of the row (MPZCH_RESET_DEFERRED: same observable state, one row write).
#include <cuda_runtime.h>

#include "common.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

// init: grid-stride over (row, quad) for dim % 4 == 0, else over elements
__global__ void __launch_bounds__(256) k_draw_all(TableDev t) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t held = t.row_hi - t.row_lo;
    if ((t.dim & 3u) == 0) {
        const uint64_t quads = t.dim / 4;
        const uint64_t nq = held * quads;
        float4* w4 = reinterpret_cast<float4*>(t.weights + t.row_lo * t.dim);
        for (uint64_t q = tid; q < nq; q += stride) {
            const uint64_t row = t.row_lo + q / quads;
            const uint64_t j = (q % quads) * 4;
            const uint64_t s0 = mix64(row, t.init_seed);
            float4 w;
            w.x = draw_elem(s0, j, t.bound);
            w.y = draw_elem(s0, j + 1, t.bound);
            w.z = draw_elem(s0, j + 2, t.bound);
            w.w = draw_elem(s0, j + 3, t.bound);
            w4[q] = w;
        }
    } else {
        const uint64_t ne = held * t.dim;
        for (uint64_t x = tid; x < ne; x += stride) {
            const uint64_t row = t.row_lo + x / t.dim;
            const uint64_t j = x % t.dim;
            t.weights[row * t.dim + j] = draw_elem(mix64(row, t.init_seed), j, t.bound);
        }
    }
}

// one row's reset by a warp: draw_row from the row's SplitMix64 seed s0 = mix64(row, init_seed),
// momentum 0 (embedding_store.cpp:62-68); the trained bit is the caller's
__device__ __forceinline__ void reset_row_body(const TableDev& t, uint64_t row, uint64_t s0, unsigned lane) {
    float* w = t.weights + row * t.dim;
    float* m = t.momentum + row * t.dim;
    if ((t.dim & 3u) == 0) {
        float4* w4 = reinterpret_cast<float4*>(w);
        float4* m4 = reinterpret_cast<float4*>(m);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t q = lane; q < t.dim / 4; q += 32) {
            w4[q] = draw_quad(s0, q, t.bound);
            m4[q] = z;
        }
    } else {
        for (uint32_t j = lane; j < t.dim; j += 32) {
            w[j] = draw_elem(s0, j, t.bound);
            m[j] = 0.f;
        }
    }
}

__device__ __forceinline__ void reset_row_warp(const TableDev& t, uint64_t row, unsigned lane) {
    reset_row_body(t, row, mix64(row, t.init_seed), lane);
    if (lane == 0) clear_trained(t, row);
}

// reset: a warp takes 32 listed rows at a time (one coalesced load of their indices, so no
// row waits on its own index load) and resets them one after another, a row's dim floats
// spread over the lanes; rows may repeat (LRU double eviction), the operation is idempotent.
__global__ void __launch_bounds__(256) k_reset_rows(TableDev t, const uint64_t* __restrict__ rows,
                                                    const unsigned* __restrict__ count) {
    pdl_wait();
    const unsigned n = *count;
    const unsigned lane = lane_id();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r0 = warp * 32; r0 < n; r0 += nwarps * 32) {
        const bool have = r0 + lane < n;
        const uint64_t mine = have ? rows[r0 + lane] : 0;
        // each lane derives its own row's seed and clears its own row's trained bit, so the
        // per-row work left is the draw and the stores (the kernel is issue-bound: ncu 69% of
        // issue slots busy with the seed recomputed by every lane for every row)
        const uint64_t s0m = mix64(mine, t.init_seed);
        if (have) clear_trained(t, mine);
        const unsigned cnt = n - r0 < 32 ? (unsigned)(n - r0) : 32u;
        for (unsigned k = 0; k < cnt; ++k)
            reset_row_body(t, __shfl_sync(0xffffffffu, mine, k), __shfl_sync(0xffffffffu, s0m, k), lane);
    }
}

// deferred mode: the batch only marks its evicted rows reset-pending (one bit per row); the
// next sgd_step that touches a row computes from the closed-form draw instead of reading the
// row (train.cu), gathers draw it on the fly, other readers flush first (k_flush_pending)
__global__ void __launch_bounds__(256) k_mark_pending(TableDev t, const uint64_t* __restrict__ rows,
                                                      const unsigned* __restrict__ count) {
    pdl_wait();
    const unsigned n = *count;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = rows[i] - t.row_lo;
        atomicOr(t.pend_bits + (r >> 5), 1u << (r & 31));
    }
}

// materialise every pending reset: a warp reads 32 bitmap words (1024 rows) per step and
// resets the pending rows among them, then clears the words
__global__ void __launch_bounds__(256) k_flush_pending(TableDev t) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t words = (t.row_hi - t.row_lo + 31) / 32;
    for (uint64_t w0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; w0 < words; w0 += warps * 32) {
        const uint32_t mine = w0 + lane < words ? t.pend_bits[w0 + lane] : 0u;
        unsigned any = __ballot_sync(0xffffffffu, mine != 0);
        while (any) {
            const unsigned src = __ffs(any) - 1;
            any &= any - 1;
            uint32_t bits = __shfl_sync(0xffffffffu, mine, src);
            const uint64_t rb = t.row_lo + (w0 + src) * 32;
            while (bits) {
                const unsigned b = __ffs(bits) - 1;
                bits &= bits - 1;
                reset_row_warp(t, rb + b, lane);
            }
        }
        if (mine) t.pend_bits[w0 + lane] = 0u;
    }
}

__global__ void k_write_slots(TableDev t, const uint64_t* __restrict__ g, const uint64_t* __restrict__ ids,
                              const uint64_t* __restrict__ metas, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        t.ident[g[i]] = ids[i];
        t.meta[g[i]] = metas[i];
    }
}

// the tags of written slots, from the identity array once every store above has landed (a slot
// listed twice holds one of its writers' ids; the tag follows whichever it is)
__global__ void k_retag_slots(TableDev t, const uint64_t* __restrict__ g, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        store_tag(t, g[i], t.ident[g[i]]);
}

// Hole check: every id stored inside its own probe window at
// offset o must see neither EMPTY nor another copy of itself in [home, home+o).
__global__ void __launch_bounds__(256) k_hole_check(TableDev t, unsigned* bad) {
    for (uint64_t g = t.row_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < t.row_hi;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t id = t.ident[g];
        if (id == kEmpty) continue;
        if (id >> 63) { atomicExch(bad, 1u); continue; }  // stray claim word
        const uint32_t s = shard_of(id, t);
        const ShardDev sd = t.shards[s];
        // the id must live in its own shard's segment to be reachable; if it does
        // not, it is a foreign occupant for everybody and cannot create a hole
        if (g < sd.offset || g >= sd.offset + sd.cap.d) continue;
        const uint64_t h = home_of(id, sd, t.seed);
        const uint64_t loc = g - sd.offset;
        const uint64_t o = loc >= h ? loc - h : loc + sd.cap.d - h;
        if (o >= t.P) continue;  // outside its window: invisible, harmless
        uint64_t x = h;
        for (uint64_t k = 0; k < o; ++k) {
            const uint64_t v = t.ident[sd.offset + x];
            if (v == kEmpty || v == id) { atomicExch(bad, 1u); break; }
            if (++x == sd.cap.d) x = 0;
        }
    }
}

// Delta cut gather (DeltaSource::cut, proj/src/publish.cpp:288-305): for each dirty row,
// its identity word and its weights.  One warp per row, 16-byte copies.
__global__ void __launch_bounds__(256) k_gather_rows(TableDev t, const uint64_t* __restrict__ rows,
                                                     uint64_t n, uint64_t* __restrict__ out_ids,
                                                     float* __restrict__ out_w) {
    const unsigned lane = lane_id();
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t row = rows[r];
        if (lane == 0) out_ids[r] = t.ident[row];
        if (!out_w) continue;
        const float* src = t.weights + row * t.dim;
        float* dst = out_w + r * t.dim;
        if ((t.dim & 3u) == 0) {
            for (uint32_t q = lane; q < t.dim / 4; q += 32)
                reinterpret_cast<float4*>(dst)[q] = reinterpret_cast<const float4*>(src)[q];
        } else {
            for (uint32_t j = lane; j < t.dim; j += 32) dst[j] = src[j];
        }
    }
}

}  // namespace

__global__ void k_trained_bytes(TableDev t, uint64_t row0, uint64_t n, uint8_t* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = row0 + i - t.row_lo;
        out[i] = (uint8_t)((t.trained[r >> 5] >> (r & 31)) & 1u);
    }
}

__global__ void k_set_trained_flag(TableDev t, uint64_t row, int v) {
    if (v) set_trained(t, row);
    else clear_trained(t, row);
}

// the trained flags of rows [row0, row0 + n) as bytes (the reference's layout), synchronous
void copy_trained_bytes(Table& t, uint64_t row0, uint64_t n, uint8_t* host_out) {
    if (!n) return;
    t.sb_buf.reserve(n);
    k_trained_bytes<<<grid_for(n, 256, 148u * 8u), 256, 0, t.stream>>>(t.dev, row0, n, t.sb_buf.as<uint8_t>());
    ++t.launches;
    MPZCH_CUDA(cudaGetLastError());
    MPZCH_CUDA(cudaMemcpyAsync(host_out, t.sb_buf.p, n, cudaMemcpyDeviceToHost, t.stream));
    MPZCH_CUDA(cudaStreamSynchronize(t.stream));
}

void set_trained_flag(Table& t, uint64_t row, bool v) {
    k_set_trained_flag<<<1, 1, 0, t.stream>>>(t.dev, row, v ? 1 : 0);
    ++t.launches;
    MPZCH_CUDA(cudaGetLastError());
    MPZCH_CUDA(cudaStreamSynchronize(t.stream));
}

void preload_row_kernels() {
    preload_kernel((const void*)k_reset_rows);
    preload_kernel((const void*)k_mark_pending);
    preload_kernel((const void*)k_flush_pending);
}

void run_gather_rows(const Table& t, const uint64_t* rows, uint64_t n, uint64_t* out_ids, float* out_w,
                     cudaStream_t st) {
    if (!n) return;
    k_gather_rows<<<grid_for(n * 32, 256, 148u * 16u), 256, 0, st>>>(t.dev, rows, n, out_ids, out_w);
}

void launch_init_table(Table& t) {
    if (t.dim == 0 || t.held_rows() == 0) return;
    k_draw_all<<<148 * 16, 256, 0, t.stream>>>(t.dev);
    ++t.launches;
    MPZCH_CUDA(cudaGetLastError());
}

void launch_reset_rows(Table& t, const uint64_t* rows, const unsigned* count, cudaStream_t st) {
    if (t.dev.pend_bits) {
        launch_pdl(k_mark_pending, 148 * 8, 256, st, t.dev, rows, count);
        t.resets_pending = true;
    } else {
        launch_pdl(k_reset_rows, 148 * 8, 256, st, t.dev, rows, count);
    }
    ++t.launches;
}

void flush_resets(Table& t, cudaStream_t st) {
    if (!t.resets_pending || t.dim == 0) return;
    k_flush_pending<<<grid_for((t.held_rows() + 1023) / 1024 * 32, 256, 148u * 16u), 256, 0, st>>>(t.dev);
    ++t.launches;
    MPZCH_CUDA(cudaGetLastError());
    t.resets_pending = false;
}

void launch_write_slots(Table& t, const uint64_t* g, const uint64_t* ids, const uint64_t* metas,
                        uint64_t n, cudaStream_t st) {
    if (!n) return;
    k_write_slots<<<grid_for(n, 256), 256, 0, st>>>(t.dev, g, ids, metas, n);
    ++t.launches;
    if (t.dev.tag) {
        k_retag_slots<<<grid_for(n, 256), 256, 0, st>>>(t.dev, g, n);
        ++t.launches;
    }
}

bool run_hole_check(Table& t) {
    unsigned* d_bad = nullptr;
    MPZCH_CUDA(cudaMallocAsync((void**)&d_bad, sizeof(unsigned), t.stream));
    MPZCH_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), t.stream));
    k_hole_check<<<grid_for(t.held_rows(), 256), 256, 0, t.stream>>>(t.dev, d_bad);
    ++t.launches;
    unsigned bad = 0;
    MPZCH_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, t.stream));
    MPZCH_CUDA(cudaFreeAsync(d_bad, t.stream));
    MPZCH_CUDA(cudaStreamSynchronize(t.stream));
    return bad == 0;
}

}  // namespace mpzch_b200
