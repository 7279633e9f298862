// sharded.cu -- the row-sharded table as one C-ABI object per rank, with the whole
// per-batch protocol enqueued on the rank's stream: ONE host wait per batch (the caller's).
//
// The S logical shards of one TableLayout (proj/include/mpzch/shard_router.hpp:13-29) are spread
// over G ranks in contiguous blocks (rank r holds {s : s*G/S == r}); global rows are those of the
// single table, so every slot is identical for any G.  A batch is split into G contiguous slices
// (rank r holds global positions [base_r, base_r + n_r)).  It replaces the reference's in-process
// shard loop (proj/src/batch_engine.cpp:160-211): every probe / claim / commit is shard-local
// (proj/include/mpzch/batch_engine.hpp:39-43), so the only exchange is ids out and slots back.
//
// Each rank owns an EXCHANGE REGION in its HBM that the other ranks write over NVLink (P2P in
// one process, CUDA IPC across processes): a header of per-source control records and epoch
// flags, receive buffers (ids, features, source positions), result buffers (slots, outcomes,
// first-evicted marks) and the global evicted list.  Phases, all kernels on the rank's stream:
//
//   P1  validate the slice (first invalid position; per-feature TTL overflow) and count its
//       positions per owner (stable partition counts, route.cu); publish {n, bad, over, counts}
//       into every rank's control record + release flag (system scope); wait for every rank's
//       record (acquire spin on the local flags) and derive, identically on every rank, the
//       batch's fate (length > invalid id > overflow: batch_engine.cpp:82-94, eviction.cpp:26-28,
//       the first invalid GLOBAL position), this slice's base, its offsets in every owner's
//       receive buffer and the received count R;
//   P2  route-scatter: partition + store (id, feature, source position) straight into the
//       owners' receive buffers (one kernel, route.cu), fence, flag; wait for every source;
//   P3  the owner remaps its R received positions (the fast path with the count on the device:
//       k_sh_adopt; sources arrive rank-ordered and each stably partitioned, so receive order is
//       global first-occurrence order and the claim ranks are the single table's);
//   P4  return-scatter: every result (slot, outcome, first-evicted mark) stored straight into
//       the source's result buffers at the source position, fence, flag; wait;
//   P5  (TTL / LRU) the canonical evicted list: each rank compacts its slice's marks in
//       position order, publishes its count, writes its segment into every rank's list at the
//       rank-ordered offset; wait -- the list is the global one on every rank.
//
// Errors are decided on the device by every rank alike, so every rank takes the same branch,
// skips the same work and still raises every flag (no rank can be left waiting).  Waits time
// out (MPZCH_PEER_TIMEOUT_MS, default 60 s) into a sticky error instead of hanging.  Batches the
// device-count fast path cannot run (LRU's claim-vs-rounds decision, tables with raw-imported
// holes, forced paths, per-feature TTLs that may overflow) take one extra host round trip to
// learn R and run the ordinary remap.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "compact.cuh"
#include "table.hpp"

namespace mpzch_b200 {

namespace {

constexpr uint32_t kMaxG = 64;
enum : uint32_t { kFCtrl = 0, kFScat = 1, kFRes = 2, kFEvc = 3, kFEv = 4, kNFlags = 5 };

// written by source s into every rank's header (ctrl[s])
struct ShCtrl {
    uint64_t n, bad, over, evc;
    uint64_t counts[kMaxG];
};
struct ShHeader {
    uint64_t flag[kNFlags][kMaxG];  // epoch of the phase's last signal from rank s
    ShCtrl ctrl[kMaxG];
};

// this rank's per-batch device state (its prefix is ShStateView, read by the owner's remap)
struct ShState {
    unsigned long long failed, R;
    unsigned long long local_bad, local_over;
    unsigned long long err_len, err_cap, err_bad, err_over, timeout;
    unsigned long long base, ntotal;
    unsigned int ev_mine, done;  // done: k_sh_finish's finished-block count
    unsigned long long ev_off, ev_total;
    unsigned long long my_off[kMaxG];
    unsigned long long roff[kMaxG + 1];
};
static_assert(offsetof(ShState, failed) == offsetof(ShStateView, failed), "ShStateView prefix");
static_assert(offsetof(ShState, R) == offsetof(ShStateView, R), "ShStateView prefix");

struct Layout {
    size_t ids, feats, src, rslots, roc, rmark, ev, bytes;
};

Layout layout_for(uint64_t cap) {
    auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
    Layout L{};
    size_t o = up(sizeof(ShHeader));
    L.ids = o;    o = up(o + cap * 8);
    L.feats = o;  o = up(o + cap * 4);
    L.src = o;    o = up(o + cap * 4);
    L.rslots = o; o = up(o + cap * 8);
    L.roc = o;    o = up(o + cap);
    L.rmark = o;  o = up(o + cap);
    L.ev = o;     o = up(o + cap * 8);
    L.bytes = o;
    return L;
}

struct ShPeers {
    unsigned long long region[kMaxG];  // every rank's exchange region (addresses valid here)
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ ShHeader* hdr(const ShPeers& P, uint32_t q) {
    return reinterpret_cast<ShHeader*>(P.region[q]);
}

// thread s < G spins on flags[s] until it reaches `e`; true if every flag arrived in time
__device__ bool wait_all(const uint64_t* flags, uint32_t G, uint64_t e, uint64_t timeout_ns, ShState* st,
                         uint32_t kind, uint32_t rank) {
    __shared__ int late;
    if (threadIdx.x == 0) late = 0;
    __syncthreads();
    const uint32_t s = threadIdx.x;
    if (s < G && !st->timeout) {
        const uint64_t t0 = globaltimer();
        unsigned k = 0;
        while (ld_acquire_sys(flags + s) < e) {
            if ((++k & 255u) == 0 && globaltimer() - t0 > timeout_ns) {
                atomicExch(&late, 1);
                printf("mpzch row-sharded: rank %u timed out in phase %u waiting for rank %u "
                       "(flag %llu, batch %llu)\n", rank, kind, s,
                       (unsigned long long)ld_acquire_sys(flags + s), (unsigned long long)e);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
    if (late || st->timeout) {
        if (threadIdx.x == 0) {
            st->timeout = 1;
            st->failed = 1;
        }
        return false;
    }
    return true;
}

// the per-batch state back to its start (run by the previous batch's last kernel, and once at
// creation): a rank that stopped answering fails every later batch
__device__ __forceinline__ void reset_state(ShState* st) {
    st->failed = st->timeout ? 1 : 0;
    st->R = 0;
    st->local_bad = ~0ull;
    st->local_over = 0;
    st->err_len = st->err_cap = st->err_over = 0;
    st->err_bad = ~0ull;
    st->ev_mine = 0;
    st->ev_off = st->ev_total = 0;
}

__global__ void k_sh_reset(ShState* st) {
    if (threadIdx.x == 0) reset_state(st);
}

// P1a' (per-feature TTLs that can overflow at this `now` only): does any position's feature
// (eviction.cpp:20-30).  The first invalid position is found by the route count (route.cu).
__global__ void __launch_bounds__(256) k_sh_overflow(const uint32_t* __restrict__ feats, uint64_t n,
                                                     uint64_t limit, uint64_t def_ttl, const uint32_t* keys,
                                                     const uint64_t* vals, uint32_t nk, ShState* st) {
    pdl_wait();
    bool over = false;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t f = feats ? feats[i] : 0;
        uint64_t ttl = def_ttl;
        for (uint32_t k = 0; k < nk; ++k)
            if (keys[k] == f) ttl = vals[k];
        over |= ttl > limit;
    }
    if (__any_sync(0xffffffffu, over) && lane_id() == 0) atomicExch(&st->local_over, 1ull);
}

// P1b: publish this slice's record into every rank's header, raise the control flags, wait for
// every rank's record and derive the batch's fate, this slice's offsets and the received count
__global__ void k_sh_publish_plan(ShPeers P, ShHeader* mine, uint32_t rank, uint32_t G, uint64_t e, uint64_t n,
                                  uint64_t over_all, const unsigned* part_totals, uint64_t cap,
                                  uint64_t timeout_ns, ShState* st) {
    pdl_wait();
    const uint32_t q = threadIdx.x;
    if (q < G) {
        ShCtrl* c = &hdr(P, q)->ctrl[rank];
        c->n = n;
        c->bad = st->local_bad;
        c->over = over_all | st->local_over;
        for (uint32_t p = 0; p < G; ++p) c->counts[p] = (n && part_totals) ? part_totals[p] : 0;
        __threadfence_system();
        st_release_sys(&hdr(P, q)->flag[kFCtrl][rank], e);
    }
    if (!wait_all(mine->flag[kFCtrl], G, e, timeout_ns, st, kFCtrl, rank)) return;
    if (threadIdx.x != 0) return;
    const volatile ShCtrl* c = mine->ctrl;
    unsigned long long base = 0, total = 0, bad = ~0ull, over = 0;
    for (uint32_t s = 0; s < G; ++s) {
        const unsigned long long ns = c[s].n, bs = c[s].bad;
        if (s == rank) base = total;
        if (bs != ~0ull) bad = min(bad, total + bs);
        over |= c[s].over;
        total += ns;
    }
    st->base = base;
    st->ntotal = total;
    if (total > 0xffffffffull) st->err_len = 1;        // batch_engine.cpp:82-83
    else if (total > cap) st->err_cap = 1;             // the exchange buffers' capacity
    else if (bad != ~0ull) st->err_bad = bad;          // batch_engine.cpp:90-94
    else if (over) st->err_over = 1;                   // eviction.cpp:26-28
    if (st->err_len || st->err_cap || st->err_bad != ~0ull || st->err_over) {
        st->failed = 1;
        return;
    }
    for (uint32_t q2 = 0; q2 < G; ++q2) {
        unsigned long long off = 0;
        for (uint32_t s = 0; s < rank; ++s) off += c[s].counts[q2];
        st->my_off[q2] = off;
    }
    unsigned long long r = 0;
    for (uint32_t s = 0; s < G; ++s) {
        st->roff[s] = r;
        r += c[s].counts[rank];
    }
    st->roff[G] = r;
    st->R = r;
}

// raise this rank's `kind` flag in every rank's header (the previous kernel's peer stores are
// flushed: PDL waits for its completion, and the release is system scope), then wait for
// every rank's
__global__ void k_sh_signal_wait(ShPeers P, ShHeader* mine, uint32_t kind, uint32_t rank, uint32_t G, uint64_t e,
                                 uint64_t timeout_ns, ShState* st) {
    pdl_wait();
    const uint32_t q = threadIdx.x;
    if (q < G) {
        __threadfence_system();
        st_release_sys(&hdr(P, q)->flag[kind][rank], e);
    }
    wait_all(mine->flag[kind], G, e, timeout_ns, st, kind, rank);
}

// P4: every received position's result straight into its source's result buffers
__global__ void __launch_bounds__(256) k_sh_return(const ShState* st, const uint32_t* __restrict__ src,
                                                   const uint64_t* __restrict__ slots,
                                                   const uint8_t* __restrict__ oc, uint8_t* mark, int clear,
                                                   ShPeers P, Layout L, uint32_t G) {
    pdl_wait();
    __shared__ unsigned long long roff[kMaxG + 1];
    for (uint32_t s = threadIdx.x; s <= G; s += blockDim.x) roff[s] = st->roff[s];
    __syncthreads();
    if (st->failed) return;
    const uint64_t R = st->R;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < R; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = G;  // roff[lo] <= j < roff[hi]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (roff[mid] <= j) lo = mid; else hi = mid;
        }
        const uint32_t p = src[j];
        const unsigned long long b = P.region[lo];
        reinterpret_cast<uint64_t*>(b + L.rslots)[p] = slots[j];
        reinterpret_cast<uint8_t*>(b + L.roc)[p] = oc[j];
        uint8_t m = 0;
        if (mark) {
            m = mark[j];
            if (clear && m) mark[j] = 0;
        }
        reinterpret_cast<uint8_t*>(b + L.rmark)[p] = m;
    }
    __threadfence_system();
}

// P5a: the evicted-list counts (published + planned in one kernel)
__global__ void k_sh_evc_plan(ShPeers P, ShHeader* mine, uint32_t rank, uint32_t G, uint64_t e,
                              uint64_t timeout_ns, ShState* st) {
    pdl_wait();
    const uint32_t q = threadIdx.x;
    if (q < G) {
        hdr(P, q)->ctrl[rank].evc = st->failed ? 0 : st->ev_mine;
        __threadfence_system();
        st_release_sys(&hdr(P, q)->flag[kFEvc][rank], e);
    }
    if (!wait_all(mine->flag[kFEvc], G, e, timeout_ns, st, kFEvc, rank)) return;
    if (threadIdx.x != 0) return;
    const volatile ShCtrl* c = mine->ctrl;
    unsigned long long off = 0, total = 0;
    for (uint32_t s = 0; s < G; ++s) {
        if (s == rank) off = total;
        total += c[s].evc;
    }
    st->ev_off = off;
    st->ev_total = total;
}

// P5b: this slice's segment of the canonical evicted list into every rank's list
__global__ void __launch_bounds__(256) k_sh_ev_scatter(const ShState* st, const uint64_t* __restrict__ mine,
                                                       ShPeers P, size_t ev_at, uint32_t G) {
    pdl_wait();
    if (st->failed) return;
    const uint64_t m = st->ev_mine, off = st->ev_off;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < m * G; x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = x / G;
        const uint32_t q = (uint32_t)(x % G);
        reinterpret_cast<uint64_t*>(P.region[q] + ev_at)[off + k] = mine[k];
    }
    __threadfence_system();
}

// last kernel of a batch: this slice's results (and the evicted list) to the caller's buffers,
// the batch's state and owner-side counters straight into the pinned result slot (mapped host
// memory: no copy operation), then the state back to its start for the next batch
__global__ void __launch_bounds__(256) k_sh_finish(ShState* st, const BatchCounters* ctr, uint64_t n,
                                                   const uint64_t* __restrict__ rslots,
                                                   const uint8_t* __restrict__ roc, uint64_t* __restrict__ out_slots,
                                                   uint8_t* __restrict__ out_oc, const uint64_t* __restrict__ ev_all,
                                                   uint64_t* __restrict__ out_ev, uint64_t ev_cap, ShState* h_st,
                                                   BatchCounters* h_ctr, unsigned* done) {
    pdl_wait();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (!st->failed) {
        for (uint64_t i = tid; i < n; i += stride) {
            out_slots[i] = rslots[i];
            out_oc[i] = roc[i];
        }
        if (out_ev) {
            const uint64_t m = min((uint64_t)st->ev_total, ev_cap);
            for (uint64_t k = tid; k < m; k += stride) out_ev[k] = ev_all[k];
        }
    }
    if (tid == 0) {
        *h_st = *st;
        if (ctr) *h_ctr = *ctr;
    }
    // the last block to finish resets the state for the next batch (every block has read it)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {
            reset_state(st);
            *done = 0;
        }
    }
}

struct EmitSlots {
    const uint64_t* slots;
    uint64_t* out;
    __device__ void operator()(uint64_t i, unsigned k) const { out[k] = slots[i]; }
};

struct ShRecord {  // what mpzch_sharded_export hands to the other ranks
    cudaIpcMemHandle_t handle;
    uint64_t bytes, cap;
    uint32_t rank, world;
    uint8_t pad[MPZCH_SHARDED_RECORD_BYTES - sizeof(cudaIpcMemHandle_t) - 24];
};
static_assert(sizeof(ShRecord) == MPZCH_SHARDED_RECORD_BYTES, "sharded record size");

}  // namespace

struct ShardedRank {
    static constexpr int kRing = 8;
    std::unique_ptr<Table> t;
    uint32_t rank = 0, G = 1;
    uint64_t cap = 0;
    int device = 0;
    Layout L{};
    uint8_t* region = nullptr;
    ShPeers peers{};
    std::vector<void*> imported;
    bool connected = false;
    uint64_t epoch = 0;
    uint64_t timeout_ns = 60ull * 1000 * 1000 * 1000;
    ShState* d_state = nullptr;
    BatchCounters* d_ctr = nullptr;
    DevBuf loc_slots, loc_oc, loc_mark, my_ev, blk;
    DevBuf g_ids, g_feats, g_slots, g_oc, g_ev;  // host-buffer group call staging
    cudaStream_t g_stream = nullptr;
    std::vector<uint32_t> s2p;
    struct Slot {
        bool busy = false;
        uint64_t ticket = 0, n = 0;
        int host_waits = 1, path = MPZCH_PATH_AUTO;
        cudaEvent_t done = nullptr;
        std::string fallback_msg;
        mpzch_status fallback_status = MPZCH_OK;
    };
    Slot slots[kRing];
    ShState* h_state = nullptr;         // pinned ring (mapped)
    BatchCounters* h_ctr = nullptr;     // pinned ring (mapped)
    ShState* hd_state = nullptr;        // their device addresses
    BatchCounters* hd_ctr = nullptr;
    cudaStream_t last_stream = nullptr;
    cudaEvent_t last_done = nullptr;
    // results of completed batches (by ticket, like the table's ring)
    struct Result {
        uint64_t ticket = ~0ull;
        mpzch_status status = MPZCH_OK;
        std::string msg;
        uint64_t ev_total = 0;
        mpzch_batch_stats stats{};
        int host_waits = 0;
    };
    Result results[64];
    mpzch_batch_stats last{};
    int last_host_waits = 0;

    ShardedRank(const uint64_t* caps, uint32_t S, uint32_t P, uint64_t seed, uint32_t dim, uint64_t init_seed,
                int dev, uint32_t r, uint32_t world, uint64_t max_batch) {
        if (world == 0 || world > kMaxG) throw Error{MPZCH_EINVAL, "row-sharded mode: 1..64 ranks"};
        if (r >= world) throw Error{MPZCH_EINVAL, "rank out of range"};
        if (S < world)
            throw Error{MPZCH_EINVAL, "row-sharded mode needs at least one logical shard per rank"};
        if (max_batch == 0 || max_batch > 0xffffffffull)
            throw Error{MPZCH_EINVAL, "max_batch must lie in [1, 2^32 - 1]"};
        rank = r;
        G = world;
        cap = max_batch;
        device = dev;
        s2p.resize(S);
        uint32_t lo = S, hi = 0;
        for (uint32_t s = 0; s < S; ++s) {
            s2p[s] = (uint32_t)((uint64_t)s * world / S);
            if (s2p[s] == r) {
                lo = std::min(lo, s);
                hi = s + 1;
            }
        }
        t.reset(new Table(caps, S, P, seed, dim, init_seed, dev, lo, hi));
        MPZCH_CUDA(cudaSetDevice(dev));
        // a kernel loaded lazily at its first launch could wait for a peer's spinning kernel
        preload_all_kernels();
        for (const void* k : {(const void*)k_sh_reset, (const void*)k_sh_overflow, (const void*)k_sh_publish_plan,
                              (const void*)k_sh_signal_wait, (const void*)k_sh_return, (const void*)k_sh_evc_plan,
                              (const void*)k_sh_ev_scatter, (const void*)k_sh_finish})
            preload_kernel(k);
        preload_compact<EmitSlots>();
        upload_route_map(*t, s2p.data(), G);
        L = layout_for(cap);
        MPZCH_CUDA(cudaMalloc(&region, L.bytes));
        MPZCH_CUDA(cudaMemset(region, 0, L.bytes));
        MPZCH_CUDA(cudaMalloc(&d_state, sizeof(ShState)));
        MPZCH_CUDA(cudaMemset(d_state, 0, sizeof(ShState)));
        MPZCH_CUDA(cudaMalloc(&d_ctr, sizeof(BatchCounters)));
        // pinned result slots the last kernel of a batch writes directly (mapped host memory)
        MPZCH_CUDA(cudaHostAlloc(&h_state, sizeof(ShState) * kRing, cudaHostAllocMapped));
        MPZCH_CUDA(cudaHostAlloc(&h_ctr, sizeof(BatchCounters) * kRing, cudaHostAllocMapped));
        MPZCH_CUDA(cudaHostGetDevicePointer((void**)&hd_state, h_state, 0));
        MPZCH_CUDA(cudaHostGetDevicePointer((void**)&hd_ctr, h_ctr, 0));
        std::memset(h_ctr, 0, sizeof(BatchCounters) * kRing);
        k_sh_reset<<<1, 32>>>(d_state);
        for (auto& s : slots) MPZCH_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
        loc_slots.reserve(cap * 8);
        loc_oc.reserve(cap);
        loc_mark.reserve(cap);
        MPZCH_CUDA(cudaMemset(loc_mark.p, 0, cap));
        my_ev.reserve(cap * 8);
        blk.reserve(((cap + kCompactChunk - 1) / kCompactChunk + 1) * 4);
        // every buffer a batch can touch is sized here, once: growing one later would cudaFree,
        // which synchronises the device -- with several ranks on one device (tests) that waits
        // for a peer's spin that waits for this rank
        Table& T = *t;
        T.ensure_fast_scratch(cap);  // the owner's remap runs with n = cap as its bound
        T.ensure_pf_scratch(cap);    // per-feature TTL / LRU tables
        T.rt_cnt.reserve(std::max<uint64_t>(1, (cap + 1023) / 1024 * G) * 4);
        T.rt_tot.reserve(kMaxG * 4);
        T.s_featk.reserve(1024 * 4);
        T.s_featv.reserve(1024 * 8);
        if (std::getenv("MPZCH_SHARDED_ALL_PATHS")) reserve_all_paths();
        if (const char* e = std::getenv("MPZCH_PEER_TIMEOUT_MS")) timeout_ns = std::strtoull(e, nullptr, 10) * 1000000ull;
        MPZCH_CUDA(cudaDeviceSynchronize());
    }

    ~ShardedRank() {
        cudaSetDevice(device);
        cudaDeviceSynchronize();
        for (void* p : imported) cudaIpcCloseMemHandle(p);
        for (auto& s : slots)
            if (s.done) cudaEventDestroy(s.done);
        if (g_stream) cudaStreamDestroy(g_stream);
        cudaFree(region);
        cudaFree(d_state);
        cudaFree(d_ctr);
        cudaFreeHost(h_state);
        cudaFreeHost(h_ctr);
    }

    // the host-synchronous fallback's scratch too (ranks sharing a device in one process)
    void reserve_all_paths() {
        Table& T = *t;
        MPZCH_CUDA(cudaSetDevice(device));
        T.ensure_ordered_scratch(cap);
        ensure_rounds_scratch(T, cap, T.stream);
        MPZCH_CUDA(cudaStreamSynchronize(T.stream));
    }

    void set_peer(uint32_t q, uint8_t* base) { peers.region[q] = (unsigned long long)(uintptr_t)base; }

    ShRecord record() const {
        ShRecord r{};
        MPZCH_CUDA(cudaSetDevice(device));
        MPZCH_CUDA(cudaIpcGetMemHandle(&r.handle, region));
        r.bytes = L.bytes;
        r.cap = cap;
        r.rank = rank;
        r.world = G;
        return r;
    }

    void connect_ipc(const uint8_t* recs) {
        if (connected) throw Error{MPZCH_ELOGIC, "rank is already connected"};
        MPZCH_CUDA(cudaSetDevice(device));
        for (uint32_t q = 0; q < G; ++q) {
            ShRecord r;
            std::memcpy(&r, recs + (size_t)q * sizeof(ShRecord), sizeof r);
            if (r.rank != q || r.world != G || r.cap != cap || r.bytes != L.bytes)
                throw Error{MPZCH_EINVAL, "sharded records disagree (rank order, world, or max_batch)"};
            if (q == rank) {
                set_peer(q, region);
                continue;
            }
            void* p = nullptr;
            MPZCH_CUDA(cudaIpcOpenMemHandle(&p, r.handle, cudaIpcMemLazyEnablePeerAccess));
            imported.push_back(p);
            set_peer(q, (uint8_t*)p);
        }
        connected = true;
    }

    // the rest of the batch is enqueued; `fail` (fallback path) records a host-side error
    void finish_slot(int si);
    uint64_t enqueue(const uint64_t* ids, const uint32_t* feats, uint64_t n, uint64_t now, const Policy& pol,
                     uint64_t* out_slots, uint8_t* out_oc, uint64_t* out_ev, uint64_t ev_cap, cudaStream_t st);
    uint64_t wait(uint64_t ticket);
};

void ShardedRank::finish_slot(int si) {
    Slot& sl = slots[si];
    if (!sl.busy) return;
    MPZCH_CUDA(cudaEventSynchronize(sl.done));
    const ShState& s = h_state[si];
    const BatchCounters& c = h_ctr[si];
    Result r;
    r.ticket = sl.ticket;
    r.host_waits = sl.host_waits;
    if (s.timeout) {
        r.status = MPZCH_ENCCL;
        r.msg = "row-sharded batch: a peer rank did not answer in time (the ranks' batches diverged or a rank died)";
    } else if (s.err_len) {
        r.status = MPZCH_ELENGTH;
        r.msg = "batch exceeds 2^32 - 1 positions";
    } else if (s.err_cap) {
        r.status = MPZCH_EINVAL;
        r.msg = "batch exceeds the row-sharded exchange capacity (max_batch)";
    } else if (s.err_bad != ~0ull) {
        r.status = MPZCH_EINVAL;
        r.msg = "invalid id at batch position " + std::to_string(s.err_bad);
    } else if (s.err_over) {
        r.status = MPZCH_EOVERFLOW;
        r.msg = "TTL expiry overflows the 64-bit timestamp range";
    } else if (sl.fallback_status != MPZCH_OK) {
        r.status = sl.fallback_status;
        r.msg = sl.fallback_msg;
    } else if (sl.path == MPZCH_PATH_AUTO && c.err.too_many == 2) {
        r.status = MPZCH_ECUDA;
        r.msg = "internal error: claim invariant violated";
    }
    if (r.status == MPZCH_OK) {
        r.ev_total = s.ev_total;
        mpzch_batch_stats& b = r.stats;
        b.positions = sl.n;
        if (sl.path == MPZCH_PATH_AUTO) {  // the owner side of the batch (its received positions)
            b.new_positions = c.new_count;
            b.new_ids = c.entry_count;
            b.found = c.found;
            b.inserted = c.inserted;
            b.evicted = c.evicted;
            b.collision = c.collision;
            b.evicted_rows = c.reset_count;
        }
        b.path = sl.path;
    }
    results[r.ticket % 64] = std::move(r);
    sl.busy = false;
}

uint64_t ShardedRank::enqueue(const uint64_t* ids, const uint32_t* feats, uint64_t n, uint64_t now,
                              const Policy& pol, uint64_t* out_slots, uint8_t* out_oc, uint64_t* out_ev,
                              uint64_t ev_cap, cudaStream_t st) {
    if (!connected) throw Error{MPZCH_ELOGIC, "row-sharded rank is not connected to its peers"};
    // a slice larger than the exchange buffers still takes part (its n makes every rank fail
    // with the capacity error), so no peer is left waiting
    const bool too_big = n > cap;
    Table& T = *t;
    MPZCH_CUDA(cudaSetDevice(device));
    const uint64_t e = ++epoch;
    const int si = (int)(e % kRing);
    finish_slot(si);
    if (last_done && st != last_stream) MPZCH_CUDA(cudaStreamWaitEvent(st, last_done, 0));
    Slot& sl = slots[si];
    sl.n = n;
    sl.host_waits = 1;
    sl.fallback_status = MPZCH_OK;
    sl.fallback_msg.clear();

    BatchArgs a{};
    a.pol = &pol;
    a.now = now;
    fill_policy_args(T, pol, now, feats, a, st);
    const bool fast = T.path_override == MPZCH_PATH_AUTO && T.hole_free && (a.uniform || a.per_feature) &&
                      pol.mode != kModeLru && cap <= (1ull << 29);
    sl.path = fast ? MPZCH_PATH_AUTO : (T.hole_free && T.path_override != MPZCH_PATH_ORDERED ? MPZCH_PATH_ROUNDS
                                                                                              : MPZCH_PATH_ORDERED);
    // per-feature TTLs that may overflow at this `now`: decided per position on the device
    const uint64_t limit = ~0ull - now;
    bool may_over = pol.mode == kModeTtl && !a.uniform && pol.default_ttl > limit;
    for (uint64_t v : pol.ttls) may_over = may_over || (pol.mode == kModeTtl && !a.uniform && v > limit);
    const unsigned B = 256;
    ShHeader* mh = reinterpret_cast<ShHeader*>(region);

    // P1: the route count with the validation pass fused in, then publish + plan
    if (n && !too_big) {
        if (may_over)
            launch_pdl(k_sh_overflow, grid_for(n, B, 148u * 8u), B, st, feats, n, limit, pol.default_ttl,
                       (const uint32_t*)a.d_featk, (const uint64_t*)a.d_featv, a.nk, d_state);
        enqueue_route_count(T, ids, n, G, st, &d_state->local_bad);
    }
    launch_pdl(k_sh_publish_plan, 1, kMaxG, st, peers, mh, rank, G, e, n,
               (uint64_t)((pol.mode == kModeTtl && a.uniform && a.overflow_all) ? 1 : 0),
               (const unsigned*)((n && !too_big) ? T.rt_tot.as<unsigned>() : nullptr), cap, timeout_ns, d_state);
    T.launches += 1;
    // P2: route-scatter straight into the owners' receive buffers
    if (n && !too_big) {
        std::vector<uint64_t> ids_to(G), feats_to(G), src_to(G);
        for (uint32_t q = 0; q < G; ++q) {
            ids_to[q] = peers.region[q] + L.ids;
            feats_to[q] = peers.region[q] + L.feats;
            src_to[q] = peers.region[q] + L.src;
        }
        PeerScatter d{ids_to.data(), feats ? feats_to.data() : nullptr, src_to.data(), nullptr};
        d.dev_offset = reinterpret_cast<const uint64_t*>(&d_state->my_off[0]);
        d.gate = reinterpret_cast<const uint64_t*>(&d_state->failed);
        run_route_scatter(T, ids, feats, n, G, d, st);
    }
    launch_pdl(k_sh_signal_wait, 1, kMaxG, st, peers, mh, (uint32_t)kFScat, rank, G, e, timeout_ns, d_state);
    T.launches += 1;
    // P3: the owner's remap of its received positions
    const uint64_t* rids = reinterpret_cast<const uint64_t*>(region + L.ids);
    const uint32_t* rfeats = feats ? reinterpret_cast<const uint32_t*>(region + L.feats) : nullptr;
    uint8_t* mark = nullptr;
    int clear = 0;
    if (fast) {
        a.ids = rids;
        a.feats = rfeats;
        a.n = cap;
        a.out_slots = loc_slots.as<uint64_t>();
        a.out_oc = loc_oc.as<uint8_t>();
        a.out_ev = nullptr;
        a.ev_cap = 0;
        a.overflow_all = false;  // decided by the ranks together (P1)
        a.sh_state = d_state;
        T.d_ctr = d_ctr;
        const bool prof = T.profiling;
        T.profiling = false;
        enqueue_fast_batch(T, a, st);
        T.profiling = prof;
        if (pol.mode != kModeDisabled) {
            mark = T.s_evflag.as<uint8_t>();
            clear = 1;
        }
    } else {
        // one more host round trip: the ordinary remap needs R on the host
        MPZCH_CUDA(cudaMemcpyAsync(&h_state[si], d_state, sizeof(ShState), cudaMemcpyDeviceToHost, st));
        MPZCH_CUDA(cudaStreamSynchronize(st));
        const ShState hs = h_state[si];
        ++sl.host_waits;
        if (!hs.failed && hs.R) {
            try {
                const uint64_t tk = enqueue_batch(T, rids, rfeats, hs.R, now, pol, loc_slots.as<uint64_t>(),
                                                  loc_oc.as<uint8_t>(), nullptr, 0, st, loc_mark.as<uint8_t>(),
                                                  /*host_waits*/ true);
                wait_batch(T, tk);
                ++sl.host_waits;
            } catch (const Error& err) {
                sl.fallback_status = err.code;
                sl.fallback_msg = err.msg;
            }
        }
        if (pol.mode != kModeDisabled) mark = loc_mark.as<uint8_t>();
    }
    // P4: results straight back into the sources' result buffers
    launch_pdl(k_sh_return, grid_for(cap, B, 148u * 8u), B, st, (const ShState*)d_state,
               (const uint32_t*)(region + L.src), (const uint64_t*)loc_slots.as<uint64_t>(),
               (const uint8_t*)loc_oc.as<uint8_t>(), mark, clear, peers, L, G);
    launch_pdl(k_sh_signal_wait, 1, kMaxG, st, peers, mh, (uint32_t)kFRes, rank, G, e, timeout_ns, d_state);
    T.launches += 2;
    // P5: the canonical evicted list (only TTL / LRU batches can evict; the policy is the same on
    // every rank, so every rank runs this phase or none does)
    if (pol.mode != kModeDisabled) {
        if (n && !too_big) {
            EmitSlots em{reinterpret_cast<const uint64_t*>(region + L.rslots), my_ev.as<uint64_t>()};
            compact_flags(region + L.rmark, n, blk.as<unsigned>(), &d_state->ev_mine, true, em, st, T.launches);
        }
        launch_pdl(k_sh_evc_plan, 1, kMaxG, st, peers, mh, rank, G, e, timeout_ns, d_state);
        launch_pdl(k_sh_ev_scatter, 148u * 4u, B, st, (const ShState*)d_state, (const uint64_t*)my_ev.as<uint64_t>(),
                   peers, L.ev, G);
        launch_pdl(k_sh_signal_wait, 1, kMaxG, st, peers, mh, (uint32_t)kFEv, rank, G, e, timeout_ns, d_state);
        T.launches += 3;
    }
    // results to the caller, the state to the mapped result slot, then reset for the next batch
    const bool want_ev = pol.mode != kModeDisabled && out_ev && ev_cap;
    launch_pdl(k_sh_finish, grid_for(std::max<uint64_t>(too_big ? 0 : n, want_ev ? ev_cap : 0), B, 148u * 8u), B, st,
               d_state, (const BatchCounters*)(fast ? d_ctr : nullptr), too_big ? 0 : n,
               (const uint64_t*)(region + L.rslots), (const uint8_t*)(region + L.roc), out_slots, out_oc,
               (const uint64_t*)(region + L.ev), want_ev ? out_ev : nullptr, ev_cap, hd_state + si, hd_ctr + si,
               &d_state->done);
    T.launches += 1;
    MPZCH_CUDA(cudaGetLastError());
    MPZCH_CUDA(cudaEventRecord(sl.done, st));
    sl.busy = true;
    sl.ticket = e;
    last_stream = st;
    last_done = sl.done;
    return e;
}

uint64_t ShardedRank::wait(uint64_t ticket) {
    MPZCH_CUDA(cudaSetDevice(device));
    const int si = (int)(ticket % kRing);
    if (slots[si].busy && slots[si].ticket == ticket) finish_slot(si);
    const Result& r = results[ticket % 64];
    if (r.ticket != ticket) throw Error{MPZCH_EINVAL, "unknown or expired batch ticket"};
    last = r.stats;
    last_host_waits = r.host_waits;
    if (r.status != MPZCH_OK) throw Error{r.status, r.msg};
    return r.ev_total;
}

}  // namespace mpzch_b200

using namespace mpzch_b200;

struct mpzch_sharded {
    ShardedRank* r;
    mpzch_table view;  // the rank's table for the accessors (not owned through this)
};

extern "C" {

mpzch_status mpzch_sharded_create(const uint64_t* caps, uint32_t num_shards, uint32_t max_probe, uint64_t seed,
                                  uint32_t dim, uint64_t init_seed, int device, uint32_t rank, uint32_t world,
                                  uint64_t max_batch, mpzch_sharded** out) {
    if (!out) return MPZCH_EINVAL;
    *out = nullptr;
    return run_guarded([&] {
        std::unique_ptr<ShardedRank> r(
            new ShardedRank(caps, num_shards, max_probe, seed, dim, init_seed, device, rank, world, max_batch));
        mpzch_sharded* h = new mpzch_sharded;
        h->view.t = r->t.get();
        h->r = r.release();
        *out = h;
    });
}

mpzch_status mpzch_sharded_destroy(mpzch_sharded* s) {
    if (!s) return MPZCH_OK;
    delete s->r;
    delete s;
    return MPZCH_OK;
}

mpzch_table* mpzch_sharded_table(mpzch_sharded* s) { return s ? &s->view : nullptr; }

mpzch_status mpzch_sharded_export(const mpzch_sharded* s, uint8_t* out_record) {
    if (!s || !out_record) return MPZCH_EINVAL;
    return run_guarded([&] {
        const ShRecord r = s->r->record();
        std::memcpy(out_record, &r, sizeof r);
    });
}

mpzch_status mpzch_sharded_connect_ipc(mpzch_sharded* s, const uint8_t* records) {
    if (!s || !records) return MPZCH_EINVAL;
    return run_guarded([&] { s->r->connect_ipc(records); });
}

mpzch_status mpzch_sharded_connect_local(mpzch_sharded* const* ranks, uint32_t world) {
    if (!ranks || world == 0) return MPZCH_EINVAL;
    return run_guarded([&] {
        for (uint32_t q = 0; q < world; ++q) {
            ShardedRank& r = *ranks[q]->r;
            if (r.rank != q || r.G != world) throw Error{MPZCH_EINVAL, "ranks must be given in rank order"};
            if (r.connected) throw Error{MPZCH_ELOGIC, "rank is already connected"};
            if (r.cap != ranks[0]->r->cap) throw Error{MPZCH_EINVAL, "ranks disagree on max_batch"};
        }
        for (uint32_t q = 0; q < world; ++q) {
            ShardedRank& r = *ranks[q]->r;
            MPZCH_CUDA(cudaSetDevice(r.device));
            for (uint32_t p = 0; p < world; ++p) {
                ShardedRank& o = *ranks[p]->r;
                if (o.device != r.device) {
                    int ok = 0;
                    MPZCH_CUDA(cudaDeviceCanAccessPeer(&ok, r.device, o.device));
                    if (!ok) throw Error{MPZCH_ECUDA, "GPUs " + std::to_string(r.device) + " and " +
                                                          std::to_string(o.device) + " have no peer access"};
                    const cudaError_t err = cudaDeviceEnablePeerAccess(o.device, 0);
                    if (err == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
                    else MPZCH_CUDA(err);
                }
                r.set_peer(p, o.region);
            }
        }
        // ranks sharing a device: no batch may grow a buffer later (cudaFree synchronises the
        // device, which would wait for a peer's spin that waits for this rank)
        for (uint32_t q = 0; q < world; ++q)
            for (uint32_t p = 0; p < world; ++p)
                if (p != q && ranks[p]->r->device == ranks[q]->r->device) {
                    ranks[q]->r->reserve_all_paths();
                    break;
                }
        for (uint32_t q = 0; q < world; ++q) ranks[q]->r->connected = true;
    });
}

mpzch_status mpzch_sharded_process_batch_async(mpzch_sharded* s, const uint64_t* ids, const uint32_t* features,
                                               uint64_t n, uint64_t now, const mpzch_policy* policy,
                                               uint64_t* out_slots, uint8_t* out_outcomes, uint64_t* out_evicted,
                                               uint64_t evicted_cap, void* stream, uint64_t* out_ticket) {
    if (!s) return MPZCH_EINVAL;
    return run_guarded([&] {
        const Policy pol = parse_policy(policy);
        *out_ticket = s->r->enqueue(ids, features, n, now, pol, out_slots, out_outcomes, out_evicted, evicted_cap,
                                    (cudaStream_t)stream);
    });
}

mpzch_status mpzch_sharded_wait(mpzch_sharded* s, uint64_t ticket, uint64_t* out_evicted_n) {
    if (!s) return MPZCH_EINVAL;
    return run_guarded([&] {
        const uint64_t ev = s->r->wait(ticket);
        if (out_evicted_n) *out_evicted_n = ev;
    });
}

mpzch_status mpzch_sharded_process_batch(mpzch_sharded* s, const uint64_t* ids, const uint32_t* features,
                                         uint64_t n, uint64_t now, const mpzch_policy* policy, uint64_t* out_slots,
                                         uint8_t* out_outcomes, uint64_t* out_evicted, uint64_t evicted_cap,
                                         uint64_t* out_evicted_n, void* stream) {
    uint64_t tk = 0;
    const mpzch_status st = mpzch_sharded_process_batch_async(s, ids, features, n, now, policy, out_slots,
                                                              out_outcomes, out_evicted, evicted_cap, stream, &tk);
    if (st != MPZCH_OK) return st;
    return mpzch_sharded_wait(s, tk, out_evicted_n);
}

mpzch_status mpzch_sharded_group_process_batch(mpzch_sharded* const* ranks, uint32_t world, const uint64_t* ids,
                                               const uint32_t* features, uint64_t n, uint64_t now,
                                               const mpzch_policy* policy, uint64_t* out_slots,
                                               uint8_t* out_outcomes, uint64_t* out_evicted, uint64_t evicted_cap,
                                               uint64_t* out_evicted_n) {
    if (!ranks || world == 0) return MPZCH_EINVAL;
    return run_guarded([&] {
        if (n > 0xffffffffull) throw Error{MPZCH_ELENGTH, "batch exceeds 2^32 - 1 positions"};  // batch_engine.cpp:82-83
        const Policy pol = parse_policy(policy);
        std::vector<ShardedRank*> R(world);
        for (uint32_t q = 0; q < world; ++q) {
            R[q] = ranks[q]->r;
            if (R[q]->rank != q || R[q]->G != world) throw Error{MPZCH_EINVAL, "ranks must be given in rank order"};
        }
        auto lo = [&](uint32_t q) { return (uint64_t)q * n / world; };
        // 1. every allocation first (growing a buffer later would synchronise a device that
        //    may hold a peer's spinning wait), then every host -> device copy
        for (uint32_t q = 0; q < world; ++q) {
            ShardedRank& r = *R[q];
            MPZCH_CUDA(cudaSetDevice(r.device));
            const uint64_t m = lo(q + 1) - lo(q);
            if (!r.g_stream) MPZCH_CUDA(cudaStreamCreateWithFlags(&r.g_stream, cudaStreamNonBlocking));
            r.g_ids.reserve(std::max<uint64_t>(m, 1) * 8);
            r.g_feats.reserve(std::max<uint64_t>(m, 1) * 4);
            r.g_slots.reserve(std::max<uint64_t>(m, 1) * 8);
            r.g_oc.reserve(std::max<uint64_t>(m, 1));
            if (q == 0 && out_evicted) r.g_ev.reserve(std::max<uint64_t>(evicted_cap, 1) * 8);
        }
        for (uint32_t q = 0; q < world; ++q) {
            ShardedRank& r = *R[q];
            MPZCH_CUDA(cudaSetDevice(r.device));
            const uint64_t m = lo(q + 1) - lo(q);
            if (m) {
                MPZCH_CUDA(cudaMemcpyAsync(r.g_ids.p, ids + lo(q), m * 8, cudaMemcpyHostToDevice, r.g_stream));
                if (features)
                    MPZCH_CUDA(cudaMemcpyAsync(r.g_feats.p, features + lo(q), m * 4, cudaMemcpyHostToDevice, r.g_stream));
            }
        }
        // 2. one host thread per rank enqueues and waits its batch (a batch on the host-synchronous
        //    fallback path waits mid-protocol; with one thread for all ranks that wait would stall
        //    the ranks not yet enqueued)
        std::vector<uint64_t> ev(world, 0);
        std::vector<Error> errs(world, Error{MPZCH_OK, ""});
        std::vector<std::thread> th;
        for (uint32_t q = 0; q < world; ++q)
            th.emplace_back([&, q] {
                ShardedRank& r = *R[q];
                const uint64_t m = lo(q + 1) - lo(q);
                try {
                    const uint64_t tk = r.enqueue(r.g_ids.as<uint64_t>(), features ? r.g_feats.as<uint32_t>() : nullptr,
                                                  m, now, pol, r.g_slots.as<uint64_t>(), r.g_oc.as<uint8_t>(),
                                                  (q == 0 && out_evicted) ? r.g_ev.as<uint64_t>() : nullptr,
                                                  (q == 0 && out_evicted) ? evicted_cap : 0, r.g_stream);
                    ev[q] = r.wait(tk);
                } catch (const Error& err) {
                    errs[q] = err;
                } catch (const std::exception& e) {
                    errs[q] = Error{MPZCH_ECUDA, e.what()};
                }
            });
        for (auto& x : th) x.join();
        for (uint32_t q = 0; q < world; ++q)
            if (errs[q].code != MPZCH_OK) throw errs[q];
        const uint64_t nev = ev[0];
        // 3. results back to the host
        for (uint32_t q = 0; q < world; ++q) {
            ShardedRank& r = *R[q];
            MPZCH_CUDA(cudaSetDevice(r.device));
            const uint64_t m = lo(q + 1) - lo(q);
            if (m) {
                MPZCH_CUDA(cudaMemcpyAsync(out_slots + lo(q), r.g_slots.p, m * 8, cudaMemcpyDeviceToHost, r.g_stream));
                MPZCH_CUDA(cudaMemcpyAsync(out_outcomes + lo(q), r.g_oc.p, m, cudaMemcpyDeviceToHost, r.g_stream));
            }
            if (q == 0 && out_evicted && nev)
                MPZCH_CUDA(cudaMemcpyAsync(out_evicted, r.g_ev.p, std::min(nev, evicted_cap) * 8,
                                           cudaMemcpyDeviceToHost, r.g_stream));
        }
        for (uint32_t q = 0; q < world; ++q) MPZCH_CUDA(cudaStreamSynchronize(R[q]->g_stream));
        if (out_evicted_n) *out_evicted_n = nev;
    });
}

mpzch_status mpzch_sharded_last_stats(const mpzch_sharded* s, mpzch_batch_stats* out, int* out_host_waits) {
    if (!s) return MPZCH_EINVAL;
    if (out) *out = s->r->last;
    if (out_host_waits) *out_host_waits = s->r->last_host_waits;
    return MPZCH_OK;
}

mpzch_status mpzch_sharded_held_shards(const mpzch_sharded* s, uint32_t* shard_lo, uint32_t* shard_hi) {
    if (!s) return MPZCH_EINVAL;
    if (shard_lo) *shard_lo = s->r->t->shard_lo;
    if (shard_hi) *shard_hi = s->r->t->shard_hi;
    return MPZCH_OK;
}

}  // extern "C"
