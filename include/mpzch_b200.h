/*
 * mpzch_b200.h -- the C-ABI drop-in boundary of the B200 MPZCH remap path.
 *
 * Plain pointers and sizes only (no torch / C++ types).  The reference has no
 * C ABI (it is a static C++ library); every entry point below names the
 * reference C++ interface it replaces, relative to /root/reference/.  The
 * C++ surface that keeps the reference's names and exception types sits on
 * top of this header in include/mpzch_b200.hpp.
 *
 * Device model: one handle = one table resident on one B200 (or, for the
 * row-sharded mode, the part of a table one rank owns).  Calls on a handle
 * are stream-ordered and must be externally serialized, exactly like the
 * reference's "mutations on a live table must be externally serialized"
 * (proj/include/mpzch/table.hpp:38-40).  Validation errors are raised before
 * any mutation (proj/src/batch_engine.cpp:146-147): the kernels carry a device
 * error word and every mutating kernel is a no-op once it is set.
 */
#ifndef MPZCH_B200_H
#define MPZCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The C++ wrapper maps each to the reference's exception type
 * with the identical message text (mpzch_last_error()). */
typedef enum mpzch_status {
    MPZCH_OK = 0,
    MPZCH_EINVAL = 1,    /* std::invalid_argument */
    MPZCH_EOVERFLOW = 2, /* std::overflow_error   */
    MPZCH_ELENGTH = 3,   /* std::length_error     */
    MPZCH_ELOGIC = 4,    /* std::logic_error      */
    MPZCH_ERANGE = 5,    /* std::out_of_range     */
    MPZCH_ECUDA = 6,     /* CUDA runtime failure  */
    MPZCH_ENOMEM = 7,    /* std::bad_alloc / cudaErrorMemoryAllocation */
    MPZCH_ENCCL = 8      /* NCCL failure (row-sharded mode) */
} mpzch_status;

/* EvictionMode, proj/include/mpzch/eviction.hpp:25 (same order) */
enum { MPZCH_MODE_DISABLED = 0, MPZCH_MODE_TTL = 1, MPZCH_MODE_LRU = 2 };

/* Outcome, proj/include/mpzch/probe_core.hpp:56 (same order, u8) */
enum { MPZCH_FOUND = 0, MPZCH_INSERTED = 1, MPZCH_EVICTED = 2, MPZCH_COLLISION = 3 };

/* Execution path (default AUTO): the claim path for Disabled / single-TTL batches on
 * hole-free tables, the A.4 rounds path for LRU and per-feature-TTL batches on hole-free
 * tables, the per-shard ordered kernel for tables with raw-imported holes.  ORDERED and
 * ROUNDS force those paths (all three are exact for every batch). */
enum { MPZCH_PATH_AUTO = 0, MPZCH_PATH_ORDERED = 1, MPZCH_PATH_ROUNDS = 2 };

/* EvictionPolicy / TtlPolicy, proj/include/mpzch/eviction.hpp:13-46.
 * per-feature TTLs are given as parallel arrays (feat_keys[i] -> feat_ttls[i]). */
typedef struct mpzch_policy {
    int32_t mode;          /* MPZCH_MODE_* */
    uint32_t n_feat;       /* entries in the per-feature map */
    uint64_t default_ttl;  /* TtlPolicy::default_ttl_seconds (TTL mode only) */
    const uint32_t* feat_keys;
    const uint64_t* feat_ttls;
} mpzch_policy;

/* Per-batch counters of the last process_batch call on a handle. */
typedef struct mpzch_batch_stats {
    uint64_t positions;
    uint64_t new_positions;  /* positions that missed the pre-batch table */
    uint64_t new_ids;        /* distinct ids among them (claim participants) */
    uint64_t found, inserted, evicted, collision; /* per position */
    uint64_t evicted_rows;   /* canonical evicted-list length */
    uint32_t path;           /* MPZCH_PATH_* actually taken */
    uint32_t rounds;         /* rounds run by the rounds path */
} mpzch_batch_stats;

typedef struct mpzch_table mpzch_table;

/* ---- construction: MpzchTable(TableConfig), proj/include/mpzch/table.hpp:43,
 *      proj/src/table.cpp:34-56; TableConfig proj/include/mpzch/table.hpp:18-28.
 * Allocates identity (EMPTY), metadata (0), row_generation (0) and, when
 * dim > 0, weights (draw_row for every row, bit-exact), momentum (0) and the
 * trained flags (0) in HBM of `device`. */
mpzch_status mpzch_table_create(const uint64_t* shard_capacities, uint32_t num_shards,
                                uint32_t max_probe, uint64_t seed, uint32_t dim,
                                uint64_t init_seed, int device, mpzch_table** out);
mpzch_status mpzch_table_destroy(mpzch_table* t);

/* layout accessors: table.hpp:48-56, TableLayout shard_router.hpp:13-29 */
uint64_t mpzch_total_rows(const mpzch_table* t);
uint32_t mpzch_num_shards(const mpzch_table* t);
uint32_t mpzch_max_probe(const mpzch_table* t);
uint32_t mpzch_dim(const mpzch_table* t);
mpzch_status mpzch_shard_layout(const mpzch_table* t, uint64_t* capacities, uint64_t* offsets);

/* ---- the hot path: process_batch(MpzchTable&, const IdBatch&, const EvictionPolicy&,
 *      ExecMode) -> vector<ProbeResult>, proj/include/mpzch/batch_engine.hpp:44-46,
 *      proj/src/batch_engine.cpp:141-221.
 * ids[n], features[n] (NULL = feature 0 everywhere, IdBatch::ids BatchEntry),
 * now = IdBatch::now.  Outputs per position: out_slots[n] (global row,
 * ProbeResult::slot), out_outcomes[n] (ProbeResult::outcome; evicted ==
 * (outcome == MPZCH_EVICTED)).  out_evicted receives the canonical evicted
 * list: global rows of the (id, feature) uniques whose outcome is Evicted, in
 * first-occurrence order, with multiplicity; *out_evicted_n is its full length
 * even when it exceeds evicted_cap.  out_evicted / out_evicted_n may be NULL.
 *
 * mpzch_process_batch: HOST buffers; copies in, runs, copies out, returns when
 * done (the reference call's semantics).
 * mpzch_process_batch_device: DEVICE buffers on the table's device, enqueued on
 * `stream` (cudaStream_t; 0 = the legacy default stream, the CUDA convention, so
 * work the caller queued on it is ordered before the batch); returns after the batch
 * completed on that stream (it reports validation errors synchronously, like
 * the reference).  out_evicted is a device pointer here. */
mpzch_status mpzch_process_batch(mpzch_table* t, const uint64_t* ids, const uint32_t* features,
                                 uint64_t n, uint64_t now, const mpzch_policy* policy,
                                 uint64_t* out_slots, uint8_t* out_outcomes, uint64_t* out_evicted,
                                 uint64_t evicted_cap, uint64_t* out_evicted_n);
mpzch_status mpzch_process_batch_device(mpzch_table* t, const uint64_t* ids,
                                        const uint32_t* features, uint64_t n, uint64_t now,
                                        const mpzch_policy* policy, uint64_t* out_slots,
                                        uint8_t* out_outcomes, uint64_t* out_evicted,
                                        uint64_t evicted_cap, uint64_t* out_evicted_n,
                                        void* stream);

/* Asynchronous variant: enqueues the batch on `stream` and returns a ticket without
 * waiting (host-side argument errors are still returned immediately).  mpzch_batch_wait
 * blocks until the ticket's batch is done and returns ITS status (invalid id, TTL overflow,
 * ... exactly as the synchronous call would have) and evicted-list length.  Batches of one
 * handle run in enqueue order; a batch that fails validation mutates nothing, so later
 * batches see the table as if the failed call had thrown.  Up to 8 batches may be in flight;
 * results of the last 64 tickets stay retrievable. */
mpzch_status mpzch_process_batch_device_async(mpzch_table* t, const uint64_t* ids,
                                              const uint32_t* features, uint64_t n, uint64_t now,
                                              const mpzch_policy* policy, uint64_t* out_slots,
                                              uint8_t* out_outcomes, uint64_t* out_evicted,
                                              uint64_t evicted_cap, void* stream,
                                              uint64_t* out_ticket);
mpzch_status mpzch_batch_wait(mpzch_table* t, uint64_t ticket, uint64_t* out_evicted_n);
/* Batched read-only lookup (MpzchTable::lookup per position) enqueued on `stream` without
 * waiting; the ticket shares the batch ring, and mpzch_batch_wait reports the status the
 * synchronous mpzch_lookup_device would have returned (invalid id: the reference's
 * require_valid_id text; id of a shard this handle does not hold: MPZCH_ERANGE).  Ordered after
 * this handle's pending batches. */
mpzch_status mpzch_lookup_device_async(mpzch_table* t, const uint64_t* ids, uint64_t n,
                                       uint64_t* out_slots, uint8_t* out_outcomes, void* stream,
                                       uint64_t* out_ticket);

/* ---- lookup-only: MpzchTable::lookup(Id) const, table.hpp:65, table.cpp:150-156,
 *      batched (semantics = one lookup per position, no writes). */
mpzch_status mpzch_lookup(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                          uint64_t* out_slots, uint8_t* out_outcomes);
mpzch_status mpzch_lookup_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                 uint64_t* out_slots, uint8_t* out_outcomes, void* stream);

/* ---- single-id training path: MpzchTable::lookup_or_insert(Id, FeatureOrdinal,
 *      Timestamp, const EvictionPolicy&), table.hpp:61-62, table.cpp:98-110 */
mpzch_status mpzch_lookup_or_insert(mpzch_table* t, uint64_t id, uint32_t feature, uint64_t now,
                                    const mpzch_policy* policy, uint64_t* out_slot,
                                    uint8_t* out_outcome);

/* ---- state download (parity): identities(s)/metadata(s) table.hpp:89-90 (all
 *      shards, concatenated in global-row order), embeddings() :92 weights,
 *      momentum_row :87, row_trained :86; row_generation_ table.cpp:55. */
mpzch_status mpzch_copy_identities(const mpzch_table* t, uint64_t* host_out);
mpzch_status mpzch_copy_metadata(const mpzch_table* t, uint64_t* host_out);
mpzch_status mpzch_copy_weights(const mpzch_table* t, uint64_t row0, uint64_t nrows,
                                float* host_out);
mpzch_status mpzch_copy_momentum(const mpzch_table* t, uint64_t row0, uint64_t nrows,
                                 float* host_out);
mpzch_status mpzch_copy_trained(const mpzch_table* t, uint8_t* host_out);
mpzch_status mpzch_copy_row_generation(const mpzch_table* t, uint64_t* host_out);
/* device pointers of the resident arrays (for fused consumers and the bench): READ views --
 * identities and metadata change only through the calls of this header (raw writes through
 * mpzch_write_slots, which also keeps the identity tags of max_probe >= 256 tables) */
mpzch_status mpzch_device_arrays(const mpzch_table* t, uint64_t** identities,
                                 uint64_t** metadata, float** weights);

/* ---- raw state import (the reference's scenario tests write the arrays
 *      directly, e.g. proj/tests/test_probe_core.cpp:113-121).  Writing raw
 *      slots may create probe-window holes, so it switches the handle to the
 *      hole-tolerant full-window semantics until mpzch_check_hole_free()
 *      proves the no-hole invariant again.  Tables with max_probe >= 256 retag
 *      the written slots (the probe's identity-tag index). */
mpzch_status mpzch_write_slots(mpzch_table* t, uint32_t shard, const uint64_t* local_slots,
                               const uint64_t* identities, const uint64_t* metadata, uint64_t n);
mpzch_status mpzch_check_hole_free(mpzch_table* t, int* out_hole_free);
/* row payload write (stands in for training writes when testing resets) */
mpzch_status mpzch_write_row(mpzch_table* t, uint64_t row, const float* weights,
                             const float* momentum, uint8_t trained);

/* ---- dirty tracking: make_cursor / dirty_rows_since, table.hpp:95-96,
 *      table.cpp:209-225 (cursor = generation; the table uid is the handle). */
mpzch_status mpzch_make_cursor(mpzch_table* t, uint64_t* out_generation);
mpzch_status mpzch_dirty_rows_since(const mpzch_table* t, uint64_t generation, uint64_t* out,
                                    uint64_t cap, uint64_t* out_n);

/* ---- row-sharded mode: one handle per rank holds the logical shards
 *      [shard_lo, shard_hi) of the layout (global row numbering unchanged, so results are
 *      identical for every number of ranks).  A rank routes its positions to owners with
 *      mpzch_route_device + an all-to-all (NCCL) or over peer memory (below), owners remap with
 *      mpzch_process_batch_device_marked, results travel back; see
 *      paper_2602_17050_b200/sharded.py.  Copies (mpzch_copy_*) return the held rows only. */
mpzch_status mpzch_table_create_sharded(const uint64_t* shard_capacities, uint32_t num_shards,
                                        uint32_t max_probe, uint64_t seed, uint32_t dim,
                                        uint64_t init_seed, int device, uint32_t shard_lo,
                                        uint32_t shard_hi, mpzch_table** out);
mpzch_status mpzch_held_rows(const mpzch_table* t, uint64_t* row_lo, uint64_t* row_hi,
                             uint32_t* shard_lo, uint32_t* shard_hi);
/* validation pass only (batch_engine.cpp:90-94): *out_bad_pos = first invalid position or ~0 */
mpzch_status mpzch_validate_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                   uint64_t* out_bad_pos, void* stream);
/* stable partition of positions by owning part: perm[n] (device) lists positions part by part
 * in input order; counts[parts] (host) the part sizes; shard_to_part[S] (host) the owners */
mpzch_status mpzch_route_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                const uint32_t* shard_to_part, uint32_t parts, uint32_t* perm,
                                uint64_t* counts, void* stream);
/* ---- peer-memory transport of the row-sharded mode (replaces the NCCL all-to-all pair; the
 *      reference has no counterpart -- its shards live in one process, batch_engine.cpp:141-221).
 *      Addresses are device addresses valid in the calling process: local buffers, buffers of
 *      another GPU reachable by P2P, or another process's buffers mapped by mpzch_ipc_import.
 *   1. mpzch_route_count_device: per-part counts[parts] (host) of this rank's positions (the
 *      count and scan phases of mpzch_route_device; arms step 2 for the same ids/n/parts);
 *   2. mpzch_route_scatter_device: every position i of part q stores ids[i], features[i] and
 *      i into part q's receive buffers ids_to[q] (u64), features_to[q] (u32), src_to[q] (u32)
 *      at offset[q] + (its rank among this rank's part-q positions): stable, so an owner that
 *      gives each source rank the offset sum of the lower ranks' counts receives the global
 *      batch's part-q positions in global order.  One kernel: partition + NVLink stores;
 *   3. (owners remap their received positions with mpzch_process_batch_device_marked)
 *   4. mpzch_return_scatter_device: received position j (source rank r: recv_offset[r] <= j <
 *      recv_offset[r+1]) stores slots[j], outcomes[j], marks[j] into slots_to[r][src[j]],
 *      outcomes_to[r][src[j]], marks_to[r][src[j]] (marks_to / marks nullable).
 * The caller orders the phases across ranks (stream sync + a barrier). */
mpzch_status mpzch_route_count_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                      const uint32_t* shard_to_part, uint32_t parts, uint64_t* counts,
                                      void* stream);
mpzch_status mpzch_route_scatter_device(const mpzch_table* t, const uint64_t* ids,
                                        const uint32_t* features, uint64_t n, uint32_t parts,
                                        const uint64_t* ids_to, const uint64_t* features_to,
                                        const uint64_t* src_to, const uint64_t* offset, void* stream);
mpzch_status mpzch_return_scatter_device(int device, uint64_t n_recv, const uint64_t* slots,
                                         const uint8_t* outcomes, const uint8_t* marks,
                                         const uint32_t* src, uint32_t parts, const uint64_t* recv_offset,
                                         const uint64_t* slots_to, const uint64_t* outcomes_to,
                                         const uint64_t* marks_to, void* stream);
/* CUDA IPC for the transport: a 72-byte record (allocation handle + offset, so buffers inside a
 * caching allocator's block work); imports are reference counted per allocation. */
#define MPZCH_IPC_RECORD_BYTES 72
mpzch_status mpzch_ipc_export(const void* device_ptr, uint8_t* out_record);
mpzch_status mpzch_ipc_import(int device, const uint8_t* record, uint64_t* out_addr);
mpzch_status mpzch_ipc_close(uint64_t addr);

/* process_batch on device buffers; out_first_evicted[n] (device, nullable) gets 1 at the first
 * position of every Evicted (id, feature) unique (how the sharded evicted list is assembled) */
mpzch_status mpzch_process_batch_device_marked(mpzch_table* t, const uint64_t* ids,
                                               const uint32_t* features, uint64_t n, uint64_t now,
                                               const mpzch_policy* policy, uint64_t* out_slots,
                                               uint8_t* out_outcomes, uint8_t* out_first_evicted,
                                               uint64_t* out_evicted_n, void* stream);

/* ---- in-library CUDA-event profiling (bench evidence).  When on, every batch records
 * events on its own launch stream around the probe kernel, the claim/commit kernels
 * and the whole batch, and the probe kernel counts the 32-byte sectors it reads. */
typedef struct mpzch_profile {
    uint64_t batches;       /* profiled batches since mpzch_set_profiling(t, 1) */
    uint64_t probe_launches;
    double probe_ms;        /* sum of probe-kernel event times */
    double claim_ms;        /* dedup + claim + commit kernels */
    double tail_ms;         /* finalize, metadata, reset, evicted list, cleanup */
    double batch_ms;        /* first to last kernel of each batch */
    uint64_t probe_sectors; /* 32-byte identity/metadata sectors the probe read */
    uint64_t probe_bytes;   /* algorithmic bytes of the probe kernel (sectors + position I/O) */
    uint64_t batch_bytes;   /* algorithmic bytes of the whole batch (SURVEY 8d terms) */
    double validate_ms;     /* per-kernel split of the fast path */
    double dedup_ms, claimk_ms, commit_ms, finalize_ms;
} mpzch_profile;
mpzch_status mpzch_set_profiling(mpzch_table* t, int on);
mpzch_status mpzch_get_profile(const mpzch_table* t, mpzch_profile* out);

/* ---- SURVEY 8f "next" rows built on the same tables:
 * fused lookup + gather (frozen-replica read path): MpzchTable::lookup (table.cpp:150-156)
 * followed by gather of the resolved rows (table.cpp:158-163); out_rows is n x dim fp32
 * (device).  Misses gather the home row, as a lookup -> gather pipeline would. */
mpzch_status mpzch_lookup_gather_device(const mpzch_table* t, const uint64_t* ids, uint64_t n,
                                        uint64_t* out_slots, uint8_t* out_outcomes,
                                        float* out_rows, void* stream);
/* delta cut (DeltaSource::cut, publish.cpp:288-305): the rows dirtied since `generation`
 * (a cursor from mpzch_make_cursor), each with its identity word and weights (host buffers,
 * row-major), in row order; *out_n is the full count.  When it fits in `cap` a new cursor is
 * taken and returned in *out_next_generation (the cut's successor cursor). */
mpzch_status mpzch_delta_cut(mpzch_table* t, uint64_t generation, uint64_t* out_rows,
                             uint64_t* out_identities, float* out_weights, uint64_t cap,
                             uint64_t* out_n, uint64_t* out_next_generation);

/* sgd_step: MpzchTable::sgd_step (proj/src/table.cpp:174-179) over
 * EmbeddingTable::sgd_step (proj/src/embedding_store.cpp:70-93).  For i = 0..n-1 in order:
 * momentum[rows[i]] := beta*momentum + grads[i]; weights[rows[i]] -= lr*momentum (fp32,
 * separately rounded), trained := 1; then every row is stamped dirty.  grads is n x dim,
 * row-major; n_grads = its element count.  Errors in the reference's order: dim 0 ->
 * MPZCH_ELOGIC; n_grads != n*dim, !(lr > 0), beta outside [0, 1) -> MPZCH_EINVAL; a row out of
 * range -> MPZCH_ERANGE after the rows before it were updated (none stamped).  Repeated rows
 * compound in position order.  _device: rows/grads in device memory, enqueued on `stream`
 * (0 = legacy default stream) after this handle's pending batches; returns when done. */
mpzch_status mpzch_sgd_step(mpzch_table* t, const uint64_t* rows, uint64_t n, const float* grads,
                            uint64_t n_grads, float lr, float beta);
mpzch_status mpzch_sgd_step_device(mpzch_table* t, const uint64_t* rows, uint64_t n,
                                   const float* grads, uint64_t n_grads, float lr, float beta,
                                   void* stream);

/* ---- publish: .mpzc / .mpzd images (proj/README.md:129-145) built from HBM,
 * CRC-32 computed on the device.
 * crc32 (publish.cpp:110-124) of n bytes of DEVICE memory, enqueued on `stream`; returns when done. */
mpzch_status mpzch_crc32_device(const void* bytes, uint64_t n, uint32_t* out_crc, void* stream);
/* serialize_snapshot (publish.cpp:126-155) into a host buffer.  *out_len = image size; out NULL:
 * size query.  cap too small: MPZCH_ELENGTH.  dim 0: MPZCH_ELOGIC.  Row-sharded handles:
 * MPZCH_EINVAL (a snapshot covers every shard).  The trailer CRC is the lineage checksum
 * (snapshot_checksum, publish.cpp:157-162). */
mpzch_status mpzch_serialize_snapshot(const mpzch_table* t, uint8_t* out, uint64_t cap,
                                      uint64_t* out_len);
/* DeltaSource::cut (publish.cpp:288-305) + serialize_delta (publish.cpp:212-230) in one pass:
 * the rows dirtied since `generation`, ascending, each record (row u64, identity u64, dim f32)
 * packed on the device, CRC on the device.  out NULL: size query (cursor unchanged); otherwise
 * a fresh cursor is returned in *out_next_generation. */
mpzch_status mpzch_serialize_delta(mpzch_table* t, uint64_t generation, uint32_t base_checksum,
                                   uint64_t sequence, uint8_t* out, uint64_t cap,
                                   uint64_t* out_len, uint64_t* out_next_generation);


/* ---- the rest of the kept surface, csrc/surface.cu ---------------------------
 * MpzchTable::process_shard_batch(shard, span<const Id> ids, span<const u64> metas, now,
 * policy, span<ProbeResult> out), proj/include/mpzch/table.hpp:71-73, proj/src/table.cpp:112-148:
 * the serialized probe of one shard, positions in order (no dedup: a repeated id probes again
 * and refreshes with its own metadata word), each with the caller's metadata word.  ids must
 * route to `shard` (the reference's precondition; not checked).  Errors: shard >= S ->
 * MPZCH_ERANGE "shard index out of range" before anything runs; a metadata word that
 * make_metadata could not have produced -> MPZCH_EINVAL with the reference's text
 * (probe_core.cpp:49-58, 76-77) AFTER the positions before it took effect (their results are
 * in out_slots / out_outcomes), exactly like the exception thrown inside the reference's loop;
 * an invalid id -> MPZCH_EINVAL at the START of its 256-position chunk (the reference hoists
 * home_slot, which validates, over each chunk before probing it: table.cpp:129-133,
 * probe_core.cpp:27-30), so only the chunks before it took effect.
 * Host buffers; returns when done. */
mpzch_status mpzch_process_shard_batch(mpzch_table* t, uint32_t shard, const uint64_t* ids,
                                       const uint64_t* metas, uint64_t n, uint64_t now,
                                       const mpzch_policy* policy, uint64_t* out_slots,
                                       uint8_t* out_outcomes);
/* dedup(span<const BatchEntry>) -> DedupResult{uniques, inverse}, proj/include/mpzch/
 * batch_engine.hpp:35, proj/src/batch_engine.cpp:79-108, 133-139: first-occurrence uniques keyed
 * on (id, feature) (features NULL = 0) and inverse[n] (u32 index into the uniques).  Errors:
 * n > 2^32 - 1 -> MPZCH_ELENGTH "batch exceeds 2^32 - 1 positions"; an invalid id ->
 * MPZCH_EINVAL "invalid id at batch position <first bad position>".  mpzch_dedup: host buffers
 * (unique arrays sized n), runs on `device`; _device: device buffers on `stream`, returns when
 * done. */
mpzch_status mpzch_dedup(int device, const uint64_t* ids, const uint32_t* features, uint64_t n,
                         uint64_t* out_unique_ids, uint32_t* out_unique_features, uint32_t* out_inverse,
                         uint64_t* out_u);
mpzch_status mpzch_dedup_device(int device, const uint64_t* ids, const uint32_t* features, uint64_t n,
                                uint64_t* unique_ids, uint32_t* unique_features, uint32_t* inverse,
                                uint64_t* out_u, void* stream);
/* MpzchTable::reset_row(global_row), table.hpp:83, table.cpp:181-186: draw_row weights,
 * momentum 0, trained 0, row stamped dirty.  dim 0 -> MPZCH_ELOGIC; row out of range ->
 * MPZCH_ERANGE "embedding row out of range". */
mpzch_status mpzch_reset_row(mpzch_table* t, uint64_t row);
/* MpzchTable::state_equals(other), table.hpp:106, table.cpp:249-260: capacities and dim equal,
 * identities of every shard and the weights bit-equal (compared on the device). */
mpzch_status mpzch_state_equals(const mpzch_table* a, const mpzch_table* b, int* out_equal);
/* single-word / range reads for the C++ accessors: row_identity (table.hpp:85, one 8-byte copy),
 * identities(s) / metadata(s) (table.hpp:89-90, only shard s's rows), row_trained (table.hpp:86),
 * gather (table.hpp:77, table.cpp:158-163: one kernel + one copy; a row out of range ->
 * MPZCH_ERANGE "embedding row out of range" before anything is copied). */
mpzch_status mpzch_read_identity(const mpzch_table* t, uint64_t row, uint64_t* out);
mpzch_status mpzch_copy_identities_range(const mpzch_table* t, uint64_t row0, uint64_t nrows,
                                         uint64_t* host_out);
mpzch_status mpzch_copy_metadata_range(const mpzch_table* t, uint64_t row0, uint64_t nrows,
                                       uint64_t* host_out);
mpzch_status mpzch_copy_trained_range(const mpzch_table* t, uint64_t row0, uint64_t nrows,
                                      uint8_t* host_out);
mpzch_status mpzch_gather(const mpzch_table* t, const uint64_t* rows, uint64_t n, float* host_out);
/* MpzchTable::shard_config(s) (table.hpp:91, ShardConfig probe_core.hpp:11-18): capacity,
 * max_probe, seed (shard_id = s); shard >= S -> MPZCH_ERANGE "shard index out of range". */
mpzch_status mpzch_shard_config(const mpzch_table* t, uint32_t shard, uint64_t* capacity,
                                uint32_t* max_probe, uint64_t* seed);

/* ---- row-sharded table, device-side protocol (replaces the reference's shard loop
 * proj/src/batch_engine.cpp:160-211 across GPUs).  One mpzch_sharded per rank (one process per
 * GPU, or several ranks in one process): rank r of G holds the logical shards {s : s*G/S == r}
 * (global rows of the single-table layout, so every slot is identical for any G).  Each rank
 * passes its contiguous slice of the global batch (slices in rank order); ids go to their
 * owners and results come back by stores into peer memory (NVLink P2P / CUDA IPC), with every
 * phase enqueued on `stream`: one host wait per batch (the wait call).  Errors are agreed on the
 * device and raised on every rank with the reference's text and precedence ("invalid id at
 * batch position N" with the GLOBAL position, length, TTL overflow).  The evicted list is the
 * global canonical one on every rank.  max_batch bounds the GLOBAL batch (exchange buffers).
 * Every rank must call process_batch the same number of times (a collective); a peer that
 * stops answering fails the batch after MPZCH_PEER_TIMEOUT_MS (default 60000) with MPZCH_ENCCL.
 * LRU batches, tables with raw-imported holes and forced paths take one extra host round trip. */
typedef struct mpzch_sharded mpzch_sharded;
#define MPZCH_SHARDED_RECORD_BYTES 128
mpzch_status mpzch_sharded_create(const uint64_t* capacities, uint32_t num_shards, uint32_t max_probe,
                                  uint64_t seed, uint32_t dim, uint64_t init_seed, int device,
                                  uint32_t rank, uint32_t world, uint64_t max_batch,
                                  mpzch_sharded** out);
mpzch_status mpzch_sharded_destroy(mpzch_sharded* s);
/* the rank's table (held shards only) for the accessors; owned by `s`, never destroy it */
mpzch_table* mpzch_sharded_table(mpzch_sharded* s);
mpzch_status mpzch_sharded_held_shards(const mpzch_sharded* s, uint32_t* shard_lo, uint32_t* shard_hi);
/* multi-process: export this rank's exchange region (CUDA IPC), gather every rank's record in
 * rank order by any host channel, then connect */
mpzch_status mpzch_sharded_export(const mpzch_sharded* s, uint8_t* out_record);
mpzch_status mpzch_sharded_connect_ipc(mpzch_sharded* s, const uint8_t* records);
/* single process: connect `world` ranks (rank order; P2P is enabled between their GPUs) */
mpzch_status mpzch_sharded_connect_local(mpzch_sharded* const* ranks, uint32_t world);
/* device buffers, stream-ordered; the ticket is waited by mpzch_sharded_wait */
mpzch_status mpzch_sharded_process_batch_async(mpzch_sharded* s, const uint64_t* ids,
                                               const uint32_t* features, uint64_t n, uint64_t now,
                                               const mpzch_policy* policy, uint64_t* out_slots,
                                               uint8_t* out_outcomes, uint64_t* out_evicted,
                                               uint64_t evicted_cap, void* stream, uint64_t* out_ticket);
mpzch_status mpzch_sharded_wait(mpzch_sharded* s, uint64_t ticket, uint64_t* out_evicted_n);
mpzch_status mpzch_sharded_process_batch(mpzch_sharded* s, const uint64_t* ids, const uint32_t* features,
                                         uint64_t n, uint64_t now, const mpzch_policy* policy,
                                         uint64_t* out_slots, uint8_t* out_outcomes,
                                         uint64_t* out_evicted, uint64_t evicted_cap,
                                         uint64_t* out_evicted_n, void* stream);
/* single process, whole batch: process_batch (batch_engine.hpp:44-46) over `world` connected
 * ranks (rank order) with HOST buffers -- the batch is split into contiguous slices, staged,
 * every rank's batch enqueued before any wait, results copied back (the evicted list from
 * rank 0; every rank holds the same one).  The reference's call, spread over the GPUs. */
mpzch_status mpzch_sharded_group_process_batch(mpzch_sharded* const* ranks, uint32_t world,
                                               const uint64_t* ids, const uint32_t* features, uint64_t n,
                                               uint64_t now, const mpzch_policy* policy,
                                               uint64_t* out_slots, uint8_t* out_outcomes,
                                               uint64_t* out_evicted, uint64_t evicted_cap,
                                               uint64_t* out_evicted_n);
/* the last waited batch: this rank's owner-side counts; host_waits = host round trips it took */
mpzch_status mpzch_sharded_last_stats(const mpzch_sharded* s, mpzch_batch_stats* out, int* out_host_waits);

/* ---- execution control / introspection */
mpzch_status mpzch_set_path(mpzch_table* t, int path);
/* Embedding-row reset of evicted slots ("fused sgd_step with reset").
 * EAGER (default): the batch writes every evicted row -- draw_row, momentum 0, trained 0 --
 * as the reference does inside process_batch (table.cpp:142 -> embedding_store.cpp:62-68).
 * DEFERRED: the batch only marks the row reset-pending; the next sgd_step that touches it
 * computes from the closed-form draw_row and momentum 0 without reading the row (reset and
 * update share one write of the row), gathers (mpzch_gather, mpzch_lookup_gather_device)
 * return the drawn row, and every other reader (copies, snapshot, delta, state_equals,
 * mpzch_device_arrays' weights pointer) materialises the pending resets first.  Every
 * observable value is bit-identical to EAGER.  Switching back to EAGER flushes. */
enum { MPZCH_RESET_EAGER = 0, MPZCH_RESET_DEFERRED = 1 };
mpzch_status mpzch_set_reset_mode(mpzch_table* t, int mode);
/* write every pending reset now (DEFERRED mode; a no-op otherwise) */
mpzch_status mpzch_flush_resets(mpzch_table* t);
mpzch_status mpzch_last_stats(const mpzch_table* t, mpzch_batch_stats* out);
/* number of kernels this handle launched since creation (bench gpu_launches) */
uint64_t mpzch_kernel_launches(const mpzch_table* t);
/* thread-local text of the last error (the reference exception's what()) */
const char* mpzch_last_error(void);
/* library build string: "sm_100a <git-describe>" */
const char* mpzch_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* MPZCH_B200_H */
