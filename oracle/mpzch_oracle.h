/*
 * mpzch_oracle.h -- CPU restatement of the MPZCH batched remap path.
 *
 * TEST INFRASTRUCTURE ONLY.  This header and mpzch_oracle.c are the parity
 * checker for the CUDA path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load them.  The product
 * path (paper_2602_17050_b200/) never links, loads or calls anything here.
 *
 * Parity pinning: the restatement is checked against (a) every golden vector
 * the reference's own tests hold for this path (tests/golden/known_answers.json,
 * copied from proj/tests/test_probe_core.cpp:37-43, :78, test_shard_router.cpp:33,
 * test_rng.cpp:11-23, test_eviction.cpp:11-31) and (b) the reference library
 * itself, compiled from /root/reference/proj/src by oracle/Makefile into
 * oracle/_ref/libmpzch_ref.so (same C ABI as below, prefix ref_ instead of
 * orc_), on randomized batch streams (tests/test_oracle_vs_ref.py) and on
 * fixtures generated from it (tests/golden/gen_golden.py).
 *
 * The function set mirrors the reference C++ API one-to-one:
 *   orc_table_create        <- MpzchTable::MpzchTable(TableConfig)   proj/src/table.cpp:34-56
 *   orc_process_batch       <- process_batch(...)                    proj/src/batch_engine.cpp:141-221
 *   orc_lookup              <- MpzchTable::lookup(Id)                proj/src/table.cpp:150-156
 *   orc_lookup_or_insert    <- MpzchTable::lookup_or_insert(...)     proj/src/table.cpp:98-110
 *   orc_probe               <- lookup_or_insert (probe core)         proj/src/probe_core.cpp:69-134
 *   orc_probe_readonly      <- lookup_readonly                       proj/src/probe_core.cpp:32-43
 * Status codes are shared with include/mpzch_b200.h (MPZCH_OK ...).
 */
#ifndef MPZCH_ORACLE_H
#define MPZCH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: identical numbering to include/mpzch_b200.h */
#define ORC_OK 0
#define ORC_EINVAL 1    /* std::invalid_argument */
#define ORC_EOVERFLOW 2 /* std::overflow_error */
#define ORC_ELENGTH 3   /* std::length_error */
#define ORC_ELOGIC 4    /* std::logic_error */
#define ORC_ERANGE 5    /* std::out_of_range */
#define ORC_ENOMEM 7

/* policy modes: EvictionMode order, proj/include/mpzch/eviction.hpp:25 */
#define ORC_MODE_DISABLED 0
#define ORC_MODE_TTL 1
#define ORC_MODE_LRU 2

/* outcome codes: Outcome order, proj/include/mpzch/probe_core.hpp:56 */
#define ORC_FOUND 0
#define ORC_INSERTED 1
#define ORC_EVICTED 2
#define ORC_COLLISION 3

typedef struct orc_table orc_table;

/* primitives (ids.hpp, rng.hpp) */
uint64_t orc_mix64(uint64_t id, uint64_t seed);
uint64_t orc_splitmix_next(uint64_t* state);
uint64_t orc_distinct_id_at(uint64_t seed, uint64_t index);
void orc_distinct_ids(uint64_t seed, uint64_t start, uint64_t count, uint64_t* out);
uint64_t orc_home_slot(uint64_t id, uint64_t capacity, uint64_t seed);
uint32_t orc_shard_of(uint64_t id, uint32_t num_shards, uint64_t seed);
void orc_draw_row(float* dst, uint32_t dim, uint64_t row, uint64_t init_seed);
void orc_draw_rows(float* dst, uint32_t dim, const uint64_t* rows, uint64_t n, uint64_t init_seed);

/* table */
int orc_table_create(const uint64_t* capacities, uint32_t num_shards, uint32_t max_probe,
                     uint64_t seed, uint32_t dim, uint64_t init_seed, orc_table** out);
void orc_table_destroy(orc_table* t);
uint64_t orc_total_rows(const orc_table* t);
uint64_t orc_shard_offset(const orc_table* t, uint32_t shard);

/* batched insert-with-eviction remap; out_* sized n; evicted list in unique-rank
 * order with multiplicity (derived as in SURVEY 8b). threads: 0 = serial. */
int orc_process_batch(orc_table* t, const uint64_t* ids, const uint32_t* features, uint64_t n,
                      uint64_t now, int mode, uint64_t default_ttl, uint32_t n_feat,
                      const uint32_t* feat_keys, const uint64_t* feat_ttls,
                      uint64_t* out_slots, uint8_t* out_outcomes, uint64_t* out_evicted,
                      uint64_t evicted_cap, uint64_t* out_evicted_n);

/* read-only lookup of each id (no batching semantics; per-id MpzchTable::lookup) */
int orc_lookup(const orc_table* t, const uint64_t* ids, uint64_t n, uint64_t* out_slots,
               uint8_t* out_outcomes);

/* the single-id training path */
int orc_lookup_or_insert(orc_table* t, uint64_t id, uint32_t feature, uint64_t now, int mode,
                         uint64_t default_ttl, uint32_t n_feat, const uint32_t* feat_keys,
                         const uint64_t* feat_ttls, uint64_t* out_slot, uint8_t* out_outcome);

/* probe core on raw arrays (one shard), for the scenario tests */
int orc_probe(uint64_t id, uint64_t meta_in, uint64_t now, uint64_t* identities,
              uint64_t* metadata, uint64_t capacity, uint32_t max_probe, uint64_t seed, int mode,
              uint64_t* out_slot, uint8_t* out_outcome);
int orc_probe_readonly(uint64_t id, const uint64_t* identities, uint64_t capacity,
                       uint32_t max_probe, uint64_t seed, uint64_t* out_slot,
                       uint8_t* out_outcome);

/* state access (global row order: shard offsets are prefix sums) */
uint64_t* orc_identities(orc_table* t);
uint64_t* orc_metadata(orc_table* t);
float* orc_weights(orc_table* t);
float* orc_momentum(orc_table* t);
uint8_t* orc_trained(orc_table* t);
uint64_t* orc_row_generation(orc_table* t);
uint64_t orc_make_cursor(orc_table* t);
/* MpzchTable::sgd_step (proj/src/table.cpp:174-179) over EmbeddingTable::sgd_step
 * (proj/src/embedding_store.cpp:70-93): momentum := beta*momentum + grad,
 * weights := weights - lr*momentum (fp32, separately rounded), trained := 1, in position
 * order; then touch_row for every row.  A row out of range throws after the rows before it
 * were updated (and before any touch). */
int orc_sgd_step(orc_table* t, const uint64_t* rows, uint64_t n, const float* grads,
                 uint64_t n_grads, float lr, float beta);

/* copies of the state (same entry points exist in oracle/_ref, prefix ref_) */
void orc_copy_identities(const orc_table* t, uint64_t* out);
void orc_copy_metadata(const orc_table* t, uint64_t* out);
void orc_copy_weights(const orc_table* t, float* out);
void orc_copy_momentum(const orc_table* t, float* out);
void orc_copy_trained(const orc_table* t, uint8_t* out);
/* MpzchTable::dirty_rows_since proj/src/table.cpp:216-225 */
int orc_dirty_rows_since(const orc_table* t, uint64_t cursor, uint64_t* out, uint64_t cap,
                         uint64_t* out_n);

/* last error text (thread-local) */
/* ---- publish, proj/src/publish.cpp */
/* crc32, publish.cpp:110-124: reflected, polynomial 0xEDB88320, init/final ~0 */
uint32_t orc_crc32(const uint8_t* bytes, uint64_t n);
/* serialize_snapshot, publish.cpp:126-155 (.mpzc).  *out_len = full size even when it
 * exceeds cap (then nothing is written and ORC_ELENGTH is returned). */
int orc_serialize_snapshot(const orc_table* t, uint8_t* out, uint64_t cap, uint64_t* out_len);
/* DeltaSource::cut (publish.cpp:288-305) + serialize_delta (publish.cpp:212-230): the rows
 * dirtied since `cursor`, then a fresh cursor in *out_next_cursor. */
int orc_serialize_delta(orc_table* t, uint64_t cursor, uint32_t base_checksum, uint64_t sequence,
                        uint8_t* out, uint64_t cap, uint64_t* out_len, uint64_t* out_next_cursor);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
