/*
 * mpzch_oracle.c -- plain-C restatement of the MPZCH batched remap path.
 *
 * TEST INFRASTRUCTURE ONLY (see mpzch_oracle.h).  Parity is pinned against
 * the reference's golden vectors and against the reference library compiled
 * from /root/reference (oracle/_ref), see tests/test_oracle_*.py.
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/.
 */
#include "mpzch_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

#define EMPTY_SLOT (~(uint64_t)0)                 /* proj/include/mpzch/ids.hpp:16 */
#define HOME_SALT 0x9E3779B97F4A7C15ull           /* proj/include/mpzch/ids.hpp:20 */
#define SHARD_SALT 0xD1B54A32D192ED03ull          /* proj/include/mpzch/ids.hpp:21 */
#define GOLDEN 0x9E3779B97F4A7C15ull              /* proj/include/mpzch/rng.hpp:16 */

/* proj/include/mpzch/ids.hpp:35-43 */
uint64_t orc_mix64(uint64_t id, uint64_t seed) {
    uint64_t x = id ^ seed;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

/* proj/include/mpzch/ids.hpp:23 */
static int is_valid_id(uint64_t id) { return (id >> 63) == 0; }

/* SplitMix64::next, proj/include/mpzch/rng.hpp:15-21 */
uint64_t orc_splitmix_next(uint64_t* state) {
    *state += GOLDEN;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* DistinctIdStream::at, proj/include/mpzch/rng.hpp:40-50 */
uint64_t orc_distinct_id_at(uint64_t seed, uint64_t index) {
    const uint64_t half = (1ull << 31) - 1;
    uint64_t left = (index >> 31) & half;
    uint64_t right = index & half;
    for (uint64_t round = 0; round < 4; ++round) {
        uint64_t f = orc_mix64(right | (round << 32), seed) & half;
        uint64_t next_right = left ^ f;
        left = right;
        right = next_right;
    }
    return (left << 31) | right;
}

void orc_distinct_ids(uint64_t seed, uint64_t start, uint64_t count, uint64_t* out) {
    for (uint64_t i = 0; i < count; ++i) out[i] = orc_distinct_id_at(seed, start + i);
}

/* home_slot, proj/src/probe_core.cpp:27-30 (validity is checked by callers) */
uint64_t orc_home_slot(uint64_t id, uint64_t capacity, uint64_t seed) {
    return orc_mix64(id ^ HOME_SALT, seed) % capacity;
}

/* shard_of, proj/src/shard_router.cpp:42-46 */
uint32_t orc_shard_of(uint64_t id, uint32_t num_shards, uint64_t seed) {
    return (uint32_t)(orc_mix64(id ^ SHARD_SALT, seed) % num_shards);
}

/* draw_row, proj/src/embedding_store.cpp:12-18; SplitMix64::next_unit rng.hpp:23 */
void orc_draw_row(float* dst, uint32_t dim, uint64_t row, uint64_t init_seed) {
    uint64_t st = orc_mix64(row, init_seed);
    const double bound = 1.0 / sqrt((double)dim);
    for (uint32_t j = 0; j < dim; ++j) {
        double u = (double)(orc_splitmix_next(&st) >> 11) * 0x1.0p-53;
        dst[j] = (float)((2.0 * u - 1.0) * bound);
    }
}

/* draw_row for n rows: dst[k * dim ...] = draw_row(rows[k]) */
void orc_draw_rows(float* dst, uint32_t dim, const uint64_t* rows, uint64_t n, uint64_t init_seed) {
    for (uint64_t k = 0; k < n; ++k) orc_draw_row(dst + k * dim, dim, rows[k], init_seed);
}

/* ---------------------------------------------------------------- table */

struct orc_table {
    uint32_t num_shards;
    uint32_t max_probe;
    uint64_t seed;
    uint32_t dim;
    uint64_t init_seed;
    uint64_t* caps;     /* TableLayout::shard_capacities */
    uint64_t* offsets;  /* TableLayout::shard_offsets, num_shards + 1 */
    uint64_t total;
    uint64_t* ident;    /* IdentityArray per shard, concatenated in global-row order */
    uint64_t* meta;     /* MetadataArray per shard, concatenated */
    float* weights;     /* EmbeddingTable weights_, rows x dim */
    float* momentum;    /* EmbeddingTable momentum_ */
    uint8_t* trained;   /* EmbeddingTable trained_ */
    uint64_t* row_gen;  /* MpzchTable::row_generation_ (table.cpp:55) */
    uint64_t gen_clock; /* MpzchTable::generation_clock_ = 1 (table.hpp:125) */
};

/* MpzchTable ctor proj/src/table.cpp:34-56, TableLayout::with_capacities
 * proj/src/shard_router.cpp:8-25, ShardConfig::validate proj/src/probe_core.cpp:8-15,
 * EmbeddingTable ctor proj/src/embedding_store.cpp:22-33 */
int orc_table_create(const uint64_t* caps, uint32_t num_shards, uint32_t max_probe,
                     uint64_t seed, uint32_t dim, uint64_t init_seed, orc_table** out) {
    *out = NULL;
    if (num_shards == 0) return fail(ORC_EINVAL, "layout needs at least one shard");
    for (uint32_t s = 0; s < num_shards; ++s)
        if (caps[s] == 0) return fail(ORC_EINVAL, "shard capacity must be >= 1");
    for (uint32_t s = 0; s < num_shards; ++s)
        if (max_probe < 1 || max_probe > caps[s])
            return fail(ORC_EINVAL, "max_probe must satisfy 1 <= max_probe <= capacity");
    orc_table* t = (orc_table*)calloc(1, sizeof *t);
    if (!t) return fail(ORC_ENOMEM, "out of host memory");
    t->num_shards = num_shards;
    t->max_probe = max_probe;
    t->seed = seed;
    t->dim = dim;
    t->init_seed = init_seed;
    t->caps = (uint64_t*)malloc(sizeof(uint64_t) * num_shards);
    t->offsets = (uint64_t*)malloc(sizeof(uint64_t) * (num_shards + 1));
    t->offsets[0] = 0;
    for (uint32_t s = 0; s < num_shards; ++s) {
        t->caps[s] = caps[s];
        t->offsets[s + 1] = t->offsets[s] + caps[s];
    }
    t->total = t->offsets[num_shards];
    t->ident = (uint64_t*)malloc(sizeof(uint64_t) * t->total);
    t->meta = (uint64_t*)calloc(t->total, sizeof(uint64_t));
    t->row_gen = (uint64_t*)calloc(t->total, sizeof(uint64_t));
    if (!t->ident || !t->meta || !t->row_gen) {
        orc_table_destroy(t);
        return fail(ORC_ENOMEM, "out of host memory");
    }
    memset(t->ident, 0xff, sizeof(uint64_t) * t->total);
    t->gen_clock = 1;
    if (dim > 0) {
        t->weights = (float*)malloc(sizeof(float) * t->total * dim);
        t->momentum = (float*)calloc(t->total * dim, sizeof(float));
        t->trained = (uint8_t*)calloc(t->total, 1);
        if (!t->weights || !t->momentum || !t->trained) {
            orc_table_destroy(t);
            return fail(ORC_ENOMEM, "out of host memory");
        }
        for (uint64_t r = 0; r < t->total; ++r)
            orc_draw_row(t->weights + r * dim, dim, r, init_seed);
    }
    *out = t;
    return ORC_OK;
}

void orc_table_destroy(orc_table* t) {
    if (!t) return;
    free(t->caps);
    free(t->offsets);
    free(t->ident);
    free(t->meta);
    free(t->weights);
    free(t->momentum);
    free(t->trained);
    free(t->row_gen);
    free(t);
}

uint64_t orc_total_rows(const orc_table* t) { return t->total; }
uint64_t orc_shard_offset(const orc_table* t, uint32_t s) { return t->offsets[s]; }
uint64_t* orc_identities(orc_table* t) { return t->ident; }
uint64_t* orc_metadata(orc_table* t) { return t->meta; }
float* orc_weights(orc_table* t) { return t->weights; }
float* orc_momentum(orc_table* t) { return t->momentum; }
uint8_t* orc_trained(orc_table* t) { return t->trained; }
uint64_t* orc_row_generation(orc_table* t) { return t->row_gen; }

/* MpzchTable::make_cursor proj/src/table.cpp:209-214 */
uint64_t orc_make_cursor(orc_table* t) { return t->gen_clock++; }

/* MpzchTable::sgd_step, proj/src/table.cpp:174-179 -> embedding_store.cpp:70-93 */
int orc_sgd_step(orc_table* t, const uint64_t* rows, uint64_t n, const float* grads,
                 uint64_t n_grads, float lr, float beta) {
    /* check_embeddings, table.cpp:94-96 (check_mutable: no frozen replicas here) */
    if (t->dim == 0) return fail(ORC_ELOGIC, "table has no embedding payload (dim = 0)");
    /* embedding_store.cpp:72-81 */
    if (n_grads != n * t->dim)
        return fail(ORC_EINVAL, "gradient shape does not match rows * dim");
    if (!(lr > 0.0f)) return fail(ORC_EINVAL, "learning rate must be positive");
    if (beta < 0.0f || beta >= 1.0f)
        return fail(ORC_EINVAL, "momentum coefficient must lie in [0, 1)");
    for (uint64_t i = 0; i < n; ++i) { /* embedding_store.cpp:82-92 */
        if (rows[i] >= t->total) return fail(ORC_ERANGE, "embedding row out of range");
        float* w = t->weights + rows[i] * t->dim;
        float* m = t->momentum + rows[i] * t->dim;
        const float* g = grads + i * t->dim;
        for (uint32_t j = 0; j < t->dim; ++j) {
            volatile float bm = beta * m[j]; /* x86-64 baseline: no FMA contraction */
            m[j] = bm + g[j];
            volatile float lm = lr * m[j];
            w[j] = w[j] - lm;
        }
        t->trained[rows[i]] = 1;
    }
    for (uint64_t i = 0; i < n; ++i) t->row_gen[rows[i]] = t->gen_clock; /* table.cpp:179 */
    return ORC_OK;
}

void orc_copy_identities(const orc_table* t, uint64_t* out) {
    memcpy(out, t->ident, sizeof(uint64_t) * t->total);
}
void orc_copy_metadata(const orc_table* t, uint64_t* out) {
    memcpy(out, t->meta, sizeof(uint64_t) * t->total);
}
void orc_copy_weights(const orc_table* t, float* out) {
    if (t->dim) memcpy(out, t->weights, sizeof(float) * t->total * t->dim);
}
void orc_copy_momentum(const orc_table* t, float* out) {
    if (t->dim) memcpy(out, t->momentum, sizeof(float) * t->total * t->dim);
}
void orc_copy_trained(const orc_table* t, uint8_t* out) {
    if (t->dim) memcpy(out, t->trained, t->total);
}

/* MpzchTable::dirty_rows_since proj/src/table.cpp:216-225 */
int orc_dirty_rows_since(const orc_table* t, uint64_t cursor, uint64_t* out, uint64_t cap,
                         uint64_t* out_n) {
    if (cursor == 0 || cursor >= t->gen_clock)
        return fail(ORC_EINVAL, "stale or unknown publication cursor");
    uint64_t k = 0;
    for (uint64_t r = 0; r < t->total; ++r) {
        if (t->row_gen[r] > cursor) {
            if (k < cap) out[k] = r;
            ++k;
        }
    }
    *out_n = k;
    return ORC_OK;
}

/* --------------------------------------------------------------- publish */

uint32_t orc_crc32(const uint8_t* bytes, uint64_t n) { /* publish.cpp:110-124 */
    static uint32_t table[256];
    static int ready = 0;
    if (!ready) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        ready = 1;
    }
    uint32_t crc = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n; ++i) crc = table[(crc ^ bytes[i]) & 0xFFu] ^ (crc >> 8);
    return crc ^ 0xFFFFFFFFu;
}

/* ByteWriter, publish.cpp:17-38: little-endian appends */
typedef struct {
    uint8_t* p;
    uint64_t n;
} bw;
static void bw_u32(bw* w, uint32_t v) {
    for (int i = 0; i < 4; ++i) w->p[w->n++] = (uint8_t)(v >> (8 * i));
}
static void bw_u64(bw* w, uint64_t v) {
    for (int i = 0; i < 8; ++i) w->p[w->n++] = (uint8_t)(v >> (8 * i));
}
static void bw_f32(bw* w, float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    bw_u32(w, u);
}
static void bw_magic(bw* w, const char* m) {
    for (int i = 0; i < 4; ++i) w->p[w->n++] = (uint8_t)m[i];
}

int orc_serialize_snapshot(const orc_table* t, uint8_t* out, uint64_t cap, uint64_t* out_len) {
    if (t->dim == 0) return fail(ORC_ELOGIC, "index-only tables (dim = 0) cannot be published");
    const uint64_t need = 48 + 8ull * t->num_shards + 8 * t->total + 4ull * t->dim * t->total;
    *out_len = need;
    if (!out || cap < need) return fail(ORC_ELENGTH, "output buffer too small");
    bw w = {out, 0};
    bw_magic(&w, "MPZC");
    bw_u32(&w, 1); /* kFormatVersion */
    bw_u64(&w, t->seed);
    bw_u32(&w, t->max_probe);
    bw_u32(&w, t->dim);
    bw_u32(&w, t->num_shards);
    for (uint32_t s = 0; s < t->num_shards; ++s) bw_u64(&w, t->caps[s]);
    bw_u64(&w, t->total);
    for (uint64_t r = 0; r < t->total; ++r) bw_u64(&w, t->ident[r]); /* shards in order */
    bw_u64(&w, t->total * t->dim);
    for (uint64_t i = 0; i < t->total * t->dim; ++i) bw_f32(&w, t->weights[i]);
    bw_u32(&w, orc_crc32(out, w.n)); /* trailer */
    return ORC_OK;
}

int orc_serialize_delta(orc_table* t, uint64_t cursor, uint32_t base_checksum, uint64_t sequence,
                        uint8_t* out, uint64_t cap, uint64_t* out_len, uint64_t* out_next_cursor) {
    if (t->dim == 0) return fail(ORC_ELOGIC, "index-only tables (dim = 0) cannot be published");
    if (cursor == 0 || cursor >= t->gen_clock)
        return fail(ORC_EINVAL, "stale or unknown publication cursor");
    uint64_t k = 0;
    for (uint64_t r = 0; r < t->total; ++r) k += t->row_gen[r] > cursor;
    const uint64_t rec = 16 + 4ull * t->dim;
    const uint64_t need = 32 + k * rec + 4;
    *out_len = need;
    if (!out || cap < need) return fail(ORC_ELENGTH, "output buffer too small");
    *out_next_cursor = orc_make_cursor(t); /* cut: cursor_ = make_cursor() */
    bw w = {out, 0};
    bw_magic(&w, "MPZD");
    bw_u32(&w, 1);
    bw_u32(&w, base_checksum);
    bw_u64(&w, sequence);
    bw_u32(&w, t->dim);
    bw_u64(&w, k);
    for (uint64_t r = 0; r < t->total; ++r) { /* dirty rows ascending, publish.cpp:297-303 */
        if (t->row_gen[r] <= cursor) continue;
        bw_u64(&w, r);
        bw_u64(&w, t->ident[r]);
        for (uint32_t j = 0; j < t->dim; ++j) bw_f32(&w, t->weights[r * t->dim + j]);
    }
    bw_u32(&w, orc_crc32(out, w.n));
    return ORC_OK;
}

/* --------------------------------------------------------------- probe core */

/* lookup_readonly, proj/src/probe_core.cpp:32-43 (full window, no early exit) */
static void probe_readonly(uint64_t id, const uint64_t* I, uint64_t cap, uint32_t P,
                           uint64_t home, uint64_t* slot_out, uint8_t* oc_out) {
    uint64_t slot = home;
    for (uint32_t i = 0; i < P; ++i) {
        if (I[slot] == id) {
            *slot_out = slot;
            *oc_out = ORC_FOUND;
            return;
        }
        if (++slot == cap) slot = 0;
    }
    *slot_out = home;
    *oc_out = ORC_COLLISION;
}

/* lookup_or_insert, proj/src/probe_core.cpp:69-134 (two passes) */
static void probe(uint64_t id, uint64_t meta_in, uint64_t now, uint64_t* I, uint64_t* M,
                  uint64_t cap, uint32_t P, int mode, uint64_t home, uint64_t* slot_out,
                  uint8_t* oc_out) {
    /* Pass 1: discovery, probe_core.cpp:78-86 */
    int exists = 0;
    uint64_t slot = home;
    for (uint32_t i = 0; i < P; ++i) {
        if (I[slot] == id) {
            exists = 1;
            break;
        }
        if (++slot == cap) slot = 0;
    }
    /* Pass 2: update / insert / evict, probe_core.cpp:89-121 */
    const int ttl = mode == ORC_MODE_TTL, lru = mode == ORC_MODE_LRU;
    int have_victim = 0;
    uint64_t victim = 0, victim_stored = 0;
    slot = home;
    for (uint32_t i = 0; i < P; ++i) {
        const uint64_t occ = I[slot];
        if (occ == id) {
            M[slot] = meta_in;
            *slot_out = slot;
            *oc_out = ORC_FOUND;
            return;
        }
        if (occ == EMPTY_SLOT) {
            I[slot] = id;
            M[slot] = meta_in;
            *slot_out = slot;
            *oc_out = ORC_INSERTED;
            return;
        }
        if (!exists) {
            if (ttl && M[slot] < now) { /* is_expired, eviction.hpp:53 */
                I[slot] = id;
                M[slot] = meta_in;
                *slot_out = slot;
                *oc_out = ORC_EVICTED;
                return;
            }
            if (lru && (!have_victim || M[slot] < victim_stored)) {
                have_victim = 1;
                victim = slot;
                victim_stored = M[slot];
            }
        }
        if (++slot == cap) slot = 0;
    }
    /* LRU fallback, probe_core.cpp:125-129 */
    if (lru && have_victim) {
        I[victim] = id;
        M[victim] = meta_in;
        *slot_out = victim;
        *oc_out = ORC_EVICTED;
        return;
    }
    /* Collision fallback, probe_core.cpp:132-133 */
    M[home] = meta_in;
    *slot_out = home;
    *oc_out = ORC_COLLISION;
}

/* require_valid_id, proj/include/mpzch/ids.hpp:25-31 */
static int require_valid_id(uint64_t id) {
    if (is_valid_id(id)) return ORC_OK;
    return fail(ORC_EINVAL, id == EMPTY_SLOT ? "id is the empty-slot sentinel"
                                             : "id exceeds the 63-bit ID space");
}

/* check_metadata_input, proj/src/probe_core.cpp:49-58 */
static int check_metadata_input(int mode, uint64_t meta_in, uint64_t now) {
    if (mode == ORC_MODE_TTL) {
        if (meta_in <= now) return fail(ORC_EINVAL, "TTL metadata must be an expiry in the future");
    } else if (meta_in != now) {
        return fail(ORC_EINVAL, "non-TTL metadata must equal the current timestamp");
    }
    return ORC_OK;
}

int orc_probe(uint64_t id, uint64_t meta_in, uint64_t now, uint64_t* identities,
              uint64_t* metadata, uint64_t capacity, uint32_t max_probe, uint64_t seed, int mode,
              uint64_t* out_slot, uint8_t* out_outcome) {
    if (capacity < 1) return fail(ORC_EINVAL, "shard capacity must be >= 1");
    if (max_probe < 1 || max_probe > capacity)
        return fail(ORC_EINVAL, "max_probe must satisfy 1 <= max_probe <= capacity");
    int rc = require_valid_id(id);
    if (rc) return rc;
    rc = check_metadata_input(mode, meta_in, now);
    if (rc) return rc;
    probe(id, meta_in, now, identities, metadata, capacity, max_probe, mode,
          orc_home_slot(id, capacity, seed), out_slot, out_outcome);
    return ORC_OK;
}

int orc_probe_readonly(uint64_t id, const uint64_t* identities, uint64_t capacity,
                       uint32_t max_probe, uint64_t seed, uint64_t* out_slot,
                       uint8_t* out_outcome) {
    int rc = require_valid_id(id);
    if (rc) return rc;
    probe_readonly(id, identities, capacity, max_probe, orc_home_slot(id, capacity, seed),
                   out_slot, out_outcome);
    return ORC_OK;
}

/* ---------------------------------------------------------------- policy */

/* TtlPolicy::validate proj/src/eviction.cpp:8-18 (+ a duplicate-key check the
 * unordered_map makes unrepresentable in the reference) */
static int validate_policy(int mode, uint64_t default_ttl, uint32_t n_feat,
                           const uint32_t* keys, const uint64_t* ttls) {
    if (mode < 0 || mode > 2) return fail(ORC_EINVAL, "unknown eviction mode");
    if (mode != ORC_MODE_TTL) return ORC_OK;
    if (default_ttl == 0) return fail(ORC_EINVAL, "default TTL must be strictly positive");
    for (uint32_t i = 0; i < n_feat; ++i) {
        if (ttls[i] == 0) {
            snprintf(g_err, sizeof g_err,
                     "per-feature TTL must be strictly positive (feature %u)", keys[i]);
            return ORC_EINVAL;
        }
        for (uint32_t j = 0; j < i; ++j)
            if (keys[j] == keys[i]) return fail(ORC_EINVAL, "duplicate feature in per-feature TTL map");
    }
    return ORC_OK;
}

/* TtlPolicy::ttl_for proj/include/mpzch/eviction.hpp:17-20 */
static uint64_t ttl_for(uint64_t default_ttl, uint32_t n_feat, const uint32_t* keys,
                        const uint64_t* ttls, uint32_t f) {
    for (uint32_t i = 0; i < n_feat; ++i)
        if (keys[i] == f) return ttls[i];
    return default_ttl;
}

/* make_metadata proj/src/eviction.cpp:20-30 */
static int make_metadata(int mode, uint64_t now, uint64_t ttl, uint64_t* out) {
    if (mode != ORC_MODE_TTL) {
        *out = now;
        return ORC_OK;
    }
    if (ttl > ~(uint64_t)0 - now)
        return fail(ORC_EOVERFLOW, "TTL expiry overflows the 64-bit timestamp range");
    *out = now + ttl;
    return ORC_OK;
}

/* EmbeddingTable::reset_row proj/src/embedding_store.cpp:62-68 */
static void reset_row(orc_table* t, uint64_t row) {
    orc_draw_row(t->weights + row * t->dim, t->dim, row, t->init_seed);
    memset(t->momentum + row * t->dim, 0, sizeof(float) * t->dim);
    t->trained[row] = 0;
}

/* ---------------------------------------------------------------- batch */

/* DedupMap / dedup_into proj/src/batch_engine.cpp:17-108: first-occurrence
 * dedup keyed on (id, feature). Any exact first-occurrence map gives the same
 * uniques/inverse; a plain open-addressed table is used here. */
typedef struct {
    uint64_t id;
    uint32_t feat;
    uint32_t uniq; /* UINT32_MAX = empty */
} dslot;

int orc_process_batch(orc_table* t, const uint64_t* ids, const uint32_t* features, uint64_t n,
                      uint64_t now, int mode, uint64_t default_ttl, uint32_t n_feat,
                      const uint32_t* feat_keys, const uint64_t* feat_ttls,
                      uint64_t* out_slots, uint8_t* out_outcomes, uint64_t* out_evicted,
                      uint64_t evicted_cap, uint64_t* out_evicted_n) {
    int rc = validate_policy(mode, default_ttl, n_feat, feat_keys, feat_ttls);
    if (rc) return rc;
    if (out_evicted_n) *out_evicted_n = 0;
    /* batch_engine.cpp:82-83 */
    if (n > 0xffffffffull) return fail(ORC_ELENGTH, "batch exceeds 2^32 - 1 positions");
    /* validation pass, batch_engine.cpp:90-94 */
    for (uint64_t i = 0; i < n; ++i) {
        if (!is_valid_id(ids[i])) {
            snprintf(g_err, sizeof g_err, "invalid id at batch position %llu",
                     (unsigned long long)i);
            return ORC_EINVAL;
        }
    }
    /* first-occurrence dedup, batch_engine.cpp:100-106 */
    uint64_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    dslot* map = (dslot*)malloc(sizeof(dslot) * cap);
    uint32_t* inverse = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint64_t* u_id = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint32_t* u_feat = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint64_t* u_meta = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint64_t* u_slot = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint8_t* u_oc = (uint8_t*)malloc(n ? n : 1);
    if (!map || !inverse || !u_id || !u_feat || !u_meta || !u_slot || !u_oc) {
        free(map); free(inverse); free(u_id); free(u_feat); free(u_meta); free(u_slot); free(u_oc);
        return fail(ORC_ENOMEM, "out of host memory");
    }
    for (uint64_t h = 0; h < cap; ++h) map[h].uniq = 0xffffffffu;
    uint32_t count = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t f = features ? features[i] : 0;
        uint64_t h = orc_mix64(ids[i] ^ ((uint64_t)f << 32), 0) & (cap - 1);
        for (;;) {
            if (map[h].uniq == 0xffffffffu) {
                map[h].id = ids[i];
                map[h].feat = f;
                map[h].uniq = count;
                u_id[count] = ids[i];
                u_feat[count] = f;
                inverse[i] = count++;
                break;
            }
            if (map[h].id == ids[i] && map[h].feat == f) {
                inverse[i] = map[h].uniq;
                break;
            }
            h = (h + 1) & (cap - 1);
        }
    }
    free(map);
    /* TTL metas, batch_engine.cpp:153-158 */
    for (uint32_t u = 0; u < count; ++u) {
        rc = make_metadata(mode, now, ttl_for(default_ttl, n_feat, feat_keys, feat_ttls, u_feat[u]),
                           &u_meta[u]);
        if (rc) {
            free(inverse); free(u_id); free(u_feat); free(u_meta); free(u_slot); free(u_oc);
            return rc;
        }
    }
    /* Stable partition by shard then per-shard probes in dedup order
     * (batch_engine.cpp:160-211, table.cpp:112-148).  Shards touch disjoint
     * state, so visiting shard by shard over the dedup order is equivalent. */
    for (uint32_t s = 0; s < t->num_shards; ++s) {
        uint64_t* I = t->ident + t->offsets[s];
        uint64_t* M = t->meta + t->offsets[s];
        for (uint32_t u = 0; u < count; ++u) {
            if (orc_shard_of(u_id[u], t->num_shards, t->seed) != s) continue;
            uint64_t local;
            uint8_t oc;
            probe(u_id[u], u_meta[u], now, I, M, t->caps[s], t->max_probe, mode,
                  orc_home_slot(u_id[u], t->caps[s], t->seed), &local, &oc);
            const uint64_t global = t->offsets[s] + local;
            if (oc == ORC_EVICTED && t->dim > 0) reset_row(t, global); /* table.cpp:142 */
            if (oc == ORC_INSERTED || oc == ORC_EVICTED)
                t->row_gen[global] = t->gen_clock; /* touch_row table.cpp:262-264 */
            u_slot[u] = global;
            u_oc[u] = oc;
        }
    }
    /* scatter, batch_engine.cpp:213-220 */
    for (uint64_t i = 0; i < n; ++i) {
        out_slots[i] = u_slot[inverse[i]];
        out_outcomes[i] = u_oc[inverse[i]];
    }
    /* canonical evicted list: uniques with outcome Evicted, unique-rank order */
    uint64_t ne = 0;
    for (uint32_t u = 0; u < count; ++u) {
        if (u_oc[u] != ORC_EVICTED) continue;
        if (out_evicted && ne < evicted_cap) out_evicted[ne] = u_slot[u];
        ++ne;
    }
    if (out_evicted_n) *out_evicted_n = ne;
    free(inverse); free(u_id); free(u_feat); free(u_meta); free(u_slot); free(u_oc);
    return ORC_OK;
}

/* MpzchTable::lookup proj/src/table.cpp:150-156 */
int orc_lookup(const orc_table* t, const uint64_t* ids, uint64_t n, uint64_t* out_slots,
               uint8_t* out_outcomes) {
    for (uint64_t i = 0; i < n; ++i) {
        int rc = require_valid_id(ids[i]);
        if (rc) return rc;
        const uint32_t s = orc_shard_of(ids[i], t->num_shards, t->seed);
        uint64_t local;
        probe_readonly(ids[i], t->ident + t->offsets[s], t->caps[s], t->max_probe,
                       orc_home_slot(ids[i], t->caps[s], t->seed), &local, &out_outcomes[i]);
        out_slots[i] = t->offsets[s] + local;
    }
    return ORC_OK;
}

/* MpzchTable::lookup_or_insert proj/src/table.cpp:98-110 */
int orc_lookup_or_insert(orc_table* t, uint64_t id, uint32_t feature, uint64_t now, int mode,
                         uint64_t default_ttl, uint32_t n_feat, const uint32_t* feat_keys,
                         const uint64_t* feat_ttls, uint64_t* out_slot, uint8_t* out_outcome) {
    int rc = validate_policy(mode, default_ttl, n_feat, feat_keys, feat_ttls);
    if (rc) return rc;
    rc = require_valid_id(id);
    if (rc) return rc;
    const uint32_t s = orc_shard_of(id, t->num_shards, t->seed);
    uint64_t meta;
    rc = make_metadata(mode, now, ttl_for(default_ttl, n_feat, feat_keys, feat_ttls, feature), &meta);
    if (rc) return rc;
    uint64_t local;
    probe(id, meta, now, t->ident + t->offsets[s], t->meta + t->offsets[s], t->caps[s],
          t->max_probe, mode, orc_home_slot(id, t->caps[s], t->seed), &local, out_outcome);
    const uint64_t global = t->offsets[s] + local;
    if (*out_outcome == ORC_EVICTED && t->dim > 0) reset_row(t, global);
    if (*out_outcome == ORC_INSERTED || *out_outcome == ORC_EVICTED)
        t->row_gen[global] = t->gen_clock;
    *out_slot = global;
    return ORC_OK;
}
