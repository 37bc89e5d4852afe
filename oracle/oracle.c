/*
 * oracle.c -- CPU restatement of the recsparse hot path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use
 * this file; the product (librsgpu.so) never links it.  Each function cites
 * the reference code it restates (paths relative to /root/reference/proj).
 * Must be compiled with -ffp-contract=off: the reference's Adam result bits
 * depend on it (SURVEY.md §8c "Build-flag hazard").
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ======================================================================== */
/* L0: hash.hpp:26-33 (fmix64), hash.hpp:46-52 (Eq. 5 probe step)          */
/* ======================================================================== */
uint64_t or_hash64(uint64_t key) {
  key ^= key >> 33;
  key *= 0xff51afd7ed558ccdULL;
  key ^= key >> 33;
  key *= 0xc4ceb9fe1a85ec53ULL;
  key ^= key >> 33;
  return key;
}

int or_probe_step(uint64_t key, uint64_t capacity, uint64_t groups, uint64_t* step) {
  if (groups == 0 || capacity / groups < 2) return 1; /* hash.hpp:47-49 ConfigError */
  const uint64_t modulus = capacity / groups - 1;
  *step = ((key % modulus + 1) | 1) * groups;
  return 0;
}

void or_hash64_batch(const uint64_t* keys, size_t n, uint64_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = or_hash64(keys[i]); /* hash.cpp:32-38 */
}

/* ======================================================================== */
/* Small open-addressing u64 -> size_t map used by the dedup restatements   */
/* (stands in for std::unordered_map in exchange_sim.cpp:87-115).           */
/* ======================================================================== */
typedef struct {
  uint64_t* keys;
  size_t* vals;
  uint8_t* used;
  size_t mask;
} u64map;

static void map_init(u64map* m, size_t n) {
  size_t cap = 16;
  while (cap < 2 * n + 2) cap <<= 1;
  m->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
  m->vals = (size_t*)malloc(cap * sizeof(size_t));
  m->used = (uint8_t*)calloc(cap, 1);
  m->mask = cap - 1;
}
static void map_free(u64map* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
}
/* try_emplace: returns pointer to value; *fresh = 1 when inserted */
static size_t* map_try_emplace(u64map* m, uint64_t key, size_t val, int* fresh) {
  size_t i = (size_t)or_hash64(key ^ 0x5bd1e9955bd1e995ULL) & m->mask;
  for (;;) {
    if (!m->used[i]) {
      m->used[i] = 1;
      m->keys[i] = key;
      m->vals[i] = val;
      *fresh = 1;
      return &m->vals[i];
    }
    if (m->keys[i] == key) {
      *fresh = 0;
      return &m->vals[i];
    }
    i = (i + 1) & m->mask;
  }
}

/* ======================================================================== */
/* L1: EmbedTable restatement (embed_table.hpp:73-211, embed_table.cpp)     */
/* ======================================================================== */
enum { ST_EMPTY = 0, ST_OCC = 1, ST_TOMB = 2 }; /* embed_table.hpp:47 */

typedef struct {
  uint32_t fresh, freed;
  int retired;
} chunk_meta;

struct or_table {
  uint64_t capacity;
  uint32_t dim, groups, chunk_rows;
  double lf;
  /* key structure (AoS KeySlot, embed_table.hpp:49-53) */
  uint64_t* skey;
  int64_t* srow;
  uint8_t* sstate;
  /* embedding structure: chunks of chunk_rows rows (embed_table.hpp:164-173) */
  size_t nchunks, chunk_cap;
  chunk_meta* chunks;
  float **emb, **m, **v;
  uint64_t **ts, **step;
  int64_t* freelist; /* LIFO (embed_table.hpp:205) */
  size_t nfree, free_cap;
  uint32_t current, next;
  uint64_t occupied, tombstones, tick;
};

static void add_chunk(or_table* t) { /* make_chunk, embed_table.cpp:99-109 */
  if (t->nchunks == t->chunk_cap) {
    size_t nc = t->chunk_cap ? 2 * t->chunk_cap : 4;
    t->chunks = (chunk_meta*)realloc(t->chunks, nc * sizeof(chunk_meta));
    t->emb = (float**)realloc(t->emb, nc * sizeof(float*));
    t->m = (float**)realloc(t->m, nc * sizeof(float*));
    t->v = (float**)realloc(t->v, nc * sizeof(float*));
    t->ts = (uint64_t**)realloc(t->ts, nc * sizeof(uint64_t*));
    t->step = (uint64_t**)realloc(t->step, nc * sizeof(uint64_t*));
    t->chunk_cap = nc;
  }
  size_t c = t->nchunks++;
  size_t rd = (size_t)t->chunk_rows * t->dim;
  t->chunks[c].fresh = 0;
  t->chunks[c].freed = 0;
  t->chunks[c].retired = 0;
  t->emb[c] = (float*)calloc(rd, sizeof(float));
  t->m[c] = (float*)calloc(rd, sizeof(float));
  t->v[c] = (float*)calloc(rd, sizeof(float));
  t->ts[c] = (uint64_t*)calloc(t->chunk_rows, sizeof(uint64_t));
  t->step[c] = (uint64_t*)calloc(t->chunk_rows, sizeof(uint64_t));
}

static int is_pow2(uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }

int or_table_create(uint64_t capacity, uint32_t dim, uint32_t groups, double lf,
                    uint32_t chunk_rows, or_table** out) {
  /* TableConfig::validate, embed_table.cpp:23-38 */
  if (!is_pow2(capacity) || !is_pow2(groups) || capacity < 2 * (uint64_t)groups ||
      !(lf > 0.0 && lf < 1.0) || chunk_rows < 1 || dim < 1)
    return 1;
  or_table* t = (or_table*)calloc(1, sizeof(or_table));
  t->capacity = capacity;
  t->dim = dim;
  t->groups = groups;
  t->chunk_rows = chunk_rows;
  t->lf = lf;
  t->skey = (uint64_t*)calloc(capacity, sizeof(uint64_t));
  t->srow = (int64_t*)calloc(capacity, sizeof(int64_t));
  t->sstate = (uint8_t*)calloc(capacity, 1);
  add_chunk(t); /* embed_table.cpp:43-44 */
  add_chunk(t);
  t->current = 0;
  t->next = 1;
  *out = t;
  return 0;
}

void or_table_destroy(or_table* t) {
  if (!t) return;
  for (size_t c = 0; c < t->nchunks; ++c) {
    free(t->emb[c]);
    free(t->m[c]);
    free(t->v[c]);
    free(t->ts[c]);
    free(t->step[c]);
  }
  free(t->chunks);
  free(t->emb);
  free(t->m);
  free(t->v);
  free(t->ts);
  free(t->step);
  free(t->skey);
  free(t->srow);
  free(t->sstate);
  free(t->freelist);
  free(t);
}

uint64_t or_table_capacity(const or_table* t) { return t->capacity; }
uint64_t or_table_occupied(const or_table* t) { return t->occupied; }
uint64_t or_table_tombstones(const or_table* t) { return t->tombstones; }
uint64_t or_table_tick(const or_table* t) { return t->tick; }

#define ROW_CHUNK(t, r) ((size_t)((r) / (t)->chunk_rows))
#define ROW_IDX(t, r) ((size_t)((r) % (t)->chunk_rows))
float* or_table_emb(or_table* t, int64_t r) {
  return t->emb[ROW_CHUNK(t, r)] + ROW_IDX(t, r) * t->dim;
}
float* or_table_m(or_table* t, int64_t r) { return t->m[ROW_CHUNK(t, r)] + ROW_IDX(t, r) * t->dim; }
float* or_table_v(or_table* t, int64_t r) { return t->v[ROW_CHUNK(t, r)] + ROW_IDX(t, r) * t->dim; }
uint64_t* or_table_ts(or_table* t, int64_t r) { return t->ts[ROW_CHUNK(t, r)] + ROW_IDX(t, r); }
uint64_t* or_table_step(or_table* t, int64_t r) {
  return t->step[ROW_CHUNK(t, r)] + ROW_IDX(t, r);
}

typedef struct {
  uint64_t found, tomb, empty;
} probe_hit;
#define NONE_SLOT (~(uint64_t)0)

/* probe_walk, embed_table.cpp:111-142: group-major, then step-major. */
static probe_hit probe_walk(const or_table* t, uint64_t key, const uint64_t* skey,
                            const uint8_t* sstate, uint64_t m) {
  const uint64_t groups = t->groups;
  const uint64_t h0 = or_hash64(key) % m;
  uint64_t step = 0;
  or_probe_step(key, m, groups, &step);
  const uint64_t per_group = m / groups;
  probe_hit hit = {NONE_SLOT, NONE_SLOT, NONE_SLOT};
  for (uint64_t g = 0; g < groups; ++g) {
    uint64_t pos = h0 + g;
    if (pos >= m) pos -= m;
    for (uint64_t s = 0; s < per_group; ++s) {
      if (sstate[pos] == ST_EMPTY) {
        hit.empty = pos;
        return hit;
      }
      if (sstate[pos] == ST_OCC && skey[pos] == key) {
        hit.found = pos;
        return hit;
      }
      if (sstate[pos] == ST_TOMB && hit.tomb == NONE_SLOT) hit.tomb = pos;
      pos += step;
      if (pos >= m) pos -= m;
    }
  }
  return hit;
}

static void reset_row(or_table* t, int64_t r) { /* embed_table.cpp:173-180 */
  memset(or_table_m(t, r), 0, t->dim * sizeof(float));
  memset(or_table_v(t, r), 0, t->dim * sizeof(float));
  *or_table_ts(t, r) = 0;
  *or_table_step(t, r) = 0;
}

static int64_t alloc_row(or_table* t) { /* embed_table.cpp:144-166 */
  if (t->nfree) {
    int64_t r = t->freelist[--t->nfree];
    t->chunks[ROW_CHUNK(t, r)].freed--;
    reset_row(t, r);
    return r;
  }
  chunk_meta* cur = &t->chunks[t->current];
  if (cur->fresh < t->chunk_rows) {
    return (int64_t)t->current * t->chunk_rows + cur->fresh++;
  }
  cur->retired = 1;
  uint32_t former_next = t->next;
  int64_t r = (int64_t)former_next * t->chunk_rows + t->chunks[former_next].fresh++;
  t->current = former_next;
  add_chunk(t);
  t->next = (uint32_t)(t->nchunks - 1);
  return r;
}

static void free_row(or_table* t, int64_t r) { /* embed_table.cpp:168-171 */
  if (t->nfree == t->free_cap) {
    t->free_cap = t->free_cap ? 2 * t->free_cap : 64;
    t->freelist = (int64_t*)realloc(t->freelist, t->free_cap * sizeof(int64_t));
  }
  t->freelist[t->nfree++] = r;
  t->chunks[ROW_CHUNK(t, r)].freed++;
}

static uint64_t expand_impl(or_table* t) { /* embed_table.cpp:267-285 */
  uint64_t nc = t->capacity;
  do {
    nc <<= 1;
  } while ((double)t->occupied > t->lf * (double)nc);
  uint64_t* nkey = (uint64_t*)calloc(nc, sizeof(uint64_t));
  int64_t* nrow = (int64_t*)calloc(nc, sizeof(int64_t));
  uint8_t* nst = (uint8_t*)calloc(nc, 1);
  for (uint64_t s = 0; s < t->capacity; ++s) {
    if (t->sstate[s] != ST_OCC) continue;
    probe_hit h = probe_walk(t, t->skey[s], nkey, nst, nc);
    /* h.empty always exists: the new array is below the load ceiling */
    nkey[h.empty] = t->skey[s];
    nrow[h.empty] = t->srow[s];
    nst[h.empty] = ST_OCC;
  }
  free(t->skey);
  free(t->srow);
  free(t->sstate);
  t->skey = nkey;
  t->srow = nrow;
  t->sstate = nst;
  t->capacity = nc;
  t->tombstones = 0;
  return nc;
}

static uint64_t next_tick(or_table* t) { return ++t->tick; } /* embed_table.hpp:194 */

int64_t or_table_insert(or_table* t, uint64_t key, const float* emb) { /* :193-227 */
  const uint64_t now = next_tick(t);
  probe_hit hit = probe_walk(t, key, t->skey, t->sstate, t->capacity);
  if (hit.found != NONE_SLOT) {
    int64_t r = t->srow[hit.found];
    memcpy(or_table_emb(t, r), emb, t->dim * sizeof(float));
    *or_table_ts(t, r) = now;
    return r;
  }
  while (hit.tomb == NONE_SLOT &&
         (double)(t->occupied + t->tombstones + 1) > t->lf * (double)t->capacity) {
    expand_impl(t);
    hit = probe_walk(t, key, t->skey, t->sstate, t->capacity);
  }
  uint64_t slot;
  int reuse = 0;
  if (hit.tomb != NONE_SLOT) {
    slot = hit.tomb;
    reuse = 1;
  } else if (hit.empty != NONE_SLOT) {
    slot = hit.empty;
  } else {
    return -1; /* InvariantError */
  }
  /* place_new, embed_table.cpp:182-191 */
  int64_t r = alloc_row(t);
  memcpy(or_table_emb(t, r), emb, t->dim * sizeof(float));
  *or_table_ts(t, r) = t->tick;
  t->skey[slot] = key;
  t->srow[slot] = r;
  t->sstate[slot] = ST_OCC;
  t->occupied++;
  if (reuse) t->tombstones--;
  return r;
}

int64_t or_table_lookup(or_table* t, uint64_t key) { /* :229-235 */
  probe_hit hit = probe_walk(t, key, t->skey, t->sstate, t->capacity);
  if (hit.found == NONE_SLOT) return -1;
  int64_t r = t->srow[hit.found];
  *or_table_ts(t, r) = next_tick(t);
  return r;
}

int64_t or_table_find(const or_table* t, uint64_t key) { /* :237-241 */
  probe_hit hit = probe_walk(t, key, t->skey, t->sstate, t->capacity);
  return hit.found == NONE_SLOT ? -1 : t->srow[hit.found];
}

int64_t or_table_ensure(or_table* t, uint64_t key) { /* :243-248 */
  int64_t r = or_table_lookup(t, key);
  if (r >= 0) return r;
  float* zeros = (float*)calloc(t->dim, sizeof(float));
  r = or_table_insert(t, key, zeros);
  free(zeros);
  return r;
}

int or_table_remove(or_table* t, uint64_t key) { /* :250-260 */
  probe_hit hit = probe_walk(t, key, t->skey, t->sstate, t->capacity);
  if (hit.found == NONE_SLOT) return 0;
  next_tick(t);
  free_row(t, t->srow[hit.found]);
  t->sstate[hit.found] = ST_TOMB;
  t->occupied--;
  t->tombstones++;
  return 1;
}

uint64_t or_table_expand(or_table* t) { /* :262-265 */
  next_tick(t);
  return expand_impl(t);
}

void or_table_lookup_batch(or_table* t, const uint64_t* keys, size_t n, float* out) {
  /* lookup_batch_serial, embed_table.cpp:317-335: one tick per batch */
  const uint64_t now = next_tick(t);
  for (size_t j = 0; j < n; ++j) {
    probe_hit hit = probe_walk(t, keys[j], t->skey, t->sstate, t->capacity);
    float* dst = out + j * t->dim;
    if (hit.found != NONE_SLOT) {
      int64_t r = t->srow[hit.found];
      memcpy(dst, or_table_emb(t, r), t->dim * sizeof(float));
      *or_table_ts(t, r) = now;
    } else {
      memset(dst, 0, t->dim * sizeof(float));
    }
  }
}

typedef struct {
  uint64_t key;
  int64_t row;
  uint64_t ts;
} entry;

static int cmp_entry_key(const void* a, const void* b) {
  uint64_t x = ((const entry*)a)->key, y = ((const entry*)b)->key;
  return x < y ? -1 : x > y;
}
static int cmp_entry_ts_key(const void* a, const void* b) {
  const entry* x = (const entry*)a;
  const entry* y = (const entry*)b;
  if (x->ts != y->ts) return x->ts < y->ts ? -1 : 1;
  return x->key < y->key ? -1 : x->key > y->key;
}

static entry* collect_entries(const or_table* t, size_t* n) {
  entry* e = (entry*)malloc((t->occupied + 1) * sizeof(entry));
  size_t k = 0;
  for (uint64_t s = 0; s < t->capacity; ++s) {
    if (t->sstate[s] != ST_OCC) continue;
    e[k].key = t->skey[s];
    e[k].row = t->srow[s];
    e[k].ts = *or_table_ts((or_table*)t, t->srow[s]);
    ++k;
  }
  *n = k;
  return e;
}

size_t or_table_export(const or_table* t, uint64_t* keys, float* emb, float* m, float* v,
                       uint64_t* step, uint64_t* ts) {
  /* contents view used by collect_entries (test_checkpoint.cpp:62-78) */
  size_t n = 0;
  entry* e = collect_entries(t, &n);
  qsort(e, n, sizeof(entry), cmp_entry_key);
  or_table* mt = (or_table*)t;
  for (size_t i = 0; i < n; ++i) {
    if (keys) keys[i] = e[i].key;
    if (emb) memcpy(emb + i * t->dim, or_table_emb(mt, e[i].row), t->dim * sizeof(float));
    if (m) memcpy(m + i * t->dim, or_table_m(mt, e[i].row), t->dim * sizeof(float));
    if (v) memcpy(v + i * t->dim, or_table_v(mt, e[i].row), t->dim * sizeof(float));
    if (step) step[i] = *or_table_step(mt, e[i].row);
    if (ts) ts[i] = e[i].ts;
  }
  free(e);
  return n;
}

/* ---- batch-tick semantics (no reference counterpart for the
 *      eviction half, which is a frozen restatement) ---------------------- */
size_t or_table_evict_oldest(or_table* t, size_t k) {
  size_t n = 0;
  entry* e = collect_entries(t, &n);
  if (k > n) k = n;
  qsort(e, n, sizeof(entry), cmp_entry_ts_key);
  for (size_t i = 0; i < k; ++i) or_table_remove(t, e[i].key);
  free(e);
  return k;
}

int64_t or_table_ensure_batch(or_table* t, const uint64_t* keys, size_t n, uint64_t tick,
                              uint64_t max_keys, int64_t* rows_out) {
  int64_t* rows = (int64_t*)malloc((n + 1) * sizeof(int64_t));
  size_t found = 0;
  for (size_t i = 0; i < n; ++i) {
    rows[i] = or_table_find(t, keys[i]);
    if (rows[i] >= 0) ++found;
  }
  const size_t missing = n - found;
  int64_t evicted = 0;
  if (max_keys > 0 && t->occupied + missing > max_keys) {
    const uint64_t need = t->occupied + missing - max_keys;
    if (need > t->occupied - found) {
      free(rows);
      return -1; /* the batch alone exceeds the bound */
    }
  }
  for (size_t i = 0; i < n; ++i)
    if (rows[i] >= 0) *or_table_ts(t, rows[i]) = tick;
  if (max_keys > 0 && t->occupied + missing > max_keys) {
    evicted = (int64_t)or_table_evict_oldest(t, t->occupied + missing - max_keys);
  }
  float* zeros = (float*)calloc(t->dim, sizeof(float));
  for (size_t i = 0; i < n; ++i) {
    if (rows[i] < 0) {
      rows[i] = or_table_insert(t, keys[i], zeros);
      *or_table_ts(t, rows[i]) = tick;
    }
  }
  free(zeros);
  if (rows_out) memcpy(rows_out, rows, n * sizeof(int64_t));
  free(rows);
  return evicted;
}

/* ======================================================================== */
/* Dedup + sharded lookup (exchange_sim.cpp)                                */
/* ======================================================================== */
size_t or_stage1_dedup(const uint64_t* ids, size_t n, uint64_t* unique, int64_t* inverse) {
  /* exchange_sim.cpp:87-98: first-occurrence order */
  u64map m;
  map_init(&m, n);
  size_t nu = 0;
  for (size_t j = 0; j < n; ++j) {
    int fresh = 0;
    size_t* pos = map_try_emplace(&m, ids[j], nu, &fresh);
    if (fresh) unique[nu++] = ids[j];
    inverse[j] = (int64_t)*pos;
  }
  map_free(&m);
  return nu;
}

size_t or_stage2_dedup(const uint64_t* received, const uint64_t* counts, size_t world,
                       uint64_t* unique, uint64_t* origin_off, uint64_t* origin_src,
                       uint64_t* origin_pos) {
  /* exchange_sim.cpp:100-115: unique over the source-ordered concatenation,
   * origins per unique in (source, position) visiting order */
  size_t total = 0;
  for (size_t s = 0; s < world; ++s) total += counts[s];
  u64map m;
  map_init(&m, total);
  size_t* uidx = (size_t*)malloc((total + 1) * sizeof(size_t));
  size_t nu = 0, j = 0;
  for (size_t s = 0; s < world; ++s) {
    for (size_t p = 0; p < counts[s]; ++p, ++j) {
      int fresh = 0;
      size_t* u = map_try_emplace(&m, received[j], nu, &fresh);
      if (fresh) unique[nu++] = received[j];
      uidx[j] = *u;
    }
  }
  if (origin_off) {
    memset(origin_off, 0, (nu + 1) * sizeof(uint64_t));
    for (j = 0; j < total; ++j) origin_off[uidx[j] + 1]++;
    for (size_t u = 0; u < nu; ++u) origin_off[u + 1] += origin_off[u];
    uint64_t* cursor = (uint64_t*)malloc((nu + 1) * sizeof(uint64_t));
    memcpy(cursor, origin_off, (nu + 1) * sizeof(uint64_t));
    j = 0;
    for (size_t s = 0; s < world; ++s) {
      for (size_t p = 0; p < counts[s]; ++p, ++j) {
        uint64_t at = cursor[uidx[j]]++;
        if (origin_src) origin_src[at] = s;
        if (origin_pos) origin_pos[at] = p;
      }
    }
    free(cursor);
  }
  free(uidx);
  map_free(&m);
  return nu;
}

uint64_t or_shard_of(uint64_t id, uint64_t world) { /* exchange_sim.cpp:82-85 */
  return or_hash64(id) % world;
}

struct or_cluster {
  size_t world;
  int mode; /* 0 none, 1 comm_unique, 2 lookup_unique, 3 two_stage (exchange_sim.hpp:31) */
  uint32_t dim;
  or_table** shards;
};

int or_cluster_create(size_t world, uint64_t capacity, uint32_t dim, uint32_t groups,
                      double lf, uint32_t chunk_rows, int mode, or_cluster** out) {
  if (world == 0 || mode < 0 || mode > 3) return 1;
  or_cluster* c = (or_cluster*)calloc(1, sizeof(or_cluster));
  c->world = world;
  c->mode = mode;
  c->dim = dim;
  c->shards = (or_table**)calloc(world, sizeof(or_table*));
  for (size_t s = 0; s < world; ++s) {
    if (or_table_create(capacity, dim, groups, lf, chunk_rows, &c->shards[s])) {
      for (size_t r = 0; r < s; ++r) or_table_destroy(c->shards[r]);
      free(c->shards);
      free(c);
      return 1;
    }
  }
  *out = c;
  return 0;
}

void or_cluster_destroy(or_cluster* c) {
  if (!c) return;
  for (size_t s = 0; s < c->world; ++s) or_table_destroy(c->shards[s]);
  free(c->shards);
  free(c);
}

or_table* or_cluster_shard(or_cluster* c, size_t s) { return c->shards[s]; }

int or_distributed_lookup(or_cluster* c, const uint64_t* requests, const uint64_t* counts,
                          float* out, uint64_t* ids_sent, uint64_t* embs_sent,
                          uint64_t* lookups, uint64_t* totals) {
  /* exchange_sim.cpp:117-233 */
  const size_t W = c->world, D = c->dim;
  const int s1 = c->mode == 1 || c->mode == 3;
  const int s2 = c->mode == 2 || c->mode == 3;
  uint64_t* req_off = (uint64_t*)calloc(W + 1, sizeof(uint64_t));
  for (size_t w = 0; w < W; ++w) req_off[w + 1] = req_off[w] + counts[w];
  const uint64_t T = req_off[W];
  uint64_t* uniq = (uint64_t*)malloc((T + 1) * sizeof(uint64_t)); /* per worker, at req_off */
  int64_t* inv = (int64_t*)malloc((T + 1) * sizeof(int64_t));
  uint64_t* nuniq = (uint64_t*)calloc(W, sizeof(uint64_t));
  /* send lists: send_ids[w][s] in emission order; stored per (w,s) */
  uint64_t* send_cnt = (uint64_t*)calloc(W * W, sizeof(uint64_t));
  uint64_t* owner = (uint64_t*)malloc((T + 1) * sizeof(uint64_t));
  uint64_t tr_req = 0, tr_recv = 0;
  if (ids_sent) memset(ids_sent, 0, W * W * sizeof(uint64_t));
  if (embs_sent) memset(embs_sent, 0, W * W * sizeof(uint64_t));
  if (lookups) memset(lookups, 0, W * sizeof(uint64_t));
  for (size_t w = 0; w < W; ++w) {
    const uint64_t* r = requests + req_off[w];
    tr_req += counts[w];
    if (s1) {
      nuniq[w] = or_stage1_dedup(r, counts[w], uniq + req_off[w], inv + req_off[w]);
    } else {
      memcpy(uniq + req_off[w], r, counts[w] * sizeof(uint64_t));
      for (uint64_t j = 0; j < counts[w]; ++j) inv[req_off[w] + j] = (int64_t)j;
      nuniq[w] = counts[w];
    }
    for (uint64_t u = 0; u < nuniq[w]; ++u) {
      uint64_t o = or_shard_of(uniq[req_off[w] + u], W);
      owner[req_off[w] + u] = o;
      send_cnt[w * W + o]++;
    }
    for (size_t s = 0; s < W; ++s) {
      if (ids_sent) ids_sent[w * W + s] += send_cnt[w * W + s];
      tr_recv += send_cnt[w * W + s];
    }
  }
  /* unique_rows[w] filled by the shard answers (scatter, :211-221) */
  float* urows = (float*)calloc((T + 1) * D, sizeof(float));
  uint8_t* filled = (uint8_t*)calloc(T + 1, 1);
  for (size_t s = 0; s < W; ++s) {
    or_table* shard = c->shards[s];
    /* received[w] = send_ids[w][s] in emission order; remember (w, u) */
    uint64_t nrecv = 0;
    for (size_t w = 0; w < W; ++w) nrecv += send_cnt[w * W + s];
    uint64_t* recv = (uint64_t*)malloc((nrecv + 1) * sizeof(uint64_t));
    uint64_t* recv_w = (uint64_t*)malloc((nrecv + 1) * sizeof(uint64_t));
    uint64_t* recv_u = (uint64_t*)malloc((nrecv + 1) * sizeof(uint64_t));
    uint64_t* rc = (uint64_t*)calloc(W, sizeof(uint64_t));
    uint64_t k = 0;
    for (size_t w = 0; w < W; ++w) {
      for (uint64_t u = 0; u < nuniq[w]; ++u) {
        if (owner[req_off[w] + u] != s) continue;
        recv[k] = uniq[req_off[w] + u];
        recv_w[k] = w;
        recv_u[k] = u;
        ++k;
      }
      rc[w] = send_cnt[w * W + s];
    }
    if (s2) {
      uint64_t* u2 = (uint64_t*)malloc((nrecv + 1) * sizeof(uint64_t));
      uint64_t* ooff = (uint64_t*)malloc((nrecv + 2) * sizeof(uint64_t));
      uint64_t* osrc = (uint64_t*)malloc((nrecv + 1) * sizeof(uint64_t));
      uint64_t* opos = (uint64_t*)malloc((nrecv + 1) * sizeof(uint64_t));
      size_t nu2 = or_stage2_dedup(recv, rc, W, u2, ooff, osrc, opos);
      if (lookups) lookups[s] += nu2;
      uint64_t* src_base = (uint64_t*)calloc(W + 1, sizeof(uint64_t));
      for (size_t w = 0; w < W; ++w) src_base[w + 1] = src_base[w] + rc[w];
      for (size_t u = 0; u < nu2; ++u) {
        int64_t row = or_table_ensure(shard, u2[u]);
        if (row < 0) return 2;
        const float* emb = or_table_emb(shard, row);
        for (uint64_t o = ooff[u]; o < ooff[u + 1]; ++o) {
          uint64_t j = src_base[osrc[o]] + opos[o];
          uint64_t w = recv_w[j], uu = recv_u[j];
          memcpy(urows + (req_off[w] + uu) * D, emb, D * sizeof(float));
          filled[req_off[w] + uu] = 1;
        }
      }
      free(src_base);
      free(u2);
      free(ooff);
      free(osrc);
      free(opos);
    } else {
      for (uint64_t j = 0; j < nrecv; ++j) {
        int64_t row = or_table_ensure(shard, recv[j]);
        if (row < 0) return 2;
        memcpy(urows + (req_off[recv_w[j]] + recv_u[j]) * D, or_table_emb(shard, row),
               D * sizeof(float));
        filled[req_off[recv_w[j]] + recv_u[j]] = 1;
        if (lookups) lookups[s]++;
      }
    }
    for (size_t w = 0; w < W; ++w)
      if (embs_sent) embs_sent[s * W + w] += rc[w];
    free(recv);
    free(recv_w);
    free(recv_u);
    free(rc);
  }
  int status = 0;
  for (size_t w = 0; w < W && status == 0; ++w) {
    for (uint64_t u = 0; u < nuniq[w]; ++u)
      if (!filled[req_off[w] + u]) status = 2; /* unanswered request id */
    for (uint64_t j = 0; j < counts[w] && status == 0; ++j) {
      memcpy(out + (req_off[w] + j) * D, urows + (req_off[w] + (uint64_t)inv[req_off[w] + j]) * D,
             D * sizeof(float));
    }
  }
  if (totals) {
    totals[0] = tr_req;
    totals[1] = tr_recv;
  }
  free(req_off);
  free(uniq);
  free(inv);
  free(nuniq);
  free(send_cnt);
  free(owner);
  free(urows);
  free(filled);
  return status;
}

/* ======================================================================== */
/* Gradient accumulation + optimizers (sparse_update.cpp)                   */
/* ======================================================================== */
typedef struct {
  uint64_t id;
  size_t idx;
} id_idx;
static int cmp_id_idx(const void* a, const void* b) {
  uint64_t x = ((const id_idx*)a)->id, y = ((const id_idx*)b)->id;
  return x < y ? -1 : x > y;
}

size_t or_accumulate(const uint64_t* ids, const float* grads, size_t n, uint32_t dim,
                     uint64_t* ids_out, float* sums_out) {
  /* GradAccumulator::accumulate, sparse_update.cpp:45-56: f32 sums in token
   * order; std::map iteration gives ascending id order. */
  u64map m;
  map_init(&m, n);
  float* sums = (float*)calloc((n + 1) * (size_t)dim, sizeof(float));
  id_idx* order = (id_idx*)malloc((n + 1) * sizeof(id_idx));
  size_t nu = 0;
  for (size_t i = 0; i < n; ++i) {
    int fresh = 0;
    size_t* u = map_try_emplace(&m, ids[i], nu, &fresh);
    if (fresh) {
      order[nu].id = ids[i];
      order[nu].idx = nu;
      ++nu;
    }
    float* acc = sums + *u * dim;
    const float* g = grads + i * dim;
    for (uint32_t e = 0; e < dim; ++e) acc[e] += g[e];
  }
  qsort(order, nu, sizeof(id_idx), cmp_id_idx);
  for (size_t k = 0; k < nu; ++k) {
    ids_out[k] = order[k].id;
    memcpy(sums_out + k * dim, sums + order[k].idx * dim, dim * sizeof(float));
  }
  free(order);
  free(sums);
  map_free(&m);
  return nu;
}

void or_adam_row(float* w, float* m, float* v, uint64_t* step, const float* grad, uint32_t dim,
                 double lr, double beta1, double beta2, double eps) {
  /* adam_update_row, sparse_update.cpp:22-37 (double math, f32 state) */
  *step += 1;
  const double bc1 = 1.0 - pow(beta1, (double)*step);
  const double bc2 = 1.0 - pow(beta2, (double)*step);
  for (uint32_t e = 0; e < dim; ++e) {
    const double g = grad[e];
    const double me = beta1 * m[e] + (1.0 - beta1) * g;
    const double ve = beta2 * v[e] + (1.0 - beta2) * g * g;
    m[e] = (float)me;
    v[e] = (float)ve;
    const double m_hat = me / bc1;
    const double v_hat = ve / bc2;
    w[e] = (float)(w[e] - lr * m_hat / (sqrt(v_hat) + eps));
  }
}

void or_adagrad_row(float* w, float* acc, uint64_t* step, const float* grad, uint32_t dim,
                    double lr, double eps) {
  /* UNPINNED (no reference Adagrad): frozen restatement in the discipline of
   * adam_update_row -- f32 state kept in the opt_v slot, double math,
   * step counter bumped.  acc' = acc + g*g ; w' = w - lr*g/(sqrt(acc')+eps). */
  *step += 1;
  for (uint32_t e = 0; e < dim; ++e) {
    const double g = grad[e];
    const double a = acc[e] + g * g;
    acc[e] = (float)a;
    w[e] = (float)(w[e] - lr * g / (sqrt(a) + eps));
  }
}

size_t or_apply(or_table* t, const uint64_t* ids, const float* sums, size_t n, int optimizer,
                double lr, double beta1, double beta2, double eps) {
  /* GradAccumulator::apply_serial, sparse_update.cpp:85-98 */
  for (size_t i = 0; i < n; ++i) {
    int64_t r = or_table_ensure(t, ids[i]);
    const float* g = sums + i * t->dim;
    if (optimizer == 0)
      or_adam_row(or_table_emb(t, r), or_table_m(t, r), or_table_v(t, r), or_table_step(t, r), g,
                  t->dim, lr, beta1, beta2, eps);
    else
      or_adagrad_row(or_table_emb(t, r), or_table_v(t, r), or_table_step(t, r), g, t->dim, lr,
                     eps);
  }
  return n;
}

/* ======================================================================== */
/* Table merging (merge_registry.cpp:23-33, plan_merge :107)                */
/* ======================================================================== */
int or_encode_tagged_id(uint32_t k_bits, uint32_t index, uint32_t index_limit, uint64_t raw,
                        uint64_t* out) {
  if (index > index_limit) return 1;
  const uint32_t shift = 63 - k_bits;
  if (raw >> shift != 0) return 2;
  *out = ((uint64_t)index << shift) | raw;
  return 0;
}

int or_decode_tagged_id(uint32_t k_bits, uint32_t index_limit, uint64_t tagged,
                        uint32_t* index, uint64_t* raw) {
  if (tagged >> 63 != 0) return 1;
  const uint32_t shift = 63 - k_bits;
  const uint32_t idx = (uint32_t)(tagged >> shift);
  if (idx > index_limit) return 2;
  *index = idx;
  *raw = tagged & (((uint64_t)1 << shift) - 1);
  return 0;
}

uint32_t or_bit_width(uint64_t x) {
  uint32_t b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

/* ======================================================================== */
/* Sequence batching (seq_batcher.cpp:22-78) + cost-model partition         */
/* ======================================================================== */
size_t or_closest_prefix(const uint64_t* cumsums, size_t n, uint64_t target) {
  size_t lo = 0, hi = n; /* std::lower_bound */
  while (lo < hi) {
    size_t mid = lo + (hi - lo) / 2;
    if (cumsums[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo == n) return n;
  if (lo == 0) return 1;
  const uint64_t above = cumsums[lo] - target;
  const uint64_t below = target - cumsums[lo - 1];
  if (below <= above) return lo;
  return lo + 1;
}

size_t or_sequence_batches(const uint64_t* lengths, size_t n, uint64_t target,
                           uint64_t chunk_samples, uint64_t* batch_sizes) {
  /* SequenceBatcher::next_batch over WorkerStream's chunk source
   * (workload.cpp:378-383): buffer = [head, tail) of the length list. */
  size_t head = 0, tail = 0, nb = 0;
  uint64_t buffered = 0;
  int exhausted = 0;
  uint64_t* cums = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  for (;;) {
    while (buffered < target && !exhausted) {
      if (tail >= n) {
        exhausted = 1;
        break;
      }
      size_t end = tail + chunk_samples < n ? tail + chunk_samples : n;
      for (; tail < end; ++tail) buffered += lengths[tail];
    }
    if (head == tail) break;
    uint64_t run = 0;
    for (size_t i = head; i < tail; ++i) {
      run += lengths[i];
      cums[i - head] = run;
    }
    size_t k = or_closest_prefix(cums, tail - head, target);
    for (size_t i = 0; i < k; ++i) buffered -= lengths[head + i];
    head += k;
    batch_sizes[nb++] = k;
  }
  free(cums);
  return nb;
}

typedef struct {
  double cost;
  size_t idx;
} cost_idx;
static int cmp_cost_desc(const void* a, const void* b) {
  const cost_idx* x = (const cost_idx*)a;
  const cost_idx* y = (const cost_idx*)b;
  if (x->cost != y->cost) return x->cost > y->cost ? -1 : 1;
  return x->idx < y->idx ? -1 : x->idx > y->idx;
}

void or_cost_partition(const uint64_t* lengths, size_t n, size_t world, double a, double b,
                       uint32_t* rank_out) {
  /* UNPINNED: the reference splits ranks round-robin (workload.cpp:461-469)
   * and uses a*len+b*len^2 (workload.hpp:106-109) only for simulated time.
   * Frozen restatement: longest-processing-time-first greedy. */
  cost_idx* c = (cost_idx*)malloc((n + 1) * sizeof(cost_idx));
  for (size_t i = 0; i < n; ++i) {
    const double len = (double)lengths[i];
    c[i].cost = a * len + b * len * len;
    c[i].idx = i;
  }
  qsort(c, n, sizeof(cost_idx), cmp_cost_desc);
  double* load = (double*)calloc(world, sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    size_t best = 0;
    for (size_t r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    load[best] += c[i].cost;
    rank_out[c[i].idx] = (uint32_t)best;
  }
  free(load);
  free(c);
}

/* ======================================================================== */
/* Workload generator (workload.hpp:36-49, workload.cpp:30-39,103-152,280-307,348-355) */
/* ======================================================================== */
#define MT_N 312
#define MT_M 156
void or_rng_seed(or_rng* r, uint64_t seed) { /* std::mt19937_64 seeding */
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
}

uint64_t or_rng_next(or_rng* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double rng_unit(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_unit_pos(or_rng* r) {
  return (double)((or_rng_next(r) >> 11) + 1) * 0x1.0p-53;
}

static double normal_cdf(double z) { return 0.5 * erfc(-z / sqrt(2.0)); }
static double trunc_lognormal_mean(double mu, double sigma, double upper) {
  const double log_u = log(upper);
  const double numer =
      exp(mu + sigma * sigma / 2.0) * normal_cdf((log_u - mu - sigma * sigma) / sigma);
  const double denom = normal_cdf((log_u - mu) / sigma);
  return numer / denom;
}

static double* zipf_cdf(uint64_t vocab, double exponent) {
  double* cdf = (double*)malloc(vocab * sizeof(double));
  double total = 0;
  for (uint64_t r = 0; r < vocab; ++r) {
    total += pow((double)(r + 1), -exponent);
    cdf[r] = total;
  }
  for (uint64_t r = 0; r < vocab; ++r) cdf[r] /= total;
  cdf[vocab - 1] = 1.0;
  return cdf;
}

static uint64_t zipf_sample(const double* cdf, uint64_t vocab, or_rng* rng) {
  const double u = rng_unit(rng);
  uint64_t lo = 0, hi = vocab; /* std::upper_bound */
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (u < cdf[mid])
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo < vocab - 1 ? lo : vocab - 1;
}

int64_t or_generate_workload(uint64_t seed, uint64_t num_sequences, double mean_len,
                             uint64_t max_len, double sigma, double zipf, uint32_t tables,
                             const uint64_t* vocab, uint64_t* lengths, uint64_t* ids,
                             uint64_t max_tokens) {
  if (!(sigma > 0) || max_len < 2 || !(mean_len > 1.0) || mean_len >= (double)max_len ||
      tables == 0 || zipf < 0)
    return -1;
  /* TruncatedLognormal ctor: bisection on mu (workload.cpp:103-121) */
  double lo = -20.0, hi = log((double)max_len) + 10.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (trunc_lognormal_mean(mid, sigma, (double)max_len) < mean_len)
      lo = mid;
    else
      hi = mid;
  }
  const double mu = 0.5 * (lo + hi);
  double** cdfs = (double**)malloc(tables * sizeof(double*));
  for (uint32_t t = 0; t < tables; ++t) cdfs[t] = zipf_cdf(vocab[t], zipf);
  uint32_t kb = or_bit_width(tables);
  if (kb < 1) kb = 1; /* catalog_from, workload.cpp:171-172 */
  or_rng rng;
  or_rng_seed(&rng, seed);
  uint64_t tok = 0;
  int64_t status = 0;
  for (uint64_t sid = 1; sid <= num_sequences; ++sid) {
    uint64_t len;
    for (;;) { /* TruncatedLognormal::sample, workload.cpp:123-133 */
      const double u1 = rng_unit_pos(&rng);
      const double u2 = rng_unit(&rng);
      const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
      const double x = exp(mu + sigma * z);
      if (x > (double)max_len) continue;
      uint64_t nn = (uint64_t)llround(x);
      if (nn > max_len) nn = max_len;
      len = nn < 1 ? 1 : nn;
      break;
    }
    (void)rng_unit(&rng); /* label, workload.cpp:297 */
    lengths[sid - 1] = len;
    for (uint64_t t = 0; t < len; ++t) {
      const uint32_t ordinal = (uint32_t)(1 + t % tables);
      const uint64_t raw = zipf_sample(cdfs[ordinal - 1], vocab[ordinal - 1], &rng);
      uint64_t id = 0;
      or_encode_tagged_id(kb, ordinal, tables, raw, &id);
      if (tok >= max_tokens) {
        status = -1;
        goto done;
      }
      ids[tok++] = id;
    }
  }
done:
  for (uint32_t t = 0; t < tables; ++t) free(cdfs[t]);
  free(cdfs);
  return status < 0 ? -1 : (int64_t)tok;
}

void or_pseudo_sparse_grad(uint64_t sample_id, uint64_t step, float* out, uint32_t dim) {
  /* workload.cpp:348-355 */
  const uint64_t base =
      or_hash64(sample_id * 0x9e3779b97f4a7c15ULL + step * 0xbf58476d1ce4e5b9ULL + 1);
  for (uint32_t e = 0; e < dim; ++e) {
    const double u = (double)(or_hash64(base + e) >> 11) * 0x1.0p-53;
    out[e] = (float)((u - 0.5) * 0.1);
  }
}
