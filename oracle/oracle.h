/*
 * oracle.h -- CPU restatement of the recsparse sparse-embedding hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (librsgpu.so,
 * paper_2505_12663_b200/) may include, link or call this code.  It is used
 * by tests/ (as the parity checker), by __graft_entry__.smoke() and by the
 * cpu_baseline leg of bench.py.
 *
 * Every function restates the algorithm of the reference implementation at
 * /root/reference/proj (cited file:line, paths relative to proj/).  Parity of
 * this restatement is pinned two ways (see tests/test_oracle_*.py):
 *   1. against the known-answer vectors of the reference's own unit tests
 *      (tests/golden/kat.json, transcribed with file:line citations), and
 *   2. against the reference itself, compiled from its sources by
 *      oracle/Makefile into oracle/_ref/librsref.so, on seeded random inputs.
 * Functions with no reference counterpart (Adagrad, eviction, the cost-model
 * sequence partition, the gradient all-to-all counts) are frozen
 * restatements of the semantics written down in DESIGN.md ("unpinned").
 */
#ifndef RS_ORACLE_H
#define RS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- L0 primitives (hash.hpp) ------------------------------------------ */
uint64_t or_hash64(uint64_t key);
/* returns 0 and *step on success, 1 on ConfigError (capacity/groups < 2) */
int or_probe_step(uint64_t key, uint64_t capacity, uint64_t groups, uint64_t* step);
void or_hash64_batch(const uint64_t* keys, size_t n, uint64_t* out);

/* ---- L1 table (embed_table.hpp/.cpp) ------------------------------------ */
typedef struct or_table or_table;
/* status: 0 ok, 1 config error */
int or_table_create(uint64_t capacity, uint32_t dim, uint32_t groups, double max_load_factor,
                    uint32_t chunk_rows, or_table** out);
void or_table_destroy(or_table* t);
uint64_t or_table_capacity(const or_table* t);
uint64_t or_table_occupied(const or_table* t);
uint64_t or_table_tombstones(const or_table* t);
uint64_t or_table_tick(const or_table* t);
/* upsert; returns flat row id (chunk*chunk_rows+row) or -1 on invariant error */
int64_t or_table_insert(or_table* t, uint64_t key, const float* emb);
int64_t or_table_lookup(or_table* t, uint64_t key); /* stamps; -1 when absent */
int64_t or_table_find(const or_table* t, uint64_t key); /* no side effects */
int64_t or_table_ensure(or_table* t, uint64_t key);
int or_table_remove(or_table* t, uint64_t key); /* 1 removed, 0 absent */
uint64_t or_table_expand(or_table* t);
void or_table_lookup_batch(or_table* t, const uint64_t* keys, size_t n, float* out);
float* or_table_emb(or_table* t, int64_t row);
float* or_table_m(or_table* t, int64_t row);
float* or_table_v(or_table* t, int64_t row);
uint64_t* or_table_ts(or_table* t, int64_t row);
uint64_t* or_table_step(or_table* t, int64_t row);
/* Export live entries sorted by key: keys[occ], emb/m/v[occ*dim], step[occ], ts[occ].
 * Any pointer may be NULL.  Returns the number of entries. */
size_t or_table_export(const or_table* t, uint64_t* keys, float* emb, float* m, float* v,
                       uint64_t* step, uint64_t* ts);

/* ---- batch-tick table semantics of the GPU build ----------
 * One logical tick per batch op: every key a batch touches is stamped with
 * that tick.  ensure_batch: stamps present keys, then (if max_keys > 0 and
 * the missing keys would exceed it) evicts the smallest (ts, key) among keys
 * not touched by this batch, then inserts the missing keys as zero rows in
 * the order given.  Returns the number of evictions, or -1 if the batch
 * cannot fit.  rows_out (optional) receives the flat row per key. */
int64_t or_table_ensure_batch(or_table* t, const uint64_t* keys, size_t n, uint64_t tick,
                              uint64_t max_keys, int64_t* rows_out);
/* Evict the k entries with smallest (ts, key).  Returns number evicted. */
size_t or_table_evict_oldest(or_table* t, size_t k);

/* ---- dedup (exchange_sim.cpp:87-115) ------------------------------------ */
/* returns n_unique; unique[n] (capacity n), inverse[n] */
size_t or_stage1_dedup(const uint64_t* ids, size_t n, uint64_t* unique, int64_t* inverse);
/* received = concatenation of W lists with counts[W]; returns n_unique;
 * origin_off[n_unique+1] CSR offsets, origin_src/pos[n] in (source, position) order */
size_t or_stage2_dedup(const uint64_t* received, const uint64_t* counts, size_t world,
                       uint64_t* unique, uint64_t* origin_off, uint64_t* origin_src,
                       uint64_t* origin_pos);
uint64_t or_shard_of(uint64_t id, uint64_t world);

/* ---- sharded lookup (exchange_sim.cpp:117-233) --------------------------- */
typedef struct or_cluster or_cluster;
int or_cluster_create(size_t world, uint64_t capacity, uint32_t dim, uint32_t groups,
                      double max_load_factor, uint32_t chunk_rows, int dedup_mode,
                      or_cluster** out);
void or_cluster_destroy(or_cluster* c);
or_table* or_cluster_shard(or_cluster* c, size_t s);
/* requests: concatenation of W lists, counts[W]; out: concatenation of
 * outputs [Σcounts x dim]; trace arrays (may be NULL): ids_sent[W*W],
 * embs_sent[W*W] (row-major [src][dst]), lookups[W], totals[2] =
 * {ids_requested, ids_received}.  Returns 0, or 2 on invariant error. */
int or_distributed_lookup(or_cluster* c, const uint64_t* requests, const uint64_t* counts,
                          float* out, uint64_t* ids_sent, uint64_t* embs_sent,
                          uint64_t* lookups, uint64_t* totals);

/* ---- gradient accumulation + optimizers (sparse_update.cpp) -------------- */
/* Sums grads per id in token order (f32), output ascending by id.
 * returns number of distinct ids. */
size_t or_accumulate(const uint64_t* ids, const float* grads, size_t n, uint32_t dim,
                     uint64_t* ids_out, float* sums_out);
void or_adam_row(float* w, float* m, float* v, uint64_t* step, const float* g, uint32_t dim,
                 double lr, double beta1, double beta2, double eps);
void or_adagrad_row(float* w, float* acc, uint64_t* step, const float* g, uint32_t dim,
                    double lr, double eps);
/* apply: ascending ids (as produced by or_accumulate), ensure + row update.
 * optimizer 0 = Adam(lr,b1,b2,eps), 1 = Adagrad(lr, eps). */
size_t or_apply(or_table* t, const uint64_t* ids, const float* sums, size_t n, int optimizer,
                double lr, double beta1, double beta2, double eps);

/* ---- table merging (merge_registry.cpp) ---------------------------------- */
/* 0 ok; 1 index out of range; 2 raw id overflow */
int or_encode_tagged_id(uint32_t k_bits, uint32_t index, uint32_t index_limit, uint64_t raw,
                        uint64_t* out);
/* 0 ok; 1 top bit; 2 index out of range */
int or_decode_tagged_id(uint32_t k_bits, uint32_t index_limit, uint64_t tagged,
                        uint32_t* index, uint64_t* raw);
uint32_t or_bit_width(uint64_t x);

/* ---- sequence batching (seq_batcher.cpp) --------------------------------- */
size_t or_closest_prefix(const uint64_t* cumsums, size_t n, uint64_t target);
/* Alg. 1 over a stream of lengths arriving in chunks of chunk_samples:
 * writes batch sizes (#samples per batch) into batch_sizes, returns #batches */
size_t or_sequence_batches(const uint64_t* lengths, size_t n, uint64_t target,
                           uint64_t chunk_samples, uint64_t* batch_sizes);
/* Cost-model cross-rank partition (unpinned): LPT greedy on
 * cost a*len + b*len^2 (ties: smaller index first; least-loaded rank, ties
 * to the lower rank).  rank_out[n]. */
void or_cost_partition(const uint64_t* lengths, size_t n, size_t world, double a, double b,
                       uint32_t* rank_out);

/* ---- workload generator (workload.hpp/.cpp) ------------------------------ */
typedef struct or_rng { uint64_t mt[312]; int mti; } or_rng;
void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
/* Generates num_sequences samples exactly as generate_workload
 * (workload.cpp:280-307) with `tables` logical tables of vocabularies
 * vocab[tables] and catalog k_bits.  lengths[num_sequences];
 * ids[Σlengths] (capacity max_tokens).  Returns total tokens or -1 if
 * max_tokens too small / bad config. */
int64_t or_generate_workload(uint64_t seed, uint64_t num_sequences, double mean_len,
                             uint64_t max_len, double sigma, double zipf, uint32_t tables,
                             const uint64_t* vocab, uint64_t* lengths, uint64_t* ids,
                             uint64_t max_tokens);
void or_pseudo_sparse_grad(uint64_t sample_id, uint64_t step, float* out, uint32_t dim);

#ifdef __cplusplus
}
#endif
#endif
