/*
 * rsgpu.h -- C-ABI of the B200-native (sm_100a) sparse-embedding hot path.
 *
 * Drop-in boundary for the reference's table/lookup API
 * (/root/reference/proj/include/recsparse/ *.hpp).  Plain pointers and sizes,
 * no C++ or torch types.  Every entry point names the reference interface it
 * replaces.  Pointers prefixed d_ are device pointers; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  All calls are asynchronous on
 * `stream` unless documented as synchronizing.
 *
 * Errors: no exceptions cross the ABI.  Status codes map 1:1 onto the
 * reference's exception taxonomy (common.hpp:24-39):
 *   RS_OK 0, RS_ERR_CONFIG 1 (ConfigError / std::invalid_argument on shapes),
 *   RS_ERR_INVARIANT 2 (InvariantError), RS_ERR_IO 3 (IoError),
 *   RS_ERR_CUDA 4 (CUDA/NCCL failure), RS_ERR_CAPACITY 5 (bounded table
 *   cannot hold the batch), RS_ERR_RANGE 6 (std::out_of_range /
 *   std::overflow_error of the id encoding).  rs_last_error() returns the
 *   message of the last failure on the calling thread.
 *
 * Threading (embed_table.hpp:69-72): one writer per table per stream;
 * concurrent read-only calls (rs_table_find, rs_table_gather_rows) are safe.
 */
#ifndef RSGPU_H
#define RSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

enum {
  RS_OK = 0,
  RS_ERR_CONFIG = 1,
  RS_ERR_INVARIANT = 2,
  RS_ERR_IO = 3,
  RS_ERR_CUDA = 4,
  RS_ERR_CAPACITY = 5,
  RS_ERR_RANGE = 6
};

enum { RS_OPT_NONE = 0, RS_OPT_ADAM = 1, RS_OPT_ADAGRAD = 2 };

typedef struct rs_table rs_table;         /* one dynamic hash embedding table (one shard) */
typedef struct rs_workspace rs_workspace; /* per-stream scratch for dedup/reduce/step */

/* TableConfig (embed_table.hpp:28-36) plus the GPU build's extensions. */
typedef struct {
  uint64_t capacity;       /* initial key slots; power of two >= 16 */
  uint32_t embedding_dim;  /* floats per row, >= 1 */
  uint32_t thread_groups;  /* power of two, capacity >= 2*groups (validated like the
                              reference; the GPU probes 8-slot buckets with 8 lanes) */
  double max_load_factor;  /* (occupied + tombstones)/capacity ceiling, in (0,1) */
  uint32_t chunk_rows;     /* row-pool growth granularity, >= 1 */
  uint32_t optimizer;      /* RS_OPT_*: which state arrays rows carry */
  uint64_t initial_rows;   /* row-pool pre-allocation (0: capacity*max_load_factor) */
  uint64_t max_keys;       /* 0: unbounded (expand); >0: bounded, evict oldest (ts, key) */
} rs_table_config;

/* AdamParams (sparse_update.hpp:26-31); Adagrad uses lr and eps. */
typedef struct {
  uint32_t kind; /* RS_OPT_ADAM or RS_OPT_ADAGRAD */
  double lr, beta1, beta2, eps;
} rs_optimizer_params;

typedef struct {
  uint64_t capacity, occupied, tombstones;
  uint64_t rows_allocated, rows_free, row_capacity;
  uint64_t tick;
  uint32_t embedding_dim, optimizer;
  uint64_t host_syncs; /* stream synchronizations the capacity bookkeeping needed so far */
} rs_table_info;

/* ---- meta ---------------------------------------------------------------- */
int rs_abi_version(void);
const char* rs_status_string(int status);
const char* rs_last_error(void);
/* number of rsgpu kernel launches issued so far by this process (evidence) */
uint64_t rs_kernel_launches(void);
/* Device buffers and synchronous copies for C / C++ callers without a CUDA
 * runtime of their own (the C++ shim include/recsparse_gpu uses them). */
int rs_buffer_alloc(uint64_t bytes, void** out);
int rs_buffer_free(void* d);
int rs_copy_to_device(void* d, const void* h, uint64_t bytes);
int rs_copy_to_host(void* h, const void* d, uint64_t bytes);

/* ---- primitives (hash.hpp) --------------------------------------------- */
/* hash64_batch (hash.hpp:38, hash.cpp:21-30) */
int rs_hash64_batch(const uint64_t* d_keys, uint64_t n, uint64_t* d_out, void* stream);
/* SimCluster::shard_of (exchange_sim.cpp:82-85) */
int rs_shard_of_batch(const uint64_t* d_ids, uint64_t n, uint32_t world, uint32_t* d_owner,
                      void* stream);

/* ---- dynamic table (EmbedTable, embed_table.hpp:73-211) ------------------- */
/* EmbedTable(TableConfig) (embed_table.cpp:40-45); validation :23-38 */
int rs_table_create(const rs_table_config* cfg, rs_table** out);
int rs_table_destroy(rs_table* t);
/* capacity()/occupied()/tombstones()/tick() (embed_table.hpp:112-118). Synchronizes. */
int rs_table_stats(rs_table* t, rs_table_info* out);
/* insert (embed_table.cpp:193-227), batched upsert; duplicate keys: last wins.
 * d_emb [n x dim]. New keys get fresh zeroed optimizer state. */
int rs_table_insert(rs_table* t, const uint64_t* d_keys, uint64_t n, const float* d_emb,
                    void* stream);
/* find (embed_table.cpp:237-241): d_rows[n] = row id or -1; no side effects. */
int rs_table_find(rs_table* t, const uint64_t* d_keys, uint64_t n, int64_t* d_rows, void* stream);
/* lookup_batch (embed_table.cpp:287-315): d_out [n x dim], zeros on miss,
 * every hit stamped with one tick for the whole batch. */
int rs_table_lookup(rs_table* t, const uint64_t* d_keys, uint64_t n, float* d_out, void* stream);
/* ensure (embed_table.cpp:243-248), batched find-or-insert-zero-row; d_rows
 * optional.  Bounded tables evict the oldest (ts, key) first. */
int rs_table_ensure(rs_table* t, const uint64_t* d_keys, uint64_t n, int64_t* d_rows,
                    void* stream);
/* remove (embed_table.cpp:250-260); d_removed[n] (optional) = 1 if removed. */
int rs_table_remove(rs_table* t, const uint64_t* d_keys, uint64_t n, uint8_t* d_removed,
                    void* stream);
/* expand (embed_table.cpp:262-285): doubles the key structure at least once;
 * rows never move.  Synchronizes; *new_capacity optional. */
int rs_table_expand(rs_table* t, uint64_t* new_capacity, void* stream);
/* eviction (no reference counterpart): remove the k live entries
 * with smallest (ts, key).  Synchronizes; *evicted optional. */
int rs_table_evict(rs_table* t, uint64_t k, uint64_t* evicted, void* stream);
/* Gather rows by row id (row handles from find/ensure): d_out [n x dim]. */
int rs_table_gather_rows(rs_table* t, const int64_t* d_rows, uint64_t n, float* d_out,
                         void* stream);
/* Host export of live entries (for_each_occupied, embed_table.hpp:142-147),
 * sorted by key.  Any output may be NULL; *count = occupied.  Call with
 * max_entries = 0 to query the count.  Synchronizes. */
int rs_table_export(rs_table* t, uint64_t max_entries, uint64_t* keys, float* emb, float* m,
                    float* v, uint64_t* step, uint64_t* ts, uint64_t* count);
/* bump_tick (embed_table.hpp:159-161): fast-forward the batch tick. */
int rs_table_bump_tick(rs_table* t, uint64_t to);
/* Deep copy (EmbedTable's copy constructor, embed_table.cpp:47-97): same
 * slots, row ids, state, counters and tick.  Synchronizes. */
int rs_table_clone(rs_table* src, rs_table** out);
/* Row state of host keys (the row accessors embedding(h) / opt_m / opt_v /
 * opt_step / row_timestamp of embed_table.hpp:123-132, batched, no side
 * effects): rows[n] = row id or -1; emb/m/v [n x dim], step[n], ts[n] (the
 * key's batch tick); zeros for absent keys.  Any output may be NULL.
 * Synchronizes. */
int rs_table_read_entries(rs_table* t, const uint64_t* keys, uint64_t n, int64_t* rows, float* emb,
                          float* m, float* v, uint64_t* step, uint64_t* ts);
/* Host import of full entries (restore path, checkpoint.cpp:238-249: keys are
 * re-inserted, slots are not portable).  m/v/step/ts may be NULL. */
int rs_table_import(rs_table* t, uint64_t n, const uint64_t* keys, const float* emb,
                    const float* m, const float* v, const uint64_t* step, const uint64_t* ts);

/* ---- dedup (exchange_sim.cpp:87-115) -------------------------------------- */
int rs_workspace_create(uint64_t max_tokens, rs_workspace** out);
int rs_workspace_destroy(rs_workspace* ws);
/* stage1_dedup: first-occurrence unique ids + int32 inverse; *d_n_unique is a
 * device uint32.  Stage 2 is the same call over the source-ordered
 * concatenation of received lists (its inverse gives every origin). */
int rs_dedup(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, uint64_t* d_unique,
             int32_t* d_inverse, uint32_t* d_n_unique, void* stream);

/* ---- the fused training step (workload.cpp:506-581 for one shard) --------
 * forward : dedup -> find-or-insert (zero-vivify) -> jagged gather
 *           d_out[n x dim] (bit-exact with distributed_lookup's outputs)
 * backward: segment-reduce d_grads[n x dim] onto unique rows fused with the
 *           optimizer update (Adam sparse_update.cpp:22-37 / Adagrad) */
int rs_forward(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n, float* d_out,
               void* stream);
int rs_backward(rs_workspace* ws, rs_table* t, const float* d_grads, uint64_t n,
                const rs_optimizer_params* opt, void* stream);
int rs_step(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
            const float* d_grads, float* d_out, const rs_optimizer_params* opt, void* stream);
/* rs_step plus run_workload's per-step emb_checksum (workload.cpp:547-549):
 * *d_checksum (device f64) = the sum of every value written to d_out, computed
 * inside the gather kernel (fixed reduction tree: deterministic). */
int rs_step_checksum(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, float* d_out, const rs_optimizer_params* opt,
                     double* d_checksum, void* stream);
/* GradAccumulator::accumulate + apply for one window (sparse_update.cpp:45-83):
 * dedup ids, zero-vivify absent ids, segment-reduce grads fused with the
 * optimizer.  No gather. */
int rs_sparse_update(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, const rs_optimizer_params* opt, void* stream);
/* Unique ids of the last forward / sparse update / dedup on this workspace,
 * in the order of its internal unique index (the index of rs_accumulate's
 * rows).  The fused step numbers ids in an unspecified order; rs_dedup's is
 * first-occurrence.  d_out may be NULL to query *n_out.  Synchronizes. */
int rs_workspace_unique(rs_workspace* ws, uint64_t* d_out, uint64_t cap, uint64_t* n_out);
/* Results of the last forward on this workspace (device pointers owned by ws). */
int rs_workspace_results(rs_workspace* ws, const uint64_t** d_unique, const int32_t** d_inverse,
                         const uint32_t** d_n_unique, const int64_t** d_rows);
/* Per-kernel CUDA-event timing of rs_step (diagnostic; disables graph
 * capture).  Phases: 0 dedup, 1 table find-or-insert, 2 gather, 3 tile
 * reduce, 4 finish + optimizer.  rs_workspace_phase_ms returns the mean ms. */
int rs_workspace_set_profiling(rs_workspace* ws, int on);
/* Device-side timeline of the fast step (diagnostics; enabled when RS_TRACE=1
 * at the workspace's first rs_step): out[(kernel * 4096 + block) * 2 + {0,1}]
 * = first warp start / last warp end (%globaltimer ns) of each block of the
 * steps since the last call; kernels 0 dedup+probe, 1 CSR finish, 2 hot
 * tiles, 3 hot finish, 4 scratch clean, 5 heavy CSR ids; the sharded step
 * (rs_comm_timeline) adds 6 requester gather, 7 gradient flags, 8 wait ids,
 * 9 owner dedup, 10 owner table + respond, 11 wait rows, 12 wait gradients,
 * 13 owner update done.  16 kernel slots; *n_out = 0 when tracing is off. */
int rs_workspace_trace(rs_workspace* ws, uint64_t* out, uint64_t cap, uint64_t* n_out);
int rs_workspace_phase_ms(rs_workspace* ws, double* ms, uint32_t nphases, uint64_t* count);
/* n_unique of the last dedup on this workspace (host value).  Synchronizes. */
int rs_workspace_n_unique(rs_workspace* ws, uint64_t* out);
/* GradAccumulator::accumulate for one micro-batch (sparse_update.cpp:45-56):
 * aggregated grads per unique id of the last forward, first-occurrence order,
 * d_sums [n_unique x dim]. */
int rs_accumulate(rs_workspace* ws, const float* d_grads, uint64_t n, float* d_sums,
                  void* stream);
/* GradAccumulator::apply given aggregated grads (sparse_update.cpp:58-83):
 * ensure + one optimizer step per key, keys unique. */
int rs_apply_aggregated(rs_table* t, const uint64_t* d_keys, uint64_t n, const float* d_sums,
                        const rs_optimizer_params* opt, void* stream);

/* ---- row-sharded step over the W GPUs of one node (exchange_sim.cpp:117-233) --
 * One process per GPU.  Each rank owns the keys with hash64(key) % W == rank
 * (SimCluster::shard_of, exchange_sim.cpp:82-85) in its own rs_table shard.
 * The ID, embedding and gradient exchanges are peer stores over NVLink into a
 * symmetric arena each rank exports by CUDA IPC (rs_comm_ipc_handle /
 * rs_comm_open: the caller exchanges the 64-byte handles, e.g. with
 * torch.distributed.all_gather_object).  Every rank must call each step. */
typedef struct rs_comm rs_comm;
int rs_comm_create(int rank, int world, uint64_t max_tokens, uint32_t dim, rs_comm** out);
int rs_comm_ipc_handle(rs_comm* c, void* handle_out /* 64 bytes */);
int rs_comm_open(rs_comm* c, const void* handles /* world x 64 bytes, rank order */);
int rs_comm_destroy(rs_comm* c);
/* distributed_lookup with DedupMode::kTwoStage for this rank's tokens:
 * d_out [n x dim] bit-exact with the reference's outputs[rank]. */
int rs_dist_forward(rs_comm* c, rs_table* shard, const uint64_t* d_ids, uint64_t n, float* d_out,
                    void* stream);
/* per-token grads -> pre-reduced unique rows to the owners -> ordered
 * stage-2 sum (source, position) -> optimizer on the owners' shards. */
int rs_dist_backward(rs_comm* c, rs_table* shard, const float* d_grads, uint64_t n,
                     const rs_optimizer_params* opt, void* stream);
/* forward + backward in one call (same results), ordered so that no rank
 * idles on a flag in steady state: reduce while the peers' ids are in
 * flight, answer + update as owner, gather last.  d_out gets the rows as they
 * were before this step's update (distributed_lookup semantics). */
int rs_dist_step(rs_comm* c, rs_table* shard, const uint64_t* d_ids, uint64_t n,
                 const float* d_grads, float* d_out, const rs_optimizer_params* opt, void* stream);
/* rs_dist_step plus this rank's emb_checksum (the f64 sum of every value
 * written to d_out, computed inside the gather kernel) into *d_checksum. */
int rs_dist_step_checksum(rs_comm* c, rs_table* shard, const uint64_t* d_ids, uint64_t n,
                          const float* d_grads, float* d_out, const rs_optimizer_params* opt,
                          double* d_checksum, void* stream);
/* This rank's ExchangeTrace row (exchange_sim.hpp:37-59) for the last step:
 * ids_sent[W] (to each owner), embs_sent[W] (vectors this owner sent back to
 * each requester), lookups, ids_requested, ids_received.  Synchronizes. */
/* Per-phase device time of the sharded step (CUDA events on the step's
 * stream; synchronizes at the end of each step while on, no graphs): phases
 * req_dedup, send_ids, wait_ids, owner_dedup, owner_table_respond,
 * wait_embs, gather (rs_dist_step: gather + reduce + sums to the owners),
 * req_reduce (split API only), wait_grads, owner_update -- mean ms. */
int rs_comm_set_profiling(rs_comm* c, int on);
/* device-side barrier of the group on `stream` (all ranks call it): work
 * enqueued after it starts once every rank reached it */
int rs_comm_barrier(rs_comm* c, void* stream);
int rs_comm_phase_ms(rs_comm* c, double* ms, int n, uint64_t* count);
/* rs_workspace_trace of the sharded step's requester workspace (RS_TRACE=1). */
int rs_comm_timeline(rs_comm* c, uint64_t* out, uint64_t cap, uint64_t* n_out);
int rs_comm_trace(rs_comm* c, uint64_t* ids_sent, uint64_t* embs_sent, uint64_t* lookups,
                  uint64_t* ids_requested, uint64_t* ids_received);
/* A group of `world` logical ranks on the current GPU (one process): the
 * SimCluster of the reference (exchange_sim.hpp:63-75 -- W shards in one
 * process, exchange_sim.cpp:117-233) on the sharded step's own kernels, arena
 * layout and flag protocol, with each other's arenas as plain device
 * pointers.  comms_out[world] in rank order; destroy each with
 * rs_comm_destroy.  Drive it only with rs_dist_group_*, which enqueue every
 * phase rank by rank on one stream in data-flow order (no kernel waits on a
 * kernel that has not run). */
int rs_comm_create_local(int world, uint64_t max_tokens, uint32_t dim, rs_comm** comms_out);
/* rs_dist_forward / rs_dist_backward / rs_dist_step for all ranks of a local
 * group: arrays of `world` per-rank arguments (shards[r] owns the keys with
 * hash64 % world == r). */
int rs_dist_group_forward(rs_comm* const* comms, rs_table* const* shards, int world,
                          const uint64_t* const* d_ids, const uint64_t* n, float* const* d_out,
                          void* stream);
int rs_dist_group_backward(rs_comm* const* comms, rs_table* const* shards, int world,
                           const float* const* d_grads, const uint64_t* n,
                           const rs_optimizer_params* opt, void* stream);
int rs_dist_group_step(rs_comm* const* comms, rs_table* const* shards, int world,
                       const uint64_t* const* d_ids, const uint64_t* n, const float* const* d_grads,
                       float* const* d_out, const rs_optimizer_params* opt, void* stream);

/* ---- table merging (merge_registry.cpp:23-175) ---------------------------- */
/* encode_tagged_id on device (merge_registry.cpp:23-33); synchronizes,
 * RS_ERR_RANGE if an index or raw id is out of range. */
int rs_encode_ids(const uint64_t* d_raw, uint64_t n, uint32_t k_bits, uint32_t table_index,
                  uint32_t index_limit, uint64_t* d_out, void* stream);

/* Pooling / FeatureConfig (merge_registry.hpp:28-43) */
enum { RS_POOL_NONE = 0, RS_POOL_SUM = 1, RS_POOL_MEAN = 2 };
typedef struct {
  const char* feature_name;
  uint32_t embedding_dim;
  const char* const* lookup_tables;
  uint32_t n_lookup_tables;
  uint32_t pooling; /* RS_POOL_* */
} rs_feature_config;

/* plan_merge (merge_registry.cpp:69-110): same groups, member order, k bits
 * and ConfigError cases (RS_ERR_CONFIG, reference message text). */
typedef struct rs_merge_plan rs_merge_plan;
int rs_plan_merge(const rs_feature_config* configs, uint32_t n, rs_merge_plan** out);
int rs_merge_plan_destroy(rs_merge_plan* plan);
uint32_t rs_merge_plan_groups(const rs_merge_plan* plan);
int rs_merge_plan_group(const rs_merge_plan* plan, uint32_t group, uint32_t* embedding_dim,
                        uint32_t* k_bits, uint32_t* n_members);
/* member table i in [1, m] of a group (MergeGroup::member_tables[i - 1]); NULL if none */
const char* rs_merge_plan_member(const rs_merge_plan* plan, uint32_t group, uint32_t index);
/* MergePlan::group_index_for + MergeGroup::table_index_of (unknown table: RS_ERR_CONFIG) */
int rs_merge_plan_find(const rs_merge_plan* plan, const char* table, uint32_t* group,
                       uint32_t* index);

/* HashTableCollection (merge_registry.hpp:90-105): one device table per
 * group, the prototype config with the group's embedding dim. */
typedef struct rs_collection rs_collection;
int rs_collection_create(const rs_merge_plan* plan, const rs_table_config* prototype,
                         rs_collection** out);
int rs_collection_destroy(rs_collection* c);
rs_table* rs_collection_table(rs_collection* c, uint32_t group);
/* collection_lookup (merge_registry.cpp:112-158): per raw id, every lookup
 * table's row (zero-vivified), pooled none / sum (table order) / mean
 * (sum * (1.0f / n)); d_out [n x embedding_dim].  Synchronizes: RS_ERR_RANGE
 * if a raw id exceeds its group's payload width (no table touched then). */
int rs_collection_lookup(rs_collection* c, const rs_feature_config* feature,
                         const uint64_t* d_raw_ids, uint64_t n, float* d_out, void* stream);

/* run_workload's per-token routing (workload.cpp:431-447, 506-531): decode
 * the catalog tag (TableCatalog, ordinals 1..n_catalog in catalog order) and
 * re-encode into the merged group's id space.  rs_route_tagged is a stable
 * partition by group: d_gids / d_pos hold group 0's tokens in token order,
 * then group 1's, ...; h_counts[groups] (optional) synchronizes and reports
 * decode / encode range errors (RS_ERR_RANGE). */
typedef struct rs_router rs_router;
int rs_router_create(const rs_merge_plan* plan, const char* const* catalog_names,
                     uint32_t n_catalog, rs_router** out);
int rs_router_destroy(rs_router* r);
int rs_route_tagged(rs_router* r, const uint64_t* d_tagged, uint64_t n, uint64_t* d_gids,
                    uint32_t* d_pos, uint64_t* h_counts, void* stream);

/* ---- dynamic sequence balancing (seq_batcher.cpp, workload.cpp:368-469) --- */
/* closest_prefix (seq_batcher.cpp:22-34); n == 0: RS_ERR_CONFIG */
int rs_closest_prefix(const uint64_t* cumsums, uint64_t n, uint64_t target, uint64_t* k_out);
/* ChunkSource: fill up to cap (sample id, token count) pairs, *n_out of them;
 * return 0 once exhausted (SequenceBatcher's std::function<bool(chunk&)>). */
typedef int (*rs_chunk_source)(void* ctx, uint64_t* sample_ids, uint64_t* token_counts,
                               uint64_t cap, uint64_t* n_out);
typedef struct rs_seq_batcher rs_seq_batcher;
/* SequenceBatcher (seq_batcher.cpp:36-78, Alg. 1); target < 1: RS_ERR_CONFIG */
int rs_seq_batcher_create(uint64_t target_tokens, rs_chunk_source source, void* ctx,
                          uint64_t max_chunk, rs_seq_batcher** out);
int rs_seq_batcher_destroy(rs_seq_batcher* b);
/* next_batch: *n_out samples in arrival order, 0 when done; a zero-token
 * sample: RS_ERR_INVARIANT */
int rs_seq_batcher_next(rs_seq_batcher* b, uint64_t* sample_ids, uint64_t* token_counts,
                        uint64_t cap, uint64_t* n_out);
uint64_t rs_seq_batcher_buffered_tokens(const rs_seq_batcher* b);
uint64_t rs_seq_batcher_buffered_samples(const rs_seq_batcher* b);
/* rank per sequence: round robin (the reference's split, workload.cpp:461-469)
 * or longest-processing-time-first on CostModel::sample_compute a*len+b*len^2
 * (workload.hpp:106-109); load_out[world] (optional) the cost per rank */
enum { RS_PARTITION_ROUND_ROBIN = 0, RS_PARTITION_COST_LPT = 1 };
int rs_partition_sequences(const uint64_t* lengths, uint64_t n, uint32_t world, uint32_t policy,
                           double a, double b, uint32_t* rank_out, double* load_out);
/* imbalance_report (seq_batcher.cpp:140-152) */
int rs_imbalance_report(const uint64_t* per_worker_tokens, uint64_t n, uint64_t* max_tokens,
                        uint64_t* min_tokens, double* spread);
/* weighted_grad_combine (seq_batcher.cpp:80-138); grads [workers x dim] */
int rs_weighted_grad_combine(const uint64_t* batch_sizes, const double* grads, uint64_t workers,
                             uint64_t dim, double* out);

/* ---- one run_workload step fed from host memory (workload.cpp:506-581) ----
 * Pinned host ids + sequence lengths go to the device on a copy stream (two
 * buffer sets, the copies of step k+1 overlap step k); the gradients are
 * pseudo_sparse_grad on the device; the step runs; its embedding checksum
 * (run_workload's emb_checksum) is copied to *h_checksum.  Nothing syncs. */
typedef struct rs_feeder rs_feeder;
int rs_feeder_create(uint64_t max_tokens, uint64_t max_seqs, uint32_t dim, rs_feeder** out);
int rs_feeder_destroy(rs_feeder* f);
float* rs_feeder_out(rs_feeder* f, int which);
int rs_feeder_step(rs_feeder* f, rs_workspace* ws, rs_table* t, const uint64_t* h_ids, uint64_t n,
                   const uint64_t* h_lengths, uint64_t n_seq, uint64_t first_sample_id,
                   uint64_t step, const rs_optimizer_params* opt, double* h_checksum,
                   void* stream);
int rs_feeder_dist_step(rs_feeder* f, rs_comm* c, rs_table* shard, const uint64_t* h_ids,
                        uint64_t n, const uint64_t* h_lengths, uint64_t n_seq,
                        uint64_t first_sample_id, uint64_t step, const rs_optimizer_params* opt,
                        double* h_checksum, void* stream);

/* ---- elastic checkpoint (checkpoint.hpp:25-54, checkpoint.cpp) ----------------
 * The reference's little-endian shard file; records in key order with slot =
 * ordinal (device slots are not the reference's probe positions), so files
 * are byte-deterministic and save -> load -> save is byte-identical.  Loads
 * follow load_cluster: modulo file selection + ownership refilter when the
 * world size changes; tick fast-forwarded to the newest stamp.  All sync. */
typedef struct {
  uint32_t version, world_size, shard_rank, embedding_dim;
  uint64_t capacity, entry_count;
} rs_ckpt_header;
int rs_ckpt_shard_file_name(uint32_t rank, uint32_t world_size, char* out, uint64_t cap);
int rs_ckpt_save_shard(rs_table* t, uint32_t rank, uint32_t world_size, const char* path);
int rs_ckpt_read_header(const char* path, rs_ckpt_header* out);
int rs_ckpt_load_shard(rs_table* t, const char* dir, uint32_t saved_world, uint32_t new_world,
                       uint32_t rank);

/* ---- synthetic inputs (workload.cpp:103-152, 280-307, 348-355) ------------ */
/* generate_workload: per-sample lengths + catalog-tagged ids (k = bit_width(tables)) */
int rs_workload_generate(uint64_t seed, uint64_t num_sequences, double mean_len, uint64_t max_len,
                         double sigma, double zipf, uint32_t tables, const uint64_t* vocab,
                         uint64_t* lengths, uint64_t* ids, uint64_t max_tokens,
                         uint64_t* n_tokens);
/* generate_workload_file (workload.cpp:280-315): the same workload written in
 * the reference's text format (header line, then "sid<TAB>label<TAB>ids"). */
int rs_workload_write(const char* path, uint64_t seed, uint64_t num_sequences, double mean_len,
                      uint64_t max_len, double sigma, double zipf, uint32_t tables, const uint64_t* vocab);
/* read_workload_file (workload.cpp:317-339): host arrays sample_ids/labels/
 * lengths [cap_seq], ids [cap_tok] (any may be NULL); zero capacities return
 * the counts only.  RS_ERR_IO on open failure, "bad record", "empty sequence". */
int rs_workload_read(const char* path, uint64_t cap_seq, uint64_t cap_tok, uint64_t* sample_ids,
                     double* labels, uint64_t* lengths, uint64_t* ids, uint64_t* n_seq, uint64_t* n_tok);
/* pseudo_sparse_grad per token on device: d_out[t] = g(sample_of_token[t], step) */
int rs_pseudo_grads(const uint64_t* d_sample_of_token, uint64_t n, uint64_t step, uint32_t dim,
                    float* d_out, void* stream);
/* the same gradients for a jagged batch given by its sequence lengths (sample
 * ids first_sample_id + s, the generator's numbering): one row per sample,
 * broadcast to the sample's tokens; dim % 4 == 0 */
int rs_pseudo_grads_jagged(const uint64_t* d_lengths, uint64_t n_seq, uint64_t first_sample_id,
                           uint64_t step, uint32_t dim, uint64_t n_tokens, float* d_out,
                           void* stream);
/* the same from the token offsets of the batch (d_offsets[n_seq + 1], device):
 * one kernel, block per sample */
int rs_pseudo_grads_offsets(const uint64_t* d_offsets, uint64_t n_seq, uint64_t first_sample_id,
                            uint64_t step, uint32_t dim, float* d_out, void* stream);
/* the same from a work list of (sample, token begin, token end) u32 triples
 * (device), one balanced block per triple */
int rs_pseudo_grads_chunks(const void* d_work, uint32_t n_chunks, uint64_t first_sample_id,
                           uint64_t step, uint32_t dim, float* d_out, void* stream);
/* run_workload's emb_checksum (workload.cpp:547-549): sum of d_x[0, n) in f64,
 * fixed order (deterministic), into *d_out */
int rs_checksum(const float* d_x, uint64_t n, double* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RSGPU_H */
