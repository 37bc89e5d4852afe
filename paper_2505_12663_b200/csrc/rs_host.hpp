// rs_host.hpp -- host-side objects behind the opaque C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <vector>

#include "rs_internal.cuh"

// Counter snapshot copied device->host asynchronously after every mutating
// batch op, double-buffered so the host can bound occupancy without a sync
// (DESIGN.md §4 "sync-free capacity management").
struct rs_mirror {
  rs::TableCounters* pinned = nullptr;
  rs::TableCounters* dev_ptr = nullptr;  // the same pinned buffer as seen by kernels (mapped)
  cudaEvent_t ev = nullptr;
  uint64_t requested_at_copy = 0;  // cumulative keys requested when the copy was enqueued
  bool valid = false;
};

struct rs_table {
  uint64_t host_syncs = 0;  // read_counters calls (stream syncs)
  rs_table_config cfg{};
  rs::TableDev* dev = nullptr;   // device descriptor + counters
  rs::TableDesc desc{};          // host copy of the pointer section
  uint64_t capacity = 0;         // key slots
  // sync-free capacity bookkeeping
  rs_mirror mirror[2];
  int mirror_next = 0;
  uint64_t requested_total = 0;  // Σ n over all insert/ensure batches
  uint64_t exact_occ = 0, exact_tomb = 0, exact_rows = 0, exact_requested = 0;
  uint64_t ahead_n = 0;  // largest batch the headroom was sized for (table_prepare)
  // Adam bias-correction tables 1 - beta^step computed with the host libm
  // (bit-identical to sparse_update.cpp:25-26 on this host)
  double* d_bc = nullptr;        // [2 x bc_len]
  uint64_t bc_len = 0;
  double bc_beta1 = -1, bc_beta2 = -1;
  uint64_t applies = 0;          // optimizer applications (upper bound of any row step)
  uint64_t host_tick = 0;        // batch ops issued (device tick follows it)
  // bounded tables: probe-miss list + eviction key buffer
  uint32_t* d_missing = nullptr;
  uint64_t missing_cap = 0;
  uint64_t* d_victims = nullptr;
  uint64_t victims_cap = 0;
  // device victim selection (evict.cu)
  void* d_evict = nullptr;          // EvictState
  uint32_t* d_cand = nullptr;       // 2 x candidate lists
  uint32_t* d_victim_idx = nullptr;
  uint64_t evict_cap = 0, victim_idx_cap = 0;
  uint64_t buf_gen = 0;  // bumps when a buffer baked into captured graphs is reallocated
  bool evict_tmin_valid = false;  // the device selection may start its tick window at its last min
  // bounded tables: the stamp log (evict.cu; rs_internal.cuh LogRec)
  rs::LogRec* d_log = nullptr;
  rs::LogCtl* d_log_ctl = nullptr;
  uint64_t log_cap = 0;           // records (power of two)
  bool log_valid = false;         // the log lists every live entry (else: rebuilt before the next ensure)
  uint64_t log_tail_ub = 0;       // host upper bound of the device tail
  uint64_t log_head_lb = 0;       // host lower bound of the device head (last read)
  uint32_t* d_lg_cnt = nullptr;   // per window block: live records
  long long* d_lg_pre = nullptr;
  uint64_t lg_nb = 0;             // window blocks allocated
  uint64_t log_rebuilds = 0;
};

struct rs_graph_entry {
  // everything a captured step bakes in
  rs_table* t = nullptr;
  const void* ids = nullptr;
  const void* grads = nullptr;
  void* out = nullptr;
  double* csum = nullptr;
  uint64_t n = 0;
  int mirror = 0;
  int set = 0;
  const void* pbuf = nullptr;
  uint64_t tcap = 0, tgen = 0;  // table capacity / buffer generation baked into the graph
  unsigned char opt[128] = {0};
  cudaGraphExec_t exec = nullptr;
  uint64_t last_use = 0;
  uint64_t launches = 0;  // rsgpu kernels inside the graph
  bool fast = false;      // the step_fast.cu graph
};

// One dedup scratch hash set (SoA, S+1 slots; slot S holds the id equal to
// the empty sentinel).  Two sets alternate between calls: each call uses the
// clean set and cleans the other one (the previous call's) in its kernels,
// from the dirty list u_slot[0, cnt).
struct rs_scratch {
  unsigned long long* skey = nullptr;
  uint32_t* sfirstx = nullptr;  // ~first position (exact dedup)
  uint32_t* sntile = nullptr;   // tiles containing the id
  uint32_t* suidx = nullptr;    // unique index of the slot
  uint32_t* srow = nullptr;     // table row of the slot
  uint32_t* u_slot = nullptr;   // slot of each unique id (dirty list)
  uint32_t* cnt = nullptr;      // device [0] = unique ids in the set
};

// Scratch of the single-GPU fast step (step_fast.cu), allocated on the first
// rs_step: two alternating sets of 16-byte records {key, count, row} (each
// step cleans the other set from its dirty list), plus per-slot unique /
// hot indices, token positions (64 per slot) and the hot-id partial lists.
struct rs_fast_set {
  void* rec = nullptr;           // [S + 1] records
  uint32_t* u_slot = nullptr;    // slot of each unique id (dirty list)
  uint32_t* cnt = nullptr;       // device [0] unique ids
};
struct rs_fast {
  bool ready = false;
  rs_fast_set set[2];
  int cur = 0;                   // set the next fast step uses
  int last = 0;                  // set of the last fast step
  uint32_t* uidx = nullptr;      // [S + 1]
  uint32_t* hidx = nullptr;      // [S + 1] hot index (~0 between steps)
  uint32_t* pos = nullptr;       // [(S + 1) x 64] token positions
  uint32_t* hot_slot = nullptr;  // [max_hot]
  uint32_t* hlist = nullptr;     // [max_hot x ntiles]
  uint32_t* ctr = nullptr;       // [0] hot ids [1] partials [2] error bits
  double* tokcs = nullptr;       // [max_tokens] per-token row sums (rs_step_checksum)
  unsigned long long* trace = nullptr;  // RS_TRACE=1: per (kernel, block) start / end timeline
  uint64_t ntiles = 0, max_hot = 0;
  uint32_t hot_min = 64;         // ids with more occurrences take the hot path (RS_HOT_MIN)
  uint32_t light_max = 8;        // CSR ids with more occurrences: the heavy CSR kernel (RS_LIGHT_MAX)
  uint32_t* heavy = nullptr;     // [max_tokens] slots of the heavy CSR ids
  cudaStream_t aux2 = nullptr, aux3 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_j1 = nullptr, ev_j2 = nullptr, ev_j3 = nullptr;
};

struct rs_workspace {
  rs_fast fast;
  bool use_fast = true;     // rs_step on unbounded tables: step_fast.cu (RS_FAST_STEP=0: the split kernels)
  bool last_fast = false;   // the last op was a fast step (its unique count lives in fast.set[fast.last])
  bool last_exact = false;  // the last op was rs_dedup (first-occurrence numbering)
  // KC split (RS_SPLIT_KC=0: one pass): the hot-id pass is launched by the finish
  bool split_kc = true;
  bool kc_forked = false;  // the hot tile pass was launched on aux_stream (launch_finish joins)
  // programmatic dependent launch on the step's same-stream kernel edges (RS_PDL=0: off)
  bool pdl = true;
  bool pdl_now = false;
  // rs_step_checksum: f64 sum of the gathered rows, fused into the gather
  double* csum_dst = nullptr;
  uint32_t* tok_rank = nullptr;  // per token: rank among its id's occurrences (KA -> KC)
  bool tok_rank_ok = false;      // the last KA of this workspace produced tok_rank
  double* csum_part = nullptr;         // per-tile partials
  unsigned int* csum_ticket = nullptr;  // tiles done (the last one sums, then zeroes it)  // set while step_enqueue issues the unbounded fast step
  bool graph_fork = true;  // hot-id finish as a forked branch inside captured graphs (RS_GRAPH_FORK=0: linear)
  uint64_t max_tokens = 0;
  uint64_t S = 0;  // scratch hash capacity (power of two)
  rs_scratch set[2];
  int cur = 0;       // clean set the next call uses
  int last_set = 0;  // set used by the last call (its results)
  cudaStream_t cap_stream = nullptr;  // capture stream for the step graphs
  cudaStream_t aux_stream = nullptr;  // forked branch of the step (reserved)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<rs_graph_entry> graphs;
  std::vector<uint64_t> seen;  // bounded tables: step signatures run once eagerly (capture on the second)
  uint64_t graph_clock = 0;
  bool use_graphs = true;
  bool fork = true;  // run the hot-id finish concurrently on aux_stream
  // optional per-kernel CUDA-event timing (forces the non-graph path)
  bool profiling = false;
  cudaEvent_t prof_ev[8] = {nullptr};
  double prof_ms[8] = {0};
  uint64_t prof_count = 0;
  // per token
  uint32_t* slot_of = nullptr;
  int32_t* inverse = nullptr;
  // per unique
  uint64_t* unique = nullptr;
  uint32_t* u_ntile = nullptr;
  uint32_t* u_poff = nullptr;
  uint32_t* u_ticket = nullptr;
  uint32_t* urow = nullptr;
  int64_t* urow64 = nullptr;
  // cross-tile partial sums
  uint32_t* ptile = nullptr;
  uint32_t* porder = nullptr;
  uint32_t* hot_list = nullptr;  // ids with > kWarpMaxParts partials (KB)
  uint32_t* u_cnt = nullptr;     // occurrences per unique id
  uint32_t* csr_pos = nullptr;   // token positions grouped by id (CSR path)
  float* pbuf = nullptr;         // [pbuf_floats partials | pbuf_floats usum]
  uint64_t pbuf_floats = 0;
  // scans
  uint64_t* scan_status = nullptr;
  uint32_t* ctr = nullptr;  // [0] tile ticket [1] blocks done [4] n_hot [5] partial alloc
  // last forward
  uint64_t last_n = 0;
  uint32_t last_tile = 0;
  rs_table* last_table = nullptr;
  bool have_forward = false;
};

// Cross-GPU synchronisation folded into the step kernels (sharded step):
// a prologue wait on flags in this rank's arena, and a grid-level arrival
// whose last block raises flags at the peers (dist_sync.cuh).
struct rs_dist_sync {
  const unsigned long long* wait_flags = nullptr;  // [wait_n] flags to wait for (null: none)
  uint32_t wait_n = 0;
  const unsigned long long* epoch = nullptr;       // device step epoch
  unsigned long long* const* sig_flags = nullptr;  // [sig_n] peer flag words to raise (null: none)
  uint32_t sig_n = 0;
  unsigned int* sig_done = nullptr;                // arrival counter of the signalling kernels
  uint32_t sig_total = 0;                          // blocks arriving (set by the launcher)
  unsigned long long* error = nullptr;             // set on a wait timeout
  unsigned long long* tl = nullptr;                // device timeline (RS_TRACE=1): the owner update's slot
};

// The requester's id send folded into the table-metadata kernel (KB): the
// owner partition of the unique ids, stored straight into the owners'
// receive lists, then counts + flags raised by the last block (dist.cu).
struct rs_dist_send {
  char* const* peers = nullptr;                  // [W] arena bases (null: no send)
  size_t off_ids = 0;                            // receive lists in the arena
  uint32_t cap = 0, world = 1, rank = 0;
  uint32_t* send_cnt = nullptr;                  // [W] cursors (zero between steps)
  uint32_t* send_pos = nullptr;                  // per unique id: owner * cap + j
  uint32_t* const* cnt_ptrs = nullptr;           // [W] &peer(r)->cnt_in[rank]
  unsigned long long* const* flag_ptrs = nullptr;  // [W] &peer(r)->sig_ids[rank]
  unsigned long long* epoch = nullptr;           // requester step counter (bumped here)
  unsigned int* done = nullptr;                  // last-block counter
  unsigned long long* trace_ids_sent = nullptr;  // [W]
  unsigned long long* trace_requested = nullptr;
  uint64_t n_tokens = 0;
};

// Options of the fused kernels used by the sharded (multi-GPU) step (dist.cu).
struct rs_dist_opts {
  rs_dist_sync sync;                    // waits / signals folded into the kernels
  const uint32_t* d_n = nullptr;        // device token count (owner side); null: host n
  const uint32_t* pos_map = nullptr;    // CSR position of each token (owner: origin slot)
  bool no_stage = false;                // no hot ids possible: no gradient staging
  bool no_hot = false;                  // finish: skip the hot-id kernel (none possible)
  const uint32_t* csr_pos = nullptr;    // finish: CSR position array (null: the workspace's)
  const void* gather_view = nullptr;    // rs::TableDev* whose emb = requester receive buffer
  float* const* peer_dst = nullptr;     // device [W] peer gradient receive bases
  const uint32_t* send_pos = nullptr;   // per unique id: owner * cap + position
  uint32_t cap = 0, rank = 0;
  double* csum = nullptr;               // gather: f64 sum of the gathered rows (host token count only)
};

namespace rs {

// CUDA graphs run their kernel nodes at the priority of the stream each was
// captured on (the owner / gather streams of the sharded step), not the
// launch stream's; RS_GRAPH_PRIO=0 turns that off (experiments).
inline unsigned long long graph_flags() {
  static const bool off = getenv("RS_GRAPH_PRIO") && getenv("RS_GRAPH_PRIO")[0] == '0';
  return off ? 0ull : (unsigned long long)cudaGraphInstantiateFlagUseNodePriority;
}
// table.cu
int table_prepare(rs_table* t, uint64_t n, cudaStream_t s, int headroom = 0);  // room for n more keys
                                                                               // (+ headroom batches' worth, steps)
int table_after_op(rs_table* t, cudaStream_t s);             // enqueue counter mirror
int table_ensure_device(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                        uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                        uint32_t* d_srow, cudaStream_t s);
// evict.cu: device victim selection + removal (bounded ensure after the
// probe: explicit_k == 0; explicit evict: explicit_k = k)
int log_prepare(rs_table* t, uint64_t n_max, cudaStream_t s);  // bounded ensure: log room / rebuild
rs::LogArgs log_args(rs_table* t, int probe);                     // (null rec: no log)
void log_invalidate(rs_table* t);                                 // rebuilt before the next bounded ensure
int evict_device(rs_table* t, const uint32_t* d_n, uint64_t n_host, uint64_t explicit_k,
                 cudaStream_t s);
int evict_count(rs_table* t, uint64_t* out, cudaStream_t s);
int evict_prepare(rs_table* t, uint64_t max_victims);  // host: size the selection buffers
// bounded ensure split for graph capture: host part, then enqueue-only part
int table_bounded_prepare(rs_table* t, uint64_t n_max, cudaStream_t s);
int table_bounded_evict_insert(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                               uint32_t* d_rows32, int64_t* d_rows64, cudaStream_t s);
int table_bounded_enqueue(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                          uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                          uint32_t* d_srow, cudaStream_t s);  // victims of the last selection (syncs)
int table_ensure_any(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                     uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                     uint32_t* d_srow, cudaStream_t s);
int table_upsert_enqueue(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                         uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                         uint32_t* d_srow, cudaStream_t s);
int table_mirror_copy(rs_table* t, int which, cudaStream_t s);
int table_mirror_commit(rs_table* t, int which, cudaStream_t s);
int table_adam_tables(rs_table* t, double beta1, double beta2, uint64_t applies, cudaStream_t s);
// step.cu
uint32_t tile_tokens_for_dim(uint32_t dim);
int step_set_smem_attrs();
int step_fdedup(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, int use, cudaStream_t s,
                const uint32_t* d_n);
int step_ftable(rs_workspace* ws, rs_table* t, int use, uint64_t n_max, bool do_table,
                bool do_clean, cudaStream_t s, const rs_dist_send* send = nullptr);
int step_tile(rs_workspace* ws, rs_table* t, int use, uint64_t n, float* d_out,
              const float* d_grads, bool clean_other, cudaStream_t s, const rs_dist_opts* dopt);
int step_finish(rs_workspace* ws, rs_table* t, int use, uint64_t n, const float* d_grads,
                const void* opt_args, float* sums_out, cudaStream_t s, const rs_dist_opts* dopt);
int step_opt_args(rs_table* t, const rs_optimizer_params* p, void* out, cudaStream_t s);
int step_reduce_prepare(rs_workspace* ws, uint32_t D, uint64_t n, cudaStream_t s);
// step_fast.cu
bool fast_step_supported(const rs_table* t);
bool fast_dim_supported(uint32_t dim);
int fast_prepare(rs_workspace* ws);
int fast_check_errors(rs_workspace* ws, cudaStream_t s);
// the sharded requester on the fast kernels (step_fast.cu, used by dist.cu)
int fast_dist_front(rs_workspace* ws, uint32_t D, const uint64_t* d_ids, uint64_t n, int use, cudaStream_t s,
                    const rs_dist_send& send);
int fast_dist_reduce(rs_workspace* ws, rs::TableDev* view, uint32_t D, uint64_t n, const float* d_grads, int use,
                     cudaStream_t s, bool fork, float* const* peer_dst, uint32_t cap, uint32_t rank);
int fast_dist_gather(rs_workspace* ws, const rs::TableDev* view, uint32_t D, uint64_t n, float* d_out, int use,
                     cudaStream_t s, const rs_dist_sync& sync, double* csum, uint32_t grid);
void fast_free(rs_workspace* ws);
int fast_enqueue(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n, const float* d_grads,
                 float* d_out, const void* opt_args, int use, cudaStream_t s, cudaEvent_t* ev, bool fork,
                 rs::TableCounters* mirror_out);
}  // namespace rs
