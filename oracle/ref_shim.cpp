// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED reference library
// (TEST INFRASTRUCTURE).  oracle/Makefile compiles /root/reference/proj/src/*.cpp
// in place together with this file into oracle/_ref/librsref.so.  Nothing of
// the reference is copied into this repository; this file only calls its
// public API (proj/include/recsparse/*.hpp).  Used by tests (to pin the C
// restatement in oracle.c and as the reference of GPU parity tests) and by
// bench.py's reference arm (CPU baseline, kind "reference").
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "recsparse/checkpoint.hpp"
#include "recsparse/common.hpp"
#include "recsparse/embed_table.hpp"
#include "recsparse/exchange_sim.hpp"
#include "recsparse/hash.hpp"
#include "recsparse/merge_registry.hpp"
#include "recsparse/seq_batcher.hpp"
#include "recsparse/sparse_update.hpp"
#include "recsparse/workload.hpp"

using namespace recsparse;

namespace {
int status_of(const std::exception& e) {
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const InvariantError*>(&e)) return 2;
  if (dynamic_cast<const IoError*>(&e)) return 3;
  return 1;
}
#define GUARD(body)                  \
  try {                              \
    body;                            \
  } catch (const std::exception& e) { \
    return status_of(e);             \
  }
int64_t flat(const EmbedTable& t, RowHandle h) {
  return static_cast<int64_t>(h.chunk) * t.config().chunk_rows + h.row;
}
RowHandle unflat(const EmbedTable& t, int64_t r) {
  return RowHandle{static_cast<uint32_t>(r / t.config().chunk_rows),
                   static_cast<uint32_t>(r % t.config().chunk_rows)};
}
}  // namespace

extern "C" {

uint64_t ref_hash64(uint64_t k) { return hash64(k); }
int ref_probe_step(uint64_t key, uint64_t cap, uint64_t groups, uint64_t* out) {
  GUARD(*out = probe_step(key, cap, groups));
  return 0;
}

// ---- EmbedTable ---------------------------------------------------------
int ref_table_create(uint64_t capacity, uint32_t dim, uint32_t groups, double lf,
                     uint32_t chunk_rows, void** out) {
  GUARD({
    TableConfig c;
    c.capacity = capacity;
    c.embedding_dim = dim;
    c.thread_groups = groups;
    c.max_load_factor = lf;
    c.chunk_rows = chunk_rows;
    *out = new EmbedTable(c);
  });
  return 0;
}
void ref_table_destroy(void* t) { delete static_cast<EmbedTable*>(t); }
void* ref_table_copy(void* t) { return new EmbedTable(*static_cast<EmbedTable*>(t)); }
uint64_t ref_table_capacity(void* t) { return static_cast<EmbedTable*>(t)->capacity(); }
uint64_t ref_table_occupied(void* t) { return static_cast<EmbedTable*>(t)->occupied(); }
uint64_t ref_table_tombstones(void* t) { return static_cast<EmbedTable*>(t)->tombstones(); }
uint64_t ref_table_tick(void* t) { return static_cast<EmbedTable*>(t)->tick(); }
int64_t ref_table_insert(void* tp, uint64_t key, const float* emb) {
  auto* t = static_cast<EmbedTable*>(tp);
  try {
    return flat(*t, t->insert(key, std::span<const float>(emb, t->embedding_dim())));
  } catch (const std::exception&) {
    return -2;
  }
}
int64_t ref_table_lookup(void* tp, uint64_t key) {
  auto* t = static_cast<EmbedTable*>(tp);
  auto h = t->lookup(key);
  return h ? flat(*t, *h) : -1;
}
int64_t ref_table_find(void* tp, uint64_t key) {
  auto* t = static_cast<EmbedTable*>(tp);
  auto h = t->find(key);
  return h ? flat(*t, *h) : -1;
}
int64_t ref_table_ensure(void* tp, uint64_t key) {
  auto* t = static_cast<EmbedTable*>(tp);
  try {
    return flat(*t, t->ensure(key));
  } catch (const std::exception&) {
    return -2;
  }
}
int ref_table_remove(void* tp, uint64_t key) { return static_cast<EmbedTable*>(tp)->remove(key); }
uint64_t ref_table_expand(void* tp) { return static_cast<EmbedTable*>(tp)->expand(); }
void ref_table_lookup_batch(void* tp, const uint64_t* keys, uint64_t n, float* out, int serial) {
  auto* t = static_cast<EmbedTable*>(tp);
  std::span<const uint64_t> k(keys, n);
  std::span<float> o(out, n * t->embedding_dim());
  if (serial)
    t->lookup_batch_serial(k, o);
  else
    t->lookup_batch(k, o);
}
// Row access by flat id: which = 0 emb, 1 m, 2 v
void ref_table_row(void* tp, int64_t r, int which, float* out) {
  auto* t = static_cast<EmbedTable*>(tp);
  RowHandle h = unflat(*t, r);
  std::span<const float> s = which == 0 ? t->embedding(h) : which == 1 ? t->opt_m(h) : t->opt_v(h);
  std::memcpy(out, s.data(), s.size() * sizeof(float));
}
void ref_table_row_aux(void* tp, int64_t r, uint64_t* step, uint64_t* ts) {
  auto* t = static_cast<EmbedTable*>(tp);
  RowHandle h = unflat(*t, r);
  *step = t->opt_step(h);
  *ts = t->row_timestamp(h);
}
// Live entries in slot order: keys, emb, m, v, step, ts (any may be NULL)
uint64_t ref_table_export_slots(void* tp, uint64_t* keys, float* emb, float* m, float* v,
                                uint64_t* step, uint64_t* ts) {
  auto* t = static_cast<EmbedTable*>(tp);
  const size_t d = t->embedding_dim();
  uint64_t i = 0;
  t->for_each_occupied([&](uint64_t, uint64_t key, RowHandle h) {
    if (keys) keys[i] = key;
    if (emb) std::memcpy(emb + i * d, t->embedding(h).data(), d * 4);
    if (m) std::memcpy(m + i * d, t->opt_m(h).data(), d * 4);
    if (v) std::memcpy(v + i * d, t->opt_v(h).data(), d * 4);
    if (step) step[i] = t->opt_step(h);
    if (ts) ts[i] = t->row_timestamp(h);
    ++i;
  });
  return i;
}

// ---- dedup / exchange ---------------------------------------------------
uint64_t ref_stage1_dedup(const uint64_t* ids, uint64_t n, uint64_t* unique, int64_t* inverse) {
  Stage1Result r = stage1_dedup(std::span<const uint64_t>(ids, n));
  std::memcpy(unique, r.unique_ids.data(), r.unique_ids.size() * 8);
  for (uint64_t j = 0; j < n; ++j) inverse[j] = static_cast<int64_t>(r.inverse_index[j]);
  return r.unique_ids.size();
}
uint64_t ref_stage2_dedup(const uint64_t* received, const uint64_t* counts, uint64_t world,
                          uint64_t* unique, uint64_t* origin_off, uint64_t* origin_src,
                          uint64_t* origin_pos) {
  std::vector<std::vector<uint64_t>> lists(world);
  uint64_t j = 0;
  for (uint64_t s = 0; s < world; ++s)
    for (uint64_t p = 0; p < counts[s]; ++p) lists[s].push_back(received[j++]);
  Stage2Result r = stage2_dedup(lists);
  uint64_t o = 0;
  for (size_t u = 0; u < r.unique_ids.size(); ++u) {
    unique[u] = r.unique_ids[u];
    origin_off[u] = o;
    for (const auto& org : r.origins[u]) {
      origin_src[o] = org.source;
      origin_pos[o] = org.position;
      ++o;
    }
  }
  origin_off[r.unique_ids.size()] = o;
  return r.unique_ids.size();
}
uint64_t ref_shard_of(uint64_t id, uint64_t world) { return SimCluster::shard_of(id, world); }

int ref_cluster_create(uint64_t world, uint64_t capacity, uint32_t dim, uint32_t groups,
                       double lf, uint32_t chunk_rows, int mode, void** out) {
  GUARD({
    TableConfig c;
    c.capacity = capacity;
    c.embedding_dim = dim;
    c.thread_groups = groups;
    c.max_load_factor = lf;
    c.chunk_rows = chunk_rows;
    *out = new SimCluster(world, c, static_cast<DedupMode>(mode));
  });
  return 0;
}
void ref_cluster_destroy(void* c) { delete static_cast<SimCluster*>(c); }
void* ref_cluster_shard(void* c, uint64_t s) { return &static_cast<SimCluster*>(c)->shards[s]; }
int ref_distributed_lookup(void* cp, const uint64_t* requests, const uint64_t* counts, float* out,
                           uint64_t* ids_sent, uint64_t* embs_sent, uint64_t* lookups,
                           uint64_t* totals) {
  auto* c = static_cast<SimCluster*>(cp);
  const size_t W = c->world_size;
  std::vector<std::vector<uint64_t>> req(W);
  uint64_t j = 0;
  for (size_t w = 0; w < W; ++w)
    for (uint64_t p = 0; p < counts[w]; ++p) req[w].push_back(requests[j++]);
  GUARD({
    LookupResult r = distributed_lookup(*c, req);
    uint64_t o = 0;
    for (size_t w = 0; w < W; ++w) {
      std::memcpy(out + o, r.outputs[w].data(), r.outputs[w].size() * 4);
      o += r.outputs[w].size();
    }
    for (size_t s = 0; s < W; ++s)
      for (size_t d = 0; d < W; ++d) {
        if (ids_sent) ids_sent[s * W + d] = r.trace.ids_sent[s][d];
        if (embs_sent) embs_sent[s * W + d] = r.trace.embs_sent[s][d];
      }
    if (lookups)
      for (size_t s = 0; s < W; ++s) lookups[s] = r.trace.lookups[s];
    if (totals) {
      totals[0] = r.trace.ids_requested;
      totals[1] = r.trace.ids_received;
    }
  });
  return 0;
}

// ---- optimizer ----------------------------------------------------------
uint64_t ref_accumulate(const uint64_t* ids, const float* grads, uint64_t n, uint32_t dim,
                        uint64_t* ids_out, float* sums_out) {
  GradAccumulator acc(dim, 1);
  acc.accumulate(std::span<const uint64_t>(ids, n), std::span<const float>(grads, n * dim));
  uint64_t i = 0;
  for (const auto& [id, g] : acc.pending()) {
    ids_out[i] = id;
    std::memcpy(sums_out + i * dim, g.data(), dim * 4);
    ++i;
  }
  return i;
}
// accumulate + apply (Adam) through GradAccumulator; serial=1 uses apply_serial
uint64_t ref_accumulate_apply_adam(void* tp, const uint64_t* ids, const float* grads, uint64_t n,
                                   double lr, double b1, double b2, double eps, int serial) {
  auto* t = static_cast<EmbedTable*>(tp);
  GradAccumulator acc(t->embedding_dim(), 1);
  acc.accumulate(std::span<const uint64_t>(ids, n),
                 std::span<const float>(grads, n * t->embedding_dim()));
  AdamParams p{lr, b1, b2, eps};
  return serial ? acc.apply_serial(*t, p) : acc.apply(*t, p);
}
void ref_adam_row(float* w, float* m, float* v, uint64_t* step, const float* g, uint32_t dim,
                  double lr, double b1, double b2, double eps) {
  AdamParams p{lr, b1, b2, eps};
  adam_update_row(std::span<float>(w, dim), std::span<float>(m, dim), std::span<float>(v, dim),
                  *step, std::span<const float>(g, dim), p);
}

// ---- merge / batching ---------------------------------------------------
int ref_encode_tagged_id(uint32_t k, uint32_t idx, uint32_t lim, uint64_t raw, uint64_t* out) {
  try {
    *out = encode_tagged_id(k, idx, lim, raw);
  } catch (const std::out_of_range&) {
    return 1;
  } catch (const std::overflow_error&) {
    return 2;
  }
  return 0;
}
int ref_decode_tagged_id(uint32_t k, uint32_t lim, uint64_t tagged, uint32_t* idx,
                         uint64_t* raw) {
  try {
    auto [i, x] = decode_tagged_id(k, lim, tagged);
    *idx = i;
    *raw = x;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::out_of_range&) {
    return 2;
  }
  return 0;
}
// Feature specs cross the C boundary as text:
//   "name|dim|pooling|table1,table2;name2|..."   pooling 0 none, 1 sum, 2 mean
static std::vector<FeatureConfig> parse_features(const char* spec) {
  std::vector<FeatureConfig> out;
  std::stringstream all(spec);
  std::string item;
  while (std::getline(all, item, ';')) {
    if (item.empty()) continue;
    std::stringstream f(item);
    std::string name, dim, pool, tables;
    std::getline(f, name, '|');
    std::getline(f, dim, '|');
    std::getline(f, pool, '|');
    std::getline(f, tables, '|');
    FeatureConfig c;
    c.feature_name = name;
    c.embedding_dim = static_cast<uint32_t>(std::stoul(dim));
    const int p = std::stoi(pool);
    c.pooling = p == 0 ? Pooling::kNone : (p == 1 ? Pooling::kSum : Pooling::kMean);
    std::stringstream t(tables);
    std::string tab;
    while (std::getline(t, tab, ',')) c.lookup_tables.push_back(tab);
    out.push_back(std::move(c));
  }
  return out;
}

// plan -> "dim:k:member1,member2|dim:k:..." (group order, member order)
int ref_plan_merge(const char* spec, char* out, uint64_t cap) {
  GUARD({
    const std::vector<FeatureConfig> f = parse_features(spec);
    const MergePlan plan = plan_merge(f);
    std::string s;
    for (size_t g = 0; g < plan.groups.size(); ++g) {
      if (g) s += "|";
      s += std::to_string(plan.groups[g].embedding_dim) + ":" +
           std::to_string(plan.groups[g].k_bits) + ":";
      for (size_t i = 0; i < plan.groups[g].member_tables.size(); ++i)
        s += (i ? "," : "") + plan.groups[g].member_tables[i];
    }
    if (s.size() + 1 > cap) return 4;
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
  return 0;
}

struct RefCollection {
  std::vector<FeatureConfig> features;
  HashTableCollection coll;
};

void* ref_collection_create(const char* spec, uint64_t capacity, uint32_t chunk_rows, int* status) {
  try {
    std::vector<FeatureConfig> f = parse_features(spec);
    TableConfig proto;
    proto.capacity = capacity;
    proto.chunk_rows = chunk_rows;
    proto.embedding_dim = 1;
    MergePlan plan = plan_merge(f);
    *status = 0;
    return new RefCollection{f, HashTableCollection(std::move(plan), proto)};
  } catch (const std::exception& e) {
    *status = status_of(e);
    return nullptr;
  }
}
void ref_collection_destroy(void* h) { delete static_cast<RefCollection*>(h); }
void* ref_collection_table(void* h, uint64_t g) { return &static_cast<RefCollection*>(h)->coll.table(g); }
// out [n x feature dim]; 0, or 1 ConfigError, 5 overflow/range of an id
int ref_collection_lookup(void* h, const char* feature, const uint64_t* raw, uint64_t n, float* out) {
  RefCollection* c = static_cast<RefCollection*>(h);
  try {
    for (const FeatureConfig& f : c->features) {
      if (f.feature_name != feature) continue;
      const auto rows = c->coll.lookup(f, std::span<const uint64_t>(raw, n));
      for (uint64_t i = 0; i < n; ++i) std::memcpy(out + i * f.embedding_dim, rows[i].data(), f.embedding_dim * 4);
      return 0;
    }
    return 1;
  } catch (const std::overflow_error&) {
    return 5;
  } catch (const std::out_of_range&) {
    return 5;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- checkpoint (checkpoint.hpp) ------------------------------------------
int ref_ckpt_save_cluster(void* cluster, const char* dir) {
  GUARD(save_cluster(*static_cast<SimCluster*>(cluster), dir));
  return 0;
}
void* ref_ckpt_load_cluster(const char* dir, uint32_t saved_world, uint32_t new_world, uint64_t capacity,
                            uint32_t dim, uint32_t chunk_rows, int* status) {
  try {
    TableConfig cfg;
    cfg.capacity = capacity;
    cfg.embedding_dim = dim;
    cfg.chunk_rows = chunk_rows;
    *status = 0;
    return new SimCluster(load_cluster(dir, saved_world, new_world, cfg));
  } catch (const std::exception& e) {
    *status = status_of(e);
    return nullptr;
  }
}

uint64_t ref_closest_prefix(const uint64_t* cums, uint64_t n, uint64_t target) {
  return closest_prefix(std::span<const uint64_t>(cums, n), target);
}
uint64_t ref_sequence_batches(const uint64_t* lengths, uint64_t n, uint64_t target,
                              uint64_t chunk_samples, uint64_t* batch_sizes) {
  uint64_t cursor = 0;
  SequenceBatcher b(target, [&](std::vector<SequenceSample>& chunk) {
    if (cursor >= n) return false;
    const uint64_t end = std::min(n, cursor + chunk_samples);
    for (; cursor < end; ++cursor) {
      SequenceSample s;
      s.sample_id = cursor;
      s.feature_ids.assign(lengths[cursor], 1);
      chunk.push_back(std::move(s));
    }
    return true;
  });
  uint64_t nb = 0;
  while (auto batch = b.next_batch()) batch_sizes[nb++] = batch->size();
  return nb;
}

// ---- workload generator (the reference's own, text output parsed back) ---
// tables_vocab[tables]; features are "t<i>" of dim 1, one table each, in order.
int64_t ref_generate_workload(uint64_t seed, uint64_t num_sequences, double mean_len,
                              uint64_t max_len, double sigma, double zipf, uint32_t tables,
                              const uint64_t* vocab, uint64_t* lengths, uint64_t* ids,
                              uint64_t max_tokens) {
  try {
    WorkloadSpec spec;
    spec.seed = seed;
    spec.num_sequences = num_sequences;
    spec.length.mean = mean_len;
    spec.length.max_len = max_len;
    spec.length.sigma = sigma;
    spec.zipf_exponent = zipf;
    for (uint32_t t = 0; t < tables; ++t) {
      const std::string name = "t" + std::to_string(t);
      spec.features.push_back({"f" + std::to_string(t), 1, {name}, Pooling::kNone});
      spec.table_vocab[name] = vocab[t];
    }
    std::ostringstream os;
    generate_workload(spec, os);
    std::istringstream is(os.str());
    std::string line;
    uint64_t tok = 0, s = 0;
    while (std::getline(is, line)) {
      if (line.empty() || line[0] == '#') continue;
      std::istringstream ls(line);
      uint64_t sid;
      double label;
      ls >> sid >> label;
      uint64_t id, len = 0;
      while (ls >> id) {
        if (tok >= max_tokens) return -1;
        ids[tok++] = id;
        ++len;
      }
      lengths[s++] = len;
    }
    return static_cast<int64_t>(tok);
  } catch (const std::exception&) {
    return -1;
  }
}
// generate_workload_file / read_workload_file (workload.cpp:309-339) as they are.
int ref_write_workload_file(const char* path, uint64_t seed, uint64_t num_sequences, double mean_len,
                            uint64_t max_len, double sigma, double zipf, uint32_t tables, const uint64_t* vocab) {
  try {
    WorkloadSpec spec;
    spec.seed = seed;
    spec.num_sequences = num_sequences;
    spec.length.mean = mean_len;
    spec.length.max_len = max_len;
    spec.length.sigma = sigma;
    spec.zipf_exponent = zipf;
    for (uint32_t t = 0; t < tables; ++t) {
      const std::string name = "t" + std::to_string(t);
      spec.features.push_back({"f" + std::to_string(t), 1, {name}, Pooling::kNone});
      spec.table_vocab[name] = vocab[t];
    }
    generate_workload_file(spec, path);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
// -> number of samples (tokens in *n_tok), or -status on an exception
int64_t ref_read_workload_file(const char* path, uint64_t* sample_ids, double* labels, uint64_t* lengths,
                               uint64_t* ids, uint64_t cap_tok, uint64_t* n_tok) {
  try {
    const std::vector<SequenceSample> s = read_workload_file(path);
    uint64_t tok = 0;
    for (size_t i = 0; i < s.size(); ++i) {
      sample_ids[i] = s[i].sample_id;
      labels[i] = s[i].label;
      lengths[i] = s[i].feature_ids.size();
      for (uint64_t id : s[i].feature_ids)
        if (tok < cap_tok) ids[tok++] = id;
    }
    *n_tok = tok;
    return static_cast<int64_t>(s.size());
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}
void ref_pseudo_sparse_grad(uint64_t sample_id, uint64_t step, float* out, uint32_t dim) {
  pseudo_sparse_grad(sample_id, step, std::span<float>(out, dim));
}

// ---- CPU baseline: the reference's own single-step path ----------------------
// One C1-shaped step through the reference API on a W=1 SimCluster: stage-1
// dedup + ensure + inverse expand (distributed_lookup, exchange_sim.cpp:117-233),
// then GradAccumulator::accumulate + apply (OpenMP rows).  Adam is the
// reference's; optimizer=1 (Adagrad) has no reference and runs the frozen
// restatement of oracle.c on the reference's table rows.  Returns seconds.
// Adagrad has no reference: the frozen restatement of oracle.c on the
// reference's rows (ascending id, ensure per id, OpenMP rows like apply).
static void adagrad_apply(EmbedTable& t, const GradAccumulator& acc, double lr, double eps) {
  const uint32_t dim = t.embedding_dim();
  std::vector<RowHandle> hs;
  std::vector<const std::vector<float>*> gs;
  for (const auto& [id, g] : acc.pending()) {
    hs.push_back(t.ensure(id));
    gs.push_back(&g);
  }
  const int64_t m = static_cast<int64_t>(hs.size());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    auto w = t.embedding(hs[i]);
    auto a = t.opt_v(hs[i]);
    t.opt_step(hs[i]) += 1;
    const std::vector<float>& g = *gs[i];
    for (uint32_t e = 0; e < dim; ++e) {
      const double gd = g[e];
      const double an = a[e] + gd * gd;
      a[e] = static_cast<float>(an);
      w[e] = static_cast<float>(w[e] - lr * gd / (std::sqrt(an) + eps));
    }
  }
}

double ref_c1_step(void* cluster, const uint64_t* ids, const float* grads, uint64_t n,
                   int optimizer, double lr, double eps, float* out) {
  auto* c = static_cast<SimCluster*>(cluster);
  const uint32_t dim = c->shards[0].embedding_dim();
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::vector<uint64_t>> req(1, std::vector<uint64_t>(ids, ids + n));
  LookupResult r = distributed_lookup(*c, req);
  GradAccumulator acc(dim, 1);
  acc.accumulate(req[0], std::span<const float>(grads, n * dim));
  if (optimizer == 0)
    acc.apply(c->shards[0], AdamParams{lr, 0.9, 0.999, eps});
  else
    adagrad_apply(c->shards[0], acc, lr, eps);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (out) std::memcpy(out, r.outputs[0].data(), r.outputs[0].size() * 4);
  return sec;
}

// One W-worker step exactly as run_workload drives it (workload.cpp:506-581):
// distributed_lookup over the W workers' token lists, every token's gradient
// routed to its owner in (worker, token) order (workload.cpp:519-526), one
// GradAccumulator per owner shard (:565-569), then apply (:573-581).  The
// simulation is single-threaded by the reference's design; the row updates
// inside apply use OpenMP.  requests = the W lists concatenated, counts[W].
// Returns seconds.
double ref_dist_step(void* cluster, const uint64_t* requests, const uint64_t* counts, const float* grads,
                     int optimizer, double lr, double eps) {
  auto* c = static_cast<SimCluster*>(cluster);
  const uint64_t W = c->world_size;
  const uint32_t dim = c->shards[0].embedding_dim();
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::vector<uint64_t>> req(W);
  uint64_t off = 0;
  for (uint64_t w = 0; w < W; ++w) {
    req[w].assign(requests + off, requests + off + counts[w]);
    off += counts[w];
  }
  LookupResult r = distributed_lookup(*c, req);
  (void)r;
  std::vector<std::vector<uint64_t>> gid(W);
  std::vector<std::vector<float>> grow(W);
  off = 0;
  for (uint64_t w = 0; w < W; ++w) {
    for (uint64_t j = 0; j < counts[w]; ++j) {
      const uint64_t id = requests[off + j];
      const size_t s = SimCluster::shard_of(id, W);
      gid[s].push_back(id);
      grow[s].insert(grow[s].end(), grads + (off + j) * dim, grads + (off + j + 1) * dim);
    }
    off += counts[w];
  }
  std::vector<GradAccumulator> acc;
  for (uint64_t s = 0; s < W; ++s) acc.emplace_back(dim, 1);
  for (uint64_t s = 0; s < W; ++s)
    if (!gid[s].empty()) acc[s].accumulate(gid[s], grow[s]);
  for (uint64_t s = 0; s < W; ++s) {
    if (optimizer == 0)
      acc[s].apply(c->shards[s], AdamParams{lr, 0.9, 0.999, eps});
    else
      adagrad_apply(c->shards[s], acc[s], lr, eps);
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
int ref_omp_max_threads() { return omp_get_max_threads(); }

}  // extern "C"
