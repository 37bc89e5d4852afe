// recsparse_gpu.cpp -- the reference's C++ API (include/recsparse_gpu) over
// the C-ABI of librsgpu.so.  Host side only: every table operation, dedup,
// gather, reduce and optimizer step runs in the sm_100a kernels behind
// rsgpu.h; this file moves host spans to and from device buffers, maps
// status codes onto the reference's exceptions (common.hpp:24-39), and keeps
// the bookkeeping the reference API exposes (handles, trace counts of the
// ablation modes, the accumulation window).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <ostream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>

#include "../../include/rsgpu.h"
#include "recsparse/embed_table.hpp"
#include "recsparse/exchange_sim.hpp"
#include "recsparse/sparse_update.hpp"

namespace recsparse {

namespace gpu {
void check(int status, const char* what) {
  if (status == RS_OK) return;
  const std::string msg = std::string(what) + ": " + rs_last_error();
  switch (status) {
    case RS_ERR_CONFIG: throw ConfigError(msg);
    case RS_ERR_INVARIANT: throw InvariantError(msg);
    case RS_ERR_IO: throw IoError(msg);
    case RS_ERR_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace gpu

namespace {

using gpu::check;

// A device buffer (rs_buffer_alloc) holding a copy of host data.
class Dev {
 public:
  explicit Dev(uint64_t bytes) : bytes_(bytes) { check(rs_buffer_alloc(bytes, &p_), "rs_buffer_alloc"); }
  template <typename T>
  explicit Dev(std::span<const T> h) : Dev(h.size_bytes()) {
    check(rs_copy_to_device(p_, h.data(), h.size_bytes()), "rs_copy_to_device");
  }
  ~Dev() { rs_buffer_free(p_); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  template <typename T>
  void to_host(T* h, uint64_t bytes) const {
    check(rs_copy_to_host(h, p_, bytes), "rs_copy_to_host");
  }

 private:
  void* p_ = nullptr;
  uint64_t bytes_;
};

rs_table_info stats(rs_table* t) {
  rs_table_info i;
  check(rs_table_stats(t, &i), "rs_table_stats");
  return i;
}

rs_optimizer_params adam(const AdamParams& p) {
  rs_optimizer_params o;
  o.kind = RS_OPT_ADAM;
  o.lr = p.lr;
  o.beta1 = p.beta1;
  o.beta2 = p.beta2;
  o.eps = p.eps;
  return o;
}

}  // namespace

// ---- hash.hpp ------------------------------------------------------------------
void hash64_batch(std::span<const uint64_t> keys, std::span<uint64_t> out) {
  if (keys.size() != out.size()) throw std::invalid_argument("hash64_batch: size mismatch");
  if (keys.empty()) return;
  Dev k(keys), o(out.size_bytes());
  check(rs_hash64_batch(k.as<uint64_t>(), keys.size(), o.as<uint64_t>(), nullptr), "rs_hash64_batch");
  o.to_host(out.data(), out.size_bytes());
}

void hash64_batch_serial(std::span<const uint64_t> keys, std::span<uint64_t> out) {
  if (keys.size() != out.size()) throw std::invalid_argument("hash64_batch_serial: size mismatch");
  for (size_t i = 0; i < keys.size(); ++i) out[i] = hash64(keys[i]);
}

// ---- embed_table.hpp ----------------------------------------------------------
void TableConfig::validate() const {
  if (!is_power_of_two(capacity)) throw ConfigError("TableConfig: capacity must be a power of two");
  if (!is_power_of_two(thread_groups)) throw ConfigError("TableConfig: thread_groups must be a power of two");
  if (capacity < 2ull * thread_groups) throw ConfigError("TableConfig: capacity must be >= 2 * thread_groups");
  if (!(max_load_factor > 0.0 && max_load_factor < 1.0))
    throw ConfigError("TableConfig: max_load_factor must be in (0, 1)");
  if (embedding_dim == 0) throw ConfigError("TableConfig: embedding_dim must be >= 1");
  if (chunk_rows == 0) throw ConfigError("TableConfig: chunk_rows must be >= 1");
}

EmbedTable::EmbedTable(TableConfig config) : config_(config) {
  config_.validate();
  rs_table_config c;
  std::memset(&c, 0, sizeof(c));
  c.capacity = config_.capacity;
  c.embedding_dim = config_.embedding_dim;
  c.thread_groups = config_.thread_groups;
  c.max_load_factor = config_.max_load_factor;
  c.chunk_rows = config_.chunk_rows;
  c.optimizer = RS_OPT_ADAM;  // rows carry emb, m, v, step (embed_table.hpp:164-173)
  check(rs_table_create(&c, &t_), "EmbedTable");
}

EmbedTable::EmbedTable(const EmbedTable& o) : config_(o.config_), keys_(o.keys_) {
  check(rs_table_clone(o.t_, &t_), "EmbedTable(copy)");
}
EmbedTable::EmbedTable(EmbedTable&& o) noexcept
    : config_(o.config_), t_(o.t_), keys_(std::move(o.keys_)), rows_(std::move(o.rows_)) {
  o.t_ = nullptr;
}
EmbedTable& EmbedTable::operator=(const EmbedTable& o) {
  if (this != &o) {
    EmbedTable tmp(o);
    *this = std::move(tmp);
  }
  return *this;
}
EmbedTable& EmbedTable::operator=(EmbedTable&& o) noexcept {
  if (this != &o) {
    if (t_) rs_table_destroy(t_);
    config_ = o.config_;
    t_ = o.t_;
    keys_ = std::move(o.keys_);
    rows_ = std::move(o.rows_);
    o.t_ = nullptr;
  }
  return *this;
}
EmbedTable::~EmbedTable() {
  if (t_) rs_table_destroy(t_);
}

void EmbedTable::invalidate() const { rows_.clear(); }

RowHandle EmbedTable::handle_of(int64_t row) const {
  const uint64_t r = static_cast<uint64_t>(row);
  return RowHandle{static_cast<uint32_t>(r / config_.chunk_rows), static_cast<uint32_t>(r % config_.chunk_rows)};
}

std::optional<RowHandle> EmbedTable::probe(uint64_t key, int stamp) const {
  if (stamp) {  // lookup: one batch of one key stamps the tick
    Dev k(std::span<const uint64_t>(&key, 1)), out(uint64_t{4} * config_.embedding_dim);
    check(rs_table_lookup(t_, k.as<uint64_t>(), 1, out.as<float>(), nullptr), "lookup");
    invalidate();
  }
  int64_t row = -1;
  check(rs_table_read_entries(t_, &key, 1, &row, nullptr, nullptr, nullptr, nullptr, nullptr), "find");
  if (row < 0) return std::nullopt;
  const RowHandle h = handle_of(row);
  keys_[h] = key;
  return h;
}

RowHandle EmbedTable::insert(uint64_t key, std::span<const float> embedding) {
  if (embedding.size() != config_.embedding_dim)
    throw std::invalid_argument("insert: embedding length != embedding_dim");
  {
    Dev k(std::span<const uint64_t>(&key, 1)), e(embedding);
    check(rs_table_insert(t_, k.as<uint64_t>(), 1, e.as<float>(), nullptr), "insert");
  }
  invalidate();
  const auto h = probe(key, 0);
  if (!h) throw InvariantError("insert: key not found after insert");
  return *h;
}

std::optional<RowHandle> EmbedTable::lookup(uint64_t key) { return probe(key, 1); }
std::optional<RowHandle> EmbedTable::find(uint64_t key) const { return probe(key, 0); }

RowHandle EmbedTable::ensure(uint64_t key) {
  int64_t row = -1;
  {
    Dev k(std::span<const uint64_t>(&key, 1)), r(8);
    check(rs_table_ensure(t_, k.as<uint64_t>(), 1, r.as<int64_t>(), nullptr), "ensure");
    r.to_host(&row, 8);
  }
  invalidate();
  if (row < 0) throw InvariantError("ensure: no usable slot");
  const RowHandle h = handle_of(row);
  keys_[h] = key;
  return h;
}

bool EmbedTable::remove(uint64_t key) {
  uint8_t removed = 0;
  {
    Dev k(std::span<const uint64_t>(&key, 1)), r(1);
    check(rs_table_remove(t_, k.as<uint64_t>(), 1, r.as<uint8_t>(), nullptr), "remove");
    r.to_host(&removed, 1);
  }
  if (removed) {
    invalidate();
    for (auto it = keys_.begin(); it != keys_.end();)
      it = it->second == key ? keys_.erase(it) : std::next(it);
  }
  return removed != 0;
}

uint64_t EmbedTable::expand() {
  uint64_t cap = 0;
  check(rs_table_expand(t_, &cap, nullptr), "expand");
  return cap;
}

void EmbedTable::lookup_batch(std::span<const uint64_t> keys, std::span<float> out) {
  if (out.size() != keys.size() * config_.embedding_dim)
    throw std::invalid_argument("lookup_batch: output size != keys * embedding_dim");
  if (keys.empty()) return;
  Dev k(keys), o(out.size_bytes());
  check(rs_table_lookup(t_, k.as<uint64_t>(), keys.size(), o.as<float>(), nullptr), "lookup_batch");
  o.to_host(out.data(), out.size_bytes());
  invalidate();
}

void EmbedTable::lookup_batch_serial(std::span<const uint64_t> keys, std::span<float> out) {
  lookup_batch(keys, out);  // one implementation: the GPU batch (one tick per batch)
}

double EmbedTable::load_factor() const {
  const rs_table_info i = stats(t_);
  return static_cast<double>(i.occupied + i.tombstones) / static_cast<double>(i.capacity);
}
uint64_t EmbedTable::capacity() const { return stats(t_).capacity; }
uint64_t EmbedTable::occupied() const { return stats(t_).occupied; }
uint64_t EmbedTable::tombstones() const { return stats(t_).tombstones; }
uint64_t EmbedTable::tick() const { return stats(t_).tick; }

uint64_t EmbedTable::key_of(RowHandle h) const {
  auto it = keys_.find(h);
  if (it == keys_.end()) {  // a handle this object has not seen: learn the live set
    for (const auto& e : live_entries()) keys_[e.second] = e.first;
    it = keys_.find(h);
    if (it == keys_.end()) throw std::out_of_range("EmbedTable: unknown row handle");
  }
  return it->second;
}

EmbedTable::RowView& EmbedTable::view(RowHandle h) const {
  const uint64_t key = key_of(h);
  auto it = rows_.find(key);
  if (it != rows_.end()) return it->second;
  const uint32_t D = config_.embedding_dim;
  RowView v;
  v.emb.resize(D);
  v.m.resize(D);
  v.v.resize(D);
  int64_t row = -1;
  check(rs_table_read_entries(t_, &key, 1, &row, v.emb.data(), v.m.data(), v.v.data(), &v.step, &v.ts),
        "row accessor");
  if (row < 0) throw std::out_of_range("EmbedTable: row handle of a removed key");
  return rows_.emplace(key, std::move(v)).first->second;
}

std::span<float> EmbedTable::embedding(RowHandle h) { return view(h).emb; }
std::span<const float> EmbedTable::embedding(RowHandle h) const { return view(h).emb; }
std::span<float> EmbedTable::opt_m(RowHandle h) { return view(h).m; }
std::span<const float> EmbedTable::opt_m(RowHandle h) const { return view(h).m; }
std::span<float> EmbedTable::opt_v(RowHandle h) { return view(h).v; }
std::span<const float> EmbedTable::opt_v(RowHandle h) const { return view(h).v; }
uint64_t& EmbedTable::row_timestamp(RowHandle h) { return view(h).ts; }
uint64_t EmbedTable::row_timestamp(RowHandle h) const { return view(h).ts; }
uint64_t& EmbedTable::opt_step(RowHandle h) { return view(h).step; }
uint64_t EmbedTable::opt_step(RowHandle h) const { return view(h).step; }

uint32_t EmbedTable::current_chunk_id() const {
  return static_cast<uint32_t>(stats(t_).rows_allocated / config_.chunk_rows);
}
size_t EmbedTable::chunk_count() const {
  return static_cast<size_t>((stats(t_).row_capacity + config_.chunk_rows - 1) / config_.chunk_rows);
}
uint64_t EmbedTable::chunk_free_rows(uint32_t chunk_id) const {
  const rs_table_info i = stats(t_);
  const uint64_t lo = uint64_t{chunk_id} * config_.chunk_rows, hi = lo + config_.chunk_rows;
  const uint64_t carved = i.rows_allocated > lo ? std::min(i.rows_allocated, hi) - lo : 0;
  return config_.chunk_rows - carved;
}

std::vector<std::pair<uint64_t, RowHandle>> EmbedTable::live_entries() const {
  uint64_t n = 0;
  check(rs_table_export(t_, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &n), "export");
  std::vector<uint64_t> keys(n);
  std::vector<int64_t> rows(n);
  if (n) {
    check(rs_table_export(t_, n, keys.data(), nullptr, nullptr, nullptr, nullptr, nullptr, &n), "export");
    check(rs_table_read_entries(t_, keys.data(), n, rows.data(), nullptr, nullptr, nullptr, nullptr, nullptr),
          "export rows");
  }
  std::vector<std::pair<uint64_t, RowHandle>> out;
  out.reserve(n);
  for (uint64_t i = 0; i < n; ++i) out.emplace_back(keys[i], handle_of(rows[i]));
  return out;
}

std::vector<RowHandle> EmbedTable::restore_entries(std::span<const uint64_t> slots, std::span<const uint64_t> keys) {
  if (occupied() != 0) throw InvariantError("restore_entries: table is not empty");
  if (slots.size() != keys.size()) throw std::invalid_argument("restore_entries: slots / keys size mismatch");
  std::vector<RowHandle> hs;
  hs.reserve(keys.size());
  for (uint64_t k : keys) hs.push_back(ensure(k));  // slots are not portable: keys are re-inserted
  return hs;
}

void EmbedTable::bump_tick(uint64_t to) {
  check(rs_table_bump_tick(t_, to), "bump_tick");
  invalidate();
}

// ---- sparse_update.hpp ---------------------------------------------------------
void adam_update_row(std::span<float> weights, std::span<float> m, std::span<float> v, uint64_t& step,
                     std::span<const float> grad, const AdamParams& params) {
  const uint32_t D = static_cast<uint32_t>(weights.size());
  if (m.size() != D || v.size() != D || grad.size() != D)
    throw std::invalid_argument("adam_update_row: span sizes differ");
  TableConfig c;
  c.capacity = 16;
  c.embedding_dim = D;
  c.chunk_rows = 16;
  EmbedTable t(c);
  const uint64_t key = 0;
  check(rs_table_import(t.gpu_handle(), 1, &key, weights.data(), m.data(), v.data(), &step, nullptr), "import");
  const rs_optimizer_params o = adam(params);
  {
    Dev k(std::span<const uint64_t>(&key, 1)), g(grad);
    check(rs_apply_aggregated(t.gpu_handle(), k.as<uint64_t>(), 1, g.as<float>(), &o, nullptr), "adam_update_row");
  }
  int64_t row = -1;
  check(rs_table_read_entries(t.gpu_handle(), &key, 1, &row, weights.data(), m.data(), v.data(), &step, nullptr),
        "adam_update_row");
}

GradAccumulator::GradAccumulator(uint32_t embedding_dim, uint64_t accum_steps)
    : dim_(embedding_dim), accum_steps_(accum_steps) {
  if (embedding_dim == 0) throw ConfigError("GradAccumulator: embedding_dim must be >= 1");
}

void GradAccumulator::accumulate(std::span<const uint64_t> ids, std::span<const float> grads) {
  if (grads.size() != ids.size() * dim_) throw std::invalid_argument("accumulate: grads size != ids * dim");
  ids_.insert(ids_.end(), ids.begin(), ids.end());
  grads_.insert(grads_.end(), grads.begin(), grads.end());
  ++seen_;
  sums_valid_ = false;
}

// The window's per-id sums from the GPU reduce (rs_forward on a scratch
// table for the dedup, rs_accumulate for the token-order sums).
const std::map<uint64_t, std::vector<float>>& GradAccumulator::pending() const {
  if (sums_valid_) return sums_;
  sums_.clear();
  const uint64_t n = ids_.size();
  if (n) {
    TableConfig c;
    c.capacity = 16;
    while (c.capacity < 2 * n) c.capacity <<= 1;
    c.embedding_dim = dim_;
    c.chunk_rows = 1024;
    EmbedTable scratch(c);
    rs_workspace* ws = nullptr;
    check(rs_workspace_create(n, &ws), "rs_workspace_create");
    try {
      Dev k{std::span<const uint64_t>(ids_)}, g{std::span<const float>(grads_)};
      Dev out(n * dim_ * 4), sums(n * dim_ * 4), uniq(n * 8);
      check(rs_forward(ws, scratch.gpu_handle(), k.as<uint64_t>(), n, out.as<float>(), nullptr), "pending");
      check(rs_accumulate(ws, g.as<float>(), n, sums.as<float>(), nullptr), "pending");
      uint64_t nu = 0;
      check(rs_workspace_unique(ws, uniq.as<uint64_t>(), n, &nu), "pending");
      std::vector<uint64_t> hu(nu);
      std::vector<float> hs(nu * dim_);
      uniq.to_host(hu.data(), nu * 8);
      sums.to_host(hs.data(), nu * dim_ * 4);
      for (uint64_t u = 0; u < nu; ++u) sums_[hu[u]].assign(hs.begin() + u * dim_, hs.begin() + (u + 1) * dim_);
    } catch (...) {
      rs_workspace_destroy(ws);
      throw;
    }
    rs_workspace_destroy(ws);
  }
  sums_valid_ = true;
  return sums_;
}

size_t GradAccumulator::apply(EmbedTable& table, const AdamParams& params) {
  if (table.embedding_dim() != dim_) throw ConfigError("apply: table dim != accumulator dim");
  const uint64_t n = ids_.size();
  uint64_t updated = 0;
  if (n) {
    rs_workspace* ws = nullptr;
    check(rs_workspace_create(n, &ws), "rs_workspace_create");
    try {
      Dev k{std::span<const uint64_t>(ids_)}, g{std::span<const float>(grads_)};
      const rs_optimizer_params o = adam(params);
      check(rs_sparse_update(ws, table.gpu_handle(), k.as<uint64_t>(), n, g.as<float>(), &o, nullptr), "apply");
      check(rs_workspace_n_unique(ws, &updated), "apply");
    } catch (...) {
      rs_workspace_destroy(ws);
      throw;
    }
    rs_workspace_destroy(ws);
    table.invalidate();
  }
  ids_.clear();
  grads_.clear();
  sums_.clear();
  sums_valid_ = true;
  seen_ = 0;
  return updated;
}

// ---- exchange_sim.hpp ----------------------------------------------------------
const char* to_string(DedupMode mode) {
  switch (mode) {
    case DedupMode::kNone: return "none";
    case DedupMode::kCommUnique: return "comm_unique";
    case DedupMode::kLookupUnique: return "lookup_unique";
    case DedupMode::kTwoStage: return "two_stage";
  }
  return "unknown";
}

static uint64_t grid_sum(const std::vector<std::vector<uint64_t>>& g) {
  uint64_t s = 0;
  for (const auto& r : g)
    for (uint64_t x : r) s += x;
  return s;
}
uint64_t ExchangeTrace::ids_sent_total() const { return grid_sum(ids_sent); }
uint64_t ExchangeTrace::embs_sent_total() const { return grid_sum(embs_sent); }
uint64_t ExchangeTrace::lookups_total() const {
  uint64_t s = 0;
  for (uint64_t x : lookups) s += x;
  return s;
}
double ExchangeTrace::stage1_ratio() const {
  return ids_requested ? static_cast<double>(ids_sent_total()) / static_cast<double>(ids_requested) : 1.0;
}
double ExchangeTrace::stage2_ratio() const {
  return ids_received ? static_cast<double>(lookups_total()) / static_cast<double>(ids_received) : 1.0;
}
void ExchangeTrace::write_records(std::ostream& os) const {
  char line[160];
  for (size_t s = 0; s < world_size; ++s)
    for (size_t d = 0; d < world_size; ++d) {
      std::snprintf(line, sizeof(line), "src=%zu dst=%zu stage=ids count=%llu bytes=%llu\n", s, d,
                    (unsigned long long)ids_sent[s][d], (unsigned long long)(ids_sent[s][d] * id_bytes));
      os << line;
      std::snprintf(line, sizeof(line), "src=%zu dst=%zu stage=embs count=%llu bytes=%llu\n", s, d,
                    (unsigned long long)embs_sent[s][d], (unsigned long long)(embs_sent[s][d] * emb_bytes));
      os << line;
    }
}

SimCluster::SimCluster(size_t world, const TableConfig& shard_config, DedupMode mode)
    : world_size(world), dedup_mode(mode) {
  if (world == 0) throw ConfigError("SimCluster: world_size must be >= 1");
  shards.reserve(world);
  for (size_t r = 0; r < world; ++r) shards.emplace_back(shard_config);
}

size_t SimCluster::shard_of(uint64_t global_id, size_t world) { return hash64(global_id) % world; }

Stage1Result stage1_dedup(std::span<const uint64_t> ids) {
  Stage1Result r;
  const uint64_t n = ids.size();
  if (n == 0) return r;
  rs_workspace* ws = nullptr;
  check(rs_workspace_create(n, &ws), "rs_workspace_create");
  std::vector<int32_t> inv(n);
  try {
    Dev k(ids), u(n * 8), iv(n * 4), nu(16);
    check(rs_dedup(ws, k.as<uint64_t>(), n, u.as<uint64_t>(), iv.as<int32_t>(), nu.as<uint32_t>(), nullptr),
          "stage1_dedup");
    uint32_t m = 0;
    nu.to_host(&m, 4);
    r.unique_ids.resize(m);
    u.to_host(r.unique_ids.data(), uint64_t{m} * 8);
    iv.to_host(inv.data(), n * 4);
  } catch (...) {
    rs_workspace_destroy(ws);
    throw;
  }
  rs_workspace_destroy(ws);
  r.inverse_index.assign(inv.begin(), inv.end());
  return r;
}

// Stage 2 = the first-occurrence dedup of the source-ordered concatenation;
// each unique id's origins are its (source, position) pairs in that order.
Stage2Result stage2_dedup(const std::vector<std::vector<uint64_t>>& received) {
  std::vector<uint64_t> flat;
  std::vector<std::pair<size_t, size_t>> where;
  for (size_t s = 0; s < received.size(); ++s)
    for (size_t j = 0; j < received[s].size(); ++j) {
      flat.push_back(received[s][j]);
      where.emplace_back(s, j);
    }
  Stage1Result s1 = stage1_dedup(flat);
  Stage2Result r;
  r.unique_ids = std::move(s1.unique_ids);
  r.origins.resize(r.unique_ids.size());
  for (size_t p = 0; p < flat.size(); ++p)
    r.origins[s1.inverse_index[p]].push_back({where[p].first, where[p].second});
  return r;
}

struct SimCluster::Group {
  std::vector<rs_comm*> comms;
  uint64_t cap = 0;
  ~Group() {
    for (rs_comm* c : comms) rs_comm_destroy(c);
  }
};

LookupResult distributed_lookup(SimCluster& cluster, const std::vector<std::vector<uint64_t>>& requests) {
  const size_t W = cluster.world_size;
  if (requests.size() != W) throw std::invalid_argument("distributed_lookup: one request list per worker required");
  const uint32_t D = cluster.shards.front().embedding_dim();
  uint64_t n_max = 1;
  for (const auto& r : requests) n_max = std::max<uint64_t>(n_max, r.size());
  if (!cluster.group_ || cluster.group_->cap < n_max) {
    auto g = std::make_shared<SimCluster::Group>();
    g->cap = std::max<uint64_t>(n_max, cluster.group_ ? 2 * cluster.group_->cap : 1024);
    g->comms.assign(W, nullptr);
    check(rs_comm_create_local(static_cast<int>(W), g->cap, D, g->comms.data()), "rs_comm_create_local");
    cluster.group_ = g;
  }
  // the GPU step: owner routing, stage-2 dedup, find-or-insert at the owner,
  // the embedding exchange and the inverse expand, for every rank
  std::vector<std::unique_ptr<Dev>> ids, outs;
  std::vector<const uint64_t*> pid(W);
  std::vector<float*> pout(W);
  std::vector<uint64_t> n(W);
  std::vector<rs_table*> tabs(W);
  for (size_t w = 0; w < W; ++w) {
    n[w] = requests[w].size();
    ids.push_back(std::make_unique<Dev>(std::span<const uint64_t>(requests[w])));
    outs.push_back(std::make_unique<Dev>(n[w] * D * 4));
    pid[w] = ids[w]->as<uint64_t>();
    pout[w] = outs[w]->as<float>();
    tabs[w] = cluster.shards[w].gpu_handle();
  }
  check(rs_dist_group_forward(cluster.group_->comms.data(), tabs.data(), static_cast<int>(W), pid.data(), n.data(),
                              pout.data(), nullptr),
        "distributed_lookup");
  LookupResult res;
  res.outputs.resize(W);
  for (size_t w = 0; w < W; ++w) {
    res.outputs[w].resize(n[w] * D);
    outs[w]->to_host(res.outputs[w].data(), n[w] * D * 4);
    cluster.shards[w].invalidate();
  }
  ExchangeTrace& tr = res.trace;
  tr.world_size = W;
  tr.id_bytes = cluster.id_bytes;
  tr.emb_bytes = cluster.emb_bytes();
  tr.ids_sent.assign(W, std::vector<uint64_t>(W, 0));
  tr.embs_sent.assign(W, std::vector<uint64_t>(W, 0));
  tr.lookups.assign(W, 0);
  for (size_t w = 0; w < W; ++w) tr.ids_requested += n[w];
  if (cluster.dedup_mode == DedupMode::kTwoStage) {  // the device's own counters
    std::vector<uint64_t> sent(W), embs(W);
    for (size_t r = 0; r < W; ++r) {
      uint64_t lookups = 0, requested = 0, received = 0;
      check(rs_comm_trace(cluster.group_->comms[r], sent.data(), embs.data(), &lookups, &requested, &received),
            "rs_comm_trace");
      for (size_t d = 0; d < W; ++d) {
        tr.ids_sent[r][d] = sent[d];
        tr.embs_sent[r][d] = embs[d];
      }
      tr.lookups[r] = lookups;
      tr.ids_received += received;
    }
    return res;
  }
  // ablation modes: what they would send, counted from the requests
  // (stage 1 = per-worker unique before the id exchange, stage 2 = per-owner
  // unique before the probes; the answers are positional)
  const bool st1 = cluster.dedup_mode == DedupMode::kCommUnique;
  const bool st2 = cluster.dedup_mode == DedupMode::kLookupUnique;
  std::vector<std::unordered_set<uint64_t>> at_owner(W);
  for (size_t w = 0; w < W; ++w) {
    std::unordered_set<uint64_t> seen;
    for (uint64_t id : requests[w]) {
      if (st1 && !seen.insert(id).second) continue;
      const size_t o = SimCluster::shard_of(id, W);
      tr.ids_sent[w][o] += 1;
      tr.embs_sent[o][w] += 1;
      at_owner[o].insert(id);
    }
  }
  for (size_t o = 0; o < W; ++o) {
    uint64_t recv = 0;
    for (size_t w = 0; w < W; ++w) recv += tr.ids_sent[w][o];
    tr.ids_received += recv;
    tr.lookups[o] = st2 ? at_owner[o].size() : recv;
  }
  return res;
}

PipelineTrace pipeline_drive(std::span<const StageCosts>) {
  throw std::logic_error("pipeline_drive: the discrete-time pipeline simulator is outside the GPU hot path");
}

}  // namespace recsparse
