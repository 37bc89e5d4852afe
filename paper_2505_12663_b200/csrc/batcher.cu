// batcher.cu -- dynamic sequence balancing on the host.
//
// Reference: closest_prefix and SequenceBatcher::next_batch
// (seq_batcher.cpp:22-78, Alg. 1), the round-robin worker split and
// WorkerStream (workload.cpp:368-402, 461-469), CostModel::sample_compute
// (workload.hpp:106-109), imbalance_report and weighted_grad_combine
// (seq_batcher.cpp:80-152).  This is sequence metadata (a few thousand
// lengths per step), so it stays on the CPU next to the data loader; the
// batches it forms feed the device step.
//
// rs_partition_sequences adds the cost-model rank assignment the north star
// asks for (longest-processing-time-first on a*len + b*len^2); the
// reference's own split is round-robin (policy RS_PARTITION_ROUND_ROBIN).
#include <algorithm>
#include <cmath>
#include <deque>
#include <numeric>
#include <string>
#include <vector>

#include "rs_internal.cuh"

using namespace rs;

struct rs_seq_batcher {
  uint64_t target = 0;
  rs_chunk_source source = nullptr;
  void* ctx = nullptr;
  std::deque<std::pair<uint64_t, uint64_t>> buffer;  // (sample id, tokens)
  uint64_t buffered = 0;
  bool exhausted = false;
  std::vector<uint64_t> chunk_ids, chunk_tokens;
};

extern "C" {

int rs_closest_prefix(const uint64_t* cumsums, uint64_t n, uint64_t target, uint64_t* k_out) {
  if (!k_out) return fail(RS_ERR_CONFIG, "closest_prefix: null output");
  if (n == 0 || !cumsums) return fail(RS_ERR_CONFIG, "closest_prefix: cumsums must be non-empty");
  const uint64_t* it = std::lower_bound(cumsums, cumsums + n, target);
  if (it == cumsums + n) {
    *k_out = n;  // every prefix sum < target
  } else if (it == cumsums) {
    *k_out = 1;
  } else {
    const uint64_t above = *it - target, below = target - *(it - 1);
    *k_out = (uint64_t)(it - cumsums) + (below <= above ? 0 : 1);  // ties: the shorter prefix
  }
  return RS_OK;
}

int rs_seq_batcher_create(uint64_t target_tokens, rs_chunk_source source, void* ctx,
                          uint64_t max_chunk, rs_seq_batcher** out) {
  if (!out || !source) return fail(RS_ERR_CONFIG, "SequenceBatcher: null argument");
  if (target_tokens < 1) return fail(RS_ERR_CONFIG, "SequenceBatcher: target token count must be >= 1");
  auto* b = new rs_seq_batcher();
  b->target = target_tokens;
  b->source = source;
  b->ctx = ctx;
  b->chunk_ids.resize(std::max<uint64_t>(1, max_chunk));
  b->chunk_tokens.resize(std::max<uint64_t>(1, max_chunk));
  *out = b;
  return RS_OK;
}

int rs_seq_batcher_destroy(rs_seq_batcher* b) {
  delete b;
  return RS_OK;
}

// next_batch: *n_out sample ids in arrival order (0 once source and buffer
// are empty).  cap must hold the batch (RS_ERR_CONFIG otherwise, nothing
// consumed).
int rs_seq_batcher_next(rs_seq_batcher* b, uint64_t* sample_ids, uint64_t* token_counts,
                        uint64_t cap, uint64_t* n_out) {
  if (!b || !n_out) return fail(RS_ERR_CONFIG, "SequenceBatcher: null argument");
  while (b->buffered < b->target && !b->exhausted) {
    uint64_t got = 0;
    if (!b->source(b->ctx, b->chunk_ids.data(), b->chunk_tokens.data(), b->chunk_ids.size(), &got)) {
      b->exhausted = true;
      break;
    }
    for (uint64_t i = 0; i < got; ++i) {
      if (b->chunk_tokens[i] == 0) return fail(RS_ERR_INVARIANT, "SequenceBatcher: sample with zero tokens");
      b->buffered += b->chunk_tokens[i];
      b->buffer.emplace_back(b->chunk_ids[i], b->chunk_tokens[i]);
    }
  }
  if (b->buffer.empty()) {
    *n_out = 0;
    return RS_OK;
  }
  std::vector<uint64_t> cums(b->buffer.size());
  uint64_t run = 0;
  for (size_t i = 0; i < b->buffer.size(); ++i) cums[i] = run += b->buffer[i].second;
  uint64_t k = 0;
  rs_closest_prefix(cums.data(), cums.size(), b->target, &k);
  if (k > cap) return fail(RS_ERR_CONFIG, "SequenceBatcher: output capacity too small");
  for (uint64_t i = 0; i < k; ++i) {
    if (sample_ids) sample_ids[i] = b->buffer.front().first;
    if (token_counts) token_counts[i] = b->buffer.front().second;
    b->buffered -= b->buffer.front().second;
    b->buffer.pop_front();
  }
  *n_out = k;
  return RS_OK;
}

uint64_t rs_seq_batcher_buffered_tokens(const rs_seq_batcher* b) { return b ? b->buffered : 0; }
uint64_t rs_seq_batcher_buffered_samples(const rs_seq_batcher* b) { return b ? b->buffer.size() : 0; }

// Rank of every sequence.  ROUND_ROBIN: i % world (workload.cpp:461-469).
// COST_LPT: sequences by descending cost a*len + b*len^2 (ties: lower index
// first), each to the currently least-loaded rank (ties: lower rank).
int rs_partition_sequences(const uint64_t* lengths, uint64_t n, uint32_t world, uint32_t policy,
                           double a, double b, uint32_t* rank_out, double* load_out) {
  if (world < 1 || (n && (!lengths || !rank_out)))
    return fail(RS_ERR_CONFIG, "rs_partition_sequences: bad arguments");
  std::vector<double> load(world, 0.0);
  auto cost = [&](uint64_t i) {
    const double len = (double)lengths[i];
    return a * len + b * len * len;  // CostModel::sample_compute
  };
  if (policy == RS_PARTITION_ROUND_ROBIN) {
    for (uint64_t i = 0; i < n; ++i) {
      rank_out[i] = (uint32_t)(i % world);
      load[i % world] += cost(i);
    }
  } else if (policy == RS_PARTITION_COST_LPT) {
    std::vector<uint64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> c(n);
    for (uint64_t i = 0; i < n; ++i) c[i] = cost(i);
    std::stable_sort(order.begin(), order.end(), [&](uint64_t x, uint64_t y) { return c[x] > c[y]; });
    for (uint64_t i : order) {
      uint32_t best = 0;
      for (uint32_t r = 1; r < world; ++r)
        if (load[r] < load[best]) best = r;
      load[best] += c[i];
      rank_out[i] = best;
    }
  } else {
    return fail(RS_ERR_CONFIG, "rs_partition_sequences: unknown policy");
  }
  if (load_out) std::copy(load.begin(), load.end(), load_out);
  return RS_OK;
}

// imbalance_report (seq_batcher.cpp:140-152)
int rs_imbalance_report(const uint64_t* per_worker_tokens, uint64_t n, uint64_t* max_tokens,
                        uint64_t* min_tokens, double* spread) {
  if (n == 0 || !per_worker_tokens)
    return fail(RS_ERR_CONFIG, "imbalance_report: need at least one worker");
  const uint64_t mx = *std::max_element(per_worker_tokens, per_worker_tokens + n);
  const uint64_t mn = *std::min_element(per_worker_tokens, per_worker_tokens + n);
  if (max_tokens) *max_tokens = mx;
  if (min_tokens) *min_tokens = mn;
  if (spread) *spread = mx == 0 ? 0.0 : (double)(mx - mn) / (double)mx;
  return RS_OK;
}

// weighted_grad_combine (seq_batcher.cpp:80-138): per element, workers in a
// fixed order, acc += (double)b_i * g_i[e]; out[e] = acc * (1 / total).
// grads: workers x dim, row-major.
int rs_weighted_grad_combine(const uint64_t* batch_sizes, const double* grads, uint64_t workers,
                             uint64_t dim, double* out) {
  if (workers == 0 || !batch_sizes || !grads || !out)
    return fail(RS_ERR_CONFIG, "weighted_grad_combine: need matching, non-empty inputs");
  uint64_t total = 0;
  for (uint64_t i = 0; i < workers; ++i) {
    if (batch_sizes[i] < 1) return fail(RS_ERR_CONFIG, "weighted_grad_combine: batch sizes must be >= 1");
    total += batch_sizes[i];
  }
  const double inv = 1.0 / (double)total;
  for (uint64_t e = 0; e < dim; ++e) {
    double acc = 0.0;
    for (uint64_t i = 0; i < workers; ++i) acc += (double)batch_sizes[i] * grads[i * dim + e];
    out[e] = acc * inv;
  }
  return RS_OK;
}

}  // extern "C"
