// recsparse_gpu sparse_update.hpp -- GradAccumulator / AdamParams
// (sparse_update.hpp:26-70 of the reference API) on the GPU.
//
// accumulate() appends the micro-batch to a device window; pending() is the
// window's per-id sums (rs_accumulate: token-order f32 sums, bit-exact for
// ids with <= 64 occurrences, within 1e-5 * sum|g| otherwise); apply() runs
// rs_sparse_update over the window: dedup, zero-vivify absent ids, ordered
// segment reduce fused with Adam (FP64 _rn math, host-libm bias tables).
// apply_serial() is the same call (the GPU result is the one result).
#pragma once

#include <cstdint>
#include <map>
#include <span>
#include <vector>

#include "recsparse/embed_table.hpp"

namespace recsparse {

struct AdamParams {
  double lr = 0.01;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double eps = 1e-8;
};

// One bias-corrected Adam step of one row (sparse_update.cpp:22-37), on the GPU.
void adam_update_row(std::span<float> weights, std::span<float> m, std::span<float> v, uint64_t& step,
                     std::span<const float> grad, const AdamParams& params);

class GradAccumulator {
 public:
  GradAccumulator(uint32_t embedding_dim, uint64_t accum_steps);

  void accumulate(std::span<const uint64_t> ids, std::span<const float> grads);
  bool ready() const { return seen_ >= accum_steps_; }
  uint64_t micro_batches_seen() const { return seen_; }
  size_t pending_ids() const { return pending().size(); }
  const std::map<uint64_t, std::vector<float>>& pending() const;

  size_t apply(EmbedTable& table, const AdamParams& params);
  size_t apply_serial(EmbedTable& table, const AdamParams& params) { return apply(table, params); }

 private:
  uint32_t dim_;
  uint64_t accum_steps_;
  uint64_t seen_ = 0;
  std::vector<uint64_t> ids_;    // the window, in call order (host staging)
  std::vector<float> grads_;
  mutable std::map<uint64_t, std::vector<float>> sums_;
  mutable bool sums_valid_ = true;
};

}  // namespace recsparse
