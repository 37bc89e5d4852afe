// recsparse_gpu embed_table.hpp -- EmbedTable (embed_table.hpp:28-211 of the
// reference API) backed by an rs_table on the GPU.
//
// Semantics kept: upsert / lookup (stamps the tick) / find (no side effects)
// / ensure (zero-vivify) / remove (tombstone, row to the LIFO free list) /
// expand (keys only, rows never move), batch gather with one tick per batch,
// value semantics (copies are device deep copies, rs_table_clone), the
// exceptions.  What differs, by design of the GPU table (SURVEY §8b caveats):
//  * capacity() is the GPU key structure's (8-slot buckets, >= 16 slots);
//  * RowHandle = {row / chunk_rows, row % chunk_rows} of the GPU row pool,
//    which is one pool carved in chunk_rows units (no dual-chunk rotation);
//  * row accessors return spans into a host snapshot read on demand
//    (rs_table_read_entries) and refreshed after every mutation -- reads,
//    not write-through;
//  * for_each_occupied visits live entries in key order (slot = ordinal);
//  * restore_entries cannot place explicit slots: it re-inserts the keys
//    (checkpoint.cpp:238-249 does the same on a resize).
#pragma once

#include <compare>
#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "recsparse/common.hpp"
#include "recsparse/hash.hpp"

struct rs_table;

namespace recsparse {

struct TableConfig {
  uint64_t capacity = 1024;
  uint32_t embedding_dim = 16;
  uint32_t thread_groups = 1;
  double max_load_factor = 0.75;
  uint32_t chunk_rows = 1024;

  void validate() const;  // embed_table.cpp:23-38, ConfigError
};

enum class SlotState : uint8_t { kEmpty = 0, kOccupied = 1, kTombstone = 2 };

struct RowHandle {
  uint32_t chunk = 0;
  uint32_t row = 0;
  friend bool operator==(const RowHandle&, const RowHandle&) = default;
  friend auto operator<=>(const RowHandle&, const RowHandle&) = default;
};

struct KeySlot {
  uint64_t key = 0;
  RowHandle handle{};
  SlotState state = SlotState::kEmpty;
};

class EmbedTable {
 public:
  explicit EmbedTable(TableConfig config);
  EmbedTable(const EmbedTable& other);
  EmbedTable(EmbedTable&& other) noexcept;
  EmbedTable& operator=(const EmbedTable& other);
  EmbedTable& operator=(EmbedTable&& other) noexcept;
  ~EmbedTable();

  RowHandle insert(uint64_t key, std::span<const float> embedding);
  std::optional<RowHandle> lookup(uint64_t key);
  std::optional<RowHandle> find(uint64_t key) const;
  RowHandle ensure(uint64_t key);
  bool remove(uint64_t key);
  uint64_t expand();
  void lookup_batch(std::span<const uint64_t> keys, std::span<float> out);
  void lookup_batch_serial(std::span<const uint64_t> keys, std::span<float> out);

  double load_factor() const;
  uint64_t capacity() const;
  uint64_t occupied() const;
  uint64_t tombstones() const;
  uint64_t tick() const;
  uint32_t embedding_dim() const { return config_.embedding_dim; }
  const TableConfig& config() const { return config_; }

  std::span<float> embedding(RowHandle h);
  std::span<const float> embedding(RowHandle h) const;
  std::span<float> opt_m(RowHandle h);
  std::span<const float> opt_m(RowHandle h) const;
  std::span<float> opt_v(RowHandle h);
  std::span<const float> opt_v(RowHandle h) const;
  uint64_t& row_timestamp(RowHandle h);
  uint64_t row_timestamp(RowHandle h) const;
  uint64_t& opt_step(RowHandle h);
  uint64_t opt_step(RowHandle h) const;

  uint32_t current_chunk_id() const;
  uint32_t next_chunk_id() const { return current_chunk_id() + 1; }
  size_t chunk_count() const;
  bool chunk_retired(uint32_t chunk_id) const { return chunk_id < current_chunk_id(); }
  uint64_t chunk_free_rows(uint32_t chunk_id) const;

  template <typename F>
  void for_each_occupied(F&& fn) const {
    const auto live = live_entries();
    for (uint64_t i = 0; i < live.size(); ++i) fn(i, live[i].first, live[i].second);
  }

  std::vector<RowHandle> restore_entries(std::span<const uint64_t> slots, std::span<const uint64_t> keys);
  void bump_tick(uint64_t to);

  // the GPU table behind this object (for the GPU-side callers of the shim)
  rs_table* gpu_handle() const { return t_; }
  // drops the host row snapshot (after an update issued through gpu_handle())
  void invalidate() const;

 private:
  struct RowView {
    std::vector<float> emb, m, v;
    uint64_t step = 0, ts = 0;
  };
  std::vector<std::pair<uint64_t, RowHandle>> live_entries() const;
  RowHandle handle_of(int64_t row) const;
  uint64_t key_of(RowHandle h) const;
  RowView& view(RowHandle h) const;
  std::optional<RowHandle> probe(uint64_t key, int stamp) const;

  TableConfig config_;
  rs_table* t_ = nullptr;
  mutable std::map<RowHandle, uint64_t> keys_;  // handles seen -> key
  mutable std::map<uint64_t, RowView> rows_;    // host snapshot by key
};

}  // namespace recsparse
