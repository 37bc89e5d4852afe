// table_dev.cuh -- device building blocks of the dynamic table shared by the
// table kernels (table.cu) and the fused step kernels (step.cu): grouped
// bucket probing, the lock-free row allocator, row initialisation and the
// last-block counter epilogue.  See table.cu for the reference mapping.
#pragma once

#include "rs_internal.cuh"

namespace rs {
namespace tdev {

constexpr unsigned kGroupsPerBlock = 32;  // 8-lane groups per 256-thread block
constexpr unsigned kProbeThreads = kGroupsPerBlock * kBucket;

__device__ __forceinline__ uint4 ld_slot_cg(const Slot* p) {
  return __ldcg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint4 ld_slot(const Slot* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

struct Probe {
  bool found;
  uint64_t slot;      // slot of the key when found
  uint32_t row;       // row when found
  uint32_t tick;      // slot tick when found
  uint64_t ins;       // insertion slot when not found (~0 = table full)
  bool ins_tomb;      // insertion slot is a tombstone
};

// Cooperative probe by the 8 lanes of a group.  `g` = lane within the group,
// `gbase` = first warp lane of the group, `gmask` = the group's lane mask.
template <bool kCoherent>
__device__ __forceinline__ Probe probe_group(const Slot* __restrict__ slots, uint64_t nb_mask,
                                             uint64_t key, unsigned g, unsigned gbase,
                                             unsigned gmask) {
  const uint64_t h = hash64(key);
  uint64_t b = (h >> 32) & nb_mask;  // high hash bits: decorrelated from shard_of = h % W
  const uint64_t step = (h | 1ull) & nb_mask;  // odd -> full cycle over nb = 2^k buckets
  uint64_t tomb = ~0ull;
  Probe r;
  r.found = false;
  r.ins = ~0ull;
  r.ins_tomb = false;
  r.row = kNoRow;
  r.tick = 0;
  r.slot = ~0ull;
  for (uint64_t t = 0; t <= nb_mask; ++t) {
    const uint4 v = kCoherent ? ld_slot_cg(slots + b * kBucket + g) : ld_slot(slots + b * kBucket + g);
    const uint64_t k = (uint64_t)v.x | ((uint64_t)v.y << 32);
    const unsigned bm = (__ballot_sync(gmask, k == key) >> gbase) & 0xFFu;
    const unsigned be = (__ballot_sync(gmask, k == kEmptyKey) >> gbase) & 0xFFu;
    const unsigned bt = (__ballot_sync(gmask, k == kTombKey) >> gbase) & 0xFFu;
    if (bm) {
      const unsigned l = __ffs(bm) - 1;
      r.found = true;
      r.slot = b * kBucket + l;
      r.row = __shfl_sync(gmask, v.z, gbase + l);
      r.tick = __shfl_sync(gmask, v.w, gbase + l);
      return r;
    }
    if (tomb == ~0ull && bt) tomb = b * kBucket + (__ffs(bt) - 1);
    if (be) {
      r.ins = tomb != ~0ull ? tomb : b * kBucket + (__ffs(be) - 1);
      r.ins_tomb = tomb != ~0ull;
      return r;
    }
    b = (b + step) & nb_mask;
  }
  r.ins = tomb;
  r.ins_tomb = tomb != ~0ull;
  return r;
}

__device__ __forceinline__ uint32_t alloc_row(TableDev* td, unsigned long long free_n0,
                                              unsigned long long fresh0, uint64_t row_cap) {
  const unsigned long long i = atomicAdd(&td->c.alloc_ctr, 1ull);
  if (i < free_n0) return td->d.free_stack[free_n0 - 1 - i];  // LIFO reuse first
  const unsigned long long r = fresh0 + (i - free_n0);
  if (r >= row_cap) {
    atomicOr(&td->c.error, kErrRowPool);
    return kNoRow;
  }
  return (uint32_t)r;
}

// A row allocated for a key that a concurrent duplicate inserted first goes
// back to the free stack (above the launch's free_n0; the epilogue moves it
// down to the top of the surviving stack).
__device__ __forceinline__ void return_row(TableDev* td, unsigned long long free_n0, uint32_t row) {
  const unsigned int k = atomicAdd(&td->c.returned, 1u);
  td->d.free_stack[free_n0 + k] = row;
}

// New-row initialisation by the 8 lanes of a group: emb from src (or zeros),
// optimizer state zeroed (alloc_row + reset_row, embed_table.cpp:144-180).
__device__ __forceinline__ void init_row(const TableDesc& d, uint32_t row, const float* src,
                                         unsigned g) {
  const uint32_t D = d.dim;
  float* e = d.emb + (size_t)row * D;
  if ((D & 3u) == 0) {
    const uint32_t D4 = D >> 2;
    for (uint32_t i = g; i < D4; i += kBucket) {
      float4 v = src ? reinterpret_cast<const float4*>(src)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(e)[i] = v;
      if (d.s1) reinterpret_cast<float4*>(d.s1 + (size_t)row * D)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (d.s2) reinterpret_cast<float4*>(d.s2 + (size_t)row * D)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    for (uint32_t i = g; i < D; i += kBucket) {
      e[i] = src ? src[i] : 0.f;
      if (d.s1) d.s1[(size_t)row * D + i] = 0.f;
      if (d.s2) d.s2[(size_t)row * D + i] = 0.f;
    }
  }
  if (g == 0) d.step[row] = 0;
}

__device__ __forceinline__ void copy_row_group(const TableDesc& d, uint32_t row, float* dst,
                                               unsigned g) {
  const uint32_t D = d.dim;
  const float* e = d.emb + (size_t)row * D;
  if ((D & 3u) == 0) {
    for (uint32_t i = g; i < (D >> 2); i += kBucket)
      reinterpret_cast<float4*>(dst)[i] = __ldg(reinterpret_cast<const float4*>(e) + i);
  } else {
    for (uint32_t i = g; i < D; i += kBucket) dst[i] = e[i];
  }
}

// A slot whose key was just claimed by a concurrent insert of the same key in
// this launch still has row == kNoRow (empty and tombstoned slots always do):
// wait for the inserter to publish it.
__device__ __forceinline__ uint32_t wait_row(Slot* slots, uint64_t slot) {
  uint32_t r;
  while ((r = ld_acquire32(&slots[slot].row)) == kNoRow) __nanosleep(32);
  return r;
}

// Find-or-insert-zero of one key by an 8-lane group (grouped bucket probing;
// duplicate keys within a launch resolve to the same row).  Returns the row (kNoRow on a full
// table / exhausted row pool, with the error bit set); stamps the batch tick.
__device__ __forceinline__ uint32_t find_or_insert_group(TableDev* td, const TableDesc& d,
                                                         uint64_t key, unsigned g, unsigned gbase,
                                                         unsigned gmask, uint32_t tick_now,
                                                         unsigned long long free_n0,
                                                         unsigned long long fresh0,
                                                         unsigned long long* s_ins,
                                                         unsigned long long* s_reuse) {
  uint32_t row = kNoRow;
  const int sp = key == kEmptyKey ? 0 : (key == kTombKey ? 1 : -1);
  if (sp >= 0) {
    uint32_t r = kNoRow;
    int fresh = 0;
    if (g == 0) {
      r = td->c.special_row[sp];
      if (r == kNoRow) {
        const uint32_t nr = alloc_row(td, free_n0, fresh0, d.row_cap);
        if (nr != kNoRow) {
          const unsigned int prev = atomicCAS(&td->c.special_row[sp], kNoRow, nr);
          r = prev == kNoRow ? nr : prev;
          fresh = prev == kNoRow;
          if (fresh) atomicAdd(s_ins, 1ull);
        }
      }
      if (r != kNoRow) td->c.special_tick[sp] = tick_now;
    }
    r = __shfl_sync(gmask, r, gbase);
    fresh = __shfl_sync(gmask, fresh, gbase);
    if (fresh) init_row(d, r, nullptr, g);
    row = r;
  } else {
    uint32_t new_row = kNoRow;
    for (;;) {
      const Probe p = probe_group<true>(d.slots, d.nb_mask, key, g, gbase, gmask);
      if (p.found) {
        row = p.row == kNoRow ? wait_row(d.slots, p.slot) : p.row;
        if (g == 0 && new_row != kNoRow) return_row(td, free_n0, new_row);
        if (g == 0 && p.tick != tick_now) d.slots[p.slot].tick = tick_now;
        break;
      }
      if (p.ins == ~0ull) {
        if (g == 0) atomicOr(&td->c.error, kErrTableFull);
        break;
      }
      if (new_row == kNoRow) {
        uint32_t r = 0;
        if (g == 0) r = alloc_row(td, free_n0, fresh0, d.row_cap);
        new_row = __shfl_sync(gmask, r, gbase);
        if (new_row == kNoRow) break;
      }
      int ok = 0;
      if (g == 0) {
        const unsigned long long expect = p.ins_tomb ? kTombKey : kEmptyKey;
        ok = atomicCAS(&d.slots[p.ins].key, expect, (unsigned long long)key) == expect;
      }
      ok = __shfl_sync(gmask, ok, gbase);
      if (!ok) continue;
      if (g == 0) {
        *reinterpret_cast<uint2*>(&d.slots[p.ins].row) = make_uint2(new_row, tick_now);
        atomicAdd(s_ins, 1ull);
        if (p.ins_tomb) atomicAdd(s_reuse, 1ull);
      }
      init_row(d, new_row, nullptr, g);
      row = new_row;
      break;
    }
  }
  return row;
}

// Last-block epilogue: folds this launch's per-launch counters into the
// table counters (the "fix-up" of the lock-free row allocator).
// bump_tick: 0 keep the tick, 1 advance it, 2 advance it iff this launch
// removed a key (remove of absent keys leaves the table identical,
// embed_table.cpp:250-260)
// mirror_out (optional): the folded counters are also stored into the host's
// pinned mirror (mapped memory), so no copy node follows the kernel.
__device__ __forceinline__ void launch_epilogue(TableDev* td, unsigned long long free_n0,
                                                unsigned long long fresh0, int bump_tick,
                                                uint32_t tick_now, TableCounters* mirror_out = nullptr,
                                                LogCtl* log_open = nullptr, uint32_t log_n = 0,
                                                const uint32_t* log_n_ptr = nullptr) {
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s_last = atomicAdd(&td->c.blocks_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    TableCounters& c = td->c;
    const unsigned long long used = c.alloc_ctr;
    if (used <= free_n0) {
      c.free_n = free_n0 - used;
    } else {
      c.free_n = 0;
      unsigned long long f = fresh0 + (used - free_n0);
      c.fresh_next = f > td->d.row_cap ? td->d.row_cap : f;
    }
    // rows handed back by lost duplicate inserts sit at [free_n0, +returned)
    for (unsigned int k = 0; k < c.returned; ++k)
      td->d.free_stack[c.free_n + k] = td->d.free_stack[free_n0 + k];
    c.free_n += c.returned;
    c.returned = 0;
    // removals push rows above free_n0 (remove kernel); fold them in
    const bool any_removed = c.removed != 0;
    c.free_n += c.removed;
    c.occupied = c.occupied + c.inserted - c.removed;
    c.tombstones = c.tombstones - c.reused + c.removed;
    c.alloc_ctr = 0;
    c.inserted = 0;
    c.reused = 0;
    c.removed = 0;
    if (bump_tick == 1 || (bump_tick == 2 && any_removed)) c.tick = tick_now;
    c.blocks_done = 0;
    if (log_open) {  // the stamp log: this op's records took [tail, tail + n)
      log_open->op_base = log_open->tail;
      log_open->tail += log_n_ptr ? *log_n_ptr : log_n;  // (a device count: read by the last block)
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (mirror_out) {
      *mirror_out = c;
      __threadfence_system();
    }
  }
}

// Keys equal to the two sentinels live in the descriptor (rare path).
__device__ __forceinline__ int special_index(uint64_t key) {
  return key == kEmptyKey ? 0 : (key == kTombKey ? 1 : -1);
}


}  // namespace tdev
}  // namespace rs
