// table.cu -- the dynamic hash embedding table on sm_100a.
//
// Replaces EmbedTable (reference embed_table.hpp:73-211, embed_table.cpp).
// Key structure: 8-slot buckets of 16-byte slots, probed by 8-lane groups
// (grouped parallel probing, Eq. 5 with G = 8 lanes); bucket walk
// b_t = (b0 + t*S) mod nb with S odd, so every bucket is visited
// (hash.hpp:54-56).  Stop rules follow probe_walk (embed_table.cpp:111-142):
// stop at the key or at the first bucket holding an empty slot, remember the
// first tombstone, insert into the first tombstone else the first empty.
// Embedding structure: SoA row pool; expansion rehashes keys only
// (embed_table.cpp:267-285), rows never move.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "rs_host.hpp"
#include "table_dev.cuh"

namespace rs {
namespace {

using namespace tdev;

// mode: 0 = ensure (find-or-insert zero row), 1 = insert (upsert src rows),
//       2 = probe-only (stamp hits, report misses; bounded tables)
__global__ void __launch_bounds__(kProbeThreads)
    k_table_upsert(TableDev* __restrict__ td, const uint64_t* __restrict__ keys,
                   const uint32_t* __restrict__ d_n, uint32_t n_host,
                   const float* __restrict__ src, int mode, uint32_t* rows32, int64_t* rows64,
                   const uint32_t* __restrict__ uslot, uint32_t* srow, uint32_t* missing_list,
                   const uint32_t* __restrict__ sel, LogArgs lg = LogArgs{}) {
  const TableDesc d = td->d;
  // the stamp log (bounded tables): this op's records at base + key index
  const unsigned long long lbase = lg.rec ? (lg.probe ? lg.ctl->tail : lg.ctl->op_base) : 0ull;
  const unsigned long long free_n0 = td->c.free_n;
  const unsigned long long fresh0 = td->c.fresh_next;
  const uint32_t tick_now = td->c.tick + 1;
  const uint32_t n = d_n ? *d_n : n_host;
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  __shared__ unsigned long long s_ins, s_reuse;
  if (threadIdx.x == 0) {
    s_ins = 0;
    s_reuse = 0;
  }
  __syncthreads();
  const uint64_t group = (uint64_t)blockIdx.x * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * kGroupsPerBlock;
  for (uint64_t ii = group; ii < n; ii += ngroups) {
    const uint64_t i = sel ? sel[ii] : ii;
    const uint64_t key = keys[i];
    const float* srow_src = (mode == 1) ? src + i * (uint64_t)d.dim : nullptr;
    uint32_t row = kNoRow;
    const int sp = special_index(key);
    if (sp >= 0) {
      uint32_t r = kNoRow;
      int fresh = 0;
      if (g == 0) {
        r = td->c.special_row[sp];
        if (r == kNoRow && mode != 2) {
          const uint32_t nr = alloc_row(td, free_n0, fresh0, d.row_cap);
          if (nr != kNoRow) {
            const unsigned int prev = atomicCAS(&td->c.special_row[sp], kNoRow, nr);
            if (prev == kNoRow) {
              r = nr;
              fresh = 1;
              atomicAdd(&s_ins, 1ull);
            } else {
              r = prev;
            }
          }
        }
        bool logged = false;
        if (r != kNoRow) {
          const unsigned int old = atomicExch(&td->c.special_tick[sp], tick_now);
          logged = old != tick_now || fresh;
        }
        if (lg.rec)
          lg.rec[(lbase + i) & lg.mask] = LogRec{key, logged ? (uint32_t)(lg.cap + sp) : kNoLogSlot, tick_now};
        if (r == kNoRow && mode == 2 && missing_list) {
          const unsigned idx = atomicAdd(&td->c.missing, 1u);
          missing_list[idx] = (uint32_t)i;
        }
      }
      r = __shfl_sync(gmask, r, gbase);
      fresh = __shfl_sync(gmask, fresh, gbase);
      if (fresh) {
        init_row(d, r, srow_src, g);
      } else if (mode == 1 && r != kNoRow) {
        for (uint32_t e = g; e < d.dim; e += kBucket) d.emb[(size_t)r * d.dim + e] = srow_src[e];
      }
      row = r;
    } else {
      uint32_t new_row = kNoRow;
      for (;;) {
        const Probe p = probe_group<true>(d.slots, d.nb_mask, key, g, gbase, gmask);
        if (p.found) {
          row = p.row == kNoRow ? wait_row(d.slots, p.slot) : p.row;
          if (g == 0 && new_row != kNoRow) return_row(td, free_n0, new_row);
          if (g == 0 && lg.rec) {  // one record per stamp: the tick CAS picks it
            const bool won = p.tick != tick_now && atomicCAS(&d.slots[p.slot].tick, p.tick, tick_now) == p.tick;
            lg.rec[(lbase + i) & lg.mask] = LogRec{key, won ? (uint32_t)p.slot : kNoLogSlot, tick_now};
          } else if (g == 0 && p.tick != tick_now) {
            d.slots[p.slot].tick = tick_now;
          }
          if (mode == 1) {  // upsert: overwrite the embedding in place
            float* e = d.emb + (size_t)row * d.dim;
            for (uint32_t k = g; k < d.dim; k += kBucket) e[k] = srow_src[k];
          }
          break;
        }
        if (mode == 2) {  // probe only
          if (g == 0 && missing_list) {
            const unsigned idx = atomicAdd(&td->c.missing, 1u);
            missing_list[idx] = (uint32_t)i;
          }
          if (g == 0 && lg.rec) lg.rec[(lbase + i) & lg.mask] = LogRec{key, kNoLogSlot, tick_now};
          break;
        }
        if (p.ins == ~0ull) {
          if (g == 0) atomicOr(&td->c.error, kErrTableFull);
          if (g == 0 && lg.rec) lg.rec[(lbase + i) & lg.mask] = LogRec{key, kNoLogSlot, tick_now};
          break;
        }
        if (new_row == kNoRow) {
          uint32_t r = 0;
          if (g == 0) r = alloc_row(td, free_n0, fresh0, d.row_cap);
          new_row = __shfl_sync(gmask, r, gbase);
          if (new_row == kNoRow) {
            if (g == 0 && lg.rec) lg.rec[(lbase + i) & lg.mask] = LogRec{key, kNoLogSlot, tick_now};
            break;
          }
        }
        int ok = 0;
        if (g == 0) {
          const unsigned long long expect = p.ins_tomb ? kTombKey : kEmptyKey;
          ok = atomicCAS(&d.slots[p.ins].key, expect, (unsigned long long)key) == expect;
        }
        ok = __shfl_sync(gmask, ok, gbase);
        if (!ok) continue;  // lost the slot to another key: walk again
        if (g == 0) {
          uint2 rt = make_uint2(new_row, tick_now);
          *reinterpret_cast<uint2*>(&d.slots[p.ins].row) = rt;
          atomicAdd(&s_ins, 1ull);
          if (p.ins_tomb) atomicAdd(&s_reuse, 1ull);
          if (lg.rec) lg.rec[(lbase + i) & lg.mask] = LogRec{key, (uint32_t)p.ins, tick_now};
        }
        init_row(d, new_row, srow_src, g);
        row = new_row;
        break;
      }
    }
    if (g == 0) {
      if (rows32) rows32[i] = row;
      if (rows64) rows64[i] = row == kNoRow ? -1 : (int64_t)row;
      if (srow) srow[uslot[i]] = row;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_ins) atomicAdd(&td->c.inserted, s_ins);
    if (s_reuse) atomicAdd(&td->c.reused, s_reuse);
  }
  // a probe launch opens the op in the log: its last block (every block has
  // read the old tail) moves the tail past the op's n records
  launch_epilogue(td, free_n0, fresh0, true, tick_now, nullptr, lg.rec && lg.probe ? lg.ctl : nullptr, n);
}

// find (no side effects) / lookup_batch (stamp hits, copy or zero rows)
__global__ void __launch_bounds__(kProbeThreads)
    k_table_find(TableDev* __restrict__ td, const uint64_t* __restrict__ keys, uint64_t n,
                 int64_t* rows64, float* out, int stamp) {
  const TableDesc d = td->d;
  const uint32_t tick_now = td->c.tick + 1;
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  const uint64_t group = (uint64_t)blockIdx.x * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * kGroupsPerBlock;
  for (uint64_t i = group; i < n; i += ngroups) {
    const uint64_t key = keys[i];
    uint32_t row = kNoRow;
    const int sp = special_index(key);
    if (sp >= 0) {
      row = td->c.special_row[sp];
      if (stamp && g == 0 && row != kNoRow) td->c.special_tick[sp] = tick_now;
    } else {
      const Probe p = probe_group<false>(d.slots, d.nb_mask, key, g, gbase, gmask);
      if (p.found) {
        row = p.row;
        if (stamp && g == 0 && p.tick != tick_now) d.slots[p.slot].tick = tick_now;
      }
    }
    if (rows64 && g == 0) rows64[i] = row == kNoRow ? -1 : (int64_t)row;
    if (out) {
      float* dst = out + i * (uint64_t)d.dim;
      if (row != kNoRow) {
        copy_row_group(d, row, dst, g);
      } else {
        for (uint32_t e = g; e < d.dim; e += kBucket) dst[e] = 0.f;
      }
    }
  }
  if (stamp) {
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      s_last = atomicAdd(&td->c.blocks_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      td->c.tick = tick_now;
      td->c.blocks_done = 0;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
}

// Row state of given keys (no side effects): row id or -1, emb / m / v rows,
// step counter and tick; zeros for absent keys.  8-lane group per key.
__global__ void __launch_bounds__(kProbeThreads)
    k_read_entries(const TableDev* __restrict__ td, const uint64_t* __restrict__ keys, uint64_t n,
                   int64_t* rows64, float* emb, float* m, float* v, uint64_t* step, uint64_t* ts) {
  const TableDesc d = td->d;
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  const uint64_t group = (uint64_t)blockIdx.x * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * kGroupsPerBlock;
  for (uint64_t i = group; i < n; i += ngroups) {
    const uint64_t key = keys[i];
    uint32_t row = kNoRow, tick = 0;
    const int sp = special_index(key);
    if (sp >= 0) {
      row = td->c.special_row[sp];
      tick = td->c.special_tick[sp];
    } else {
      const Probe p = probe_group<true>(d.slots, d.nb_mask, key, g, gbase, gmask);
      if (p.found) {
        row = p.row;
        tick = p.tick;
      }
    }
    const uint64_t D = d.dim;
    for (uint32_t e = g; e < D; e += kBucket) {
      const bool live = row != kNoRow;
      emb[i * D + e] = live ? d.emb[(uint64_t)row * D + e] : 0.f;
      m[i * D + e] = live && d.s1 ? d.s1[(uint64_t)row * D + e] : 0.f;
      v[i * D + e] = live && d.s2 ? d.s2[(uint64_t)row * D + e] : 0.f;
    }
    if (g == 0) {
      rows64[i] = row == kNoRow ? -1 : (int64_t)row;
      step[i] = row == kNoRow ? 0 : d.step[row];
      ts[i] = tick;
    }
  }
}

__global__ void __launch_bounds__(kProbeThreads)
    k_table_remove(TableDev* __restrict__ td, const uint64_t* __restrict__ keys, uint64_t n,
                   uint8_t* removed) {
  const TableDesc d = td->d;
  const unsigned long long free_n0 = td->c.free_n;
  const unsigned long long fresh0 = td->c.fresh_next;
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  const uint64_t group = (uint64_t)blockIdx.x * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * kGroupsPerBlock;
  for (uint64_t i = group; i < n; i += ngroups) {
    const uint64_t key = keys[i];
    uint32_t row = kNoRow;
    const int sp = special_index(key);
    if (sp >= 0) {
      if (g == 0) row = atomicExch(&td->c.special_row[sp], kNoRow);
    } else {
      const Probe p = probe_group<true>(d.slots, d.nb_mask, key, g, gbase, gmask);
      if (p.found && g == 0) {
        if (atomicCAS(&d.slots[p.slot].key, (unsigned long long)key, kTombKey) == key) {
          row = p.row;
          d.slots[p.slot].row = kNoRow;
        }
      }
    }
    if (g == 0) {
      if (row != kNoRow) {
        // push above the launch's free_n0; the epilogue adds `removed`
        const unsigned long long k = atomicAdd(&td->c.removed, 1ull);
        d.free_stack[free_n0 + k] = row;
        if (sp >= 0) atomicAdd(&td->c.tombstones, ~0ull);  // sentinel keys leave no tombstone
      }
      if (removed) removed[i] = row != kNoRow;
    }
  }
  launch_epilogue(td, free_n0, fresh0, 2, td->c.tick + 1);
}

// Rehash every occupied slot of `old` into the (empty) new key structure.
__global__ void __launch_bounds__(kProbeThreads)
    k_rehash(const Slot* __restrict__ old, uint64_t old_nb, Slot* __restrict__ fresh,
             uint64_t nb_mask) {
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  const uint64_t group = (uint64_t)blockIdx.x * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * kGroupsPerBlock;
  for (uint64_t b = group; b < old_nb; b += ngroups) {
    const uint4 mine = ld_slot(old + b * kBucket + g);
    const uint64_t mykey = (uint64_t)mine.x | ((uint64_t)mine.y << 32);
    unsigned live = (__ballot_sync(gmask, mykey != kEmptyKey && mykey != kTombKey) >> gbase) & 0xFFu;
    while (live) {
      const unsigned j = __ffs(live) - 1;
      live &= live - 1;
      const uint64_t key = __shfl_sync(gmask, mykey, gbase + j);
      const uint32_t row = __shfl_sync(gmask, mine.z, gbase + j);
      const uint32_t tick = __shfl_sync(gmask, mine.w, gbase + j);
      for (;;) {
        const Probe p = probe_group<true>(fresh, nb_mask, key, g, gbase, gmask);
        int ok = 0;
        if (g == 0 && p.ins != ~0ull)
          ok = atomicCAS(&fresh[p.ins].key, kEmptyKey, (unsigned long long)key) == kEmptyKey;
        ok = __shfl_sync(gmask, ok, gbase);
        if (ok) {
          if (g == 0) *reinterpret_cast<uint2*>(&fresh[p.ins].row) = make_uint2(row, tick);
          break;
        }
      }
    }
  }
}

__global__ void k_fill_slots(Slot* s, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Slot v;
    v.key = kEmptyKey;
    v.row = kNoRow;
    v.tick = 0;
    s[i] = v;
  }
}

__global__ void k_gather_rows(TableDev* __restrict__ td, const int64_t* __restrict__ rows,
                              uint64_t n, float* __restrict__ out) {
  const TableDesc d = td->d;
  const unsigned g = lane_id() & (kBucket - 1);
  const uint64_t group = (uint64_t)blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * (blockDim.x >> 3);
  for (uint64_t i = group; i < n; i += ngroups) {
    const int64_t r = rows[i];
    float* dst = out + i * (uint64_t)d.dim;
    if (r >= 0)
      copy_row_group(d, (uint32_t)r, dst, g);
    else
      for (uint32_t e = g; e < d.dim; e += kBucket) dst[e] = 0.f;
  }
}

__global__ void k_scatter_state(TableDev* __restrict__ td, const int64_t* __restrict__ rows,
                                uint64_t n, const float* m, const float* v,
                                const uint64_t* step) {
  const TableDesc d = td->d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * d.dim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = i / d.dim, e = i % d.dim;
    const int64_t r = rows[k];
    if (r < 0) continue;
    if (m && d.s1) d.s1[(size_t)r * d.dim + e] = m[i];
    if (v && d.s2) d.s2[(size_t)r * d.dim + e] = v[i];
    if (step && e == 0) d.step[r] = (uint32_t)step[k];
  }
}

__global__ void k_set_ticks(TableDev* __restrict__ td, const uint64_t* __restrict__ keys,
                            const uint64_t* __restrict__ ticks, uint64_t n) {
  const TableDesc d = td->d;
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  const uint64_t group = (uint64_t)blockIdx.x * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint64_t ngroups = (uint64_t)gridDim.x * kGroupsPerBlock;
  for (uint64_t i = group; i < n; i += ngroups) {
    const int sp = special_index(keys[i]);
    if (sp >= 0) {
      if (g == 0) td->c.special_tick[sp] = (uint32_t)ticks[i];
      continue;
    }
    const Probe p = probe_group<false>(d.slots, d.nb_mask, keys[i], g, gbase, gmask);
    if (p.found && g == 0) d.slots[p.slot].tick = (uint32_t)ticks[i];
  }
}

// Batched insert with duplicate keys: the reference inserts one key at a time,
// so the LAST occurrence's row wins (embed_table.cpp:193-227).  A temporary
// open-addressed set keyed by the key keeps the highest index + 1 of each key
// (slot `mask + 1` holds the key equal to the empty sentinel); the selection
// then lists the winning indices for one upsert launch.
__device__ __forceinline__ uint64_t last_slot(unsigned long long* hkey, uint64_t mask, uint64_t key, bool claim) {
  if (key == kEmptyKey) return mask + 1;
  uint64_t h = hash64(key) & mask;
  for (;;) {
    const unsigned long long cur = claim ? atomicCAS(&hkey[h], kEmptyKey, (unsigned long long)key) : hkey[h];
    if (cur == key || (claim && cur == kEmptyKey)) return h;
    h = (h + 1) & mask;
  }
}
__global__ void k_last_of_key(const uint64_t* __restrict__ keys, uint64_t n, unsigned long long* hkey,
                              uint32_t* hidx, uint64_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicMax(&hidx[last_slot(hkey, mask, keys[i], true)], (uint32_t)(i + 1));
}
__global__ void k_select_last(const uint64_t* __restrict__ keys, uint64_t n, unsigned long long* hkey,
                              const uint32_t* hidx, uint64_t mask, uint32_t* sel, uint32_t* cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (hidx[last_slot(hkey, mask, keys[i], false)] == i + 1) sel[atomicAdd(cnt, 1u)] = (uint32_t)i;
}

__global__ void k_hash64(const uint64_t* __restrict__ k, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = hash64(k[i]);
}
__global__ void k_shard_of(const uint64_t* __restrict__ k, uint64_t n, uint32_t world,
                           uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(hash64(k[i]) % world);
}

// ---- host helpers ----------------------------------------------------------
int alloc_rows(rs_table* t, uint64_t new_cap, cudaStream_t s) {
  TableDesc& d = t->desc;
  const uint64_t old = d.row_cap;
  const size_t D = d.dim;
  float *emb = nullptr, *s1 = nullptr, *s2 = nullptr;
  uint32_t *step = nullptr, *fs = nullptr;
  RS_CUDA(cudaMallocAsync(&emb, new_cap * D * sizeof(float), s));
  if (d.opt == RS_OPT_ADAM) RS_CUDA(cudaMallocAsync(&s1, new_cap * D * sizeof(float), s));
  if (d.opt != RS_OPT_NONE) RS_CUDA(cudaMallocAsync(&s2, new_cap * D * sizeof(float), s));
  RS_CUDA(cudaMallocAsync(&step, new_cap * sizeof(uint32_t), s));
  RS_CUDA(cudaMallocAsync(&fs, new_cap * sizeof(uint32_t), s));
  if (old) {
    RS_CUDA(cudaMemcpyAsync(emb, d.emb, old * D * sizeof(float), cudaMemcpyDeviceToDevice, s));
    if (s1) RS_CUDA(cudaMemcpyAsync(s1, d.s1, old * D * sizeof(float), cudaMemcpyDeviceToDevice, s));
    if (s2) RS_CUDA(cudaMemcpyAsync(s2, d.s2, old * D * sizeof(float), cudaMemcpyDeviceToDevice, s));
    RS_CUDA(cudaMemcpyAsync(step, d.step, old * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    RS_CUDA(cudaMemcpyAsync(fs, d.free_stack, old * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    RS_CUDA(cudaFreeAsync(d.emb, s));
    if (d.s1) RS_CUDA(cudaFreeAsync(d.s1, s));
    if (d.s2) RS_CUDA(cudaFreeAsync(d.s2, s));
    RS_CUDA(cudaFreeAsync(d.step, s));
    RS_CUDA(cudaFreeAsync(d.free_stack, s));
  }
  d.emb = emb;
  d.s1 = s1;
  d.s2 = s2;
  d.step = step;
  d.free_stack = fs;
  d.row_cap = new_cap;
  RS_CUDA(cudaMemcpyAsync(&t->dev->d, &t->desc, sizeof(TableDesc), cudaMemcpyHostToDevice, s));
  t->buf_gen++;  // captured steps that baked the row pointers in are stale
  return RS_OK;
}

int read_counters(rs_table* t, TableCounters* out, cudaStream_t s) {
  t->host_syncs++;
  RS_CUDA(cudaStreamSynchronize(s));
  RS_CUDA(cudaMemcpy(out, &t->dev->c, sizeof(TableCounters), cudaMemcpyDeviceToHost));
  if (out->error) {
    const unsigned e = out->error;
    return fail(e & kErrCapacity ? RS_ERR_CAPACITY : RS_ERR_INVARIANT,
                std::string("table device error bits ") + std::to_string(e) +
                    ((e & kErrRowPool) ? " (row pool exhausted)" : "") +
                    ((e & kErrTableFull) ? " (probe found no usable slot)" : ""));
  }
  t->exact_occ = out->occupied;
  t->exact_tomb = out->tombstones;
  t->exact_rows = out->fresh_next;
  t->exact_requested = t->requested_total;
  return RS_OK;
}

int rehash_to(rs_table* t, uint64_t new_cap, cudaStream_t s) {
  log_invalidate(t);  // slot indices change
  Slot* fresh = nullptr;
  RS_CUDA(cudaMallocAsync(&fresh, new_cap * sizeof(Slot), s));
  k_fill_slots<<<grid_for(new_cap, 256, 148 * 16), 256, 0, s>>>(fresh, new_cap);
  RS_LAUNCH_CHECK("k_fill_slots");
  const uint64_t old_nb = t->capacity / kBucket;
  k_rehash<<<grid_for(old_nb, kGroupsPerBlock, 148 * 16), kProbeThreads, 0, s>>>(
      t->desc.slots, old_nb, fresh, new_cap / kBucket - 1);
  RS_LAUNCH_CHECK("k_rehash");
  RS_CUDA(cudaFreeAsync(t->desc.slots, s));
  t->desc.slots = fresh;
  t->desc.nb_mask = new_cap / kBucket - 1;
  t->capacity = new_cap;
  RS_CUDA(cudaMemcpyAsync(&t->dev->d, &t->desc, sizeof(TableDesc), cudaMemcpyHostToDevice, s));
  // tombstones are dropped by the rehash (embed_table.cpp:283)
  RS_CUDA(cudaMemsetAsync(&t->dev->c.tombstones, 0, sizeof(unsigned long long), s));
  t->exact_tomb = 0;
  t->buf_gen++;
  return RS_OK;
}

}  // namespace

// Best upper bound on (occupied, rows) from the newest completed mirror.
static void refresh_from_mirror(rs_table* t) {
  for (int k = 0; k < 2; ++k) {
    int i = (t->mirror_next + 1 + k) & 1;  // newest first
    rs_mirror& m = t->mirror[i];
    if (!m.valid) continue;
    if (cudaEventQuery(m.ev) != cudaSuccess) continue;
    if (m.requested_at_copy >= t->exact_requested) {
      t->exact_occ = m.pinned->occupied;
      t->exact_tomb = m.pinned->tombstones;
      t->exact_rows = m.pinned->fresh_next;
      t->exact_requested = m.requested_at_copy;
    }
    break;
  }
  (void)cudaGetLastError();
}

int table_prepare(rs_table* t, uint64_t n, cudaStream_t s, int headroom) {
  refresh_from_mirror(t);
  const double lf = t->cfg.max_load_factor;
  // training steps on unbounded tables (headroom > 0) keep room for that
  // many more batches of the largest size seen: grown once (the first batch
  // of a new size: one exact read), the in-flight bound below then rarely
  // trips and waits
  const uint64_t ahead = t->cfg.max_keys || headroom <= 0 ? 0 : std::min<uint64_t>(headroom * n, 1ull << 22);
  // (only while a regrowth is cheap: the row pool and the slots are copied
  // when they grow, and at 100 M rows a copy would not fit beside the original)
  const uint64_t pool_bytes = t->desc.row_cap * (uint64_t)t->desc.dim * 4 * (t->desc.s1 ? 3 : 2) +
                              t->capacity * sizeof(Slot);
  if (ahead && n > t->ahead_n && pool_bytes < (16ull << 30)) {
    TableCounters c;
    int st = read_counters(t, &c, s);
    if (st) return st;
    t->ahead_n = n + n / 4;  // (batch sizes jitter: not one exact read per new maximum)
    if ((double)(c.occupied + c.tombstones + n + ahead) > lf * (double)t->capacity) {
      uint64_t nc = t->capacity;
      while ((double)(c.occupied + n + ahead) > lf * (double)nc) nc <<= 1;
      if (nc != t->capacity || c.tombstones) {
        st = rehash_to(t, nc, s);
        if (st) return st;
      }
    }
    if (c.fresh_next + n + ahead > t->desc.row_cap) {  // (exactly the headroom: pools can be huge)
      uint64_t want = c.fresh_next + n + ahead;
      const uint64_t cr = std::max<uint32_t>(1, t->cfg.chunk_rows);
      want = (want + cr - 1) / cr * cr;
      st = alloc_rows(t, want, s);
      if (st) return st;
    }
  }
  auto occ_ub = [&]() { return t->exact_occ + (t->requested_total - t->exact_requested); };
  auto rows_ub = [&]() { return t->exact_rows + (t->requested_total - t->exact_requested); };
  bool slots_ok = (double)(occ_ub() + t->exact_tomb + n) <= lf * (double)t->capacity;
  bool rows_ok = rows_ub() + n <= t->desc.row_cap;
  if ((!slots_ok || !rows_ok) && t->exact_requested < t->requested_total) {
    // the bound includes steps still in flight: wait for the newest committed
    // mirror (the last op's completion -- work queued after it keeps the
    // device busy) before draining the stream for an exact read
    rs_mirror& m = t->mirror[t->mirror_next ^ 1];
    if (m.valid && m.requested_at_copy > t->exact_requested) {
      RS_CUDA(cudaEventSynchronize(m.ev));
      t->host_syncs++;
      refresh_from_mirror(t);
      slots_ok = (double)(occ_ub() + t->exact_tomb + n) <= lf * (double)t->capacity;
      rows_ok = rows_ub() + n <= t->desc.row_cap;
    }
  }
  if (!slots_ok || !rows_ok) {
    TableCounters c;
    int st = read_counters(t, &c, s);
    if (st) return st;
    if ((double)(c.occupied + c.tombstones + n) > lf * (double)t->capacity) {
      uint64_t nc = t->capacity;
      do {
        nc <<= 1;
      } while ((double)(c.occupied + n) > lf * (double)nc);
      st = rehash_to(t, nc, s);
      if (st) return st;
    }
    if (c.fresh_next + n > t->desc.row_cap) {
      uint64_t want = std::max<uint64_t>(t->desc.row_cap * 2, c.fresh_next + n);
      const uint64_t cr = std::max<uint32_t>(1, t->cfg.chunk_rows);
      want = (want + cr - 1) / cr * cr;
      st = alloc_rows(t, want, s);
      if (st) return st;
    }
  }
  t->requested_total += n;
  return RS_OK;
}

int table_after_op(rs_table* t, cudaStream_t s) {
  rs_mirror& m = t->mirror[t->mirror_next];
  RS_CUDA(cudaMemcpyAsync(m.pinned, &t->dev->c, sizeof(TableCounters), cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaEventRecord(m.ev, s));
  m.requested_at_copy = t->requested_total;
  m.valid = true;
  t->mirror_next ^= 1;
  t->host_tick++;
  return RS_OK;
}

int table_ensure_device(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                        uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                        uint32_t* d_srow, cudaStream_t s) {
  if (n_max == 0) return RS_OK;
  int st = table_prepare(t, n_max, s);
  if (st) return st;
  k_table_upsert<<<grid_for(n_max, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, s>>>(
      t->dev, d_keys, d_n, (uint32_t)n_max, nullptr, 0, d_rows32, d_rows64, d_uslot, d_srow,
      nullptr, nullptr);
  RS_LAUNCH_CHECK("k_table_upsert");
  return table_after_op(t, s);
}

// Graph-capturable halves of table_ensure_device (no host work inside).
int table_upsert_enqueue(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                         uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                         uint32_t* d_srow, cudaStream_t s) {
  k_table_upsert<<<grid_for(n_max, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, s>>>(
      t->dev, d_keys, d_n, (uint32_t)n_max, nullptr, 0, d_rows32, d_rows64, d_uslot, d_srow,
      nullptr, nullptr);
  RS_LAUNCH_CHECK("k_table_upsert");
  return RS_OK;
}

int table_mirror_copy(rs_table* t, int which, cudaStream_t s) {
  RS_CUDA(cudaMemcpyAsync(t->mirror[which].pinned, &t->dev->c, sizeof(TableCounters),
                          cudaMemcpyDeviceToHost, s));
  return RS_OK;
}

int table_mirror_commit(rs_table* t, int which, cudaStream_t s) {
  rs_mirror& m = t->mirror[which];
  RS_CUDA(cudaEventRecord(m.ev, s));
  m.requested_at_copy = t->requested_total;
  m.valid = true;
  t->mirror_next = which ^ 1;
  t->host_tick++;
  return RS_OK;
}

int table_adam_tables(rs_table* t, double beta1, double beta2, uint64_t applies,
                      cudaStream_t s) {
  // bias corrections 1 - beta^step for step in [0, len), host libm pow
  // (sparse_update.cpp:25-26), so device results match the reference bits.
  if (t->d_bc && t->bc_beta1 == beta1 && t->bc_beta2 == beta2 && applies + 2 < t->bc_len)
    return RS_OK;
  uint64_t len = std::max<uint64_t>(4096, t->bc_len);
  while (applies + 2 >= len) len *= 2;
  std::vector<double> h(2 * len);
  for (uint64_t k = 0; k < len; ++k) {
    h[k] = 1.0 - std::pow(beta1, static_cast<double>(k));
    h[len + k] = 1.0 - std::pow(beta2, static_cast<double>(k));
  }
  if (t->d_bc) RS_CUDA(cudaFreeAsync(t->d_bc, s));
  RS_CUDA(cudaMallocAsync(&t->d_bc, 2 * len * sizeof(double), s));
  RS_CUDA(cudaMemcpyAsync(t->d_bc, h.data(), 2 * len * sizeof(double), cudaMemcpyHostToDevice, s));
  RS_CUDA(cudaStreamSynchronize(s));  // h goes out of scope
  t->bc_len = len;
  t->bc_beta1 = beta1;
  t->bc_beta2 = beta2;
  return RS_OK;
}


// ---- bounded tables: evict the oldest (tick, key) before inserting ----------
// No reference counterpart (SPEC.md:156,165 leave eviction out); semantics
// frozen in DESIGN.md §3 and restated in oracle.c (or_table_ensure_batch).
static int grow_u32(uint32_t** p, uint64_t* cap, uint64_t n, cudaStream_t s) {
  if (*cap >= n) return RS_OK;
  if (*p) RS_CUDA(cudaFreeAsync(*p, s));
  *cap = std::max<uint64_t>(n, 1024);
  RS_CUDA(cudaMallocAsync(p, *cap * sizeof(uint32_t), s));
  return RS_OK;
}

// Host-side selection of the k live entries with smallest (tick, key) among
// those with tick < tick_limit, then a device remove.  Synchronizes.
// Bounded ensure, host part: missing list, capacity for the misses (from the
// async counter mirror; no synchronization in steady state), selection buffers.
int table_bounded_prepare(rs_table* t, uint64_t n_max, cudaStream_t s) {
  const uint64_t cap0 = t->missing_cap;
  int st = grow_u32(&t->d_missing, &t->missing_cap, n_max, s);
  if (st) return st;
  if (t->missing_cap != cap0) t->buf_gen++;
  if ((st = table_prepare(t, n_max, s))) return st;
  if ((st = evict_prepare(t, n_max))) return st;
  return log_prepare(t, n_max, s);
}

// Bounded ensure, device part: probe (stamp hits, list misses), the device
// victim selection (oldest (tick, key) beyond the bound) with the tick
// rewound to the batch tick, then the insert of the misses.
int table_bounded_enqueue(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                          uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                          uint32_t* d_srow, cudaStream_t s) {
  RS_CUDA(cudaMemsetAsync(&t->dev->c.missing, 0, sizeof(unsigned int), s));
  // both passes write the op's stamp-log records (probe: hits + placeholders,
  // insert: the misses' records over their placeholders)
  k_table_upsert<<<grid_for(n_max, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, s>>>(
      t->dev, d_keys, d_n, (uint32_t)n_max, nullptr, 2, d_rows32, d_rows64, d_uslot, d_srow,
      t->d_missing, nullptr, log_args(t, 1));
  RS_LAUNCH_CHECK("k_table_upsert(probe)");
  int st = evict_device(t, d_n, n_max, 0, s);
  if (st) return st;
  k_table_upsert<<<grid_for(n_max, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, s>>>(
      t->dev, d_keys, &t->dev->c.missing, (uint32_t)n_max, nullptr, 0, d_rows32, d_rows64, d_uslot,
      d_srow, nullptr, t->d_missing, log_args(t, 0));
  RS_LAUNCH_CHECK("k_table_upsert(insert missing)");
  // a big op (a fill) leaves one huge unsorted group: the next op rebuilds
  // the log (tick, key)-sorted instead of selecting inside it every time
  if (n_max > (1u << 18)) log_invalidate(t);
  return RS_OK;
}

// The bounded ensure after an external probe (the fast step's KA probed,
// stamped and listed the misses in t->d_missing): victims, then the misses.
int table_bounded_evict_insert(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                               uint32_t* d_rows32, int64_t* d_rows64, cudaStream_t s) {
  int st = evict_device(t, d_n, n_max, 0, s);
  if (st) return st;
  k_table_upsert<<<grid_for(n_max, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, s>>>(
      t->dev, d_keys, &t->dev->c.missing, (uint32_t)n_max, nullptr, 0, d_rows32, d_rows64, nullptr, nullptr,
      nullptr, t->d_missing, log_args(t, 0));
  RS_LAUNCH_CHECK("k_table_upsert(insert missing)");
  if (n_max > (1u << 18)) log_invalidate(t);
  return RS_OK;
}

// ensure for any table; bounded tables probe, evict, then insert the misses.
int table_ensure_any(rs_table* t, const uint64_t* d_keys, const uint32_t* d_n, uint64_t n_max,
                     uint32_t* d_rows32, int64_t* d_rows64, const uint32_t* d_uslot,
                     uint32_t* d_srow, cudaStream_t s) {
  if (!t->cfg.max_keys)
    return table_ensure_device(t, d_keys, d_n, n_max, d_rows32, d_rows64, d_uslot, d_srow, s);
  if (n_max == 0) return RS_OK;
  int st = table_bounded_prepare(t, n_max, s);
  if (!st) st = table_bounded_enqueue(t, d_keys, d_n, n_max, d_rows32, d_rows64, d_uslot, d_srow, s);
  if (st) return st;
  return table_after_op(t, s);
}

}  // namespace rs

using namespace rs;

static cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

extern "C" {

int rs_hash64_batch(const uint64_t* d_keys, uint64_t n, uint64_t* d_out, void* stream) {
  if (n == 0) return RS_OK;
  k_hash64<<<grid_for(n, 256, 148 * 16), 256, 0, S(stream)>>>(d_keys, n, d_out);
  RS_LAUNCH_CHECK("k_hash64");
  return RS_OK;
}

int rs_shard_of_batch(const uint64_t* d_ids, uint64_t n, uint32_t world, uint32_t* d_owner,
                      void* stream) {
  if (world == 0) return fail(RS_ERR_CONFIG, "shard_of: world_size must be >= 1");
  if (n == 0) return RS_OK;
  k_shard_of<<<grid_for(n, 256, 148 * 16), 256, 0, S(stream)>>>(d_ids, n, world, d_owner);
  RS_LAUNCH_CHECK("k_shard_of");
  return RS_OK;
}

int rs_table_create(const rs_table_config* cfg, rs_table** out) {
  if (!cfg || !out) return fail(RS_ERR_CONFIG, "rs_table_create: null argument");
  const rs_table_config c = *cfg;
  auto pow2 = [](uint64_t x) { return x && !(x & (x - 1)); };
  // TableConfig::validate (embed_table.cpp:23-38)
  if (!pow2(c.capacity)) return fail(RS_ERR_CONFIG, "TableConfig: capacity must be a power of two");
  if (!pow2(c.thread_groups))
    return fail(RS_ERR_CONFIG, "TableConfig: thread_groups must be a power of two >= 1");
  if (c.capacity < 2ull * c.thread_groups)
    return fail(RS_ERR_CONFIG, "TableConfig: capacity must be >= 2 * thread_groups");
  if (!(c.max_load_factor > 0.0 && c.max_load_factor < 1.0))
    return fail(RS_ERR_CONFIG, "TableConfig: max_load_factor must be in (0, 1)");
  if (c.chunk_rows < 1) return fail(RS_ERR_CONFIG, "TableConfig: chunk_rows must be >= 1");
  if (c.embedding_dim < 1) return fail(RS_ERR_CONFIG, "TableConfig: embedding_dim must be >= 1");
  if (c.optimizer > RS_OPT_ADAGRAD) return fail(RS_ERR_CONFIG, "TableConfig: unknown optimizer");
  rs_table* t = new rs_table();
  t->cfg = c;
  t->capacity = std::max<uint64_t>(c.capacity, kBucket);  // >= one bucket
  t->desc.dim = c.embedding_dim;
  t->desc.opt = c.optimizer;
  cudaStream_t s = nullptr;
  auto cleanup = [&](int st) {
    rs_table_destroy(t);
    return st;
  };
  if (cudaMalloc(&t->dev, sizeof(TableDev)) != cudaSuccess)
    return cleanup(cuda_fail(cudaGetLastError(), "cudaMalloc(TableDev)"));
  if (cudaMalloc(&t->desc.slots, t->capacity * sizeof(Slot)) != cudaSuccess)
    return cleanup(cuda_fail(cudaGetLastError(), "cudaMalloc(slots)"));
  t->desc.nb_mask = t->capacity / kBucket - 1;
  k_fill_slots<<<grid_for(t->capacity, 256, 148 * 16), 256, 0, s>>>(t->desc.slots, t->capacity);
  count_launch();
  TableCounters c0;
  std::memset(&c0, 0, sizeof(c0));
  c0.special_row[0] = c0.special_row[1] = kNoRow;
  if (cudaMemcpy(&t->dev->c, &c0, sizeof(c0), cudaMemcpyHostToDevice) != cudaSuccess)
    return cleanup(cuda_fail(cudaGetLastError(), "init counters"));
  uint64_t rows = c.initial_rows ? c.initial_rows
                                 : (uint64_t)std::ceil((double)t->capacity * c.max_load_factor);
  if (c.max_keys) rows = std::max<uint64_t>(rows, c.max_keys);
  rows = std::max<uint64_t>(rows, 16);
  int st = alloc_rows(t, rows, s);
  if (st) return cleanup(st);
  for (auto& m : t->mirror) {
    if (cudaMallocHost(&m.pinned, sizeof(TableCounters)) != cudaSuccess ||
        cudaEventCreateWithFlags(&m.ev, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(cuda_fail(cudaGetLastError(), "mirror alloc"));
    // kernels may store the counters straight into it (mapped pinned memory)
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&m.dev_ptr), m.pinned, 0) != cudaSuccess) {
      cudaGetLastError();
      m.dev_ptr = nullptr;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess)
    return cleanup(cuda_fail(cudaGetLastError(), "rs_table_create"));
  *out = t;
  return RS_OK;
}

int rs_table_destroy(rs_table* t) {
  if (!t) return RS_OK;
  cudaDeviceSynchronize();
  cudaFree(t->desc.slots);
  cudaFree(t->desc.emb);
  cudaFree(t->desc.s1);
  cudaFree(t->desc.s2);
  cudaFree(t->desc.step);
  cudaFree(t->desc.free_stack);
  cudaFree(t->d_bc);
  cudaFree(t->dev);
  if (t->d_evict) cudaFree(t->d_evict);
  if (t->d_cand) cudaFree(t->d_cand);
  if (t->d_victim_idx) cudaFree(t->d_victim_idx);
  void* lgp[] = {t->d_log, t->d_log_ctl, t->d_lg_cnt, t->d_lg_pre};
  for (void* p : lgp)
    if (p) cudaFree(p);
  for (auto& m : t->mirror) {
    if (m.pinned) cudaFreeHost(m.pinned);
    if (m.ev) cudaEventDestroy(m.ev);
  }
  delete t;
  return RS_OK;
}

int rs_table_stats(rs_table* t, rs_table_info* out) {
  if (!t || !out) return fail(RS_ERR_CONFIG, "rs_table_stats: null argument");
  TableCounters c;
  int st = read_counters(t, &c, nullptr);
  t->host_syncs--;  // the stats call itself is not bookkeeping
  RS_CUDA(cudaDeviceSynchronize());
  RS_CUDA(cudaMemcpy(&c, &t->dev->c, sizeof(c), cudaMemcpyDeviceToHost));
  if (st) return st;
  out->host_syncs = t->host_syncs;
  out->capacity = t->capacity;
  out->occupied = c.occupied;
  out->tombstones = c.tombstones;
  out->rows_allocated = c.fresh_next;
  out->rows_free = c.free_n;
  out->row_capacity = t->desc.row_cap;
  out->tick = c.tick;
  out->embedding_dim = t->desc.dim;
  out->optimizer = t->desc.opt;
  return RS_OK;
}

int rs_table_insert(rs_table* t, const uint64_t* d_keys, uint64_t n, const float* d_emb,
                    void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_insert: null table");
  if (n == 0) return RS_OK;
  if (!d_emb) return fail(RS_ERR_CONFIG, "insert: embedding length != embedding_dim");
  if (t->cfg.max_keys) return fail(RS_ERR_CONFIG, "insert on a bounded table: use rs_table_ensure");
  cudaStream_t s = S(stream);
  int st = table_prepare(t, n, s);
  if (st) return st;
  // duplicate keys in the batch: the last occurrence wins (one upsert per key)
  uint64_t S_ = 16;
  while (S_ < 2 * n) S_ <<= 1;
  unsigned long long* hkey = nullptr;
  uint32_t *hidx = nullptr, *sel = nullptr;
  RS_CUDA(cudaMallocAsync(&hkey, (S_ + 2) * 8, s));
  RS_CUDA(cudaMallocAsync(&hidx, (S_ + 2) * 4 + n * 4 + 16, s));
  sel = hidx + S_ + 2;
  uint32_t* cnt = sel + n;
  RS_CUDA(cudaMemsetAsync(hkey, 0xFF, (S_ + 2) * 8, s));
  RS_CUDA(cudaMemsetAsync(hidx, 0, (S_ + 2) * 4, s));
  RS_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
  k_last_of_key<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(d_keys, n, hkey, hidx, S_ - 1);
  RS_LAUNCH_CHECK("k_last_of_key");
  k_select_last<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(d_keys, n, hkey, hidx, S_ - 1, sel, cnt);
  RS_LAUNCH_CHECK("k_select_last");
  k_table_upsert<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, s>>>(
      t->dev, d_keys, cnt, (uint32_t)n, d_emb, 1, nullptr, nullptr, nullptr, nullptr, nullptr, sel);
  RS_LAUNCH_CHECK("k_table_upsert(insert)");
  RS_CUDA(cudaFreeAsync(hkey, s));
  RS_CUDA(cudaFreeAsync(hidx, s));
  return table_after_op(t, s);
}

int rs_table_find(rs_table* t, const uint64_t* d_keys, uint64_t n, int64_t* d_rows, void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_find: null table");
  if (n == 0) return RS_OK;
  k_table_find<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, S(stream)>>>(
      t->dev, d_keys, n, d_rows, nullptr, 0);
  RS_LAUNCH_CHECK("k_table_find");
  return RS_OK;
}

int rs_table_lookup(rs_table* t, const uint64_t* d_keys, uint64_t n, float* d_out, void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_lookup: null table");
  if (n == 0) return RS_OK;
  k_table_find<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, S(stream)>>>(
      t->dev, d_keys, n, nullptr, d_out, 1);
  RS_LAUNCH_CHECK("k_table_find(lookup)");
  t->host_tick++;
  if (t->cfg.max_keys) log_invalidate(t);  // stamps without log records
  return RS_OK;
}

int rs_table_gather_rows(rs_table* t, const int64_t* d_rows, uint64_t n, float* d_out,
                         void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_gather_rows: null table");
  if (n == 0) return RS_OK;
  k_gather_rows<<<grid_for(n, 32, 148 * 8), 256, 0, S(stream)>>>(t->dev, d_rows, n, d_out);
  RS_LAUNCH_CHECK("k_gather_rows");
  return RS_OK;
}

int rs_table_remove(rs_table* t, const uint64_t* d_keys, uint64_t n, uint8_t* d_removed,
                    void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_remove: null table");
  if (n == 0) return RS_OK;
  k_table_remove<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads, 0, S(stream)>>>(
      t->dev, d_keys, n, d_removed);
  RS_LAUNCH_CHECK("k_table_remove");
  return table_after_op(t, S(stream));
}

int rs_table_expand(rs_table* t, uint64_t* new_capacity, void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_expand: null table");
  cudaStream_t s = S(stream);
  TableCounters c;
  int st = read_counters(t, &c, s);
  if (st) return st;
  // expand_impl (embed_table.cpp:267-272): double at least once, keep
  // doubling while occupied/capacity exceeds the load ceiling
  uint64_t nc = t->capacity;
  do {
    nc <<= 1;
  } while ((double)c.occupied > t->cfg.max_load_factor * (double)nc);
  st = rehash_to(t, nc, s);
  if (st) return st;
  RS_CUDA(cudaStreamSynchronize(s));
  if (new_capacity) *new_capacity = nc;
  return RS_OK;
}

int rs_table_ensure(rs_table* t, const uint64_t* d_keys, uint64_t n, int64_t* d_rows,
                    void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_ensure: null table");
  return table_ensure_any(t, d_keys, nullptr, n, nullptr, d_rows, nullptr, nullptr, S(stream));
}

int rs_table_evict(rs_table* t, uint64_t k, uint64_t* evicted, void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_evict: null table");
  if (evicted) *evicted = 0;
  if (k == 0) return RS_OK;
  cudaStream_t s = S(stream);
  int st = evict_prepare(t, k);
  if (!st) st = evict_device(t, nullptr, 0, k, s);
  if (!st) st = table_after_op(t, s);
  if (!st) st = evict_count(t, evicted, s);  // synchronizes
  return st;
}

// EmbedTable's copy constructor (embed_table.cpp:47-97): a device-side deep
// copy -- same key slots, row ids, row pool, free stack, counters and tick --
// so handles, contents and every later operation behave identically.
int rs_table_clone(rs_table* src, rs_table** out) {
  if (!src || !out) return fail(RS_ERR_CONFIG, "rs_table_clone: null argument");
  RS_CUDA(cudaDeviceSynchronize());
  rs_table_config c = src->cfg;
  c.capacity = src->capacity;
  c.initial_rows = src->desc.row_cap;
  rs_table* t = nullptr;
  int st = rs_table_create(&c, &t);
  if (st) return st;
  auto cp = [&](void* d, const void* s_, size_t b) {
    return b && d && s_ ? cudaMemcpy(d, s_, b, cudaMemcpyDeviceToDevice) : cudaSuccess;
  };
  const TableDesc& a = src->desc;
  TableDesc& b = t->desc;
  const size_t D = a.dim, R = a.row_cap;
  cudaError_t e = cp(b.slots, a.slots, src->capacity * sizeof(Slot));
  if (e == cudaSuccess) e = cp(b.emb, a.emb, R * D * 4);
  if (e == cudaSuccess) e = cp(b.s1, a.s1, R * D * 4);
  if (e == cudaSuccess) e = cp(b.s2, a.s2, R * D * 4);
  if (e == cudaSuccess) e = cp(b.step, a.step, R * 4);
  if (e == cudaSuccess) e = cp(b.free_stack, a.free_stack, R * 4);
  if (e == cudaSuccess) e = cp(&t->dev->c, &src->dev->c, sizeof(TableCounters));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    rs_table_destroy(t);
    return cuda_fail(e, "rs_table_clone");
  }
  t->cfg = src->cfg;
  t->requested_total = src->requested_total;
  t->exact_occ = src->exact_occ;
  t->exact_tomb = src->exact_tomb;
  t->exact_rows = src->exact_rows;
  t->exact_requested = src->exact_requested;
  t->applies = src->applies;
  t->host_tick = src->host_tick;
  *out = t;
  return RS_OK;
}

// EmbedTable::bump_tick (embed_table.hpp:159-161): the batch tick never moves backwards.
int rs_table_bump_tick(rs_table* t, uint64_t to) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_bump_tick: null table");
  if (to >> 32) return fail(RS_ERR_CONFIG, "rs_table_bump_tick: the device tick is 32 bits");
  RS_CUDA(cudaDeviceSynchronize());
  uint32_t cur = 0;
  RS_CUDA(cudaMemcpy(&cur, &t->dev->c.tick, 4, cudaMemcpyDeviceToHost));
  if (to > cur) {
    const uint32_t v = (uint32_t)to;
    RS_CUDA(cudaMemcpy(&t->dev->c.tick, &v, 4, cudaMemcpyHostToDevice));
  }
  return RS_OK;
}

int rs_table_read_entries(rs_table* t, const uint64_t* keys, uint64_t n, int64_t* rows, float* emb,
                          float* m, float* v, uint64_t* step, uint64_t* ts) {
  if (!t || (n && !keys)) return fail(RS_ERR_CONFIG, "rs_table_read_entries: null argument");
  if (n == 0) return RS_OK;
  const uint64_t D = t->desc.dim;
  // one device block: keys | rows | step | ts | emb | m | v
  const size_t bytes = n * (8 + 8 + 8 + 8) + 3 * n * D * 4;
  char* dbuf = nullptr;
  RS_CUDA(cudaMalloc(&dbuf, bytes));
  uint64_t* dk = reinterpret_cast<uint64_t*>(dbuf);
  int64_t* dr = reinterpret_cast<int64_t*>(dk + n);
  uint64_t* ds = reinterpret_cast<uint64_t*>(dr + n);
  uint64_t* dt = ds + n;
  float* de = reinterpret_cast<float*>(dt + n);
  float* dm = de + n * D;
  float* dv = dm + n * D;
  int st = RS_OK;
  cudaError_t e = cudaMemcpy(dk, keys, n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_read_entries<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads>>>(t->dev, dk, n, dr, de, dm, dv, ds, dt);
    count_launch();
    e = cudaGetLastError();
  }
  auto back = [&](void* h, const void* d, size_t b) {
    if (h && e == cudaSuccess) e = cudaMemcpy(h, d, b, cudaMemcpyDeviceToHost);
  };
  back(rows, dr, n * 8);
  back(emb, de, n * D * 4);
  back(m, dm, n * D * 4);
  back(v, dv, n * D * 4);
  back(step, ds, n * 8);
  back(ts, dt, n * 8);
  if (e != cudaSuccess) st = cuda_fail(e, "rs_table_read_entries");
  cudaFree(dbuf);
  return st;
}

int rs_table_export(rs_table* t, uint64_t max_entries, uint64_t* keys, float* emb, float* m,
                    float* v, uint64_t* step, uint64_t* ts, uint64_t* count) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_export: null table");
  TableCounters c;
  int st = read_counters(t, &c, nullptr);
  if (st) return st;
  std::vector<Slot> slots(t->capacity);
  RS_CUDA(cudaMemcpy(slots.data(), t->desc.slots, t->capacity * sizeof(Slot), cudaMemcpyDeviceToHost));
  struct E {
    uint64_t key;
    uint32_t row, tick;
  };
  std::vector<E> live;
  live.reserve(c.occupied + 2);
  for (const Slot& sl : slots)
    if (sl.key != kEmptyKey && sl.key != kTombKey) live.push_back({sl.key, sl.row, sl.tick});
  for (int sp = 0; sp < 2; ++sp)
    if (c.special_row[sp] != kNoRow)
      live.push_back({sp == 0 ? kEmptyKey : kTombKey, c.special_row[sp], c.special_tick[sp]});
  std::sort(live.begin(), live.end(), [](const E& a, const E& b) { return a.key < b.key; });
  if (count) *count = live.size();
  if (max_entries == 0) return RS_OK;
  if (max_entries < live.size()) return fail(RS_ERR_CONFIG, "rs_table_export: buffer too small");
  const size_t D = t->desc.dim;
  uint64_t nrows = 0;
  for (const E& e : live) nrows = std::max<uint64_t>(nrows, (uint64_t)e.row + 1);
  std::vector<float> he, hm, hv;
  std::vector<uint32_t> hs;
  auto pull = [&](std::vector<float>& h, const float* src) -> int {
    h.resize(nrows * D);
    if (src && nrows)
      RS_CUDA(cudaMemcpy(h.data(), src, nrows * D * 4, cudaMemcpyDeviceToHost));
    else
      std::fill(h.begin(), h.end(), 0.f);
    return RS_OK;
  };
  if (emb && (st = pull(he, t->desc.emb))) return st;
  if (m && (st = pull(hm, t->desc.s1))) return st;
  if (v && (st = pull(hv, t->desc.s2))) return st;
  if (step) {
    hs.resize(nrows);
    if (nrows) RS_CUDA(cudaMemcpy(hs.data(), t->desc.step, nrows * 4, cudaMemcpyDeviceToHost));
  }
  for (size_t i = 0; i < live.size(); ++i) {
    const E& e = live[i];
    const size_t r = e.row;
    if (keys) keys[i] = e.key;
    if (ts) ts[i] = e.tick;
    if (emb) std::memcpy(emb + i * D, he.data() + r * D, D * 4);
    if (m) std::memcpy(m + i * D, hm.data() + r * D, D * 4);
    if (v) std::memcpy(v + i * D, hv.data() + r * D, D * 4);
    if (step) step[i] = hs[r];
  }
  return RS_OK;
}

int rs_table_import(rs_table* t, uint64_t n, const uint64_t* keys, const float* emb,
                    const float* m, const float* v, const uint64_t* step, const uint64_t* ts) {
  if (t) t->evict_tmin_valid = false;  // imported ticks may lie below the last selection's min
  if (t) log_invalidate(t);              // (and the stamp log does not list them)
  if (!t) return fail(RS_ERR_CONFIG, "rs_table_import: null table");
  if (n == 0) return RS_OK;
  const size_t D = t->desc.dim;
  // the device keeps step counters and ticks in 32 bits
  uint64_t max_step = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if ((step && step[i] >> 32) || (ts && ts[i] >> 32))
      return fail(RS_ERR_CONFIG, "rs_table_import: step / ts values >= 2^32 are not representable");
    if (step) max_step = std::max(max_step, step[i]);
  }
  // duplicate keys: the last occurrence wins (insert one at a time, embed_table.cpp:193-227)
  {
    std::unordered_map<uint64_t, uint64_t> last;
    last.reserve(n * 2);
    for (uint64_t i = 0; i < n; ++i) last[keys[i]] = i;
    if (last.size() != n) {
      std::vector<uint64_t> idx;
      idx.reserve(last.size());
      for (uint64_t i = 0; i < n; ++i)
        if (last[keys[i]] == i) idx.push_back(i);
      const uint64_t u = idx.size();
      std::vector<uint64_t> k2(u), s2, t2;
      std::vector<float> e2, m2, v2;
      if (emb) e2.resize(u * D);
      if (m) m2.resize(u * D);
      if (v) v2.resize(u * D);
      if (step) s2.resize(u);
      if (ts) t2.resize(u);
      for (uint64_t j = 0; j < u; ++j) {
        const uint64_t i = idx[j];
        k2[j] = keys[i];
        if (emb) std::copy(emb + i * D, emb + (i + 1) * D, e2.begin() + j * D);
        if (m) std::copy(m + i * D, m + (i + 1) * D, m2.begin() + j * D);
        if (v) std::copy(v + i * D, v + (i + 1) * D, v2.begin() + j * D);
        if (step) s2[j] = step[i];
        if (ts) t2[j] = ts[i];
      }
      return rs_table_import(t, u, k2.data(), emb ? e2.data() : nullptr, m ? m2.data() : nullptr,
                             v ? v2.data() : nullptr, step ? s2.data() : nullptr, ts ? t2.data() : nullptr);
    }
  }
  // Adam's bias-correction table covers every imported step (host-libm bits)
  t->applies = std::max<uint64_t>(t->applies, max_step);
  uint64_t *dk = nullptr, *dstep = nullptr, *dts = nullptr;
  float *de = nullptr, *dm = nullptr, *dv = nullptr;
  int64_t* drows = nullptr;
  RS_CUDA(cudaMalloc(&dk, n * 8));
  RS_CUDA(cudaMalloc(&de, n * D * 4));
  RS_CUDA(cudaMalloc(&drows, n * 8));
  RS_CUDA(cudaMemcpy(dk, keys, n * 8, cudaMemcpyHostToDevice));
  if (emb)
    RS_CUDA(cudaMemcpy(de, emb, n * D * 4, cudaMemcpyHostToDevice));
  else
    RS_CUDA(cudaMemset(de, 0, n * D * 4));
  int st = table_prepare(t, n, nullptr);
  if (st) return st;
  k_table_upsert<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads>>>(
      t->dev, dk, nullptr, (uint32_t)n, de, 1, nullptr, drows, nullptr, nullptr, nullptr, nullptr);
  RS_LAUNCH_CHECK("k_table_upsert(import)");
  st = table_after_op(t, nullptr);
  if (st) return st;
  if (m) {
    RS_CUDA(cudaMalloc(&dm, n * D * 4));
    RS_CUDA(cudaMemcpy(dm, m, n * D * 4, cudaMemcpyHostToDevice));
  }
  if (v) {
    RS_CUDA(cudaMalloc(&dv, n * D * 4));
    RS_CUDA(cudaMemcpy(dv, v, n * D * 4, cudaMemcpyHostToDevice));
  }
  if (step) {
    RS_CUDA(cudaMalloc(&dstep, n * 8));
    RS_CUDA(cudaMemcpy(dstep, step, n * 8, cudaMemcpyHostToDevice));
  }
  if (m || v || step) {
    k_scatter_state<<<grid_for(n * D, 256, 148 * 16), 256>>>(t->dev, drows, n, dm, dv, dstep);
    RS_LAUNCH_CHECK("k_scatter_state");
  }
  if (ts) {
    RS_CUDA(cudaMalloc(&dts, n * 8));
    RS_CUDA(cudaMemcpy(dts, ts, n * 8, cudaMemcpyHostToDevice));
    k_set_ticks<<<grid_for(n, kGroupsPerBlock, 148 * 8), kProbeThreads>>>(t->dev, dk, dts, n);
    RS_LAUNCH_CHECK("k_set_ticks");
    // bump_tick(max ts) (embed_table.hpp:159-161): stamps stay monotone after a reload
    const uint64_t mx = *std::max_element(ts, ts + n);
    unsigned int cur = 0;
    RS_CUDA(cudaDeviceSynchronize());
    RS_CUDA(cudaMemcpy(&cur, &t->dev->c.tick, 4, cudaMemcpyDeviceToHost));
    if (mx > cur) {
      const unsigned int v32 = (unsigned int)mx;
      RS_CUDA(cudaMemcpy(&t->dev->c.tick, &v32, 4, cudaMemcpyHostToDevice));
    }
  }
  RS_CUDA(cudaDeviceSynchronize());
  cudaFree(dk);
  cudaFree(de);
  cudaFree(drows);
  cudaFree(dm);
  cudaFree(dv);
  cudaFree(dstep);
  cudaFree(dts);
  return RS_OK;
}

}  // extern "C"
