// evict.cu -- device victim selection for bounded tables (config 3).
//
// Frozen semantics (no reference counterpart; oracle.c:or_table_ensure_batch
// / or_table_evict_oldest): evict the `need` live entries with the smallest
// (tick, key) among the entries a batch did not touch (tick < T), where
// need = occupied + missing - max_keys.  Done without any host round trip:
//
//   k_ev_plan        need, the capacity check, state reset (1 thread)
//   tick levels      k_ev_tick_hist (full scan, 4096-bin window over the
//                    ticks from the previous selection's min tick -- a lower
//                    bound, candidate ticks never decrease; the first level
//                    also finds this selection's min tick and key range;
//                    ticks, per-block smem histograms) + k_ev_tick_pick; the
//                    window narrows 4096x per level until one tick t* is
//                    left (usually after the first level: the live ticks of
//                    a stream span far fewer than 4096 batch ops)
//   key level 0      k_ev_key_hist over the candidates with tick t* (full
//                    scan, 12-bit digit) + pick, then k_ev_emit: every
//                    candidate below the threshold becomes a victim, the ones
//                    in the threshold bin are compacted into a small list
//   key levels 1..   k_ev_select_block: the same on the compacted list, in
//                    one block (the list is one 12-bit key bin: small)
//   k_ev_remove      tombstone the victim slots, rows to the free stack
//
// Keys equal to the two sentinels live in the descriptor; they are virtual
// candidate slots capacity + {0, 1}.
#include <cuda_runtime.h>

#include <algorithm>

#include "rs_host.hpp"
#include "table_dev.cuh"

namespace rs {
namespace {

using namespace tdev;

constexpr int kBins = 4096;
constexpr int kDigitBits = 12;

struct EvictState {
  unsigned long long need;  // victims still to choose
  unsigned int T;           // candidates: live entries with tick < T
  unsigned int active;
  unsigned int tmin;
  unsigned int lo, shift, t_star_found, t_star;
  unsigned int tick_lt;     // every candidate with tick < tick_lt is a victim
  unsigned int kshift;      // key digit level: digit = (key >> kshift) & 4095
  unsigned long long kprefix;  // candidates with tick t* and key >> (kshift + 12) == kprefix
  unsigned int kdigit_lt;   // level-0 emit: victims have digit < kdigit_lt
  unsigned int all_bin;     // every candidate of the chosen bin is a victim
  unsigned int n_cand[2], n_vict, cur;
  unsigned long long kmin, kmax;  // key range of the candidates: the first key digit starts at
  unsigned int kshift0;           // the highest bit where they differ
  unsigned int level;             // tick levels done in this selection
  unsigned int tmin_prev;         // min candidate tick of the previous selection (a lower
                                  // bound of this one's: candidate ticks never decrease)
  unsigned int hist[kBins];
};

struct Cand {
  __device__ __forceinline__ static bool live(const Slot& s) {
    return s.key != kEmptyKey && s.key != kTombKey;
  }
};

// Entry i of the candidate space: slot i, or one of the 2 sentinel keys.
__device__ __forceinline__ bool entry(const TableDev* td, uint64_t i, uint64_t cap, uint64_t* key,
                                      uint32_t* tick) {
  if (i < cap) {
    const Slot s = td->d.slots[i];
    *key = s.key;
    *tick = s.tick;
    return Cand::live(s);
  }
  const int sp = (int)(i - cap);
  if (td->c.special_row[sp] == kNoRow) return false;
  *key = sp == 0 ? kEmptyKey : kTombKey;
  *tick = td->c.special_tick[sp];
  return true;
}

__global__ void __launch_bounds__(256) k_ev_plan(TableDev* td, EvictState* st, const uint32_t* d_n,
                                                 uint64_t n_host, uint64_t max_keys, uint64_t explicit_k,
                                                 int use_prev) {
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) st->hist[b] = 0;
  if (threadIdx.x != 0) return;
  const TableCounters& c = td->c;
  unsigned long long need = 0;
  if (max_keys) {  // bounded ensure: after the probe, c.tick == the batch tick T
    const uint64_t n = d_n ? *d_n : n_host;
    const uint64_t missing = c.missing, found = n - missing;
    if (c.occupied + missing > max_keys) {
      need = c.occupied + missing - max_keys;
      if (need > c.occupied - found) {  // the batch alone exceeds the bound
        atomicOr(&td->c.error, kErrCapacity);
        need = 0;
      }
    }
    st->T = c.tick;
  } else {  // explicit evict of the k oldest live entries
    need = explicit_k < c.occupied ? explicit_k : c.occupied;
    st->T = c.tick + 1;
  }
  st->need = need;
  st->active = need > 0;
  st->tmin = 0xFFFFFFFFu;
  st->t_star_found = 0;
  st->n_cand[0] = st->n_cand[1] = 0;
  st->n_vict = 0;
  st->cur = 0;
  st->all_bin = 0;
  st->kmin = ~0ull;
  st->kmax = 0;
  st->level = 0;
  // tick window: from a lower bound of the candidates' ticks (no min scan)
  uint32_t lo = use_prev ? st->tmin_prev : 0u;
  if (lo > st->T - 1) lo = 0;
  const uint32_t span = st->T - 1 - lo;
  uint32_t shift = 0;
  while (((uint64_t)span >> shift) >= (uint64_t)kBins) shift += kDigitBits;
  st->lo = lo;
  st->shift = shift;
  st->tick_lt = lo;
}

// one window level over the ticks
__global__ void __launch_bounds__(256) k_ev_tick_hist(const TableDev* td, EvictState* st, uint64_t cap) {
  __shared__ uint32_t h[kBins];
  if (!st->active || st->t_star_found) return;
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const uint32_t T = st->T, lo = st->lo, shift = st->shift;
  const bool first = st->level == 0;  // first level: also the min tick and the key range
  uint32_t m = 0xFFFFFFFFu;
  unsigned long long kmn = ~0ull, kmx = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 2;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k;
    uint32_t t;
    if (!entry(td, i, cap, &k, &t) || t >= T || t < lo) continue;
    const uint64_t b = (uint64_t)(t - lo) >> shift;
    if (b < (uint64_t)kBins) atomicAdd(&h[b], 1u);
    m = min(m, t);
    kmn = min(kmn, (unsigned long long)k);
    kmx = max(kmx, (unsigned long long)k);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (h[b]) atomicAdd(&st->hist[b], h[b]);
  if (first) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
      kmn = min(kmn, __shfl_xor_sync(0xFFFFFFFFu, kmn, o));
      kmx = max(kmx, __shfl_xor_sync(0xFFFFFFFFu, kmx, o));
    }
    if ((threadIdx.x & 31) == 0 && m != 0xFFFFFFFFu) {
      atomicMin(&st->tmin, m);
      atomicMin(&st->kmin, kmn);
      atomicMax(&st->kmax, kmx);
    }
  }
}

// Choose the bin holding the need-th smallest; candidates in lower bins are
// victims.  One block of 1024 threads: block-wide scan of 4096 bins.
__device__ __forceinline__ uint32_t pick_bin(EvictState* st, unsigned long long need,
                                             unsigned long long* below) {
  __shared__ unsigned long long part[1024];
  __shared__ uint32_t s_bin;
  __shared__ unsigned long long s_below;
  const uint32_t t = threadIdx.x;
  unsigned long long loc = 0;
  for (int j = 0; j < 4; ++j) loc += st->hist[t * 4 + j];
  part[t] = loc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive scan
    const unsigned long long v = t >= (uint32_t)o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  if (t == 0) s_bin = kBins;
  __syncthreads();
  const unsigned long long before = part[t] - loc;
  if (before < need && need <= part[t]) {
    unsigned long long run = before;
    for (int j = 0; j < 4; ++j) {
      const uint32_t hb = st->hist[t * 4 + j];
      if (run + hb >= need) {
        s_bin = t * 4 + j;
        s_below = run;
        break;
      }
      run += hb;
    }
  }
  __syncthreads();
  *below = s_below;
  const uint32_t bin = s_bin;
  __syncthreads();
  for (int b = t; b < kBins; b += blockDim.x) st->hist[b] = 0;  // ready for the next level
  return bin;
}

__global__ void __launch_bounds__(1024) k_ev_tick_pick(EvictState* st) {
  if (!st->active || st->t_star_found) return;
  unsigned long long below = 0;
  const uint32_t bin = pick_bin(st, st->need, &below);
  if (threadIdx.x != 0) return;
  if (bin >= (uint32_t)kBins) {  // fewer candidates than need (cannot happen after the plan)
    st->active = 0;
    return;
  }
  if (st->level++ == 0) {  // after the first (full) level: key range, next call's window base
    const unsigned long long x = st->kmin ^ st->kmax;
    const uint32_t nbits = x ? 64 - __clzll(x) : 0;
    st->kshift0 = nbits > (uint32_t)kDigitBits ? nbits - kDigitBits : 0;
    st->tmin_prev = st->tmin;
  }
  st->need -= below;
  st->lo = st->lo + (bin << st->shift);
  st->tick_lt = st->lo;  // everything older than the chosen bin is a victim
  if (st->shift == 0) {
    st->t_star = st->lo;
    st->t_star_found = 1;
    st->kshift = st->kshift0;  // bits above it are common to every candidate
    st->kprefix = 0;
  } else {
    st->shift = st->shift >= (uint32_t)kDigitBits ? st->shift - kDigitBits : 0;
  }
}

__device__ __forceinline__ uint32_t key_digit(uint64_t k, uint32_t kshift) {
  return (uint32_t)(k >> kshift) & (kBins - 1);
}

// key level 0: histogram of the top digit among the candidates with tick t*
__global__ void __launch_bounds__(256) k_ev_key_hist(const TableDev* td, EvictState* st, uint64_t cap) {
  __shared__ uint32_t h[kBins];
  if (!st->active) return;
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const uint32_t ts = st->t_star, ks = st->kshift;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 2;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k;
    uint32_t t;
    if (entry(td, i, cap, &k, &t) && t == ts) atomicAdd(&h[key_digit(k, ks)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (h[b]) atomicAdd(&st->hist[b], h[b]);
}

__global__ void __launch_bounds__(1024) k_ev_key_pick(EvictState* st) {
  if (!st->active) return;
  unsigned long long below = 0;
  const uint32_t bin = pick_bin(st, st->need, &below);
  if (threadIdx.x != 0) return;
  if (bin >= (uint32_t)kBins) {
    st->active = 0;
    return;
  }
  st->need -= below;
  st->kdigit_lt = bin;
}

// level-0 emit (full scan): victims = older ticks, or tick t* with a smaller
// top digit; the threshold bin's entries go to the candidate list
__global__ void __launch_bounds__(256) k_ev_emit0(const TableDev* td, EvictState* st, uint64_t cap,
                                                  uint32_t* victims, uint32_t* cand) {
  if (!st->active) return;
  const uint32_t T = st->T, lt = st->tick_lt, ts = st->t_star, ks = st->kshift, kd = st->kdigit_lt;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 2;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k;
    uint32_t t;
    bool v = false, c = false;
    if (entry(td, i, cap, &k, &t) && t < T) {
      if (t < lt) {
        v = true;
      } else if (t == ts) {
        const uint32_t d = key_digit(k, ks);
        v = d < kd;
        c = d == kd;
      }
    }
    const unsigned vm = __ballot_sync(0xFFFFFFFFu, v), cm = __ballot_sync(0xFFFFFFFFu, c);
    const unsigned lane = threadIdx.x & 31, lt_mask = (1u << lane) - 1;
    uint32_t vb = 0, cb = 0;
    if (lane == 0 && vm) vb = atomicAdd(&st->n_vict, __popc(vm));
    if (lane == 0 && cm) cb = atomicAdd(&st->n_cand[0], __popc(cm));
    vb = __shfl_sync(0xFFFFFFFFu, vb, 0);
    cb = __shfl_sync(0xFFFFFFFFu, cb, 0);
    if (v) victims[vb + __popc(vm & lt_mask)] = (uint32_t)i;
    if (c) cand[cb + __popc(cm & lt_mask)] = (uint32_t)i;
  }
}

// Key levels 1.. on the compacted candidate list (all tick t*), in ONE
// block: the list after level 0 holds one 12-bit key bin, so it is small in
// practice; each level histograms the next digit in smem, picks the bin of
// the need-th smallest, emits the keys below it and compacts the bin.
__global__ void __launch_bounds__(1024) k_ev_select_block(const TableDev* td, EvictState* st, uint32_t* cand0,
                                                          uint32_t* cand1, uint32_t* victims, uint64_t cap) {
  __shared__ uint32_t h[kBins];
  __shared__ unsigned long long part[1024];
  __shared__ uint32_t s_bin, s_nv, s_nc;
  __shared__ unsigned long long s_below;
  if (!st->active) return;
  const uint32_t tid = threadIdx.x;
  uint32_t* cand[2] = {cand0, cand1};
  for (int level = 0; level < 8; ++level) {
    const int cur = (int)st->cur;
    const uint32_t n = st->n_cand[cur];
    const unsigned long long need = st->need;
    __syncthreads();
    if (need == 0) break;
    if (need >= n) {  // the whole list goes (keys are distinct, so need == n)
      const uint32_t base = st->n_vict;
      for (uint32_t i = tid; i < n; i += blockDim.x) victims[base + i] = cand[cur][i];
      __syncthreads();
      if (tid == 0) {
        st->n_vict = base + n;
        st->need = 0;
      }
      break;
    }
    const uint32_t ks = st->kshift >= (uint32_t)kDigitBits ? st->kshift - kDigitBits : 0u;
    for (int b = tid; b < kBins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += blockDim.x) {
      uint64_t k;
      uint32_t t;
      entry(td, cand[cur][i], cap, &k, &t);
      atomicAdd(&h[key_digit(k, ks)], 1u);
    }
    __syncthreads();
    // pick the bin holding the need-th smallest
    unsigned long long loc = 0;
    for (int j = 0; j < 4; ++j) loc += h[tid * 4 + j];
    part[tid] = loc;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const unsigned long long v = tid >= (uint32_t)o ? part[tid - o] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    if (tid == 0) {
      s_bin = kBins;
      s_nv = 0;
      s_nc = 0;
    }
    __syncthreads();
    const unsigned long long before = part[tid] - loc;
    if (before < need && need <= part[tid]) {
      unsigned long long run = before;
      for (int j = 0; j < 4; ++j) {
        if (run + h[tid * 4 + j] >= need) {
          s_bin = tid * 4 + j;
          s_below = run;
          break;
        }
        run += h[tid * 4 + j];
      }
    }
    __syncthreads();
    const uint32_t bin = s_bin;
    if (bin >= (uint32_t)kBins) break;  // cannot happen: need <= n
    const uint32_t vbase = st->n_vict;
    for (uint32_t i = tid; i < n; i += blockDim.x) {
      const uint32_t idx = cand[cur][i];
      uint64_t k;
      uint32_t t;
      entry(td, idx, cap, &k, &t);
      const uint32_t d = key_digit(k, ks);
      if (d < bin) victims[vbase + atomicAdd(&s_nv, 1u)] = idx;
      else if (d == bin) cand[cur ^ 1][atomicAdd(&s_nc, 1u)] = idx;
    }
    __syncthreads();
    if (tid == 0) {
      st->n_vict = vbase + s_nv;
      st->need = need - s_below;
      st->n_cand[cur ^ 1] = s_nc;
      st->cur = cur ^ 1;
      st->kshift = ks;
    }
    __syncthreads();
    if (ks == 0 && st->need > 0) {  // every bit fixed: the remaining candidate is the victim
      const int c2 = cur ^ 1;
      const uint32_t n2 = st->n_cand[c2];
      const uint32_t base = st->n_vict;
      for (uint32_t i = tid; i < n2 && i < st->need; i += blockDim.x) victims[base + i] = cand[c2][i];
      __syncthreads();
      if (tid == 0) {
        const uint32_t take = (uint32_t)min((unsigned long long)n2, st->need);
        st->n_vict = base + take;
        st->need -= take;
      }
      break;
    }
  }
  __syncthreads();
  if (tid == 0) st->active = 0;
}

// Tombstone the victims; their rows go to the free stack.  rewind: set the
// tick to T - 1 so the insert that follows stamps the batch tick T.
__global__ void __launch_bounds__(256) k_ev_remove(TableDev* td, EvictState* st, const uint32_t* victims,
                                                   uint64_t cap, int rewind) {
  const unsigned long long free_n0 = td->c.free_n;
  const unsigned long long fresh0 = td->c.fresh_next;
  const uint32_t nv = st->n_vict;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const uint32_t idx = victims[i];
    uint32_t row;
    if (idx < cap) {
      Slot* s = td->d.slots + idx;
      row = s->row;
      s->key = kTombKey;
      s->row = kNoRow;
    } else {  // sentinel keys leave no tombstone
      row = atomicExch(&td->c.special_row[idx - cap], kNoRow);
      atomicAdd(&td->c.tombstones, ~0ull);
    }
    const unsigned long long k = atomicAdd(&td->c.removed, 1ull);
    td->d.free_stack[free_n0 + k] = row;
  }
  const uint32_t T = st->T;
  launch_epilogue(td, free_n0, fresh0, false, 0);
  if (rewind && blockIdx.x == 0 && threadIdx.x == 0) td->c.tick = T - 1;
}

}  // namespace

// Enqueue the device victim selection + removal (no host synchronization).
// Bounded ensure: max_keys > 0, n / d_n the batch's unique count (the probe
// already ran and stamped tick T).  Explicit evict: max_keys == 0, k given.
int evict_prepare(rs_table* t, uint64_t max_victims) {
  const uint64_t cap = t->capacity;
  if (!t->d_evict) {
    RS_CUDA(cudaMalloc(&t->d_evict, sizeof(EvictState)));
    RS_CUDA(cudaMemset(t->d_evict, 0, sizeof(EvictState)));
    t->evict_tmin_valid = false;
  }
  // candidate lists hold at most the entries of one key-digit bin; the worst
  // case is every live entry
  const uint64_t cand_need = cap + 2;
  const uint64_t vict_need = std::max<uint64_t>(max_victims + 2, cand_need);
  if (t->evict_cap < cand_need || t->victim_idx_cap < vict_need) {
    if (t->d_cand) RS_CUDA(cudaFree(t->d_cand));
    if (t->d_victim_idx) RS_CUDA(cudaFree(t->d_victim_idx));
    t->d_cand = nullptr;
    t->d_victim_idx = nullptr;
    RS_CUDA(cudaMalloc(&t->d_cand, 2 * cand_need * 4));
    RS_CUDA(cudaMalloc(&t->d_victim_idx, vict_need * 4));
    t->evict_cap = cand_need;
    t->victim_idx_cap = vict_need;
    t->buf_gen++;
  }
  return RS_OK;
}

// Enqueue only (graph-capturable once evict_prepare ran for this capacity).
int evict_device(rs_table* t, const uint32_t* d_n, uint64_t n_host, uint64_t explicit_k,
                 cudaStream_t s) {
  const uint64_t cap = t->capacity;
  const uint64_t bound = t->cfg.max_keys && !explicit_k ? t->cfg.max_keys : 0;
  const uint64_t max_vict = bound ? std::min<uint64_t>(n_host, cap) + 2 : explicit_k + 2;
  if (!t->d_evict || t->evict_cap < cap + 2 || t->victim_idx_cap < max_vict)
    return fail(RS_ERR_INVARIANT, "evict_device: buffers not prepared");
  const uint64_t cand_need = t->evict_cap;
  EvictState* st = reinterpret_cast<EvictState*>(t->d_evict);
  uint32_t* cand[2] = {t->d_cand, t->d_cand + cand_need};
  const unsigned scan = grid_for(cap + 2, 256, 148 * 8);
  k_ev_plan<<<1, 256, 0, s>>>(t->dev, st, d_n, n_host, bound, explicit_k, t->evict_tmin_valid ? 1 : 0);
  RS_LAUNCH_CHECK("k_ev_plan");
  t->evict_tmin_valid = true;  // from now on the window starts at the last selection's min tick
  for (int lvl = 0; lvl < 3; ++lvl) {  // 32-bit ticks: at most 3 windows of 12 bits
    k_ev_tick_hist<<<scan, 256, 0, s>>>(t->dev, st, cap);
    RS_LAUNCH_CHECK("k_ev_tick_hist");
    k_ev_tick_pick<<<1, 1024, 0, s>>>(st);
    RS_LAUNCH_CHECK("k_ev_tick_pick");
  }
  k_ev_key_hist<<<scan, 256, 0, s>>>(t->dev, st, cap);
  RS_LAUNCH_CHECK("k_ev_key_hist");
  k_ev_key_pick<<<1, 1024, 0, s>>>(st);
  RS_LAUNCH_CHECK("k_ev_key_pick");
  k_ev_emit0<<<scan, 256, 0, s>>>(t->dev, st, cap, t->d_victim_idx, cand[0]);
  RS_LAUNCH_CHECK("k_ev_emit0");
  k_ev_select_block<<<1, 1024, 0, s>>>(t->dev, st, cand[0], cand[1], t->d_victim_idx, cap);
  RS_LAUNCH_CHECK("k_ev_select_block");
  k_ev_remove<<<grid_for(max_vict, 256, 148 * 4), 256, 0, s>>>(t->dev, st, t->d_victim_idx, cap,
                                                              bound ? 1 : 0);
  RS_LAUNCH_CHECK("k_ev_remove");
  return RS_OK;
}

int evict_count(rs_table* t, uint64_t* out, cudaStream_t s) {
  unsigned int h = 0;
  RS_CUDA(cudaMemcpyAsync(&h, &reinterpret_cast<EvictState*>(t->d_evict)->n_vict, 4,
                          cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaStreamSynchronize(s));
  if (out) *out = h;
  return RS_OK;
}

}  // namespace rs
