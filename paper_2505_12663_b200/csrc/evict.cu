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

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>

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
  // stamp-log selection (k_lg_*): 1 = the log chose this op's victims
  unsigned int lg_mode, lg_sorted, lg_attempt;
  unsigned long long lg_p0, lg_p1, lg_need2, lg_head;
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
  st->lg_mode = 0;
  st->lg_attempt = 0;
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
  if (!st->active || st->lg_mode) return;
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
  if (!st->active || st->lg_mode) return;
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
  if (!st->active || st->lg_mode) return;
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

// ---- stamp-log selection (bounded tables) -----------------------------------
// The log (rs_internal.cuh LogRec) lists, per batch op in tick order, the
// entries that op stamped.  A record is live while its slot still holds
// that key with that tick; the live records are exactly the live entries,
// in tick order.  The victims -- the `need` smallest (tick, key) with tick <
// T -- are then: every live record before the tick group t* holding the
// need-th live record, plus the need2 smallest keys of group t* (the first
// need2 live records when the group lies in the rebuilt, (tick, key)-sorted
// region; else the compacted group goes to k_ev_select_block).  Reads a
// window of W records from the head instead of the table's slots; when the
// window cannot decide (t*'s group cut by the window end), the full-scan
// selection above runs instead.
constexpr uint32_t kLgPer = 4;                  // records per thread
constexpr uint32_t kLgBlock = 256 * kLgPer;     // records per block

__device__ __forceinline__ bool lg_live(const TableDev* td, const LogRec& r, uint64_t cap, uint32_t T) {
  if (r.slot == kNoLogSlot || r.tick >= T) return false;
  if (r.slot < cap) {
    const Slot sl = td->d.slots[r.slot];
    return sl.key == r.key && sl.tick == r.tick;
  }
  const int sp = (int)(r.slot - cap);
  return sp < 2 && td->c.special_row[sp] != kNoRow && td->c.special_tick[sp] == r.tick;
}

__device__ __forceinline__ unsigned long long lg_end(const LogArgs& lg, uint64_t W) {
  const unsigned long long h = lg.ctl->head, t = lg.ctl->tail;
  return min(h + W, t);
}

// live records per block of the window
__global__ void __launch_bounds__(256) k_lg_count(const TableDev* td, EvictState* st, LogArgs lg, uint64_t W,
                                                  uint32_t* cnt, uint32_t nb) {
  if (!st->active || st->lg_mode) return;  // (nothing to evict / an earlier window decided)
  const unsigned long long head = lg.ctl->head, end = lg_end(lg, W);
  const uint32_t T = st->T;
  __shared__ uint32_t ws[8];
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {  // chunk b: records head + [1024 b, 1024 b + 1024)
    const unsigned long long b0 = head + (unsigned long long)b * kLgBlock;
    uint32_t c = 0;
    if (b0 < end) {
#pragma unroll
      for (uint32_t j = 0; j < kLgPer; ++j) {
        const unsigned long long pos = b0 + threadIdx.x + j * 256;
        if (pos < end && lg_live(td, lg.rec[pos & lg.mask], lg.cap, T)) ++c;
      }
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < 8; ++w) tot += ws[w];
      cnt[b] = tot;
    }
    __syncthreads();
  }
}

// first position in [lo, hi) whose tick is > t (strict) or >= t: ticks are
// non-decreasing along the log.  One block: a strided sample, then the segment.
__device__ unsigned long long lg_bound(const LogArgs& lg, unsigned long long lo, unsigned long long hi, uint32_t t,
                                       bool strict) {
  __shared__ unsigned long long s_first;
  const uint32_t tid = threadIdx.x;
  auto after = [&](unsigned long long pos) {
    const uint32_t tk = lg.rec[pos & lg.mask].tick;
    return strict ? tk > t : tk >= t;
  };
  if (tid == 0) s_first = hi;
  __syncthreads();
  const unsigned long long n = hi - lo;
  const unsigned long long stride = (n + blockDim.x - 1) / blockDim.x;
  // sample k: position lo + k * stride; the first sample past t bounds the answer
  if (stride > 0) {
    const unsigned long long pos = lo + (unsigned long long)tid * stride;
    if (pos < hi && after(pos)) atomicMin(&s_first, pos);
  }
  __syncthreads();
  const unsigned long long s1 = s_first;
  const unsigned long long s0 = s1 >= lo + stride ? s1 - stride : lo;
  __syncthreads();
  if (tid == 0) s_first = s1;
  __syncthreads();
  for (unsigned long long pos = s0 + tid; pos < s1; pos += blockDim.x)
    if (after(pos)) atomicMin(&s_first, pos);
  __syncthreads();
  const unsigned long long r = s_first;
  __syncthreads();  // every thread read it before a next call resets it
  return r;
}

__global__ void __launch_bounds__(1024) k_lg_pick(const TableDev* td, EvictState* st, LogArgs lg, uint64_t W,
                                                  const uint32_t* cnt, long long* pre, uint32_t nb, int attempt) {
  __shared__ unsigned long long part[1024];
  __shared__ unsigned long long s_pos, s_before;
  __shared__ uint32_t s_blk;
  if (!st->active || st->lg_mode) return;
  const uint32_t tid = threadIdx.x;
  const unsigned long long need = st->need;
  const unsigned long long head = lg.ctl->head, tail = lg.ctl->tail, end = lg_end(lg, W);
  const uint32_t T = st->T;
  // the block holding the need-th live record (prefix over the block counts)
  const uint32_t per = (nb + 1023) / 1024;
  unsigned long long loc = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t b = tid * per + j;
    if (b < nb) loc += cnt[b];
  }
  part[tid] = loc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned long long v = tid >= (uint32_t)o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  if (tid == 0) s_blk = 0xFFFFFFFFu;
  __syncthreads();
  {
    unsigned long long run = part[tid] - loc;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t b = tid * per + j;
      if (b >= nb) break;
      if (run < need && need <= run + cnt[b]) {
        s_blk = b;
        s_before = run;
      }
      run += cnt[b];
    }
  }
  __syncthreads();
  if (s_blk == 0xFFFFFFFFu) return;  // fewer live records in the window than need: full scan
  // the need-th live record inside that block: its tick is t*
  const unsigned long long b0 = head + (unsigned long long)s_blk * kLgBlock;
  {
    if (tid == 0) s_pos = ~0ull;
    __syncthreads();
    const unsigned long long pos = b0 + tid;
    const bool v = tid < kLgBlock && pos < end && lg_live(td, lg.rec[pos & lg.mask], lg.cap, T);
    // in-order rank of each live record of the block
    const unsigned m = __ballot_sync(0xFFFFFFFFu, v);
    __shared__ uint32_t wsum[32];
    if ((tid & 31) == 0) wsum[tid >> 5] = __popc(m);
    __syncthreads();
    uint32_t wb = 0;
    for (uint32_t w = 0; w < (tid >> 5); ++w) wb += wsum[w];
    const uint32_t rank = wb + __popc(m & ((1u << (tid & 31)) - 1));
    if (v && s_before + rank + 1 == need) s_pos = pos;
    __syncthreads();
  }
  const unsigned long long q = s_pos;
  if (q == ~0ull) return;  // (cannot happen)
  if (q < lg.ctl->sorted_end) {
    // [head, q] lies in the rebuilt, globally (tick, key)-sorted region: the
    // victims are exactly its live records (q is the need-th) -- no group bounds
    const uint32_t per2 = (nb + 1023) / 1024;
    unsigned long long loc2 = 0;
    for (uint32_t j = 0; j < per2; ++j) {
      const uint32_t b = tid * per2 + j;
      if (b < nb) loc2 += cnt[b];
    }
    part[tid] = loc2;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const unsigned long long v = tid >= (uint32_t)o ? part[tid - o] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    long long run = (long long)(part[tid] - loc2);
    for (uint32_t j = 0; j < per2; ++j) {
      const uint32_t b = tid * per2 + j;
      if (b >= nb) break;
      pre[b] = run;
      run += cnt[b];
    }
    if (tid == 0) {
      st->lg_p0 = head;  // rank from the head: the first `need` live records
      st->lg_p1 = q + 1;
      st->lg_need2 = need;
      st->lg_sorted = 1;
      st->lg_mode = 1;
      st->lg_attempt = (uint32_t)attempt;
      st->t_star_found = 1;
      st->active = 0;
      st->lg_head = head;
      lg.ctl->head = q + 1;
    }
    return;
  }
  const uint32_t ts = lg.rec[q & lg.mask].tick;
  const unsigned long long p0 = lg_bound(lg, head, q + 1, ts, false);
  const unsigned long long p1 = lg_bound(lg, q, end, ts, true);
  const bool sorted = p0 < lg.ctl->sorted_end;
  if (!sorted && p1 == end && end < tail) return;  // the group runs past the window: full scan
  // live records before p0 (all victims): whole blocks + the part of p0's block
  const uint32_t bp = (uint32_t)((p0 - head) / kLgBlock);
  unsigned long long before = 0;
  for (uint32_t b = tid; b < bp; b += blockDim.x) before += cnt[b];
  {
    const unsigned long long pb = head + (unsigned long long)bp * kLgBlock;
    const unsigned long long pos = pb + tid;
    if (tid < kLgBlock && pos < p0 && lg_live(td, lg.rec[pos & lg.mask], lg.cap, T)) before += 1;
  }
  part[tid] = before;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < (uint32_t)o) part[tid] += part[tid + o];
    __syncthreads();
  }
  const unsigned long long vb = part[0];
  // per block: live records of group t* before the block's first record (sorted groups rank by it)
  __syncthreads();  // (part[] is reused below)
  {  // pre[b] = live records in [p0, block b) -- (p0's own block starts its group at rank 0)
    unsigned long long loc2 = 0;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t b = tid * per + j;
      if (b < nb) loc2 += cnt[b];
    }
    part[tid] = loc2;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const unsigned long long v = tid >= (uint32_t)o ? part[tid - o] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    long long run = (long long)(part[tid] - loc2) - (long long)vb;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t b = tid * per + j;
      if (b >= nb) break;
      pre[b] = run < 0 ? 0 : run;
      run += cnt[b];
    }
  }
  if (tid == 0) {
    st->lg_p0 = p0;
    st->lg_p1 = p1;
    st->lg_need2 = need - vb;
    st->lg_sorted = sorted ? 1u : 0u;
    st->lg_mode = 1;
    st->lg_attempt = (uint32_t)attempt;
    st->t_star_found = 1;  // the tick levels of the scan path stand down
    // the candidates of an unsorted group go to k_ev_select_block
    st->n_cand[0] = 0;
    st->cur = 0;
    st->need = need - vb;
    st->kshift = 64;
    if (sorted) st->active = 0;
    st->lg_head = head;
    // every live record before p0 is a victim now; in a sorted group so is
    // every live record up to q (the need-th): the next window starts after it
    lg.ctl->head = sorted ? q + 1 : p0;
  }
}

// victims: the live records before p0, and in group t* the first need2 (sorted
// group) or every live one to the candidate list (unsorted group)
__global__ void __launch_bounds__(256) k_lg_emit(const TableDev* td, EvictState* st, LogArgs lg,
                                                 const long long* pre, uint32_t* victims, uint32_t* cand,
                                                 uint32_t nb, int attempt) {
  if (st->lg_mode != 1 || st->lg_attempt != (uint32_t)attempt) return;  // (this window did not decide)
  const unsigned long long head = st->lg_head, p0 = st->lg_p0, p1 = st->lg_p1;
  const unsigned long long need2 = st->lg_need2;
  const bool sorted = st->lg_sorted != 0;
  const uint32_t T = st->T;
  for (uint32_t chunk = blockIdx.x; chunk < nb; chunk += gridDim.x) {
  const unsigned long long b0 = head + (unsigned long long)chunk * kLgBlock;
  if (b0 >= p1) break;  // (block-uniform)
  // thread t owns records b0 + 4t .. b0 + 4t + 3 (contiguous: in-order ranks)
  bool v[kLgPer], g[kLgPer];
  uint32_t slot[kLgPer];
  uint32_t ng = 0;
#pragma unroll
  for (uint32_t j = 0; j < kLgPer; ++j) {
    const unsigned long long pos = b0 + threadIdx.x * kLgPer + j;
    v[j] = g[j] = false;
    slot[j] = 0;
    if (pos < p1) {
      const LogRec r = lg.rec[pos & lg.mask];
      if (lg_live(td, r, lg.cap, T)) {
        slot[j] = r.slot;
        if (pos < p0) v[j] = true;
        else g[j] = true;
      }
    }
    ng += g[j];
  }
  // in-order rank of this thread's group-t* records within the block
  __shared__ uint32_t wsum[8];
  uint32_t x = ng;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  uint32_t wb = 0;
  for (uint32_t w = 0; w < warp; ++w) wb += wsum[w];
  long long rank = pre[chunk] + wb + x - ng;  // group-t* records before this thread's first
  uint32_t nv = 0, nc = 0;
#pragma unroll
  for (uint32_t j = 0; j < kLgPer; ++j) {
    if (g[j]) {
      if (sorted) {
        if (rank >= 0 && (unsigned long long)rank < need2) v[j] = true;
        g[j] = false;
      }
      ++rank;
    }
    nv += v[j];
    nc += g[j];
  }
  // block-aggregated appends
  __shared__ uint32_t s_nv, s_nc, s_vb, s_cb;
  if (threadIdx.x == 0) {
    s_nv = 0;
    s_nc = 0;
  }
  __syncthreads();
  const uint32_t ov = nv ? atomicAdd(&s_nv, nv) : 0u;
  const uint32_t oc = nc ? atomicAdd(&s_nc, nc) : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_vb = s_nv ? atomicAdd(&st->n_vict, s_nv) : 0u;
    s_cb = s_nc ? atomicAdd(&st->n_cand[0], s_nc) : 0u;
  }
  __syncthreads();
  uint32_t iv = s_vb + ov, ic = s_cb + oc;
#pragma unroll
  for (uint32_t j = 0; j < kLgPer; ++j) {
    if (v[j]) victims[iv++] = slot[j];
    if (g[j]) cand[ic++] = slot[j];
  }
  __syncthreads();  // (wsum / s_* of the next chunk)
  }
}
__global__ void k_lg_dbg(const EvictState* st, LogArgs lg) {
  printf("evict: T %u need %llu lg_mode %u sorted %u p0 %llu p1 %llu need2 %llu head %llu->%llu tail %llu sorted_end %llu n_vict %u n_cand %u active %u\n",
         st->T, st->need, st->lg_mode, st->lg_sorted, st->lg_p0, st->lg_p1, st->lg_need2, st->lg_head, lg.ctl->head,
         lg.ctl->tail, lg.ctl->sorted_end, st->n_vict, st->n_cand[0], st->active);
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

// ---- log rebuild: every live entry, sorted by (tick, key) ------------------
__global__ void __launch_bounds__(256) k_lg_collect(const TableDev* td, uint64_t cap, unsigned long long* keys,
                                                    uint32_t* slots, uint32_t* ticks, uint32_t* n_out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 2;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = 0;
    uint32_t t = 0;
    const bool v = entry(td, i, cap, &k, &t);
    const unsigned m = __ballot_sync(0xFFFFFFFFu, v);
    uint32_t b = 0;
    if ((threadIdx.x & 31) == 0 && m) b = atomicAdd(n_out, __popc(m));
    b = __shfl_sync(0xFFFFFFFFu, b, 0);
    if (v) {
      const uint32_t j = b + __popc(m & ((1u << (threadIdx.x & 31)) - 1));
      keys[j] = k;
      slots[j] = (uint32_t)i;
      ticks[j] = t;
    }
  }
}
__global__ void k_lg_iota(uint32_t* x, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = i;
}
__global__ void k_lg_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t* dst, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[idx[i]];
}
__global__ void k_lg_write(LogRec* rec, const unsigned long long* keys1, const uint32_t* p1, const uint32_t* slots,
                           const uint32_t* ticks2, const uint32_t* perm2, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t q = perm2[i];
    rec[i] = LogRec{keys1[q], slots[p1[q]], ticks2[i]};
  }
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

static uint64_t lg_window(const rs_table* t, uint64_t n_max);

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
  const LogArgs lg = log_args(t, 0);
  const bool use_log = lg.rec && t->lg_nb;
  if (use_log) {
    // the stamp log: a window sized by this op's batch first, then (when it
    // could not decide: t*'s group cut by the window end) the whole log --
    // which always decides, so the slot-scan path is not launched
    const uint64_t W1 = std::min<uint64_t>(lg_window(t, bound ? n_host : explicit_k), t->log_cap);
    const uint64_t Ws[2] = {W1, t->log_cap};
    for (int a = 0; a < 2; ++a) {
      const uint32_t nb = (uint32_t)((Ws[a] + kLgBlock - 1) / kLgBlock);
      if (nb > t->lg_nb) return fail(RS_ERR_INVARIANT, "evict_device: log window buffers not prepared");
      const unsigned g = std::min<unsigned>(nb, 148u * 8u);
      k_lg_count<<<g, 256, 0, s>>>(t->dev, st, lg, Ws[a], t->d_lg_cnt, nb);
      RS_LAUNCH_CHECK("k_lg_count");
      k_lg_pick<<<1, 1024, 0, s>>>(t->dev, st, lg, Ws[a], t->d_lg_cnt, t->d_lg_pre, nb, a);
      RS_LAUNCH_CHECK("k_lg_pick");
      k_lg_emit<<<g, 256, 0, s>>>(t->dev, st, lg, t->d_lg_pre, t->d_victim_idx, cand[0], nb, a);
      RS_LAUNCH_CHECK("k_lg_emit");
    }
    static const bool dbg = getenv("RS_LOG_DBG") != nullptr;
    if (dbg) k_lg_dbg<<<1, 1, 0, s>>>(st, lg);
    // an unsorted group's candidates: the key select
    k_ev_select_block<<<1, 1024, 0, s>>>(t->dev, st, cand[0], cand[1], t->d_victim_idx, cap);
    RS_LAUNCH_CHECK("k_ev_select_block");
    k_ev_remove<<<grid_for(max_vict, 256, 148), 256, 0, s>>>(t->dev, st, t->d_victim_idx, cap,
                                                            bound ? 1 : 0);
    RS_LAUNCH_CHECK("k_ev_remove");
    return RS_OK;
  }
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

// ---- the stamp log, host side ------------------------------------------------
static uint64_t lg_window(const rs_table* t, uint64_t n_max) {
  uint64_t w = std::max<uint64_t>(n_max, 1ull << 16);
  w = (w + kLgBlock - 1) / kLgBlock * kLgBlock;
  return std::min<uint64_t>(w, t->log_cap);
}

// (after any op the stamp log cannot follow)
void log_invalidate(rs_table* t) {
  if (t->log_valid) t->buf_gen++;
  t->log_valid = false;
}

LogArgs log_args(rs_table* t, int probe) {
  LogArgs a;
  if (!t->cfg.max_keys || !t->log_valid) return a;
  a.rec = t->d_log;
  a.ctl = t->d_log_ctl;
  a.mask = t->log_cap - 1;
  a.cap = t->capacity;
  a.probe = probe;
  return a;
}

// Every live entry into the log, (tick, key)-sorted (host-synchronized; after
// an op the log cannot follow -- rehash, import, stamping lookups -- or when
// the ring is full of stale records).
static int log_rebuild(rs_table* t, cudaStream_t s) {
  const uint64_t cap = t->capacity;
  const uint64_t nmax = cap + 2;
  unsigned long long *keys = nullptr, *keys1 = nullptr;
  uint32_t *slots = nullptr, *ticks = nullptr, *idx = nullptr, *p1 = nullptr, *ticks1 = nullptr,
           *ticks2 = nullptr, *perm2 = nullptr, *d_n = nullptr;
  void* tmp = nullptr;
  auto A = [&](auto** p, size_t b) { return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(b, 16)) == cudaSuccess; };
  bool ok = A(&keys, nmax * 8) && A(&keys1, nmax * 8) && A(&slots, nmax * 4) && A(&ticks, nmax * 4) &&
            A(&idx, nmax * 4) && A(&p1, nmax * 4) && A(&ticks1, nmax * 4) && A(&ticks2, nmax * 4) &&
            A(&perm2, nmax * 4) && A(&d_n, 4);
  int st = RS_OK;
  uint32_t n = 0;
  size_t tb1 = 0, tb2 = 0;
  if (!ok) {
    st = cuda_fail(cudaGetLastError(), "log rebuild: cudaMalloc");
    goto done;
  }
  RS_CUDA(cudaMemsetAsync(d_n, 0, 4, s));
  k_lg_collect<<<grid_for(nmax, 256, 148 * 8), 256, 0, s>>>(t->dev, cap, keys, slots, ticks, d_n);
  RS_LAUNCH_CHECK("k_lg_collect");
  RS_CUDA(cudaMemcpyAsync(&n, d_n, 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaStreamSynchronize(s));
  t->host_syncs++;
  if (n > t->log_cap) {
    st = fail(RS_ERR_INVARIANT, "log rebuild: more live entries than log records");
    goto done;
  }
  if (n) {
    k_lg_iota<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(idx, n);
    k_lg_iota<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(perm2, n);
    cub::DeviceRadixSort::SortPairs(nullptr, tb1, keys, keys1, idx, p1, (int)n, 0, 64, s);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, ticks1, ticks2, perm2, idx, (int)n, 0, 32, s);
    if (cudaMalloc(&tmp, std::max(tb1, tb2)) != cudaSuccess) {
      st = cuda_fail(cudaGetLastError(), "log rebuild: cudaMalloc");
      goto done;
    }
    // by key, then stably by tick: (tick, key) order
    RS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb1, keys, keys1, idx, p1, (int)n, 0, 64, s));
    k_lg_gather_u32<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(ticks, p1, ticks1, n);
    RS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb2, ticks1, ticks2, perm2, idx, (int)n, 0, 32, s));
    k_lg_write<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(t->d_log, keys1, p1, slots, ticks2, idx, n);
    RS_LAUNCH_CHECK("k_lg_write");
  }
  {
    const LogCtl c{n, 0ull, 0ull, n};
    RS_CUDA(cudaMemcpyAsync(t->d_log_ctl, &c, sizeof(c), cudaMemcpyHostToDevice, s));
  }
  RS_CUDA(cudaStreamSynchronize(s));
  t->log_valid = true;
  t->log_tail_ub = n;
  t->log_head_lb = 0;
  t->log_rebuilds++;
  t->buf_gen++;  // graphs captured without (or with a stale) log
done:
  cudaFree(tmp);
  void* ps[] = {keys, keys1, slots, ticks, idx, p1, ticks1, ticks2, perm2, d_n};
  for (void* p : ps) cudaFree(p);
  return st;
}

int log_prepare(rs_table* t, uint64_t n_max, cudaStream_t s) {
  if (!t->cfg.max_keys) return RS_OK;
  static const bool off = getenv("RS_EVICT_LOG") && getenv("RS_EVICT_LOG")[0] == '0';
  if (off) {
    if (t->log_valid) t->buf_gen++;
    t->log_valid = false;
    return RS_OK;
  }
  const uint64_t need_cap = t->cfg.max_keys + 2 + 2 * n_max;
  if (t->log_cap < need_cap) {  // (re)allocate: 4 x the bound of live records + batch room
    uint64_t c = 1;
    while (c < 4 * t->cfg.max_keys + 8 * n_max) c <<= 1;
    RS_CUDA(cudaStreamSynchronize(s));
    if (t->d_log) cudaFree(t->d_log);
    t->d_log = nullptr;
    if (!t->d_log_ctl) RS_CUDA(cudaMalloc(&t->d_log_ctl, sizeof(LogCtl)));
    RS_CUDA(cudaMalloc(&t->d_log, c * sizeof(LogRec)));
    t->log_cap = c;
    if (t->log_valid) t->buf_gen++;
    t->log_valid = false;
  }
  if (t->log_valid && t->log_tail_ub + n_max > t->log_head_lb + t->log_cap) {
    LogCtl c;  // refresh the head bound (one read); a ring still this full compacts
    RS_CUDA(cudaMemcpyAsync(&c, t->d_log_ctl, sizeof(c), cudaMemcpyDeviceToHost, s));
    RS_CUDA(cudaStreamSynchronize(s));
    t->host_syncs++;
    t->log_head_lb = c.head;
    t->log_tail_ub = c.tail;
    if (t->log_tail_ub + n_max > t->log_head_lb + t->log_cap) {
      t->log_valid = false;
      t->buf_gen++;
    }
  }
  static const bool dbg = getenv("RS_LOG_DBG") != nullptr;
  if (!t->log_valid) {
    const int st = log_rebuild(t, s);
    if (st) return st;
    if (dbg) fprintf(stderr, "log rebuild #%llu: %llu records\n", (unsigned long long)t->log_rebuilds,
                     (unsigned long long)t->log_tail_ub);
  }
  t->log_tail_ub += n_max;
  const uint64_t nb = (t->log_cap + kLgBlock - 1) / kLgBlock;  // (the whole-log window)
  if (t->lg_nb < nb) {
    RS_CUDA(cudaStreamSynchronize(s));
    if (t->d_lg_cnt) cudaFree(t->d_lg_cnt);
    if (t->d_lg_pre) cudaFree(t->d_lg_pre);
    RS_CUDA(cudaMalloc(&t->d_lg_cnt, nb * 4));
    RS_CUDA(cudaMalloc(&t->d_lg_pre, nb * 8));
    t->lg_nb = nb;
    t->buf_gen++;
  }
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
