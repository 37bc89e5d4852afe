// step.cu -- dedup, jagged gather, segment-reduce + sparse optimizer (sm_100a).
//
// One training step of one shard (reference caller: run_workload,
// workload.cpp:506-581; for W = 1 distributed_lookup reduces to
// stage1_dedup + ensure + inverse expand, exchange_sim.cpp:117-233):
//
//   K0 k_dedup_clear    reset the scratch slots used by the previous call
//   K1 k_dedup_tile     per 1 tile: smem dedup, then one global insert per
//                       (tile, distinct id): first position (atomicMax of ~pos),
//                       count, number of tiles containing the id
//   K2 k_dedup_compact  decoupled look-back scan over tokens: heads (first
//                       occurrences) get their unique index = first-occurrence
//                       order (exchange_sim.cpp:87-98), plus the offsets of
//                       the cross-tile partial-sum segments
//   K3 k_table_upsert   find-or-insert-zero of the unique ids (table.cu)
//   K4 k_gather         out[t] = emb[row(inverse[t])], 128-bit vector copies
//   K5 k_reduce_update  per tile: TMA-bulk stage of the tile's gradient rows
//                       into smem, smem grouping by unique id, position-order
//                       sums; single-tile ids update their row immediately,
//                       multi-tile ids write a partial and the last arriving
//                       tile sums the partials in tile order and updates.
//                       Adam (sparse_update.cpp:22-37) / Adagrad in FP64
//                       with explicit _rn intrinsics (no FMA contraction).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "rs_host.hpp"

namespace rs {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kWarpMaxParts = 32;  // ids with more partials finish block-cooperatively

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// ---------------------------------------------------------------------------
// K0: clear the scratch slots touched by the previous dedup (its unique list)
__global__ void k_dedup_clear(unsigned long long* skey, uint32_t* sfirstx, uint32_t* scount,
                              uint32_t* sntile, const uint32_t* u_slot, uint32_t* ctr,
                              uint64_t spare) {
  const uint32_t prev = ctr[2];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= prev;
       i += gridDim.x * blockDim.x) {
    const uint64_t s = i < prev ? u_slot[i] : spare;
    skey[s] = kEmptyKey;
    sfirstx[s] = 0;
    scount[s] = 0;
    sntile[s] = 0;
  }
}

__global__ void k_dedup_clear_all(unsigned long long* skey, uint32_t* sfirstx, uint32_t* scount,
                                  uint32_t* sntile, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    skey[i] = kEmptyKey;
    sfirstx[i] = 0;
    scount[i] = 0;
    sntile[i] = 0;
  }
}

// ---------------------------------------------------------------------------
// K1: per-tile smem dedup, then one global scratch insert per distinct id.
// blockDim.x == TT tokens per tile; dynamic smem: 2TT+1 local slots.
__global__ void k_dedup_tile(const uint64_t* __restrict__ ids, uint32_t n,
                             unsigned long long* __restrict__ skey, uint32_t* __restrict__ sfirstx,
                             uint32_t* __restrict__ scount, uint32_t* __restrict__ sntile,
                             uint64_t smask, uint64_t spare, uint32_t* __restrict__ slot_of,
                             uint32_t* __restrict__ ctr) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[4] = 0;  // hot-list count, filled by K2
  const uint32_t TT = blockDim.x;
  const uint32_t L = 2 * TT;  // local slots (power of two), index L = sentinel id
  unsigned long long* lkey = reinterpret_cast<unsigned long long*>(smem);
  uint32_t* lfirst = reinterpret_cast<uint32_t*>(lkey + L + 1);
  uint32_t* lcount = lfirst + L + 1;
  uint32_t* lgslot = lcount + L + 1;
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i <= L; i += TT) {
    lkey[i] = kEmptyKey;
    lfirst[i] = kFull;
    lcount[i] = 0;
  }
  __syncthreads();
  const uint32_t t = blockIdx.x * TT + tid;
  const bool valid = t < n;
  uint64_t id = 0, h = 0;
  uint32_t p = 0;
  if (valid) {
    id = ids[t];
    if (id == kEmptyKey) {
      p = L;
    } else {
      h = hash64(id);
      p = (uint32_t)(h >> 40) & (L - 1);
      for (;;) {
        const unsigned long long prev = atomicCAS(&lkey[p], kEmptyKey, (unsigned long long)id);
        if (prev == kEmptyKey || prev == id) break;
        p = (p + 1) & (L - 1);
      }
    }
    atomicMin(&lfirst[p], tid);
    atomicAdd(&lcount[p], 1u);
  }
  __syncthreads();
  if (valid && lfirst[p] == tid) {
    uint64_t gs;
    if (p == L) {
      gs = spare;
    } else {
      gs = h & smask;
      for (;;) {
        const unsigned long long prev = atomicCAS(&skey[gs], kEmptyKey, (unsigned long long)id);
        if (prev == kEmptyKey || prev == id) break;
        gs = (gs + 1) & smask;
      }
    }
    atomicMax(&sfirstx[gs], ~t);  // ~min(position)
    atomicAdd(&scount[gs], lcount[p]);
    atomicAdd(&sntile[gs], 1u);
    lgslot[p] = (uint32_t)gs;
  }
  __syncthreads();
  if (valid) slot_of[t] = lgslot[p];
}

// ---------------------------------------------------------------------------
// Decoupled look-back over tiles for a pair of 31-bit counters.
struct Pair {
  uint32_t a, b;
};
__device__ __forceinline__ uint64_t st_pack(uint32_t flag, Pair v) {
  return ((uint64_t)flag << 62) | ((uint64_t)(v.a & 0x7FFFFFFFu) << 31) | (v.b & 0x7FFFFFFFu);
}
__device__ __forceinline__ Pair st_unpack(uint64_t s) {
  return Pair{(uint32_t)((s >> 31) & 0x7FFFFFFFu), (uint32_t)(s & 0x7FFFFFFFu)};
}
__device__ __forceinline__ Pair warp_sum(Pair v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.a += __shfl_xor_sync(kFull, v.a, o);
    v.b += __shfl_xor_sync(kFull, v.b, o);
  }
  return v;
}
__device__ __forceinline__ Pair warp_incl_scan(Pair v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(kFull, v.a, o);
    const uint32_t b = __shfl_up_sync(kFull, v.b, o);
    if (lane >= (unsigned)o) {
      v.a += a;
      v.b += b;
    }
  }
  return v;
}

// Called by warp 0 of the block owning `tile`; returns the exclusive prefix.
__device__ Pair lookback(uint64_t* status, uint32_t tile, Pair agg) {
  const unsigned lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_release(&status[0], st_pack(2, agg));
    return Pair{0, 0};
  }
  if (lane == 0) st_release(&status[tile], st_pack(1, agg));
  Pair run{0, 0};
  int64_t j = (int64_t)tile - 1;
  for (;;) {
    const int64_t idx = j - lane;
    const uint64_t s = idx >= 0 ? ld_acquire(&status[idx]) : st_pack(2, Pair{0, 0});
    const uint32_t flag = (uint32_t)(s >> 62);
    const unsigned m0 = __ballot_sync(kFull, flag == 0);
    const unsigned m2 = __ballot_sync(kFull, flag == 2);
    const int stop = m2 ? __ffs(m2) - 1 : 31;
    const unsigned need = stop == 31 ? kFull : ((2u << stop) - 1u);
    if (m0 & need) continue;  // a predecessor inside the window has not published yet
    Pair v = (int)lane <= stop ? st_unpack(s) : Pair{0, 0};
    v = warp_sum(v);
    run.a += v.a;
    run.b += v.b;
    if (m2) break;
    j -= 32;
  }
  if (lane == 0) st_release(&status[tile], st_pack(2, Pair{agg.a + run.a, agg.b + run.b}));
  return run;
}

// K2: head = first occurrence; exclusive scan over tokens of
// (head, head && ntile > 1 ? ntile : 0) gives the unique index (first-
// occurrence order) and the offset of the id's cross-tile partial segment.
__global__ void __launch_bounds__(kScanThreads)
    k_dedup_compact(const uint64_t* __restrict__ ids, uint32_t n,
                    const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ sfirstx,
                    const uint32_t* __restrict__ sntile, uint32_t* __restrict__ suidx,
                    uint64_t* __restrict__ unique, uint32_t* __restrict__ u_slot,
                    uint32_t* __restrict__ u_ntile, uint32_t* __restrict__ u_poff,
                    uint32_t* __restrict__ u_ticket, uint32_t* __restrict__ u_done,
                    uint64_t* status, uint32_t* ctr, uint32_t ntiles, uint32_t* __restrict__ hot_list) {
  __shared__ uint32_t s_tile;
  __shared__ Pair s_warp[kScanThreads / 32];
  __shared__ Pair s_prefix;
  __shared__ bool s_last;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(&ctr[0], 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kScanTile + tid * kScanItems;
  uint32_t sl[kScanItems];
  uint32_t nt[kScanItems];
  bool hd[kScanItems];
  Pair mine{0, 0};
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint32_t t = base + k;
    hd[k] = false;
    nt[k] = 0;
    sl[k] = 0;
    if (t < n) {
      sl[k] = slot_of[t];
      hd[k] = sfirstx[sl[k]] == ~t;
      if (hd[k]) nt[k] = sntile[sl[k]];
    }
    mine.a += hd[k];
    mine.b += (hd[k] && nt[k] > 1) ? nt[k] : 0;
  }
  Pair incl = warp_incl_scan(mine);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    Pair w = lane < kScanThreads / 32 ? s_warp[lane] : Pair{0, 0};
    Pair wi = warp_incl_scan(w);
    if (lane < kScanThreads / 32) s_warp[lane] = Pair{wi.a - w.a, wi.b - w.b};
    const Pair agg{__shfl_sync(kFull, wi.a, kScanThreads / 32 - 1),
                   __shfl_sync(kFull, wi.b, kScanThreads / 32 - 1)};
    const Pair pre = lookback(status, tile, agg);
    if (lane == 0) s_prefix = pre;
  }
  __syncthreads();
  Pair run{s_prefix.a + s_warp[warp].a + incl.a - mine.a,
           s_prefix.b + s_warp[warp].b + incl.b - mine.b};
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (hd[k]) {
      const uint32_t t = base + k;
      const uint32_t ra = run.a;
      unique[ra] = ids[t];
      suidx[sl[k]] = ra;
      u_slot[ra] = sl[k];
      u_ntile[ra] = nt[k];
      if (nt[k] > kWarpMaxParts) hot_list[atomicAdd(&ctr[4], 1u)] = ra;
      u_poff[ra] = run.b;
      u_ticket[ra] = 0;
      u_done[ra] = 0;
      run.a += 1;
      run.b += nt[k] > 1 ? nt[k] : 0;
    }
  }
  if (tile == ntiles - 1 && tid == kScanThreads - 1) {
    ctr[2] = run.a;  // n_unique
    ctr[3] = run.b;  // n_part
  }
  // last block resets the tile ticket and the status words for the next call
  __syncthreads();
  if (tid == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s_last = atomicAdd(&ctr[1], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (uint32_t i = tid; i < ntiles; i += kScanThreads) status[i] = 0;
    if (tid == 0) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

__global__ void k_inverse(const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ suidx,
                          uint32_t n, int32_t* __restrict__ inverse) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    inverse[i] = (int32_t)suidx[slot_of[i]];
}

__global__ void k_copy_unique(const uint64_t* __restrict__ src, const uint32_t* __restrict__ ctr,
                              uint64_t* __restrict__ dst, uint32_t* __restrict__ n_out) {
  const uint32_t n = ctr[2];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && threadIdx.x == 0 && n_out) *n_out = n;
}

// ---------------------------------------------------------------------------
// K4: jagged gather.  A warp takes 32 consecutive tokens: each lane resolves
// one token's slot -> (unique, row) (coalesced slot_of load, two L2 loads),
// writes the int32 inverse, then the warp copies the 32 rows with LPR lanes
// per row and all 128-bit row loads of a batch issued before any store
// (up to 16 independent LDG.128 in flight per lane).
template <int LPR>
__global__ void __launch_bounds__(256, 3)
    k_gather(const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ suidx,
             const uint32_t* __restrict__ srow, const TableDev* __restrict__ td, uint32_t n,
             int32_t* __restrict__ inverse, float* __restrict__ out) {
  constexpr int RPI = 32 / LPR;        // rows per warp instruction
  constexpr int ITERS = 32 / RPI;      // instructions to cover 32 rows (one float4 per lane each)
  constexpr int BATCH = ITERS < 8 ? ITERS : 8;
  const uint32_t D4 = td->d.dim >> 2;
  const float4* __restrict__ emb = reinterpret_cast<const float4*>(td->d.emb);
  float4* __restrict__ o4 = reinterpret_cast<float4*>(out);
  const uint32_t lane = lane_id();
  const uint32_t sub = lane / LPR, l = lane % LPR;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = w * 32; base < n; base += nw * 32) {
    const uint64_t t = base + lane;
    uint32_t u = 0, r = 0;
    if (t < n) {
      const uint32_t s = __ldg(slot_of + t);
      u = __ldcg(suidx + s);
      r = __ldcg(srow + s);
      inverse[t] = (int32_t)u;
    }
    const uint32_t cnt = (n - base) < 32 ? (uint32_t)(n - base) : 32u;
#pragma unroll
    for (int b0 = 0; b0 < ITERS; b0 += BATCH) {
      uint32_t rr[BATCH];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) rr[k] = __shfl_sync(kFull, r, (b0 + k) * RPI + sub);
      for (uint32_t jj = 0; jj < D4; jj += LPR) {  // uniform trip count
        const uint32_t j = jj + l;
        float4 v[BATCH];
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          const uint32_t tok = (b0 + k) * RPI + sub;
          if (tok < cnt && j < D4) v[k] = __ldg(emb + (size_t)rr[k] * D4 + j);
        }
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          const uint32_t tok = (b0 + k) * RPI + sub;
          if (tok < cnt && j < D4) __stcs(o4 + (base + tok) * D4 + j, v[k]);
        }
      }
    }
  }
}

// scalar fallback for D % 4 != 0
__global__ void k_gather_scalar(const uint32_t* __restrict__ slot_of,
                                const uint32_t* __restrict__ suidx, const uint32_t* __restrict__ srow,
                                const TableDev* __restrict__ td, uint32_t n,
                                int32_t* __restrict__ inverse, float* __restrict__ out) {
  const uint32_t D = td->d.dim;
  const float* emb = td->d.emb;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t t = w; t < n; t += nw) {
    const uint32_t s = slot_of[t];
    const uint32_t r = __ldcg(srow + s);
    if (lane == 0) inverse[t] = (int32_t)__ldcg(suidx + s);
    for (uint32_t e = lane; e < D; e += 32) out[t * D + e] = emb[(size_t)r * D + e];
  }
}

// ---------------------------------------------------------------------------
// Optimizers: FP64 math with explicit round-to-nearest intrinsics so nvcc
// cannot contract into FMA (the reference is compiled -ffp-contract=off).
struct OptArgs {
  uint32_t kind;
  double lr, b1, b2, eps, omb1, omb2;
  const double* bc;  // [2 x bc_len]: 1 - b1^k, 1 - b2^k (host libm)
  uint64_t bc_len;
};

__device__ __forceinline__ void adagrad_elem(float& w, float& a, float gf, const OptArgs& o) {
  const double g = (double)gf;
  const double an = __dadd_rn((double)a, __dmul_rn(g, g));
  a = __double2float_rn(an);
  w = __double2float_rn(
      __dsub_rn((double)w, __ddiv_rn(__dmul_rn(o.lr, g), __dadd_rn(__dsqrt_rn(an), o.eps))));
}
__device__ __forceinline__ void adam_elem(float& w, float& m, float& v, float gf, double bc1,
                                          double bc2, const OptArgs& o) {
  const double g = (double)gf;
  const double me = __dadd_rn(__dmul_rn(o.b1, (double)m), __dmul_rn(o.omb1, g));
  const double ve = __dadd_rn(__dmul_rn(o.b2, (double)v), __dmul_rn(__dmul_rn(o.omb2, g), g));
  m = __double2float_rn(me);
  v = __double2float_rn(ve);
  const double mh = __ddiv_rn(me, bc1);
  const double vh = __ddiv_rn(ve, bc2);
  w = __double2float_rn(
      __dsub_rn((double)w, __ddiv_rn(__dmul_rn(o.lr, mh), __dadd_rn(__dsqrt_rn(vh), o.eps))));
}

// Applies one optimizer step to `row` with the lane-distributed gradient
// acc[c][j] for elements e = (c*32 + lane)*VEC + j.  Called by a full warp.
template <int VEC, int CH>
__device__ __forceinline__ void load_vec(const float* __restrict__ src, uint32_t D,
                                         float (&x)[CH][VEC], bool coherent);
template <int VEC, int CH>
__device__ __forceinline__ void store_vec(float* __restrict__ dst, uint32_t D,
                                          const float (&x)[CH][VEC]);

// Applies one optimizer step to `row` with the lane-distributed gradient
// acc[c][j] for elements e = (c*32 + lane)*VEC + j.  Called by a full warp.
// Row loads are issued before the step counter so their latencies overlap.
template <int VEC, int CH>
__device__ __forceinline__ void apply_row(const TableDesc& d, uint32_t row,
                                          const float (&acc)[CH][VEC], const OptArgs& o) {
  const unsigned lane = lane_id();
  const uint32_t D = d.dim;
  if (row == kNoRow) return;
  float* w = d.emb + (size_t)row * D;
  float* m = d.s1 ? d.s1 + (size_t)row * D : nullptr;
  float* v = d.s2 + (size_t)row * D;
  float wv[CH][VEC], mv[CH][VEC], vv[CH][VEC];
  load_vec<VEC, CH>(w, D, wv, false);
  load_vec<VEC, CH>(v, D, vv, false);
  if (m) load_vec<VEC, CH>(m, D, mv, false);
  uint32_t step = 0;
  if (lane == 0) {
    step = d.step[row] + 1;
    d.step[row] = step;
  }
  step = __shfl_sync(kFull, step, 0);
  double bc1 = 1.0, bc2 = 1.0;
  if (o.kind == RS_OPT_ADAM) {
    if (step < o.bc_len) {
      bc1 = o.bc[step];
      bc2 = o.bc[o.bc_len + step];
    } else {
      bc1 = 1.0 - pow(o.b1, (double)step);
      bc2 = 1.0 - pow(o.b2, (double)step);
    }
  }
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      if (VEC == 1 && (uint32_t)(c * 32 + lane) >= D) continue;
      if (o.kind == RS_OPT_ADAM)
        adam_elem(wv[c][j], mv[c][j], vv[c][j], acc[c][j], bc1, bc2, o);
      else
        adagrad_elem(wv[c][j], vv[c][j], acc[c][j], o);
    }
  store_vec<VEC, CH>(w, D, wv);
  store_vec<VEC, CH>(v, D, vv);
  if (m) store_vec<VEC, CH>(m, D, mv);
}

template <int VEC, int CH>
__device__ __forceinline__ void load_vec(const float* __restrict__ src, uint32_t D,
                                         float (&x)[CH][VEC], bool coherent) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const uint32_t e0 = ((uint32_t)c * 32 + lane) * VEC;
    if (VEC == 4) {
      float4 t = coherent ? __ldcg(reinterpret_cast<const float4*>(src + e0))
                          : *reinterpret_cast<const float4*>(src + e0);
      x[c][0] = t.x; x[c][1] = t.y; x[c][2] = t.z; x[c][3] = t.w;
    } else if (VEC == 2) {
      float2 t = coherent ? __ldcg(reinterpret_cast<const float2*>(src + e0))
                          : *reinterpret_cast<const float2*>(src + e0);
      x[c][0] = t.x; x[c][1] = t.y;
    } else {
      x[c][0] = e0 < D ? (coherent ? __ldcg(src + e0) : src[e0]) : 0.f;
    }
  }
}

template <int VEC, int CH>
__device__ __forceinline__ void store_vec(float* __restrict__ dst, uint32_t D,
                                          const float (&x)[CH][VEC]) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const uint32_t e0 = ((uint32_t)c * 32 + lane) * VEC;
    if (VEC == 4) {
      *reinterpret_cast<float4*>(dst + e0) = make_float4(x[c][0], x[c][1], x[c][2], x[c][3]);
    } else if (VEC == 2) {
      *reinterpret_cast<float2*>(dst + e0) = make_float2(x[c][0], x[c][1]);
    } else if (e0 < D) {
      dst[e0] = x[c][0];
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

struct ReduceArgs {
  const int32_t* inverse;
  const float* grads;
  uint32_t n;
  uint32_t ntiles;
  uint32_t bw;  // bitmap words = ceil(ntiles / 32)
  const uint32_t* u_ntile;
  const uint32_t* u_poff;
  uint32_t* u_ticket;
  const uint32_t* urow;
  const uint32_t* n_unique;  // device count of the last dedup
  const uint32_t* n_hot;     // device count of ids with > kWarpMaxParts partials
  const uint32_t* hot_list;
  float* usum;               // [U x D] sums of single-tile ids
  float* pbuf;               // [n_part x D] per-(tile, id) partial sums
  uint32_t* ptile;           // tile of each partial
  uint32_t* porder;          // scratch: partial index by rank
  TableDev* td;
  float* sums_out;  // accumulate-only mode when non-null
  bool tma;
};


template <int VEC, int CH>
__device__ __forceinline__ void zero_acc(float (&x)[CH][VEC]) {
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < VEC; ++j) x[c][j] = 0.f;
}
template <int VEC, int CH>
__device__ __forceinline__ void add_acc(float (&x)[CH][VEC], const float (&y)[CH][VEC]) {
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < VEC; ++j) x[c][j] += y[c][j];
}

template <int VEC, int CH>
__device__ __forceinline__ void finalize(const ReduceArgs& a, const TableDesc& d, uint32_t uu,
                                         const float (&acc)[CH][VEC], const OptArgs& o) {
  if (a.sums_out)
    store_vec<VEC, CH>(a.sums_out + (size_t)uu * d.dim, d.dim, acc);
  else
    apply_row<VEC, CH>(d, __ldg(a.urow + uu), acc, o);
}

// Ordered sum of partials whose indices (within the id's segment) are given
// by rank in `order` (smem or global), ranks [r0, r1), PF rows in flight.
template <int VEC, int CH>
__device__ __forceinline__ void ordered_sum(const ReduceArgs& a, const uint32_t* order,
                                            uint32_t poff, uint32_t r0, uint32_t r1, uint32_t D,
                                            float (&acc)[CH][VEC]) {
  constexpr int PF = (CH * VEC <= 4) ? 8 : (CH * VEC <= 8) ? 4 : 2;
  const unsigned lane = lane_id();
  zero_acc<VEC, CH>(acc);
  for (uint32_t r = r0; r < r1; r += 32) {
    const uint32_t cnt = min(32u, r1 - r);
    const uint32_t idx = lane < cnt ? order[r + lane] : 0;
    for (uint32_t j0 = 0; j0 < cnt; j0 += PF) {
      float x[PF][CH][VEC];
#pragma unroll
      for (int jj = 0; jj < PF; ++jj) {
        const uint32_t i = __shfl_sync(kFull, idx, (j0 + jj) & 31);
        if (j0 + jj < cnt) load_vec<VEC, CH>(a.pbuf + (size_t)(poff + i) * D, D, x[jj], false);
      }
#pragma unroll
      for (int jj = 0; jj < PF; ++jj)
        if (j0 + jj < cnt) add_acc<VEC, CH>(acc, x[jj]);
    }
  }
}

// K5.  blockDim.x == TT (tokens per tile, <= 256), one tile per block.
//  phase 0  TMA bulk copy (UBLKCP) of the tile's contiguous gradient rows
//  phase 1  group the tile's tokens by unique id in smem (first-occurrence
//           order), stable ranks -> local CSR; partial tickets
//  phase 2  warp per group: position-order f32 sum, in place into the group's
//           first row (no other group reads that row)
//  phase 3  element-parallel stores: single-tile ids -> usum[u], multi-tile
//           ids -> pbuf[poff + ticket] tagged with the tile index
template <int VEC, int CH>
__global__ void __launch_bounds__(256, 2) k_tile_reduce(ReduceArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t TT = blockDim.x;
  const uint32_t NW = TT >> 5;
  const uint32_t L = 2 * TT;
  const uint32_t D = a.td->d.dim;
  float* sg = reinterpret_cast<float*>(smem);  // [TT x D] staged gradients
  unsigned char* p = smem + (size_t)TT * D * 4;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(p);
  p += 16;
  uint32_t* lkey = reinterpret_cast<uint32_t*>(p);
  uint32_t* lfirst = lkey + L;
  uint32_t* lgroup = lfirst + L;
  uint32_t* gcnt = lgroup + L;
  uint32_t* goff = gcnt + TT;
  uint32_t* gu = goff + TT;
  uint32_t* gdst = gu + TT;        // destination row offset (floats) of each group's sum
  uint32_t* wsum = gdst + TT;      // [32]
  uint32_t* misc = wsum + 32;      // [0] ng
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(misc + 32);  // [NW x TT]
  uint16_t* csr = wcnt + (size_t)NW * TT;                    // [TT]
  float* dst_base[2] = {a.usum, a.pbuf};
  (void)dst_base;

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t tile = blockIdx.x;
  const uint32_t t0 = tile * TT;
  const uint32_t rows = min(TT, a.n - t0);

  for (uint32_t i = tid; i < L; i += TT) {
    lkey[i] = kFull;
    lfirst[i] = kFull;
  }
  for (uint32_t i = tid; i < NW * TT; i += TT) wcnt[i] = 0;
  if (a.tma) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = rows * D * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"(bytes)
                   : "memory");
      const char* src = reinterpret_cast<const char*>(a.grads + (size_t)t0 * D);
      constexpr uint32_t kChunk = 32768;
      for (uint32_t off = 0; off < bytes; off += kChunk) {
        const uint32_t sz = min(kChunk, bytes - off);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(reinterpret_cast<char*>(sg) + off)),
            "l"(src + off), "r"(sz), "r"(smem_u32(bar))
            : "memory");
      }
    }
  } else {
    const float* src = a.grads + (size_t)t0 * D;
    for (uint32_t i = tid; i < rows * D; i += TT) sg[i] = src[i];
  }
  __syncthreads();

  // ---- phase 1
  const bool valid = tid < rows;
  const uint32_t u = valid ? (uint32_t)__ldg(a.inverse + t0 + tid) : kFull;
  uint32_t ps = 0;
  if (valid) {
    ps = hash32(u) & (L - 1);
    for (;;) {
      const uint32_t prev = atomicCAS(&lkey[ps], kFull, u);
      if (prev == kFull || prev == u) break;
      ps = (ps + 1) & (L - 1);
    }
    atomicMin(&lfirst[ps], tid);
  }
  __syncthreads();
  const bool head = valid && lfirst[ps] == tid;
  const unsigned hb = __ballot_sync(kFull, head);
  if (lane == 0) wsum[warp] = __popc(hb);
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < NW ? wsum[lane] : 0;
    uint32_t x = v;
#pragma unroll
    for (int o2 = 1; o2 < 32; o2 <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o2);
      if (lane >= (unsigned)o2) x += y;
    }
    if (lane < NW) wsum[lane] = x - v;
    if (lane == 31) misc[0] = x;
  }
  __syncthreads();
  const uint32_t ng = misc[0];
  if (head) {
    const uint32_t lg = wsum[warp] + __popc(hb & lanemask_lt());
    lgroup[ps] = lg;
    gu[lg] = u;
    const uint32_t nt = __ldg(a.u_ntile + u);
    uint32_t dst;
    if (nt > 1) {
      const uint32_t tk = atomicAdd(a.u_ticket + u, 1u);
      const uint32_t slot = __ldg(a.u_poff + u) + tk;
      a.ptile[slot] = tile;
      dst = slot | 0x80000000u;  // partial buffer
    } else {
      dst = u;  // usum
    }
    gdst[lg] = dst;
  }
  __syncthreads();
  const uint32_t mylg = valid ? lgroup[ps] : (0xFFFF0000u | lane);
  const unsigned mm = __match_any_sync(kFull, mylg);
  const uint32_t rw = __popc(mm & lanemask_lt());
  if (valid && rw == 0) wcnt[warp * TT + mylg] = (uint16_t)__popc(mm);
  __syncthreads();
  if (tid < ng) {
    uint32_t run = 0;
    for (uint32_t w = 0; w < NW; ++w) {
      const uint32_t c = wcnt[w * TT + tid];
      wcnt[w * TT + tid] = (uint16_t)run;
      run += c;
    }
    gcnt[tid] = run;
  }
  __syncthreads();
  {  // exclusive scan of gcnt[0, ng) -> goff
    const uint32_t v = tid < ng ? gcnt[tid] : 0;
    uint32_t x = v;
#pragma unroll
    for (int o2 = 1; o2 < 32; o2 <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o2);
      if (lane >= (unsigned)o2) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint32_t wv = lane < NW ? wsum[lane] : 0;
      uint32_t z = wv;
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, z, o2);
        if (lane >= (unsigned)o2) z += y;
      }
      if (lane < NW) wsum[lane] = z - wv;
    }
    __syncthreads();
    if (tid < ng) goff[tid] = wsum[warp] + x - v;
  }
  __syncthreads();
  if (valid) csr[goff[mylg] + wcnt[warp * TT + mylg] + rw] = (uint16_t)tid;
  if (a.tma) {
    asm volatile(
        "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar))
        : "memory");
  }
  __syncthreads();

  // ---- phase 2: position-order sums
  for (uint32_t g = warp; g < ng; g += NW) {
    const uint32_t cnt = gcnt[g];
    if (cnt < 2) continue;
    const uint32_t base = goff[g];
    float acc[CH][VEC];
    load_vec<VEC, CH>(sg + (size_t)csr[base] * D, D, acc, false);
    for (uint32_t k = 1; k < cnt; ++k) {
      float x[CH][VEC];
      load_vec<VEC, CH>(sg + (size_t)csr[base + k] * D, D, x, false);
      add_acc<VEC, CH>(acc, x);
    }
    store_vec<VEC, CH>(sg + (size_t)csr[base] * D, D, acc);
  }
  __syncthreads();

  // ---- phase 3: element-parallel stores of sums / partials
  if ((D & 3u) == 0) {
    const uint32_t D4 = D >> 2;
    const uint32_t nchunks = ng * D4;
    for (uint32_t q = tid; q < nchunks; q += TT) {
      const uint32_t g = q / D4, c = q - g * D4;
      const float4 sum = *reinterpret_cast<const float4*>(sg + (size_t)csr[goff[g]] * D + 4 * c);
      const uint32_t dst = gdst[g];
      float* base = (dst & 0x80000000u) ? a.pbuf + (size_t)(dst & 0x7FFFFFFFu) * D
                                        : a.usum + (size_t)dst * D;
      __stcg(reinterpret_cast<float4*>(base) + c, sum);
    }
  } else {
    const uint32_t nchunks = ng * D;
    for (uint32_t q = tid; q < nchunks; q += TT) {
      const uint32_t g = q / D, e = q - g * D;
      const uint32_t dst = gdst[g];
      float* base = (dst & 0x80000000u) ? a.pbuf + (size_t)(dst & 0x7FFFFFFFu) * D
                                        : a.usum + (size_t)dst * D;
      base[e] = sg[(size_t)csr[goff[g]] * D + e];
    }
  }
}

// K6.  Finish every unique id: combine its partials in tile order, then one
// optimizer step on its row (or store the aggregated sum).
//  blocks [0, hot_blocks): one id with > kWarpMaxParts partials at a time, the
//    whole block ranks its partials (bitmap over tiles) and splits the ordered
//    sum over the warps (fixed split -> deterministic)
//  other blocks: warp per id, no block barriers (ids finish independently)
template <int VEC, int CH>
__global__ void __launch_bounds__(256, 3) k_finish(ReduceArgs a, OptArgs o, uint32_t hot_blocks) {
  extern __shared__ __align__(16) unsigned char smem2[];
  const uint32_t NW = blockDim.x >> 5;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const TableDesc d = a.td->d;
  const uint32_t D = d.dim;
  if (blockIdx.x >= hot_blocks) {
    uint32_t* order_w = reinterpret_cast<uint32_t*>(smem2) + warp * 32;  // [NW x 32]
    const uint32_t nu = *a.n_unique;
    const uint32_t stride = (gridDim.x - hot_blocks) * NW;
    for (uint32_t uu = (blockIdx.x - hot_blocks) * NW + warp; uu < nu; uu += stride) {
      const uint32_t nt = __ldg(a.u_ntile + uu);
      if (nt > kWarpMaxParts) continue;
      const uint32_t poff = __ldg(a.u_poff + uu);
      const uint32_t row = a.sums_out ? 0u : __ldg(a.urow + uu);
      float acc[CH][VEC];
      if (nt <= 1) {
        load_vec<VEC, CH>(a.usum + (size_t)uu * D, D, acc, false);
      } else {
        const uint32_t tl = lane < nt ? __ldg(a.ptile + poff + lane) : kFull;
        uint32_t r = 0;
#pragma unroll 8
        for (uint32_t j = 0; j < nt; ++j) r += __shfl_sync(kFull, tl, j) < tl;
        if (lane < nt) order_w[r] = lane;
        __syncwarp();
        ordered_sum<VEC, CH>(a, order_w, poff, 0, nt, D, acc);
        __syncwarp();
        if (lane == 0) a.u_ticket[uu] = 0;
      }
      if (a.sums_out)
        store_vec<VEC, CH>(a.sums_out + (size_t)uu * D, D, acc);
      else
        apply_row<VEC, CH>(d, row, acc, o);
    }
    return;
  }
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem2);  // [bw]
  uint32_t* wpre = bm + a.bw;                          // [bw]
  float* wpart = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(wpre + a.bw) + 15) & ~uintptr_t(15));  // [NW x D]
  const uint32_t nh = *a.n_hot;
  for (uint32_t h = blockIdx.x; h < nh; h += hot_blocks) {
    const uint32_t uu = a.hot_list[h];
    const uint32_t nt = __ldg(a.u_ntile + uu), poff = __ldg(a.u_poff + uu);
    for (uint32_t i = threadIdx.x; i < a.bw; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
      const uint32_t tl = __ldg(a.ptile + poff + i);
      atomicOr(&bm[tl >> 5], 1u << (tl & 31));
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t per = (a.bw + 31) / 32;
      const uint32_t w0 = min(lane * per, a.bw), w1 = min(w0 + per, a.bw);
      uint32_t loc = 0;
      for (uint32_t i = w0; i < w1; ++i) loc += __popc(bm[i]);
      uint32_t x = loc;
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o2);
        if (lane >= (unsigned)o2) x += y;
      }
      uint32_t runp = x - loc;
      for (uint32_t i = w0; i < w1; ++i) {
        wpre[i] = runp;
        runp += __popc(bm[i]);
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
      const uint32_t tl = __ldg(a.ptile + poff + i);
      a.porder[poff + wpre[tl >> 5] + __popc(bm[tl >> 5] & ((1u << (tl & 31)) - 1u))] = i;
    }
    __syncthreads();
    const uint32_t per = (nt + NW - 1) / NW;
    const uint32_t r0 = min(warp * per, nt), r1 = min(r0 + per, nt);
    float part[CH][VEC];
    ordered_sum<VEC, CH>(a, a.porder + poff, poff, r0, r1, D, part);
    store_vec<VEC, CH>(wpart + (size_t)warp * D, D, part);
    __syncthreads();
    if (warp == 0) {
      float tot[CH][VEC];
      zero_acc<VEC, CH>(tot);
      for (uint32_t w = 0; w < NW; ++w) {
        float x[CH][VEC];
        load_vec<VEC, CH>(wpart + (size_t)w * D, D, x, false);
        add_acc<VEC, CH>(tot, x);
      }
      if (lane == 0) a.u_ticket[uu] = 0;
      if (a.sums_out)
        store_vec<VEC, CH>(a.sums_out + (size_t)uu * D, D, tot);
      else
        apply_row<VEC, CH>(d, __ldg(a.urow + uu), tot, o);
    }
    __syncthreads();
  }
}

// Optimizer-only apply for pre-aggregated sums (GradAccumulator::apply given
// `pending`, sparse_update.cpp:58-83): warp per key.
template <int VEC, int CH>
__global__ void k_apply_sums(TableDev* __restrict__ td, const int64_t* __restrict__ rows,
                             uint64_t n, const float* __restrict__ sums, OptArgs o) {
  const TableDesc d = td->d;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w; i < n; i += nw) {
    float acc[CH][VEC];
    load_vec<VEC, CH>(sums + i * d.dim, d.dim, acc, false);
    const int64_t r = rows[i];
    if (r >= 0) apply_row<VEC, CH>(d, (uint32_t)r, acc, o);
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch helpers
struct Shape {
  int vec, ch;
};
Shape shape_for(uint32_t D) {
  if (D % 128 == 0 && D / 128 <= 4) return {4, (int)(D / 128)};
  if (D % 64 == 0 && D / 64 <= 2) return {2, (int)(D / 64)};
  return {1, (int)((D + 31) / 32)};
}

}  // namespace

uint32_t tile_tokens_for_dim(uint32_t D) {
  // keep the staged gradient tile at <= 64 KB so two tiles fit per SM
  uint32_t tt = 256;
  while (tt > 32 && (uint64_t)tt * D * 4 > 65536) tt >>= 1;
  return tt;
}

int dedup_run(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, uint32_t TT, cudaStream_t s) {
  if (n > ws->max_tokens)
    return fail(RS_ERR_CONFIG, "dedup: batch of " + std::to_string(n) +
                                   " ids exceeds workspace max_tokens " +
                                   std::to_string(ws->max_tokens));
  // K0: clear the previous call's slots (first call: full clear at creation)
  k_dedup_clear<<<grid_for(ws->last_n + 1, 256, 148 * 8), 256, 0, s>>>(
      ws->skey, ws->sfirstx, ws->scount, ws->sntile, ws->u_slot, ws->ctr, ws->S);
  RS_LAUNCH_CHECK("k_dedup_clear");
  ws->last_n = n;
  if (n == 0) {
    RS_CUDA(cudaMemsetAsync(ws->ctr + 2, 0, 2 * sizeof(uint32_t), s));
    return RS_OK;
  }
  const uint32_t ntiles = (uint32_t)((n + TT - 1) / TT);
  const size_t sm1 = (size_t)(2 * TT + 1) * (8 + 4 + 4 + 4);
  k_dedup_tile<<<ntiles, TT, sm1, s>>>(d_ids, (uint32_t)n, ws->skey, ws->sfirstx, ws->scount,
                                       ws->sntile, ws->S - 1, ws->S, ws->slot_of, ws->ctr);
  RS_LAUNCH_CHECK("k_dedup_tile");
  const uint32_t stiles = (uint32_t)((n + kScanTile - 1) / kScanTile);
  k_dedup_compact<<<stiles, kScanThreads, 0, s>>>(
      d_ids, (uint32_t)n, ws->slot_of, ws->sfirstx, ws->sntile, ws->suidx, ws->unique,
      ws->u_slot, ws->u_ntile, ws->u_poff, ws->u_ticket, ws->u_done, ws->scan_status, ws->ctr,
      stiles, ws->hot_list);
  RS_LAUNCH_CHECK("k_dedup_compact");
  ws->last_tile = TT;
  return RS_OK;
}

static int launch_gather(rs_workspace* ws, rs_table* t, uint64_t n, float* d_out,
                         cudaStream_t s) {
  const uint32_t D = t->desc.dim;
  if (D % 4 == 0) {
    const uint32_t d4 = D / 4;
    const unsigned grid = grid_for(n, 256, 148 * 16);
#define RS_GATHER(LPR)                                                                      \
  k_gather<LPR><<<grid, 256, 0, s>>>(ws->slot_of, ws->suidx, ws->srow, t->dev, (uint32_t)n, \
                                     ws->inverse, d_out)
    if (d4 >= 32)
      RS_GATHER(32);
    else if (d4 >= 16)
      RS_GATHER(16);
    else if (d4 >= 8)
      RS_GATHER(8);
    else if (d4 >= 4)
      RS_GATHER(4);
    else if (d4 >= 2)
      RS_GATHER(2);
    else
      RS_GATHER(1);
#undef RS_GATHER
    RS_LAUNCH_CHECK("k_gather");
  } else {
    k_gather_scalar<<<grid_for(n, 8, 148 * 8), 256, 0, s>>>(ws->slot_of, ws->suidx, ws->srow,
                                                            t->dev, (uint32_t)n, ws->inverse, d_out);
    RS_LAUNCH_CHECK("k_gather_scalar");
  }
  return RS_OK;
}

static int opt_args(rs_table* t, const rs_optimizer_params* p, OptArgs* o, cudaStream_t s) {
  if (!p) return fail(RS_ERR_CONFIG, "optimizer params required");
  if (p->kind != RS_OPT_ADAM && p->kind != RS_OPT_ADAGRAD)
    return fail(RS_ERR_CONFIG, "unknown optimizer kind");
  if (p->kind == RS_OPT_ADAM && t->desc.opt != RS_OPT_ADAM)
    return fail(RS_ERR_CONFIG, "table was created without Adam state (opt_m)");
  if (p->kind == RS_OPT_ADAGRAD && t->desc.opt == RS_OPT_NONE)
    return fail(RS_ERR_CONFIG, "table was created without optimizer state");
  o->kind = p->kind;
  o->lr = p->lr;
  o->b1 = p->beta1;
  o->b2 = p->beta2;
  o->eps = p->eps;
  o->omb1 = 1.0 - p->beta1;
  o->omb2 = 1.0 - p->beta2;
  o->bc = nullptr;
  o->bc_len = 0;
  if (p->kind == RS_OPT_ADAM) {
    int st = table_adam_tables(t, p->beta1, p->beta2, t->applies, s);
    if (st) return st;
    o->bc = t->d_bc;
    o->bc_len = t->bc_len;
  }
  return RS_OK;
}

// partial sums: at most one per (tile, id) pair <= n; usum: one per id <= n
static int reduce_prepare(rs_workspace* ws, uint32_t D, uint64_t n, cudaStream_t s) {
  if (ws->pbuf_floats < n * D) {
    if (ws->pbuf) RS_CUDA(cudaFreeAsync(ws->pbuf, s));
    ws->pbuf_floats = ws->max_tokens * (uint64_t)D;
    RS_CUDA(cudaMallocAsync(&ws->pbuf, 2 * ws->pbuf_floats * sizeof(float), s));
  }
  return RS_OK;
}

// one-time opt-in to large dynamic shared memory for every instantiation
static int set_smem_attrs() {
  static int done = 0;
  if (done) return RS_OK;
  const int big = 200 * 1024;
#define RS_ATTR(V, C)                                                                          \
  RS_CUDA(cudaFuncSetAttribute(k_tile_reduce<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               big));                                                          \
  RS_CUDA(cudaFuncSetAttribute(k_finish<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  RS_ATTR(4, 1) RS_ATTR(4, 2) RS_ATTR(4, 3) RS_ATTR(4, 4)
  RS_ATTR(2, 1) RS_ATTR(2, 2)
  RS_ATTR(1, 1) RS_ATTR(1, 2) RS_ATTR(1, 3) RS_ATTR(1, 4) RS_ATTR(1, 5) RS_ATTR(1, 6)
  RS_ATTR(1, 7) RS_ATTR(1, 8)
#undef RS_ATTR
  done = 1;
  return RS_OK;
}

static int launch_reduce(rs_workspace* ws, rs_table* t, const float* d_grads, uint64_t n,
                         const OptArgs& o, float* sums_out, cudaStream_t s) {
  const uint32_t D = t->desc.dim;
  const uint32_t TT = ws->last_tile;
  const uint32_t ntiles = (uint32_t)((n + TT - 1) / TT);
  int st = reduce_prepare(ws, D, n, s);
  if (st) return st;
  ReduceArgs a;
  a.inverse = ws->inverse;
  a.grads = d_grads;
  a.n = (uint32_t)n;
  a.ntiles = ntiles;
  a.bw = (ntiles + 31) / 32;
  a.u_ntile = ws->u_ntile;
  a.u_poff = ws->u_poff;
  a.u_ticket = ws->u_ticket;
  a.urow = ws->urow;
  a.n_unique = ws->ctr + 2;
  a.n_hot = ws->ctr + 4;
  a.hot_list = ws->hot_list;
  a.pbuf = ws->pbuf;
  a.usum = ws->pbuf + ws->pbuf_floats;
  a.ptile = ws->ptile;
  a.porder = ws->porder;
  a.td = t->dev;
  a.sums_out = sums_out;
  a.tma = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(d_grads) & 15u) == 0);
  const uint32_t NW = TT / 32;
  const size_t smem5 = (size_t)TT * D * 4 + 16 + (size_t)(3 * 2 * TT + 4 * TT + 64) * 4 +
                       (size_t)NW * TT * 2 + (size_t)TT * 2 + 16;
  const size_t smem6 = std::max<size_t>((size_t)8 * 32 * 4, (size_t)2 * a.bw * 4 + 16 + (size_t)8 * D * 4 + 16);
  const uint32_t hot_blocks = 2 * 148;
  const Shape sh = shape_for(D);
  const unsigned grid6 = hot_blocks + grid_for(n, 8, 148 * 24);
  auto go = [&](auto k5, auto k6) -> int {
    k5<<<ntiles, TT, smem5, s>>>(a);
    RS_LAUNCH_CHECK("k_tile_reduce");
    k6<<<grid6, 256, smem6, s>>>(a, o, hot_blocks);
    RS_LAUNCH_CHECK("k_finish");
    return RS_OK;
  };
#define RS_SHAPE(V, C) \
  if (sh.vec == V && sh.ch == C) return go(k_tile_reduce<V, C>, k_finish<V, C>);
  RS_SHAPE(4, 1) RS_SHAPE(4, 2) RS_SHAPE(4, 3) RS_SHAPE(4, 4)
  RS_SHAPE(2, 1) RS_SHAPE(2, 2)
  RS_SHAPE(1, 1) RS_SHAPE(1, 2) RS_SHAPE(1, 3) RS_SHAPE(1, 4) RS_SHAPE(1, 5) RS_SHAPE(1, 6)
  RS_SHAPE(1, 7) RS_SHAPE(1, 8)
#undef RS_SHAPE
  return fail(RS_ERR_CONFIG, "embedding_dim " + std::to_string(D) + " unsupported by the reduce");
}

}  // namespace rs

using namespace rs;

static cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

extern "C" {

int rs_workspace_create(uint64_t max_tokens, rs_workspace** out) {
  if (!out) return fail(RS_ERR_CONFIG, "rs_workspace_create: null out");
  if (max_tokens == 0 || max_tokens > (1ull << 30))
    return fail(RS_ERR_CONFIG, "rs_workspace_create: max_tokens must be in [1, 2^30]");
  rs_workspace* ws = new rs_workspace();
  ws->max_tokens = max_tokens;
  uint64_t S_ = 1024;
  while (S_ < 2 * max_tokens) S_ <<= 1;
  ws->S = S_;
  const uint64_t N = max_tokens;
  auto A = [&](auto** p, size_t bytes) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16)) == cudaSuccess;
  };
  bool ok = A(&ws->skey, (S_ + 1) * 8) && A(&ws->sfirstx, (S_ + 1) * 4) &&
            A(&ws->scount, (S_ + 1) * 4) && A(&ws->sntile, (S_ + 1) * 4) &&
            A(&ws->suidx, (S_ + 1) * 4) && A(&ws->srow, (S_ + 1) * 4) &&
            A(&ws->slot_of, N * 4) && A(&ws->inverse, N * 4) && A(&ws->unique, N * 8) &&
            A(&ws->u_slot, N * 4) && A(&ws->u_ntile, N * 4) && A(&ws->u_poff, N * 4) &&
            A(&ws->u_ticket, N * 4) && A(&ws->u_done, N * 4) && A(&ws->urow, N * 4) &&
            A(&ws->urow64, N * 8) && A(&ws->ptile, N * 4) && A(&ws->porder, N * 4) && A(&ws->hot_list, (N / 32 + 64) * 4) &&
            A(&ws->scan_status, ((N + kScanTile - 1) / kScanTile + 1) * 8) && A(&ws->ctr, 64);
  if (!ok) {
    rs_workspace_destroy(ws);
    return cuda_fail(cudaGetLastError(), "rs_workspace_create: cudaMalloc");
  }
  if (set_smem_attrs() != RS_OK || cudaStreamCreateWithFlags(&ws->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    rs_workspace_destroy(ws);
    return RS_ERR_CUDA;
  }
  k_dedup_clear_all<<<grid_for(S_ + 1, 256, 148 * 16), 256>>>(ws->skey, ws->sfirstx, ws->scount,
                                                               ws->sntile, S_ + 1);
  count_launch();
  cudaMemset(ws->scan_status, 0, ((N + kScanTile - 1) / kScanTile + 1) * 8);
  cudaMemset(ws->ctr, 0, 64);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    rs_workspace_destroy(ws);
    return cuda_fail(cudaGetLastError(), "rs_workspace_create");
  }
  *out = ws;
  return RS_OK;
}

int rs_workspace_destroy(rs_workspace* ws) {
  if (!ws) return RS_OK;
  cudaDeviceSynchronize();
  void* ptrs[] = {ws->skey,    ws->sfirstx, ws->scount,  ws->sntile,   ws->suidx,  ws->srow,
                  ws->slot_of, ws->inverse, ws->unique,  ws->u_slot,   ws->u_ntile, ws->u_poff,
                  ws->u_ticket, ws->u_done, ws->urow,    ws->urow64,   ws->ptile,  ws->porder,
                  ws->pbuf,    ws->scan_status, ws->ctr, ws->hot_list};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& g : ws->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (ws->cap_stream) cudaStreamDestroy(ws->cap_stream);
  delete ws;
  return RS_OK;
}

int rs_dedup(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, uint64_t* d_unique,
             int32_t* d_inverse, uint32_t* d_n_unique, void* stream) {
  if (!ws) return fail(RS_ERR_CONFIG, "rs_dedup: null workspace");
  cudaStream_t s = S(stream);
  int st = dedup_run(ws, d_ids, n, 512, s);
  if (st) return st;
  ws->have_forward = false;
  if (n) {
    if (d_inverse) {
      k_inverse<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(ws->slot_of, ws->suidx, (uint32_t)n,
                                                          d_inverse);
      RS_LAUNCH_CHECK("k_inverse");
    }
    k_copy_unique<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(ws->unique, ws->ctr, d_unique,
                                                            d_n_unique);
    RS_LAUNCH_CHECK("k_copy_unique");
  } else if (d_n_unique) {
    RS_CUDA(cudaMemsetAsync(d_n_unique, 0, sizeof(uint32_t), s));
  }
  return RS_OK;
}

int rs_forward(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n, float* d_out,
               void* stream) {
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_forward: null handle");
  cudaStream_t s = S(stream);
  const uint32_t TT = tile_tokens_for_dim(t->desc.dim);
  int st = dedup_run(ws, d_ids, n, TT, s);
  if (st) return st;
  ws->have_forward = true;
  ws->last_table = t;
  if (n == 0) return RS_OK;
  st = table_ensure_any(t, ws->unique, ws->ctr + 2, n, ws->urow, ws->urow64, ws->u_slot,
                           ws->srow, s);
  if (st) return st;
  return launch_gather(ws, t, n, d_out, s);
}

int rs_backward(rs_workspace* ws, rs_table* t, const float* d_grads, uint64_t n,
                const rs_optimizer_params* opt, void* stream) {
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_backward: null handle");
  if (!ws->have_forward || ws->last_table != t || ws->last_n != n)
    return fail(RS_ERR_CONFIG, "rs_backward: must follow rs_forward on the same table and batch");
  if (n == 0) return RS_OK;
  cudaStream_t s = S(stream);
  OptArgs o;
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  st = launch_reduce(ws, t, d_grads, n, o, nullptr, s);
  if (st) return st;
  t->applies++;
  ws->have_forward = false;  // rows were updated: a second backward would double-apply
  return RS_OK;
}

// All launches of one training step, no host-side work (graph capturable).
static int step_enqueue(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                        const float* d_grads, float* d_out, const OptArgs& o, uint32_t TT,
                        int mirror, cudaStream_t s) {
  int st = dedup_run(ws, d_ids, n, TT, s);
  if (st) return st;
  st = table_upsert_enqueue(t, ws->unique, ws->ctr + 2, n, ws->urow, ws->urow64, ws->u_slot,
                            ws->srow, s);
  if (st) return st;
  st = launch_gather(ws, t, n, d_out, s);
  if (st) return st;
  st = launch_reduce(ws, t, d_grads, n, o, nullptr, s);
  if (st) return st;
  return table_mirror_copy(t, mirror, s);
}

int rs_step(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
            const float* d_grads, float* d_out, const rs_optimizer_params* opt, void* stream) {
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_step: null handle");
  if (t->cfg.max_keys || n == 0 || !ws->use_graphs) {
    // bounded tables synchronize on the host to evict: no graph
    int st = rs_forward(ws, t, d_ids, n, d_out, stream);
    if (st) return st;
    return rs_backward(ws, t, d_grads, n, opt, stream);
  }
  if (n > ws->max_tokens)
    return fail(RS_ERR_CONFIG, "rs_step: batch exceeds workspace max_tokens");
  cudaStream_t s = S(stream);
  OptArgs o;
  std::memset(&o, 0, sizeof(o));
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  // host side, outside the graph: capacity bound (may rehash / grow rows on s)
  st = table_prepare(t, n, s);
  if (st) return st;
  const uint32_t TT = tile_tokens_for_dim(t->desc.dim);
  st = reduce_prepare(ws, t->desc.dim, n, s);
  if (st) return st;
  const int mirror = t->mirror_next;
  static_assert(sizeof(OptArgs) <= sizeof(((rs_graph_entry*)0)->opt), "opt key");
  rs_graph_entry* hit = nullptr;
  for (auto& g : ws->graphs) {
    if (g.t == t && g.ids == d_ids && g.grads == d_grads && g.out == d_out && g.n == n &&
        g.mirror == mirror && g.pbuf == ws->pbuf && std::memcmp(g.opt, &o, sizeof(o)) == 0) {
      hit = &g;
      break;
    }
  }
  if (!hit) {
    if (ws->graphs.size() >= 16) {  // evict the least recently used
      auto lru = std::min_element(ws->graphs.begin(), ws->graphs.end(),
                                  [](const rs_graph_entry& x, const rs_graph_entry& y) {
                                    return x.last_use < y.last_use;
                                  });
      cudaGraphExecDestroy(lru->exec);
      ws->graphs.erase(lru);
    }
    rs_graph_entry e;
    e.t = t;
    e.ids = d_ids;
    e.grads = d_grads;
    e.out = d_out;
    e.n = n;
    e.mirror = mirror;
    e.pbuf = ws->pbuf;
    std::memcpy(e.opt, &o, sizeof(o));
    cudaStream_t cs = ws->cap_stream;
    RS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    const uint64_t launches_before = launches();
    st = step_enqueue(ws, t, d_ids, n, d_grads, d_out, o, TT, mirror, cs);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    if (st) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
    const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return cuda_fail(ie, "cudaGraphInstantiate");
    e.launches = launches() - launches_before;
    ws->graphs.push_back(e);
    hit = &ws->graphs.back();
    // capture only recorded the launches: undo the launch count of the capture
    count_launch(0 - e.launches);
  }
  hit->last_use = ++ws->graph_clock;
  RS_CUDA(cudaGraphLaunch(hit->exec, s));
  count_launch(hit->launches);
  ws->last_n = n;
  ws->last_tile = TT;
  ws->last_table = t;
  ws->have_forward = false;
  t->applies++;
  return table_mirror_commit(t, mirror, s);
}

int rs_sparse_update(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, const rs_optimizer_params* opt, void* stream) {
  // GradAccumulator::accumulate + apply for one window (sparse_update.cpp:45-83):
  // dedup, zero-vivify absent ids, segment-reduce fused with the update.
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_sparse_update: null handle");
  cudaStream_t s = S(stream);
  OptArgs o;
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  const uint32_t TT = tile_tokens_for_dim(t->desc.dim);
  st = dedup_run(ws, d_ids, n, TT, s);
  if (st) return st;
  ws->have_forward = false;
  ws->last_table = t;
  if (n == 0) return RS_OK;
  st = table_ensure_any(t, ws->unique, ws->ctr + 2, n, ws->urow, ws->urow64, ws->u_slot,
                        ws->srow, s);
  if (st) return st;
  k_inverse<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(ws->slot_of, ws->suidx, (uint32_t)n,
                                                      ws->inverse);
  RS_LAUNCH_CHECK("k_inverse");
  st = launch_reduce(ws, t, d_grads, n, o, nullptr, s);
  if (st) return st;
  t->applies++;
  return RS_OK;
}

int rs_workspace_results(rs_workspace* ws, const uint64_t** d_unique, const int32_t** d_inverse,
                         const uint32_t** d_n_unique, const int64_t** d_rows) {
  if (!ws) return fail(RS_ERR_CONFIG, "rs_workspace_results: null workspace");
  if (d_unique) *d_unique = ws->unique;
  if (d_inverse) *d_inverse = ws->inverse;
  if (d_n_unique) *d_n_unique = ws->ctr + 2;
  if (d_rows) *d_rows = ws->urow64;
  return RS_OK;
}

int rs_workspace_n_unique(rs_workspace* ws, uint64_t* out) {
  if (!ws || !out) return fail(RS_ERR_CONFIG, "rs_workspace_n_unique: null argument");
  RS_CUDA(cudaDeviceSynchronize());
  uint32_t n = 0;
  RS_CUDA(cudaMemcpy(&n, ws->ctr + 2, 4, cudaMemcpyDeviceToHost));
  *out = n;
  return RS_OK;
}

int rs_accumulate(rs_workspace* ws, const float* d_grads, uint64_t n, float* d_sums,
                  void* stream) {
  if (!ws || !ws->last_table) return fail(RS_ERR_CONFIG, "rs_accumulate: no forward on workspace");
  if (ws->last_n != n) return fail(RS_ERR_CONFIG, "rs_accumulate: batch size differs from forward");
  if (n == 0) return RS_OK;
  OptArgs o;
  std::memset(&o, 0, sizeof(o));
  return launch_reduce(ws, ws->last_table, d_grads, n, o, d_sums, S(stream));
}

int rs_apply_aggregated(rs_table* t, const uint64_t* d_keys, uint64_t n, const float* d_sums,
                        const rs_optimizer_params* opt, void* stream) {
  if (!t) return fail(RS_ERR_CONFIG, "rs_apply_aggregated: null table");
  if (n == 0) return RS_OK;
  cudaStream_t s = S(stream);
  OptArgs o;
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  int64_t* rows = nullptr;
  RS_CUDA(cudaMallocAsync(&rows, n * 8, s));
  st = rs_table_ensure(t, d_keys, n, rows, stream);
  if (st) return st;
  const Shape sh = shape_for(t->desc.dim);
  const unsigned grid = grid_for(n, 8, 148 * 8);
#define RS_SHAPE(V, C)                                                                   \
  if (sh.vec == V && sh.ch == C) {                                                       \
    k_apply_sums<V, C><<<grid, 256, 0, s>>>(t->dev, rows, n, d_sums, o);                 \
    RS_LAUNCH_CHECK("k_apply_sums");                                                     \
    RS_CUDA(cudaFreeAsync(rows, s));                                                     \
    t->applies++;                                                                        \
    return RS_OK;                                                                        \
  }
  RS_SHAPE(4, 1) RS_SHAPE(4, 2) RS_SHAPE(4, 3) RS_SHAPE(4, 4)
  RS_SHAPE(2, 1) RS_SHAPE(2, 2)
  RS_SHAPE(1, 1) RS_SHAPE(1, 2) RS_SHAPE(1, 3) RS_SHAPE(1, 4) RS_SHAPE(1, 5) RS_SHAPE(1, 6)
  RS_SHAPE(1, 7) RS_SHAPE(1, 8)
#undef RS_SHAPE
  return fail(RS_ERR_CONFIG, "embedding_dim unsupported by the optimizer");
}

}  // extern "C"
