// step.cu -- dedup, jagged gather, segment-reduce + sparse optimizer (sm_100a).
//
// One training step of one shard.  Reference caller: run_workload
// (workload.cpp:506-581); for W = 1 distributed_lookup reduces to
// stage1_dedup + ensure + inverse expand (exchange_sim.cpp:117-233), then
// GradAccumulator::accumulate + apply (sparse_update.cpp:45-83).
//
// Fast step (rs_step / rs_forward / rs_backward), four kernels:
//   KA k_fdedup   per tile: smem dedup, one global scratch insert per (tile,
//                 id): slot, number of tiles containing the id; new ids get
//                 their unique index from one atomic per block
//   KB k_ftable   per unique id (8-lane group): find-or-insert-zero in the
//                 table (grouped bucket probing), partial-segment offsets
//                 (one atomic per block), hot-id list; cleans the scratch
//                 slots of the previous call (double-buffered scratch)
//   KC k_ftile    per tile: jagged gather out[t] = emb[row(t)] (128-bit row
//                 copies, 8 in flight per lane) fused with the segment
//                 reduce bookkeeping: tokens of ids with <= kCsrMax
//                 occurrences go into the id's CSR segment; tokens of hot ids
//                 are summed per (tile, id) in position order from a TMA bulk
//                 copy (cp.async.bulk -> UBLKCP) of the tile's gradient rows
//   KD k_finish   per id: CSR ids sort their positions and sum the gradient
//                 rows in the reference's token order (bit-exact); hot ids
//                 combine their tile partials in tile order; then one optimizer
//                 step per row (FP64, explicit _rn, no FMA)
// The internal unique numbering of the fast step is unspecified (atomic);
// the exact first-occurrence dedup of stage1_dedup (exchange_sim.cpp:87-98)
// is rs_dedup: tile insert with first positions + decoupled look-back scan.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "opt_dev.cuh"
#include "rs_host.hpp"
#include "dist_sync.cuh"
#include "scratch_dev.cuh"
#include "table_dev.cuh"

namespace rs {
namespace {

using namespace odev;
using namespace tdev;
using namespace sdev;

constexpr uint32_t kCsrMax = 64;  // ids with at most this many occurrences: exact-order CSR path

// ctr[] slots of the workspace counter block
enum : int { kCtrTicket = 0, kCtrDone = 1, kCtrNHot = 4, kCtrPartAlloc = 5, kCtrCsrAlloc = 6 };

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void k_clean(SetDev c) {
  clean_set(c, blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
}

__global__ void k_clear_all(SetDev c, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    c.skey[i] = kEmptyKey;
    c.sfirstx[i] = 0;
    c.sntile[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *c.cnt = 0;
}

// Block-local dedup of the tile's ids in smem.  Returns the local slot of the
// thread's id; *rep = this thread's smem CAS claimed the slot (the tile's
// representative of the id); with first_pos, first[p] = lowest thread index.
struct LocalTable {
  unsigned long long* key;
  uint32_t* first;
  uint32_t* gslot;
  uint32_t L;
};
__device__ __forceinline__ uint32_t local_insert(const LocalTable& lt, uint64_t id, uint64_t h,
                                                 uint32_t tid, bool first_pos, bool* rep) {
  uint32_t p;
  *rep = false;
  if (id == kEmptyKey) {
    p = lt.L;
    *rep = atomicCAS(&lt.key[p], kEmptyKey, 0ull) == kEmptyKey;
  } else {
    p = (uint32_t)(h >> 40) & (lt.L - 1);
    for (;;) {
      const unsigned long long prev = atomicCAS(&lt.key[p], kEmptyKey, (unsigned long long)id);
      if (prev == kEmptyKey) {
        *rep = true;
        break;
      }
      if (prev == id) break;
      p = (p + 1) & (lt.L - 1);
    }
  }
  if (first_pos) atomicMin(&lt.first[p], tid);
  return p;
}

// ---------------------------------------------------------------------------
// KA: fast dedup tile.  blockDim.x == TT.
__global__ void k_fdedup(const uint64_t* __restrict__ ids, uint32_t n_host, SetDev S,
                         uint32_t* __restrict__ slot_of, uint64_t* __restrict__ unique,
                         uint32_t* __restrict__ ctr, const uint32_t* __restrict__ d_n,
                         uint32_t* __restrict__ tok_rank) {
  pdl_trigger();  // KB may get resident (it waits for this grid)
  const uint32_t n = d_n ? *d_n : n_host;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t TT = blockDim.x;
  const uint32_t L = 2 * TT;
  LocalTable lt;
  lt.L = L;
  lt.key = reinterpret_cast<unsigned long long*>(smem);
  lt.first = reinterpret_cast<uint32_t*>(lt.key + L + 1);
  lt.gslot = lt.first + L + 1;
  uint32_t* lnew = lt.gslot + L + 1;  // [L + 1] local index of new ids (+1), 0 = not new
  uint32_t* lcnt = lnew + L + 1;      // [L + 1] occurrences of the id in the tile
  __shared__ uint32_t s_nnew, s_base;
  const uint32_t tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) {
    ctr[kCtrNHot] = 0;       // filled by KB
    ctr[kCtrCsrAlloc] = 0;
    ctr[kCtrPartAlloc] = 0;  // partial segments, allocated by KB
  }
  for (uint32_t i = tid; i <= L; i += TT) {
    lt.key[i] = kEmptyKey;
    lnew[i] = 0;
    lcnt[i] = 0;
  }
  if (tid == 0) s_nnew = 0;
  __syncthreads();
  const uint32_t t = blockIdx.x * TT + tid;
  const bool valid = t < n;
  uint64_t id = 0, h = 0;
  uint32_t p = 0;
  bool rep = false;
  unsigned long long first0 = kEmptyKey;
  uint32_t lr = 0;
  if (valid) {
    id = ids[t];
    h = hash64(id);
    // the global slot's key, read now: overlaps the tile-local dedup below
    if (id != kEmptyKey) first0 = __ldcg(&S.skey[h & S.smask]);
    p = local_insert(lt, id, h, tid, false, &rep);
    lr = atomicAdd(&lcnt[p], 1u);  // rank within the tile (any order: KD sorts)
  }
  __syncthreads();
  if (rep) {
    bool fresh = false;
    const uint64_t gs = scratch_insert(S, id, h, &fresh, &first0);
    atomicAdd(&S.sntile[gs], 1u);
    if (tok_rank)  // the tile's base within the id's occurrences (lt.first is free here)
      lt.first[p] = atomicAdd(&S.sfirstx[gs], lcnt[p]);
    else
      atomicAdd(&S.sfirstx[gs], lcnt[p]);  // occurrence count
    lt.gslot[p] = (uint32_t)gs;
    if (fresh) lnew[p] = atomicAdd(&s_nnew, 1u) + 1;
  }
  __syncthreads();
  if (tid == 0 && s_nnew) s_base = atomicAdd(S.cnt, s_nnew);
  __syncthreads();
  if (rep && lnew[p]) {
    const uint32_t u = s_base + lnew[p] - 1;
    const uint32_t gs = lt.gslot[p];
    S.suidx[gs] = u;
    S.u_slot[u] = gs;
    unique[u] = id;
  }
  if (valid) {
    slot_of[t] = lt.gslot[p];
    // the token's rank among all occurrences of its id: KC places its CSR
    // position there without an atomic
    if (tok_rank) tok_rank[t] = lt.first[p] + lr;
  }
}

// ---------------------------------------------------------------------------
// KB: per unique id find-or-insert-zero + partial segments + hot list, and
// cleaning of the other scratch set.  One id per 8-lane group; the grid
// covers every possible id (blocks beyond n_unique only clean).
struct FTableArgs {
  TableDev* td;
  SetDev use;
  SetDev clean;
  bool do_clean;
  bool do_table;  // false: metadata only (bounded tables resolve rows separately)
  const uint64_t* unique;
  uint32_t* u_ntile;
  uint32_t* u_poff;
  uint32_t* u_ticket;
  uint32_t* urow;
  int64_t* urow64;
  uint32_t* hot_list;
  uint32_t* u_cnt;
  uint32_t* ctr;
  rs_dist_send send;  // sharded requester: ids to their owners (peers == null: off)
};

constexpr unsigned kGroups = 32;  // 8-lane groups per 256-thread block

__global__ void __launch_bounds__(256, 8) k_ftable(FTableArgs a) {
  pdl_wait();
  pdl_trigger();
  TableDev* td = a.td;
  const TableDesc d = td->d;
  const unsigned long long free_n0 = td->c.free_n;
  const unsigned long long fresh0 = td->c.fresh_next;
  const uint32_t tick_now = td->c.tick + 1;
  if (a.do_clean)
    clean_set(a.clean, blockIdx.x * (uint64_t)blockDim.x + threadIdx.x,
              (uint64_t)gridDim.x * blockDim.x);
  const uint32_t nu = *a.use.cnt;
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  __shared__ unsigned long long s_ins, s_reuse;
  __shared__ uint32_t s_wc[8], s_wp[8], s_bc, s_bp;
  __shared__ uint32_t s_ocnt[64], s_obase[64];  // sharded send: per-owner block counts (world <= 64)
  if (threadIdx.x == 0) {
    s_ins = 0;
    s_reuse = 0;
  }
  for (uint32_t r = threadIdx.x; r < 64; r += blockDim.x) s_ocnt[r] = 0;
  __syncthreads();
  // every warp runs the same trip count (shuffles below are warp-wide, the
  // allocation block-wide)
  const uint32_t per_iter = gridDim.x * kGroups;
  for (uint32_t base = 0; base < nu; base += per_iter) {
    const uint32_t i = base + blockIdx.x * kGroups + (threadIdx.x >> 3);
    const bool active = i < nu;
    uint64_t key = 0;
    uint32_t slot = 0, nt = 0, cnt = 0;
    if (active) {
      key = a.unique[i];
      slot = a.use.u_slot[i];
      nt = a.use.sntile[slot];
      cnt = a.use.sfirstx[slot];
    }
    // the probe's first slot window depends only on the key: prefetch it into
    // L2 now (overlaps the scratch loads and the block-wide allocation below)
    if (a.do_table && active && g == 0) {
      const uint64_t b = (hash64(key) >> 32) & d.nb_mask;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(d.slots + b * kBucket));
    }
    const bool hot = cnt > kCsrMax;
    // segments: CSR of the id's token positions (exact-order path) or its
    // per-tile partial sums (hot path); warp-aggregated allocation
    const uint32_t want_c = (active && g == 0 && !hot) ? cnt : 0u;
    const uint32_t want_p = (active && g == 0 && hot) ? nt : 0u;
    uint32_t ic = want_c, ip = want_p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yc = __shfl_up_sync(kFull, ic, o);
      const uint32_t yp = __shfl_up_sync(kFull, ip, o);
      if (lane >= (unsigned)o) {
        ic += yc;
        ip += yp;
      }
    }
    // block-aggregated allocation: one atomic per block and counter (the
    // counters are single addresses every block hits)
    const uint32_t tc = __shfl_sync(kFull, ic, 31), tp = __shfl_sync(kFull, ip, 31);
    const uint32_t warp = threadIdx.x >> 5;
    if (lane == 0) {
      s_wc[warp] = tc;
      s_wp[warp] = tp;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t rc = 0, rp = 0;
      for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) {
        const uint32_t xc = s_wc[w], xp = s_wp[w];
        s_wc[w] = rc;
        s_wp[w] = rp;
        rc += xc;
        rp += xp;
      }
      s_bc = rc ? atomicAdd(&a.ctr[kCtrCsrAlloc], rc) : 0u;
      s_bp = rp ? atomicAdd(&a.ctr[kCtrPartAlloc], rp) : 0u;
    }
    __syncthreads();
    const uint32_t bc = s_bc + s_wc[warp], bp = s_bp + s_wp[warp];
    __syncthreads();  // s_w* / s_b* are rewritten by the next trip
    if (active && g == 0) {
      a.u_cnt[i] = cnt;
      a.u_ntile[i] = hot ? nt : 0u;  // 0 marks the CSR path
      a.u_poff[i] = hot ? bp + ip - want_p : bc + ic - want_c;
      a.u_ticket[i] = 0;
      if (hot) a.hot_list[atomicAdd(&a.ctr[kCtrNHot], 1u)] = i;
    }
    if (a.send.peers) {  // owner partition: one lane per group holds the id
      // positions: block-local counters per owner, then one global atomic per
      // (block, owner) -- the per-owner counters are hot single addresses
      const bool mine = active && g == 0;
      const uint32_t o = mine ? (uint32_t)(hash64(key) % a.send.world) : 0u;
      uint32_t jl = 0;
      if (mine) jl = atomicAdd(&s_ocnt[o], 1u);
      __syncthreads();
      for (uint32_t r = threadIdx.x; r < a.send.world; r += blockDim.x) {
        const uint32_t c = s_ocnt[r];
        s_obase[r] = c ? atomicAdd(&a.send.send_cnt[r], c) : 0u;
        s_ocnt[r] = 0;
      }
      __syncthreads();
      if (mine) {
        const uint32_t j = s_obase[o] + jl;
        reinterpret_cast<uint64_t*>(a.send.peers[o] + a.send.off_ids)[(size_t)a.send.rank * a.send.cap + j] = key;
        const uint32_t sp = o * a.send.cap + j;
        a.send.send_pos[i] = sp;
        a.use.srow[slot] = sp;  // the gather reads the received row sp
      }
    }
    if (!a.do_table || !active) continue;
    const uint32_t row = find_or_insert_group(td, d, key, g, gbase, gmask, tick_now, free_n0, fresh0,
                                              &s_ins, &s_reuse);
    if (g == 0) {
      a.urow[i] = row;
      a.urow64[i] = row == kNoRow ? -1 : (int64_t)row;
      a.use.srow[slot] = row;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_ins) atomicAdd(&td->c.inserted, s_ins);
    if (s_reuse) atomicAdd(&td->c.reused, s_reuse);
  }
  if (a.do_table) launch_epilogue(td, free_n0, fresh0, true, tick_now);
  if (a.send.peers) {  // last block: counts + ids flags at every owner (step epoch e)
    __shared__ bool last;
    __shared__ unsigned long long e;
    __syncthreads();
    if (threadIdx.x == 0) {
      e = *a.send.epoch + 1;  // read before arriving; published by the last block
      unsigned int old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.send.done) : "memory");
      last = old == gridDim.x - 1;
      if (last) fence_sys();
    }
    __syncthreads();
    if (last) {
      for (uint32_t r = threadIdx.x; r < a.send.world; r += blockDim.x) {
        *a.send.cnt_ptrs[r] = a.send.send_cnt[r];
        a.send.trace_ids_sent[r] = a.send.send_cnt[r];
      }
      if (threadIdx.x == 0) *a.send.trace_requested = a.send.n_tokens;
      __syncthreads();
      for (uint32_t r = threadIdx.x; r < a.send.world; r += blockDim.x) {
        st_release_sys(a.send.flag_ptrs[r], e);
        a.send.send_cnt[r] = 0;
      }
      if (threadIdx.x == 0) {
        *a.send.epoch = e;
        *a.send.done = 0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// KC: jagged gather fused with the tile segment-reduce.
struct TileArgs {
  const TableDev* td;
  SetDev use;
  uint32_t* clean_cnt;  // zeroed by block 0 (the other set was cleaned by KB)
  const uint32_t* slot_of;
  uint32_t n;
  int32_t* inverse;
  float* out;           // gather destination (null: no gather)
  const float* grads;   // reduce source (null: no reduce)
  bool tma;
  const uint32_t* u_ntile;
  const uint32_t* u_poff;
  uint32_t* u_ticket;
  float* pbuf;
  uint32_t* ptile;
  uint32_t* csr_pos;
  const uint32_t* d_n;      // device token count (null: n)
  const uint32_t* pos_map;  // CSR value per token (null: token index)
  const uint32_t* tok_rank; // rank of the token among its id's occurrences (null: atomic placement)
  bool stage;               // hot ids possible: stage the tile's gradient rows
  rs_dist_sync sync;        // sharded step: wait for the peers' rows before gathering
  // f64 sum of every gathered value (run_workload's emb_checksum), fused into
  // the gather: per-tile partials, the last tile sums them in tile order
  double* csum_out = nullptr;
  double* csum_part = nullptr;
  unsigned int* csum_ticket = nullptr;
  uint32_t persist_tiles = 0;  // kTileHot: > 0 = number of tiles walked by a smaller grid
};

// MODE kTileFull: gather + CSR placement + hot-id tile partials (one pass);
// kTileGatherCsr: gather + CSR placement only (no staging smem: many blocks
// per SM); kTileHot: hot-id tile partials only (runs beside the CSR finish)
enum : int { kTileFull = 0, kTileGatherCsr = 1, kTileHot = 2 };

#ifndef RS_KC1_MINB
#define RS_KC1_MINB 4
#endif
// One tile of KC (`iter`: how many tiles this block processed before -- the
// TMA barrier's phase parity).
template <int VEC, int CH, int LPR, int MODE>
__device__ __forceinline__ void ftile_body(const TileArgs& a, const uint32_t tile, const uint32_t iter) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t TT = blockDim.x;
  const uint32_t NW = TT >> 5;
  const uint32_t L = 2 * TT;
  const uint32_t D = a.td->d.dim;
  const bool red = a.grads != nullptr;
  float* sg = reinterpret_cast<float*>(smem);  // [TT x D] staged gradients (reduce)
  unsigned char* p = smem + ((MODE != kTileGatherCsr && red) ? (size_t)TT * D * 4 : 0);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(p);
  p += 16;
  uint32_t* lkey = reinterpret_cast<uint32_t*>(p);
  uint32_t* lfirst = lkey + L;
  uint32_t* lgroup = lfirst + L;
  uint32_t* gcnt = lgroup + L;
  uint32_t* goff = gcnt + TT;
  uint32_t* gu = goff + TT;
  uint32_t* gdst = gu + TT;
  uint32_t* wsum = gdst + TT;      // [32]
  uint32_t* misc = wsum + 32;      // [0] ng
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(misc + 32);  // [NW x TT]
  uint16_t* csr = wcnt + (size_t)NW * TT;                    // [TT]

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t t0 = tile * TT;
  const uint32_t nn = a.d_n ? *a.d_n : a.n;
  if (a.clean_cnt && tile == 0 && tid == 0) *a.clean_cnt = 0;
  if (t0 >= nn) return;
  dist_wait(a.sync);
  const uint32_t rows = min(TT, nn - t0);

  if (MODE != kTileGatherCsr && red && a.stage) {
    for (uint32_t i = tid; i < L; i += TT) {
      lkey[i] = kFull;
      lfirst[i] = kFull;
    }
    for (uint32_t i = tid; i < NW * TT; i += TT) wcnt[i] = 0;
    if (a.tma) {
      if (tid == 0) {
        if (iter == 0) {
          asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        // the previous tile's generic-proxy reads of sg happen before these async writes
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
  }

  // ---- resolve every token: slot -> (unique id, table row)
  const bool valid = tid < rows;
  uint32_t u = kFull, r = 0, trank = 0;
  if (valid) {
    const uint32_t s = __ldg(a.slot_of + t0 + tid);
    if (MODE != kTileHot && a.tok_rank) trank = __ldg(a.tok_rank + t0 + tid);
    u = __ldcg(a.use.suidx + s);
    r = __ldcg(a.use.srow + s);
  }
  // the id's CSR metadata, issued with the gather's row loads
  uint32_t nt = 0, upoff = 0;
  if (red && valid) {
    nt = __ldg(a.u_ntile + u);
    if (MODE != kTileHot) upoff = __ldg(a.u_poff + u);
  }

  // ---- gather: warp w copies the rows of tokens [32w, 32w + 32)
  if (MODE != kTileHot && a.out) {
    if (valid) a.inverse[t0 + tid] = (int32_t)u;
    constexpr int RPI = 32 / LPR;
    constexpr int ITERS = 32 / RPI;
    constexpr int BATCH = ITERS < 8 ? ITERS : 8;
    const uint32_t D4 = D >> 2;
    const float4* __restrict__ emb = reinterpret_cast<const float4*>(a.td->d.emb);
    float4* __restrict__ o4 = reinterpret_cast<float4*>(a.out);
    const uint32_t sub = lane / LPR, l = lane % LPR;
    const uint32_t wb = warp * 32;
    const uint32_t cnt = rows > wb ? min(32u, rows - wb) : 0u;
    const bool csum = a.csum_out != nullptr;
    double cs = 0.0;
#pragma unroll
    for (int b0 = 0; b0 < ITERS; b0 += BATCH) {
      uint32_t rr[BATCH];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) rr[k] = __shfl_sync(kFull, r, (b0 + k) * RPI + sub);
      for (uint32_t jj = 0; jj < D4; jj += LPR) {
        const uint32_t j = jj + l;
        float4 v[BATCH];
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          const uint32_t tok = (b0 + k) * RPI + sub;
          if (tok < cnt && j < D4)  // rows written by peers this step: L2 (coherent) loads
            v[k] = a.sync.wait_flags ? __ldcg(emb + (size_t)rr[k] * D4 + j) : __ldg(emb + (size_t)rr[k] * D4 + j);
        }
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          const uint32_t tok = (b0 + k) * RPI + sub;
          if (tok < cnt && j < D4) {
            __stcs(o4 + (size_t)(t0 + wb + tok) * D4 + j, v[k]);
            if (csum) cs += (double)v[k].x + (double)v[k].y + (double)v[k].z + (double)v[k].w;
          }
        }
      }
    }
    if (csum) {  // fixed reduction tree: the result does not depend on timing
      __shared__ double s_cs[32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(kFull, cs, o);
      if (lane == 0) s_cs[warp] = cs;
      __syncthreads();
      if (warp == 0) {
        double x = lane < NW ? s_cs[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        unsigned last = 0;
        if (lane == 0) {
          a.csum_part[tile] = x;
          __threadfence();
          last = atomicAdd(a.csum_ticket, 1u) == gridDim.x - 1;
        }
        if (__shfl_sync(kFull, last, 0)) {
          __threadfence();
          double y = 0.0;
          for (uint32_t b = lane; b < gridDim.x; b += 32) y += __ldcg(a.csum_part + b);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(kFull, y, o);
          if (lane == 0) {
            *a.csum_out = y;
            *a.csum_ticket = 0;
          }
        }
      }
    }
  }
  if (!red) return;

  // ---- ids with <= kCsrMax occurrences: place the token position into the
  // id's CSR segment (warp-aggregated cursor; the finish kernel sorts it)
  const bool csr_tok = valid && nt == 0;
  if (MODE != kTileHot && a.tok_rank) {
    if (csr_tok) a.csr_pos[upoff + trank] = t0 + tid;
  } else if (MODE != kTileHot) {
    const uint32_t key = csr_tok ? u : (0xFFFF0000u | lane);
    const unsigned mm0 = __match_any_sync(kFull, key);
    const uint32_t leader = __ffs(mm0) - 1;
    uint32_t base = 0;
    if (csr_tok && lane == leader) base = atomicAdd(a.u_ticket + u, (uint32_t)__popc(mm0));
    base = __shfl_sync(kFull, base, leader);
    if (csr_tok)
      a.csr_pos[upoff + base + __popc(mm0 & lanemask_lt())] =
          a.pos_map ? __ldg(a.pos_map + t0 + tid) : t0 + tid;
  }
  const bool hotv = valid && nt > 0;
  if (MODE == kTileGatherCsr || !a.stage) return;  // no hot part here / none possible
  __syncthreads();  // lkey / lfirst / wcnt initialised by all threads above

  // ---- hot ids: group the tile's tokens by unique id (first occurrence)
  uint32_t ps = 0;
  if (hotv) {
    ps = hash32(u) & (L - 1);
    for (;;) {
      const uint32_t prev = atomicCAS(&lkey[ps], kFull, u);
      if (prev == kFull || prev == u) break;
      ps = (ps + 1) & (L - 1);
    }
    atomicMin(&lfirst[ps], tid);
  }
  __syncthreads();
  const bool head = hotv && lfirst[ps] == tid;
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
    const uint32_t tk = atomicAdd(a.u_ticket + u, 1u);
    const uint32_t slot = __ldg(a.u_poff + u) + tk;
    a.ptile[slot] = tile;
    gdst[lg] = slot;
  }
  __syncthreads();
  const uint32_t mylg = hotv ? lgroup[ps] : (0xFFFF0000u | lane);
  const unsigned mm = __match_any_sync(kFull, mylg);
  const uint32_t rw = __popc(mm & lanemask_lt());
  if (hotv && rw == 0) wcnt[warp * TT + mylg] = (uint16_t)__popc(mm);
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
  if (hotv) csr[goff[mylg] + wcnt[warp * TT + mylg] + rw] = (uint16_t)tid;
  if (a.tma) {
    asm volatile(
        "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(iter & 1u)
        : "memory");
  }
  __syncthreads();

  // ---- position-order sums, in place into the group's first row
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

  // ---- element-parallel stores of sums / partials
  if ((D & 3u) == 0) {
    const uint32_t D4 = D >> 2;
    const uint32_t nchunks = ng * D4;
    for (uint32_t q = tid; q < nchunks; q += TT) {
      const uint32_t g = q / D4, c = q - g * D4;
      const float4 sum = *reinterpret_cast<const float4*>(sg + (size_t)csr[goff[g]] * D + 4 * c);
      __stcg(reinterpret_cast<float4*>(a.pbuf + (size_t)gdst[g] * D) + c, sum);
    }
  } else {
    const uint32_t nchunks = ng * D;
    for (uint32_t q = tid; q < nchunks; q += TT) {
      const uint32_t g = q / D, e = q - g * D;
      a.pbuf[(size_t)gdst[g] * D + e] = sg[(size_t)csr[goff[g]] * D + e];
    }
  }
}

template <int VEC, int CH, int LPR, int MODE>
__global__ void __launch_bounds__(256, MODE == kTileGatherCsr ? RS_KC1_MINB : 3) k_ftile(TileArgs a) {
  pdl_wait();
  pdl_trigger();
  if (MODE == kTileHot && a.persist_tiles) {
    // persistent hot pass: fewer resident blocks, each walking tiles, so the
    // concurrent main branch (gather + CSR finish) keeps most of the SMs
    uint32_t iter = 0;
    for (uint32_t tile = blockIdx.x; tile < a.persist_tiles; tile += gridDim.x, ++iter) {
      ftile_body<VEC, CH, LPR, MODE>(a, tile, iter);
      __syncthreads();
    }
    return;
  }
  ftile_body<VEC, CH, LPR, MODE>(a, blockIdx.x, 0);
}

// scalar gather for D % 4 != 0 (the reduce part of KC handles any D)
__global__ void k_gather_scalar(const uint32_t* __restrict__ slot_of, SetDev use,
                                const TableDev* __restrict__ td, uint32_t n,
                                int32_t* __restrict__ inverse, float* __restrict__ out) {
  const uint32_t D = td->d.dim;
  const float* emb = td->d.emb;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lane = lane_id();
  for (uint64_t t = w; t < n; t += nw) {
    const uint32_t s = slot_of[t];
    const uint32_t r = __ldcg(use.srow + s);
    if (lane == 0) inverse[t] = (int32_t)__ldcg(use.suidx + s);
    for (uint32_t e = lane; e < D; e += 32) out[t * D + e] = emb[(size_t)r * D + e];
  }
}

// ---------------------------------------------------------------------------
// KD: finish every unique id.
struct FinishArgs {
  const uint32_t* n_unique;
  const uint32_t* n_hot;
  const uint32_t* hot_list;
  const uint32_t* u_ntile;  // 0: CSR path; > 0: tiles holding a partial (hot path)
  const uint32_t* u_poff;   // CSR offset / partial offset
  const uint32_t* u_cnt;    // occurrences
  uint32_t* u_ticket;
  const uint32_t* urow;
  const float* grads;
  const uint32_t* csr_pos;
  const float* pbuf;
  const uint32_t* ptile;
  uint32_t* porder;
  uint32_t bw;  // bitmap words = ceil(ntiles / 32)
  TableDev* td;
  float* sums_out;  // accumulate-only mode when non-null
  // sharded requester: the aggregated row of id u goes to the owner's
  // gradient receive buffer over NVLink (peer store)
  float* const* peer_dst;
  const uint32_t* send_pos;
  uint32_t cap, rank;
  uint64_t dbg_nrows, dbg_ncsr;  // RS_BOUNDS builds: valid grad rows / csr_pos entries
  rs_dist_sync sync;             // sharded step: prologue wait / grid-level signal
};

__device__ __forceinline__ float* sum_dst(const FinishArgs& a, uint32_t uu, uint32_t D) {
  if (a.peer_dst) {
    const uint32_t sp = a.send_pos[uu];
    const uint32_t o = sp / a.cap, j = sp - o * a.cap;
    return a.peer_dst[o] + ((size_t)a.rank * a.cap + j) * D;
  }
  return a.sums_out ? a.sums_out + (size_t)uu * D : nullptr;
}

// Sum of rows src(order[k]) for k in [r0, r1) in that order, PF in flight.
template <int VEC, int CH, bool kPartial>
__device__ __forceinline__ void ordered_sum(const FinishArgs& a, const uint32_t* order,
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
        const float* src = kPartial ? a.pbuf + (size_t)(poff + i) * D : a.grads + (size_t)i * D;
        if (j0 + jj < cnt) load_vec<VEC, CH>(src, D, x[jj], false);
      }
#pragma unroll
      for (int jj = 0; jj < PF; ++jj)
        if (j0 + jj < cnt) add_acc<VEC, CH>(acc, x[jj]);
    }
  }
}

// CSR path, element-parallel: G = D/4 threads per id, each owning one float4
// chunk of the row.  The id's <= kCsrMax token positions are ranked within the
// group (shuffles), written sorted to smem, and the gradient rows are summed
// in position order (the reference's accumulate order) -> bit-exact sums.
#ifndef RS_CSR_MINB
#define RS_CSR_MINB 5  // measured: 5 (48 regs) beats 4 / 6 / 8 at config 1 (G = 16, NV = 1)
#endif
template <int G, int NV>
__global__ void __launch_bounds__(256, NV == 1 ? RS_CSR_MINB : 4) k_finish_csr(FinishArgs a, OptArgs o) {
  // G lanes per id, each owning NV float4 chunks of the row (chunk gl + j*G)
  WarpTrace wt_(a.sync.tl, 14);
  pdl_wait();
  constexpr int PPT = (int)(kCsrMax / G);  // positions held per thread
  __shared__ uint32_t order_s[(256 / G) * kCsrMax];
  const TableDesc d = a.td->d;
  const uint32_t D4 = d.dim >> 2;
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const uint32_t gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << gbase;
  const uint32_t gpb = blockDim.x / G;
  uint32_t* order = order_s + (threadIdx.x / G) * kCsrMax;
  const uint32_t gid = blockIdx.x * gpb + threadIdx.x / G;
  const uint32_t ngroups = gridDim.x * gpb;
  dist_wait(a.sync);
  const uint32_t nu = *a.n_unique;
  const float4* __restrict__ g4 = reinterpret_cast<const float4*>(a.grads);
  const bool sums = a.sums_out || a.peer_dst;
  for (uint32_t uu = gid; uu < nu; uu += ngroups) {
    // the id's metadata in one round trip (the hot test must not serialize it)
    const uint32_t nt = __ldg(a.u_ntile + uu);
    const uint32_t c = __ldg(a.u_cnt + uu), off = __ldg(a.u_poff + uu);
    const uint32_t row = sums ? 0u : __ldg(a.urow + uu);
    if (nt != 0) continue;  // hot path (group-uniform)
#ifdef RS_BOUNDS
    if (c > kCsrMax || off + c > a.dbg_ncsr) {
      if (gl == 0) printf("k_finish_csr: uu %u c %u off %u ncsr %llu\n", uu, c, off, (unsigned long long)a.dbg_ncsr);
      continue;
    }
#endif
    // issue the row loads early: independent of the gradient sum
    float4 wv[NV], vv[NV], mv[NV];
    float4* rw = reinterpret_cast<float4*>(d.emb);
    float4* rv = reinterpret_cast<float4*>(d.s2);
    float4* rm = reinterpret_cast<float4*>(d.s1);
    const size_t rbase = (size_t)row * D4 + gl;
    uint32_t st0 = 0;  // the row's step counter, also loaded early
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      wv[j] = vv[j] = mv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!sums && row != kNoRow) {
        wv[j] = rw[rbase + j * G];
        vv[j] = rv[rbase + j * G];
        if (rm) mv[j] = rm[rbase + j * G];
      }
    }
    if (!sums && row != kNoRow && gl == 0) st0 = d.step[row];
    uint32_t p[PPT], r[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const uint32_t k = gl + j * G;
      p[j] = k < c ? __ldg(a.csr_pos + off + k) : kFull;
      r[j] = 0;
    }
    // rank every held position against all c positions of the id
#pragma unroll
    for (int jq = 0; jq < PPT; ++jq) {
      if ((uint32_t)(jq * G) >= c) break;
      // lanes >= c hold the kFull sentinel, which ranks nothing: skip them
      const uint32_t lim = min((uint32_t)G, c - (uint32_t)(jq * G));
      for (uint32_t src = 0; src < lim; ++src) {
        const uint32_t q = __shfl_sync(gmask, p[jq], src, G);
#pragma unroll
        for (int j = 0; j < PPT; ++j) r[j] += q < p[j];
      }
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j)
      if (gl + j * G < c) order[r[j]] = p[j];
    __syncwarp(gmask);
#ifdef RS_BOUNDS
    {
      bool bad = false;
      for (uint32_t k2 = 0; k2 < c; ++k2) bad |= order[k2] >= a.dbg_nrows;
      if (!sums && row != kNoRow && row >= d.row_cap) bad = true;
      if (a.peer_dst && a.send_pos[uu] >= a.cap * 64u) bad = true;
      if (bad) {
        if (gl == 0) printf("k_finish_csr: uu %u c %u row %u order0 %u nrows %llu sp %u\n", uu, c, row,
                            order[0], (unsigned long long)a.dbg_nrows, a.peer_dst ? a.send_pos[uu] : 0u);
        continue;
      }
    }
#endif
    // gradient rows summed in token order (the reference's accumulate order)
    float4 acc[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int B = NV == 1 ? 4 : 2;  // rows in flight per step of the loop
    constexpr int B2 = 2 * B;           // long lists: twice as many in flight
    uint32_t k = 0;
    for (; k + B2 <= c; k += B2) {
      float4 x[B2][NV];
#pragma unroll
      for (int q = 0; q < B2; ++q)
#pragma unroll
        for (int j = 0; j < NV; ++j) x[q][j] = g4[(size_t)order[k + q] * D4 + gl + j * G];
#pragma unroll
      for (int q = 0; q < B2; ++q)
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          acc[j].x += x[q][j].x;
          acc[j].y += x[q][j].y;
          acc[j].z += x[q][j].z;
          acc[j].w += x[q][j].w;
        }
    }
    for (; k + B <= c; k += B) {
      float4 x[B][NV];
#pragma unroll
      for (int q = 0; q < B; ++q)
#pragma unroll
        for (int j = 0; j < NV; ++j) x[q][j] = g4[(size_t)order[k + q] * D4 + gl + j * G];
#pragma unroll
      for (int q = 0; q < B; ++q)
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          acc[j].x += x[q][j].x;
          acc[j].y += x[q][j].y;
          acc[j].z += x[q][j].z;
          acc[j].w += x[q][j].w;
        }
    }
    for (; k < c; ++k) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const float4 x = g4[(size_t)order[k] * D4 + gl + j * G];
        acc[j].x += x.x;
        acc[j].y += x.y;
        acc[j].z += x.z;
        acc[j].w += x.w;
      }
    }
    __syncwarp(gmask);  // (u_ticket needs no reset: KB / k_own_table zero it every step)
    if (float* dst = sum_dst(a, uu, d.dim)) {
#pragma unroll
      for (int j = 0; j < NV; ++j) reinterpret_cast<float4*>(dst)[gl + j * G] = acc[j];
      continue;
    }
    if (row == kNoRow) continue;
    uint32_t st = 0;
    if (gl == 0) {
      st = st0 + 1;
      d.step[row] = st;
    }
    st = __shfl_sync(gmask, st, 0, G);
    double bc1 = 1.0, bc2 = 1.0;
    if (o.kind == RS_OPT_ADAM) {
      if (st < o.bc_len) {
        bc1 = o.bc[st];
        bc2 = o.bc[o.bc_len + st];
      } else {
        bc1 = 1.0 - pow(o.b1, (double)st);
        bc2 = 1.0 - pow(o.b2, (double)st);
      }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float* wp = reinterpret_cast<float*>(&wv[j]);
      float* vp = reinterpret_cast<float*>(&vv[j]);
      float* mp = reinterpret_cast<float*>(&mv[j]);
      const float* gp = reinterpret_cast<const float*>(&acc[j]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (o.kind == RS_OPT_ADAM)
          adam_elem(wp[e], mp[e], vp[e], gp[e], bc1, bc2, o);
        else
          adagrad_elem(wp[e], vp[e], gp[e], o);
      }
      rw[rbase + j * G] = wv[j];
      rv[rbase + j * G] = vv[j];
      if (rm) rm[rbase + j * G] = mv[j];
    }
  }
  dist_arrive(a.sync);
}

// Roles by block index:
//  [0, hot_blocks)  hot ids (> kCsrMax occurrences), one per block: the
//                   per-tile partials are ranked by tile (bitmap + prefix
//                   popcounts) and summed in tile order, split over the warps
//                   with a fixed split (deterministic, blocked order)
//  other blocks     warp per CSR id: its <= kCsrMax token positions are
//                   sorted and the gradient rows summed in position order --
//                   exactly the reference's accumulate order
//                   (sparse_update.cpp:49-54), so these sums are bit-exact
#ifndef RS_FIN_MINB
#define RS_FIN_MINB 3
#endif
template <int VEC, int CH>
__global__ void __launch_bounds__(256, RS_FIN_MINB) k_finish(FinishArgs a, OptArgs o, uint32_t hot_blocks) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem2[];
  const uint32_t NW = blockDim.x >> 5;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const TableDesc d = a.td->d;
  const uint32_t D = d.dim;
  dist_wait(a.sync);
  if (blockIdx.x >= hot_blocks) {
    uint32_t* order_w = reinterpret_cast<uint32_t*>(smem2) + warp * kCsrMax;  // [NW x 64]
    const uint32_t nu = *a.n_unique;
    const uint32_t stride = (gridDim.x - hot_blocks) * NW;
    for (uint32_t uu = (blockIdx.x - hot_blocks) * NW + warp; uu < nu; uu += stride) {
      if (__ldg(a.u_ntile + uu) != 0) continue;  // hot path
      const uint32_t c = __ldg(a.u_cnt + uu), off = __ldg(a.u_poff + uu);
      const uint32_t row = (a.sums_out || a.peer_dst) ? 0u : __ldg(a.urow + uu);
      const uint32_t p0 = lane < c ? __ldg(a.csr_pos + off + lane) : kFull;
      const uint32_t p1 = lane + 32 < c ? __ldg(a.csr_pos + off + 32 + lane) : kFull;
      uint32_t r0 = 0, r1 = 0;
      for (uint32_t j = 0; j < min(c, 32u); ++j) {
        const uint32_t q = __shfl_sync(kFull, p0, j);
        r0 += q < p0;
        r1 += q < p1;
      }
      for (uint32_t j = 32; j < c; ++j) {
        const uint32_t q = __shfl_sync(kFull, p1, j - 32);
        r0 += q < p0;
        r1 += q < p1;
      }
      if (lane < c) order_w[r0] = p0;
      if (lane + 32 < c) order_w[r1] = p1;
      __syncwarp();
      float acc[CH][VEC];
      ordered_sum<VEC, CH, false>(a, order_w, 0, 0, c, D, acc);
      __syncwarp();
      if (lane == 0) a.u_ticket[uu] = 0;
      if (float* dst = sum_dst(a, uu, D))
        store_vec<VEC, CH>(dst, D, acc);
      else
        apply_row<VEC, CH>(d, row, acc, o);
    }
    dist_arrive(a.sync);
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
    ordered_sum<VEC, CH, true>(a, a.porder + poff, poff, r0, r1, D, part);
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
      if (float* dst = sum_dst(a, uu, D))
        store_vec<VEC, CH>(dst, D, tot);
      else
        apply_row<VEC, CH>(d, __ldg(a.urow + uu), tot, o);
    }
    __syncthreads();
  }
  dist_arrive(a.sync);
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
// Exact first-occurrence dedup (rs_dedup): tile insert with first positions,
// then a single-pass decoupled look-back scan over tokens.
__global__ void k_dedup_tile_exact(const uint64_t* __restrict__ ids, uint32_t n, SetDev S,
                                   uint32_t* __restrict__ slot_of) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t TT = blockDim.x;
  const uint32_t L = 2 * TT;
  LocalTable lt;
  lt.L = L;
  lt.key = reinterpret_cast<unsigned long long*>(smem);
  lt.first = reinterpret_cast<uint32_t*>(lt.key + L + 1);
  lt.gslot = lt.first + L + 1;
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i <= L; i += TT) {
    lt.key[i] = kEmptyKey;
    lt.first[i] = kFull;
  }
  __syncthreads();
  const uint32_t t = blockIdx.x * TT + tid;
  const bool valid = t < n;
  uint64_t id = 0, h = 0;
  uint32_t p = 0;
  bool rep = false;
  if (valid) {
    id = ids[t];
    h = hash64(id);
    p = local_insert(lt, id, h, tid, true, &rep);
  }
  __syncthreads();
  if (valid && lt.first[p] == tid) {
    bool fresh = false;
    const uint64_t gs = scratch_insert(S, id, h, &fresh);
    atomicMax(&S.sfirstx[gs], ~t);  // ~min(position)
    lt.gslot[p] = (uint32_t)gs;
  }
  __syncthreads();
  if (valid) slot_of[t] = lt.gslot[p];
}

__device__ __forceinline__ uint64_t st_pack(uint32_t flag, uint32_t v) {
  return ((uint64_t)flag << 62) | (v & 0x3FFFFFFFFFFFFFFFull);
}

// Called by warp 0 of the block owning `tile`; returns the exclusive prefix.
__device__ uint32_t lookback(uint64_t* status, uint32_t tile, uint32_t agg) {
  const unsigned lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_release(&status[0], st_pack(2, agg));
    return 0;
  }
  if (lane == 0) st_release(&status[tile], st_pack(1, agg));
  uint32_t run = 0;
  int64_t j = (int64_t)tile - 1;
  for (;;) {
    const int64_t idx = j - lane;
    const uint64_t s = idx >= 0 ? ld_acquire(&status[idx]) : st_pack(2, 0);
    const uint32_t flag = (uint32_t)(s >> 62);
    const unsigned m0 = __ballot_sync(kFull, flag == 0);
    const unsigned m2 = __ballot_sync(kFull, flag == 2);
    const int stop = m2 ? __ffs(m2) - 1 : 31;
    const unsigned need = stop == 31 ? kFull : ((2u << stop) - 1u);
    if (m0 & need) continue;  // a predecessor inside the window has not published yet
    uint32_t v = (int)lane <= stop ? (uint32_t)s : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    run += v;
    if (m2) break;
    j -= 32;
  }
  if (lane == 0) st_release(&status[tile], st_pack(2, agg + run));
  return run;
}

// Heads (first occurrences) get their unique index = rank in position order.
__global__ void __launch_bounds__(kScanThreads)
    k_dedup_compact(const uint64_t* __restrict__ ids, uint32_t n,
                    const uint32_t* __restrict__ slot_of, SetDev S, uint64_t* __restrict__ unique,
                    uint64_t* status, uint32_t* ctr, uint32_t ntiles, uint32_t* clean_cnt) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_prefix;
  __shared__ bool s_last;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(&ctr[kCtrTicket], 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  if (tile == 0 && tid == 0 && clean_cnt) *clean_cnt = 0;
  const uint32_t base = tile * kScanTile + tid * kScanItems;
  uint32_t sl[kScanItems];
  bool hd[kScanItems];
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint32_t t = base + k;
    hd[k] = false;
    sl[k] = 0;
    if (t < n) {
      sl[k] = slot_of[t];
      hd[k] = S.sfirstx[sl[k]] == ~t;
    }
    mine += hd[k];
  }
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= (unsigned)o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, wi, o);
      if (lane >= (unsigned)o) wi += y;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    const uint32_t agg = __shfl_sync(kFull, wi, kScanThreads / 32 - 1);
    const uint32_t pre = lookback(status, tile, agg);
    if (lane == 0) s_prefix = pre;
  }
  __syncthreads();
  uint32_t ra = s_prefix + s_warp[warp] + incl - mine;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (hd[k]) {
      unique[ra] = ids[base + k];
      S.suidx[sl[k]] = ra;
      S.u_slot[ra] = sl[k];
      ++ra;
    }
  }
  if (tile == ntiles - 1 && tid == kScanThreads - 1) *S.cnt = ra;
  __syncthreads();
  if (tid == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s_last = atomicAdd(&ctr[kCtrDone], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {  // reset the tile ticket and the status words for the next call
    for (uint32_t i = tid; i < ntiles; i += kScanThreads) status[i] = 0;
    if (tid == 0) {
      ctr[kCtrTicket] = 0;
      ctr[kCtrDone] = 0;
    }
  }
}

__global__ void k_inverse(const uint32_t* __restrict__ slot_of, SetDev S, uint32_t n,
                          int32_t* __restrict__ inverse) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    inverse[i] = (int32_t)S.suidx[slot_of[i]];
}

__global__ void k_copy_unique(const uint64_t* __restrict__ src, const uint32_t* __restrict__ cnt,
                              uint64_t* __restrict__ dst, uint32_t* __restrict__ n_out) {
  const uint32_t n = *cnt;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && threadIdx.x == 0 && n_out) *n_out = n;
}

// ---------------------------------------------------------------------------
struct Shape {
  int vec, ch;
};
Shape shape_for(uint32_t D) {
  if (D % 128 == 0 && D / 128 <= 4) return {4, (int)(D / 128)};
  if (D % 64 == 0 && D / 64 <= 2) return {2, (int)(D / 64)};
  return {1, (int)((D + 31) / 32)};
}

int lpr_for(uint32_t D) {
  const uint32_t d4 = D / 4;
  if (d4 >= 32) return 32;
  if (d4 >= 16) return 16;
  if (d4 >= 8) return 8;
  if (d4 >= 4) return 4;
  if (d4 >= 2) return 2;
  return 1;
}

}  // namespace

uint32_t tile_tokens_for_dim(uint32_t D) {
  // staged gradient tile <= 64 KB so two tiles fit per SM
  static const uint32_t cap = [] {
    const char* e = getenv("RS_TILE_MAX");  // experiments: 64 / 128 / 256
    const uint32_t v = e ? (uint32_t)atoi(e) : 256u;
    return (v == 64 || v == 128 || v == 256) ? v : 256u;
  }();
  uint32_t tt = cap;
  while (tt > 32 && (uint64_t)tt * D * 4 > 65536) tt >>= 1;
  return tt;
}

// ---- host side -------------------------------------------------------------

// every k_ftile / k_finish instantiation opts in to large dynamic smem once
template <int V, int C, int LPR>
static int attr_tile() {
  RS_CUDA(cudaFuncSetAttribute(k_ftile<V, C, LPR, kTileFull>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024));
  if (LPR == 1)
    RS_CUDA(cudaFuncSetAttribute(k_ftile<V, C, 1, kTileHot>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024));
  return RS_OK;
}
template <int V, int C>
static int attr_shape() {
  int st = attr_tile<V, C, 1>() | attr_tile<V, C, 2>() | attr_tile<V, C, 4>() |
           attr_tile<V, C, 8>() | attr_tile<V, C, 16>() | attr_tile<V, C, 32>();
  if (st) return st;
  RS_CUDA(cudaFuncSetAttribute(k_finish<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               200 * 1024));
  return RS_OK;
}
static int set_smem_attrs() {
  static int done = 0;
  if (done) return RS_OK;

  int st = attr_shape<4, 1>() | attr_shape<4, 2>() | attr_shape<4, 3>() | attr_shape<4, 4>() |
           attr_shape<2, 1>() | attr_shape<2, 2>() | attr_shape<1, 1>() | attr_shape<1, 2>() |
           attr_shape<1, 3>() | attr_shape<1, 4>() | attr_shape<1, 5>() | attr_shape<1, 6>() |
           attr_shape<1, 7>() | attr_shape<1, 8>();
  if (st) return st;
  done = 1;
  return RS_OK;
}

static FTableArgs ftable_args(rs_workspace* ws, rs_table* t, int use) {
  FTableArgs a;
  a.td = t->dev;
  a.use = set_dev(ws, use);
  a.clean = set_dev(ws, use ^ 1);
  a.do_clean = true;
  a.do_table = true;
  a.unique = ws->unique;
  a.u_ntile = ws->u_ntile;
  a.u_poff = ws->u_poff;
  a.u_ticket = ws->u_ticket;
  a.urow = ws->urow;
  a.urow64 = ws->urow64;
  a.hot_list = ws->hot_list;
  a.u_cnt = ws->u_cnt;
  a.ctr = ws->ctr;
  return a;
}

static int launch_fdedup(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, int use,
                         cudaStream_t s, const uint32_t* d_n = nullptr, bool ranks = false) {
  const uint32_t TT = ws->last_tile;
  const uint32_t ntiles = (uint32_t)((n + TT - 1) / TT);
  const size_t sm = (size_t)(2 * TT + 1) * (8 + 4 + 4 + 4 + 4);
  carve(k_fdedup), k_fdedup<<<ntiles, TT, sm, s>>>(d_ids, (uint32_t)n, set_dev(ws, use), ws->slot_of, ws->unique,
                                  ws->ctr, d_n, ranks ? ws->tok_rank : nullptr);
  RS_LAUNCH_CHECK("k_fdedup");
  ws->tok_rank_ok = ranks;
  return RS_OK;
}

// KA + KB of the fast step on set `use`, cleaning set `use ^ 1`.
static int fast_dedup_table(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                            int use, cudaStream_t s) {
  int st = launch_fdedup(ws, d_ids, n, use, s, nullptr, true);
  if (st) return st;
  carve(k_ftable), k_ftable<<<grid_for(n, kGroups, 148 * 8), kGroups * kBucket, 0, s>>>(ftable_args(ws, t, use));
  RS_LAUNCH_CHECK("k_ftable");
  return RS_OK;
}

// partial sums: at most one per (tile, hot id) pair <= n
static int reduce_prepare(rs_workspace* ws, uint32_t D, uint64_t n, cudaStream_t s) {
  if (ws->pbuf_floats < n * D) {
    if (ws->pbuf) RS_CUDA(cudaFreeAsync(ws->pbuf, s));
    ws->pbuf_floats = ws->max_tokens * (uint64_t)D;
    RS_CUDA(cudaMallocAsync(&ws->pbuf, 2 * ws->pbuf_floats * sizeof(float), s));
  }
  return RS_OK;
}

// KC with gather and/or reduce.
static int launch_tile(rs_workspace* ws, rs_table* t, int use, uint64_t n, float* d_out,
                       const float* d_grads, bool clean_other, cudaStream_t s,
                       const rs_dist_opts* dopt = nullptr) {
  const uint32_t D = t->desc.dim;
  const uint32_t TT = ws->last_tile;
  const uint32_t ntiles = (uint32_t)((n + TT - 1) / TT);
  TileArgs a;
  a.td = (dopt && dopt->gather_view) ? reinterpret_cast<const TableDev*>(dopt->gather_view) : t->dev;
  a.use = set_dev(ws, use);
  a.d_n = dopt ? dopt->d_n : nullptr;
  a.pos_map = dopt ? dopt->pos_map : nullptr;
  a.stage = !(dopt && dopt->no_stage);
  if (dopt) a.sync = dopt->sync;
  a.clean_cnt = clean_other ? ws->set[use ^ 1].cnt : nullptr;
  a.slot_of = ws->slot_of;
  a.n = (uint32_t)n;
  a.inverse = ws->inverse;
  a.out = (D % 4 == 0) ? d_out : nullptr;
  a.grads = d_grads;
  a.tma = a.stage && d_grads && (D % 4 == 0) &&
          ((reinterpret_cast<uintptr_t>(d_grads) & 15u) == 0);
  a.u_ntile = ws->u_ntile;
  a.u_poff = ws->u_poff;
  a.u_ticket = ws->u_ticket;
  a.pbuf = ws->pbuf;
  a.ptile = ws->ptile;
  a.csr_pos = ws->csr_pos;
  // token ranks from this workspace's KA (not for the owner's received lists)
  a.tok_rank = (d_grads && ws->tok_rank_ok && !(dopt && (dopt->pos_map || dopt->d_n))) ? ws->tok_rank : nullptr;
  double* csum = dopt ? (dopt->d_n ? nullptr : dopt->csum) : ws->csum_dst;
  if (csum && d_out && D % 4 == 0) {
    a.csum_out = csum;
    a.csum_part = ws->csum_part;
    a.csum_ticket = ws->csum_ticket;
  }
  if (d_out && D % 4 != 0) {
    carve(k_gather_scalar), k_gather_scalar<<<grid_for(n, 8, 148 * 8), 256, 0, s>>>(ws->slot_of, a.use, t->dev,
                                                            (uint32_t)n, ws->inverse, d_out);
    RS_LAUNCH_CHECK("k_gather_scalar");
    if (!d_grads) {
      if (clean_other) RS_CUDA(cudaMemsetAsync(ws->set[use ^ 1].cnt, 0, 4, s));
      return RS_OK;
    }
  }
  const uint32_t NW = TT / 32;
  const size_t smem = (d_grads && a.stage ? (size_t)TT * D * 4 : 0) + 16 +
                      (size_t)(3 * 2 * TT + 4 * TT + 64) * 4 + (size_t)NW * TT * 2 +
                      (size_t)TT * 2 + 16;
  const Shape sh = shape_for(D);
  const int lpr = lpr_for(D);
  // single-GPU reduce: gather + CSR placement now (no staging smem, many
  // blocks per SM); the hot-id partials run in launch_finish beside the CSR
  // finish, which needs only the CSR placement
  const bool split = ws->split_kc && d_grads && a.stage && !dopt && D % 4 == 0;
  if (split) {
    // the hot pass needs only KA / KB: with the fork it runs on the aux
    // stream concurrently with the gather + CSR pass (and later the CSR
    // finish); launch_finish joins
    TileArgs a2 = a;
    a2.out = nullptr;
    a2.clean_cnt = nullptr;
    a2.csum_out = nullptr;
    // RS_KC2_PER_SM: resident hot-pass blocks per SM (0: one block per tile)
    static const unsigned kc2_per_sm = getenv("RS_KC2_PER_SM") ? (unsigned)atoi(getenv("RS_KC2_PER_SM")) : 0u;
    unsigned hot_grid = ntiles;
    if (kc2_per_sm && !a.d_n && ntiles > 148u * kc2_per_sm) {
      hot_grid = 148u * kc2_per_sm;
      a2.persist_tiles = ntiles;
    }
    cudaStream_t hs = s;
    if (ws->fork) {
      RS_CUDA(cudaEventRecord(ws->ev_fork, s));
      RS_CUDA(cudaStreamWaitEvent(ws->aux_stream, ws->ev_fork, 0));
      hs = ws->aux_stream;
      ws->kc_forked = true;
    }
    bool kc2 = false;
#define RS_HOT(V, C)                                                           \
  if (!kc2 && sh.vec == V && sh.ch == C) {                                     \
    carve(k_ftile<V, C, 1, kTileHot>), k_ftile<V, C, 1, kTileHot><<<hot_grid, TT, smem, hs>>>(a2);                \
    RS_LAUNCH_CHECK("k_ftile(hot)");                                           \
    kc2 = true;                                                                \
  }
    RS_HOT(4, 1) RS_HOT(4, 2) RS_HOT(4, 3) RS_HOT(4, 4) RS_HOT(2, 1) RS_HOT(2, 2)
    RS_HOT(1, 1) RS_HOT(1, 2) RS_HOT(1, 3) RS_HOT(1, 4) RS_HOT(1, 5) RS_HOT(1, 6) RS_HOT(1, 7)
    RS_HOT(1, 8)
#undef RS_HOT
    if (!kc2) return fail(RS_ERR_INVARIANT, "launch_tile: no hot tile kernel for this shape");
  }
#define RS_TILE(V, C, LP)                                                     \
  if (sh.vec == V && sh.ch == C && lpr == LP) {                               \
    if (split)                                                                \
      RS_CUDA(launch_pdl(ws->pdl_now, k_ftile<V, C, LP, kTileGatherCsr>,      \
                         ntiles, TT, 16, s, a));                              \
    else                                                                      \
      RS_CUDA(launch_pdl(ws->pdl_now, k_ftile<V, C, LP, kTileFull>, ntiles,   \
                         TT, smem, s, a));                                    \
    RS_LAUNCH_CHECK("k_ftile");                                               \
    return RS_OK;                                                             \
  }
#define RS_TILE_ALL(V, C) \
  RS_TILE(V, C, 1) RS_TILE(V, C, 2) RS_TILE(V, C, 4) RS_TILE(V, C, 8) RS_TILE(V, C, 16) RS_TILE(V, C, 32)
  RS_TILE_ALL(4, 1) RS_TILE_ALL(4, 2) RS_TILE_ALL(4, 3) RS_TILE_ALL(4, 4)
  RS_TILE_ALL(2, 1) RS_TILE_ALL(2, 2)
  RS_TILE_ALL(1, 1) RS_TILE_ALL(1, 2) RS_TILE_ALL(1, 3) RS_TILE_ALL(1, 4) RS_TILE_ALL(1, 5)
  RS_TILE_ALL(1, 6) RS_TILE_ALL(1, 7) RS_TILE_ALL(1, 8)
#undef RS_TILE_ALL
#undef RS_TILE
  return fail(RS_ERR_CONFIG, "embedding_dim " + std::to_string(D) + " unsupported");
}

// KD.
static int launch_finish(rs_workspace* ws, rs_table* t, int use, uint64_t n, const float* d_grads,
                         const OptArgs& o, float* sums_out, cudaStream_t s,
                         const rs_dist_opts* dopt = nullptr) {
  const uint32_t D = t->desc.dim;
  const uint32_t TT = ws->last_tile;
  const uint32_t ntiles = (uint32_t)((n + TT - 1) / TT);
  FinishArgs a;
  a.n_unique = ws->set[use].cnt;
  a.n_hot = ws->ctr + kCtrNHot;
  a.hot_list = ws->hot_list;
  a.u_ntile = ws->u_ntile;
  a.u_poff = ws->u_poff;
  a.u_cnt = ws->u_cnt;
  a.u_ticket = ws->u_ticket;
  a.urow = ws->urow;
  a.grads = d_grads;
  a.csr_pos = (dopt && dopt->csr_pos) ? dopt->csr_pos : ws->csr_pos;
  a.pbuf = ws->pbuf;
  a.ptile = ws->ptile;
  a.porder = ws->porder;
  a.bw = (ntiles + 31) / 32;
  a.td = t->dev;
  a.sums_out = sums_out;
  a.peer_dst = dopt ? dopt->peer_dst : nullptr;
  a.send_pos = dopt ? dopt->send_pos : nullptr;
  a.cap = dopt ? dopt->cap : 0;
  a.rank = dopt ? dopt->rank : 0;
  a.dbg_nrows = (dopt && dopt->d_n) ? ws->max_tokens : n;
  a.dbg_ncsr = (dopt && dopt->csr_pos) ? ~0ull : ws->max_tokens;
  const uint32_t hot_blocks = 2 * 148;
  const size_t smem = std::max<size_t>((size_t)8 * kCsrMax * 4,
                                       (size_t)2 * a.bw * 4 + 16 + (size_t)8 * D * 4 + 16);
  const uint32_t g4 = D % 4 == 0 ? D / 4 : 0;
  const int G = (g4 >= 2 && g4 <= 32 && !(g4 & (g4 - 1))) ? (int)g4 : 0;
  // CSR finish shape: G lanes x 1 float4 per id; RS_CSR_NV=2 runs G/2 lanes
  // x 2 float4 (twice the ids in flight per SM -- measured ~1 % slower at
  // config 1, kept for other shapes' experiments)
  // The sharded owner's update (no hot ids, <= W origins per id) runs G/2
  // lanes x 2 float4: at 48 registers its ids then fit one wave
  // (RS_OWN_NV=1: G lanes x 1)
  static const int nv_env = getenv("RS_CSR_NV") ? atoi(getenv("RS_CSR_NV")) : 1;
  static const int nv_own = getenv("RS_OWN_NV") ? atoi(getenv("RS_OWN_NV")) : 2;
  const bool owner = dopt && dopt->no_hot;
  const int NVc = ((owner ? nv_own : nv_env) == 2 && G >= 4) ? 2 : 1;
  const int Gc = G / NVc;
  // G > 0: CSR ids on s, hot ids concurrently on the forked aux stream
  const unsigned grid = G > 0 ? hot_blocks : hot_blocks + grid_for(n, 8, 148 * 24);
  cudaStream_t hs = s;
  bool fork = G > 0 && ws->fork && !(dopt && dopt->no_hot);
  bool split_fork = false;  // the hot finish follows the hot tile pass on aux_stream
  if (ws->kc_forked) {  // the hot tile pass already runs on the aux stream
    ws->kc_forked = false;
    split_fork = G > 0;
    if (G > 0) {
      hs = ws->aux_stream;
      fork = true;
    } else {  // one finish kernel for both paths: join first
      RS_CUDA(cudaEventRecord(ws->ev_join, ws->aux_stream));
      RS_CUDA(cudaStreamWaitEvent(s, ws->ev_join, 0));
      fork = false;
    }
  } else if (fork) {
    RS_CUDA(cudaEventRecord(ws->ev_fork, s));
    RS_CUDA(cudaStreamWaitEvent(ws->aux_stream, ws->ev_fork, 0));
    hs = ws->aux_stream;
  }
  const Shape sh = shape_for(D);
  // programmatic edges only where the same-stream predecessor is our tile kernel
  const bool pdl_hot = ws->pdl_now && split_fork;
  bool launched = G > 0 && dopt && dopt->no_hot;  // owner side: no hot ids possible
  static const unsigned csr_cap = getenv("RS_CSR_GRID") ? (unsigned)atoi(getenv("RS_CSR_GRID")) : 148u * 16u;
  const unsigned eg = G > 0 ? grid_for(n * (uint64_t)Gc, 256, csr_cap) : 0;
  if (dopt) {  // the blocks of both finish kernels arrive on one counter
    a.sync = dopt->sync;
    a.sync.sig_total = (launched ? 0u : grid) + eg;
  }
#define RS_FIN(V, C)                                                   \
  if (!launched && sh.vec == V && sh.ch == C) {                        \
    RS_CUDA(launch_pdl(pdl_hot, k_finish<V, C>, grid, 256, smem, hs, a, o, \
                       hot_blocks));                                   \
    RS_LAUNCH_CHECK("k_finish");                                       \
    launched = true;                                                   \
  }
  RS_FIN(4, 1) RS_FIN(4, 2) RS_FIN(4, 3) RS_FIN(4, 4)
  RS_FIN(2, 1) RS_FIN(2, 2)
  RS_FIN(1, 1) RS_FIN(1, 2) RS_FIN(1, 3) RS_FIN(1, 4) RS_FIN(1, 5) RS_FIN(1, 6) RS_FIN(1, 7)
  RS_FIN(1, 8)
#undef RS_FIN
  if (!launched) return fail(RS_ERR_CONFIG, "embedding_dim " + std::to_string(D) + " unsupported");
  if (G > 0) {
#define RS_CSR(GG, NN)                                      \
  if (Gc == GG && NVc == NN) {                              \
    RS_CUDA(launch_pdl(ws->pdl_now, k_finish_csr<GG, NN>,   \
                       eg, 256, 0, s, a, o));               \
    RS_LAUNCH_CHECK("k_finish_csr");                        \
  }
    RS_CSR(32, 1) RS_CSR(16, 1) RS_CSR(8, 1) RS_CSR(4, 1) RS_CSR(2, 1)
    RS_CSR(16, 2) RS_CSR(8, 2) RS_CSR(4, 2) RS_CSR(2, 2)
#undef RS_CSR
    if (fork) {
      RS_CUDA(cudaEventRecord(ws->ev_join, ws->aux_stream));
      RS_CUDA(cudaStreamWaitEvent(s, ws->ev_join, 0));  // join
    }
  }
  return RS_OK;
}

static int opt_args(rs_table* t, const rs_optimizer_params* p, OptArgs* o, cudaStream_t s) {
  std::memset(o, 0, sizeof(*o));
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
  if (p->kind == RS_OPT_ADAM) {
    int st = table_adam_tables(t, p->beta1, p->beta2, t->applies, s);
    if (st) return st;
    o->bc = t->d_bc;
    o->bc_len = t->bc_len;
  }
  return RS_OK;
}

// Dedup + find-or-insert of the fast step on set `use` (bounded tables take
// the host-synchronized probe / evict / insert path), then KC.
static int forward_enqueue(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                           float* d_out, const float* d_grads, int use, cudaStream_t s) {
  int st;
  if (t->cfg.max_keys) {
    carve(k_clean), k_clean<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(set_dev(ws, use ^ 1));
    RS_LAUNCH_CHECK("k_clean");
    if ((st = launch_fdedup(ws, d_ids, n, use, s, nullptr, true))) return st;
    FTableArgs a = ftable_args(ws, t, use);
    a.do_clean = false;
    a.do_table = false;
    carve(k_ftable), k_ftable<<<grid_for(n, kGroups, 148 * 8), kGroups * kBucket, 0, s>>>(a);
    RS_LAUNCH_CHECK("k_ftable(meta)");
    st = table_ensure_any(t, ws->unique, ws->set[use].cnt, n, ws->urow, ws->urow64,
                          ws->set[use].u_slot, ws->set[use].srow, s);
    if (st) return st;
  } else {
    if ((st = fast_dedup_table(ws, t, d_ids, n, use, s))) return st;
  }
  return launch_tile(ws, t, use, n, d_out, d_grads, true, s);
}

int step_set_smem_attrs() { return set_smem_attrs(); }
int step_fdedup(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, int use, cudaStream_t s,
                const uint32_t* d_n) {
  return launch_fdedup(ws, d_ids, n, use, s, d_n, d_n == nullptr);  // host n: token ranks too
}
int step_ftable(rs_workspace* ws, rs_table* t, int use, uint64_t n_max, bool do_table,
                bool do_clean, cudaStream_t s, const rs_dist_send* send) {
  FTableArgs a = ftable_args(ws, t, use);
  a.do_table = do_table;
  a.do_clean = do_clean;
  if (send) a.send = *send;
  carve(k_ftable), k_ftable<<<grid_for(n_max, kGroups, 148 * 8), kGroups * kBucket, 0, s>>>(a);
  RS_LAUNCH_CHECK("k_ftable");
  return RS_OK;
}
int step_tile(rs_workspace* ws, rs_table* t, int use, uint64_t n, float* d_out,
              const float* d_grads, bool clean_other, cudaStream_t s, const rs_dist_opts* dopt) {
  return launch_tile(ws, t, use, n, d_out, d_grads, clean_other, s, dopt);
}
int step_finish(rs_workspace* ws, rs_table* t, int use, uint64_t n, const float* d_grads,
                const void* opt_args, float* sums_out, cudaStream_t s, const rs_dist_opts* dopt) {
  OptArgs o;
  if (opt_args)
    std::memcpy(&o, opt_args, sizeof(o));
  else
    std::memset(&o, 0, sizeof(o));
  return launch_finish(ws, t, use, n, d_grads, o, sums_out, s, dopt);
}
int step_opt_args(rs_table* t, const rs_optimizer_params* p, void* out, cudaStream_t s) {
  return opt_args(t, p, reinterpret_cast<OptArgs*>(out), s);
}
int step_reduce_prepare(rs_workspace* ws, uint32_t D, uint64_t n, cudaStream_t s) {
  return reduce_prepare(ws, D, n, s);
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
  if (const char* e = getenv("RS_NO_GRAPH")) ws->use_graphs = e[0] == '0';
  if (const char* e = getenv("RS_NO_FORK")) ws->fork = e[0] == '0';
  if (const char* e = getenv("RS_GRAPH_FORK")) ws->graph_fork = e[0] != '0';
  if (const char* e = getenv("RS_SPLIT_KC")) ws->split_kc = e[0] != '0';
  if (const char* e = getenv("RS_PDL")) ws->pdl = e[0] != '0';
  if (const char* e = getenv("RS_FAST_STEP")) ws->use_fast = e[0] != '0';
  uint64_t S_ = 1024;
  while (S_ < 2 * max_tokens) S_ <<= 1;
  ws->S = S_;
  const uint64_t N = max_tokens;
  auto A = [&](auto** p, size_t bytes) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16)) == cudaSuccess;
  };
  bool ok = true;
  for (auto& x : ws->set)
    ok = ok && A(&x.skey, (S_ + 1) * 8) && A(&x.sfirstx, (S_ + 1) * 4) &&
         A(&x.sntile, (S_ + 1) * 4) && A(&x.suidx, (S_ + 1) * 4) && A(&x.srow, (S_ + 1) * 4) &&
         A(&x.u_slot, N * 4) && A(&x.cnt, 16);
  ok = ok && A(&ws->slot_of, N * 4) && A(&ws->inverse, N * 4) && A(&ws->unique, N * 8) &&
       A(&ws->u_ntile, N * 4) && A(&ws->u_poff, N * 4) && A(&ws->u_ticket, N * 4) &&
       A(&ws->urow, N * 4) && A(&ws->urow64, N * 8) && A(&ws->ptile, N * 4) &&
       A(&ws->porder, N * 4) && A(&ws->hot_list, (N / 32 + 64) * 4) && A(&ws->u_cnt, N * 4) && A(&ws->csr_pos, N * 4) &&
       A(&ws->scan_status, ((N + kScanTile - 1) / kScanTile + 1) * 8) && A(&ws->ctr, 64) &&
       A(&ws->csum_part, (N / 32 + 2) * 8) && A(&ws->csum_ticket, 16) && A(&ws->tok_rank, N * 4) &&
       cudaMemset(ws->csum_ticket, 0, 16) == cudaSuccess;
  if (!ok) {
    rs_workspace_destroy(ws);
    return cuda_fail(cudaGetLastError(), "rs_workspace_create: cudaMalloc");
  }
  if (set_smem_attrs() != RS_OK ||
      cudaStreamCreateWithFlags(&ws->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ws->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ws->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ws->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    rs_workspace_destroy(ws);
    return RS_ERR_CUDA;
  }
  for (int k = 0; k < 2; ++k) {
    carve(k_clear_all), k_clear_all<<<grid_for(S_ + 1, 256, 148 * 16), 256>>>(set_dev(ws, k), S_ + 1);
    count_launch();
  }
  cudaMemset(ws->scan_status, 0, ((N + kScanTile - 1) / kScanTile + 1) * 8);
  cudaMemset(ws->ctr, 0, 64);
  cudaMemset(ws->u_ticket, 0, N * 4);
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
  fast_free(ws);
  for (auto& x : ws->set) {
    void* ps[] = {x.skey, x.sfirstx, x.sntile, x.suidx, x.srow, x.u_slot, x.cnt};
    for (void* p : ps)
      if (p) cudaFree(p);
  }
  void* ptrs[] = {ws->slot_of, ws->inverse, ws->unique, ws->u_ntile,  ws->u_poff,
                  ws->u_ticket, ws->urow,   ws->urow64, ws->ptile,    ws->porder,
                  ws->pbuf,    ws->scan_status, ws->ctr, ws->hot_list, ws->u_cnt, ws->csr_pos,
                  ws->csum_part, ws->csum_ticket, ws->tok_rank};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& g : ws->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& e : ws->prof_ev)
    if (e) cudaEventDestroy(e);
  if (ws->cap_stream) cudaStreamDestroy(ws->cap_stream);
  if (ws->aux_stream) cudaStreamDestroy(ws->aux_stream);
  if (ws->ev_fork) cudaEventDestroy(ws->ev_fork);
  if (ws->ev_join) cudaEventDestroy(ws->ev_join);
  delete ws;
  return RS_OK;
}

int rs_dedup(rs_workspace* ws, const uint64_t* d_ids, uint64_t n, uint64_t* d_unique,
             int32_t* d_inverse, uint32_t* d_n_unique, void* stream) {
  if (!ws) return fail(RS_ERR_CONFIG, "rs_dedup: null workspace");
  if (n > ws->max_tokens)
    return fail(RS_ERR_CONFIG, "dedup: batch of " + std::to_string(n) +
                                   " ids exceeds workspace max_tokens " +
                                   std::to_string(ws->max_tokens));
  cudaStream_t s = S(stream);
  const int use = ws->cur;
  const SetDev su = set_dev(ws, use), sc = set_dev(ws, use ^ 1);
  ws->have_forward = false;
  carve(k_clean), k_clean<<<grid_for(n + 1, 256, 148 * 8), 256, 0, s>>>(sc);
  RS_LAUNCH_CHECK("k_clean");
  if (n == 0) {
    RS_CUDA(cudaMemsetAsync(ws->set[use].cnt, 0, 4, s));
    RS_CUDA(cudaMemsetAsync(sc.cnt, 0, 4, s));
    if (d_n_unique) RS_CUDA(cudaMemsetAsync(d_n_unique, 0, sizeof(uint32_t), s));
    ws->last_set = use;
    ws->last_fast = false;
    ws->last_exact = true;
    ws->cur ^= 1;
    return RS_OK;
  }
  const uint32_t TT = 256;
  const uint32_t ntiles = (uint32_t)((n + TT - 1) / TT);
  const size_t sm = (size_t)(2 * TT + 1) * (8 + 4 + 4);
  carve(k_dedup_tile_exact), k_dedup_tile_exact<<<ntiles, TT, sm, s>>>(d_ids, (uint32_t)n, su, ws->slot_of);
  RS_LAUNCH_CHECK("k_dedup_tile_exact");
  const uint32_t stiles = (uint32_t)((n + kScanTile - 1) / kScanTile);
  carve(k_dedup_compact), k_dedup_compact<<<stiles, kScanThreads, 0, s>>>(d_ids, (uint32_t)n, ws->slot_of, su, ws->unique,
                                                  ws->scan_status, ws->ctr, stiles, sc.cnt);
  RS_LAUNCH_CHECK("k_dedup_compact");
  if (d_inverse) {
    carve(k_inverse), k_inverse<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(ws->slot_of, su, (uint32_t)n, d_inverse);
    RS_LAUNCH_CHECK("k_inverse");
  }
  carve(k_copy_unique), k_copy_unique<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(ws->unique, su.cnt, d_unique, d_n_unique);
  RS_LAUNCH_CHECK("k_copy_unique");
  ws->last_set = use;
  ws->last_fast = false;
  ws->last_exact = true;
  ws->cur ^= 1;
  ws->last_n = n;
  return RS_OK;
}

int rs_forward(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n, float* d_out,
               void* stream) {
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_forward: null handle");
  if (n > ws->max_tokens) return fail(RS_ERR_CONFIG, "rs_forward: batch exceeds workspace max_tokens");
  cudaStream_t s = S(stream);
  ws->have_forward = false;
  ws->last_n = n;
  ws->last_tile = tile_tokens_for_dim(t->desc.dim);
  ws->last_table = t;
  if (n == 0) {  // an empty batch is a forward too: its (no-op) backward may follow
    ws->have_forward = true;
    return RS_OK;
  }
  int st = set_smem_attrs();
  if (st) return st;
  if (!t->cfg.max_keys && (st = table_prepare(t, n, s))) return st;
  const int use = ws->cur;
  st = forward_enqueue(ws, t, d_ids, n, d_out, nullptr, use, s);
  if (st) return st;
  if (!t->cfg.max_keys && (st = table_after_op(t, s))) return st;
  ws->last_set = use;
  ws->last_fast = false;
  ws->last_exact = false;
  ws->cur ^= 1;
  ws->have_forward = true;
  return RS_OK;
}

int rs_backward(rs_workspace* ws, rs_table* t, const float* d_grads, uint64_t n,
                const rs_optimizer_params* opt, void* stream) {
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_backward: null handle");
  if (!ws->have_forward || ws->last_table != t || ws->last_n != n)
    return fail(RS_ERR_CONFIG, "rs_backward: must follow rs_forward on the same table and batch");
  if (n == 0) {
    ws->have_forward = false;
    return RS_OK;
  }
  cudaStream_t s = S(stream);
  OptArgs o;
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  if ((st = reduce_prepare(ws, t->desc.dim, n, s))) return st;
  if ((st = launch_tile(ws, t, ws->last_set, n, nullptr, d_grads, false, s))) return st;
  if ((st = launch_finish(ws, t, ws->last_set, n, d_grads, o, nullptr, s))) return st;
  t->applies++;
  ws->have_forward = false;  // rows were updated: a second backward would double-apply
  return RS_OK;
}

int rs_accumulate(rs_workspace* ws, const float* d_grads, uint64_t n, float* d_sums,
                  void* stream) {
  if (!ws || !ws->last_table || !ws->have_forward)
    return fail(RS_ERR_CONFIG, "rs_accumulate: no forward on workspace");
  if (ws->last_n != n) return fail(RS_ERR_CONFIG, "rs_accumulate: batch size differs from forward");
  if (n == 0) return RS_OK;
  cudaStream_t s = S(stream);
  rs_table* t = ws->last_table;
  OptArgs o;
  std::memset(&o, 0, sizeof(o));
  int st = reduce_prepare(ws, t->desc.dim, n, s);
  if (st) return st;
  if ((st = launch_tile(ws, t, ws->last_set, n, nullptr, d_grads, false, s))) return st;
  return launch_finish(ws, t, ws->last_set, n, d_grads, o, d_sums, s);
}

// All launches of one training step, no host-side work (graph capturable).
static int step_enqueue(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                        const float* d_grads, float* d_out, const OptArgs& o, int use,
                        int mirror, cudaStream_t s, cudaEvent_t* ev) {
  int st;
  struct PdlOff {  // programmatic edges only inside this call, also on error returns
    rs_workspace* w;
    ~PdlOff() { w->pdl_now = false; }
  } pdl_off{ws};
  ws->pdl_now = false;
  if (ev) RS_CUDA(cudaEventRecord(ev[0], s));
  if (t->cfg.max_keys) {  // bounded: dedup + metadata, then probe / evict / insert on the device
    carve(k_clean), k_clean<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(set_dev(ws, use ^ 1));
    RS_LAUNCH_CHECK("k_clean");
    if ((st = launch_fdedup(ws, d_ids, n, use, s, nullptr, true))) return st;
    if (ev) RS_CUDA(cudaEventRecord(ev[1], s));
    FTableArgs a = ftable_args(ws, t, use);
    a.do_clean = false;
    a.do_table = false;
    carve(k_ftable), k_ftable<<<grid_for(n, kGroups, 148 * 8), kGroups * kBucket, 0, s>>>(a);
    RS_LAUNCH_CHECK("k_ftable(meta)");
    if ((st = table_bounded_enqueue(t, ws->unique, ws->set[use].cnt, n, ws->urow, ws->urow64,
                                    ws->set[use].u_slot, ws->set[use].srow, s)))
      return st;
  } else {
    if ((st = launch_fdedup(ws, d_ids, n, use, s, nullptr, true))) return st;
    if (ev) RS_CUDA(cudaEventRecord(ev[1], s));
    ws->pdl_now = ws->pdl && !ev;  // eager profiling keeps plain launches
    RS_CUDA(launch_pdl(ws->pdl_now, k_ftable, grid_for(n, kGroups, 148 * 8), kGroups * kBucket, 0, s,
                       ftable_args(ws, t, use)));
    RS_LAUNCH_CHECK("k_ftable");
  }
  if (ev) RS_CUDA(cudaEventRecord(ev[2], s));
  if ((st = launch_tile(ws, t, use, n, d_out, d_grads, true, s))) return st;
  if (ev) RS_CUDA(cudaEventRecord(ev[3], s));
  if ((st = launch_finish(ws, t, use, n, d_grads, o, nullptr, s))) return st;
  ws->pdl_now = false;  // (the mirror copy below is not a kernel)
  if (ev) RS_CUDA(cudaEventRecord(ev[4], s));
  return table_mirror_copy(t, mirror, s);
}

static int step_call(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, float* d_out, const rs_optimizer_params* opt, void* stream);

int rs_step(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
            const float* d_grads, float* d_out, const rs_optimizer_params* opt, void* stream) {
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_step: null handle");
  ws->csum_dst = nullptr;
  return step_call(ws, t, d_ids, n, d_grads, d_out, opt, stream);
}

// rs_step + run_workload's emb_checksum of the gathered rows (workload.cpp:
// 547-549) into d_checksum (device f64), summed inside the gather kernel.
int rs_step_checksum(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, float* d_out, const rs_optimizer_params* opt,
                     double* d_checksum, void* stream) {
  if (!ws || !t || !d_checksum) return fail(RS_ERR_CONFIG, "rs_step_checksum: null argument");
  // the gather kernel sums the rows it writes when D % 4 == 0; otherwise a
  // separate reduction over d_out
  const bool fused = n > 0 && t->desc.dim % 4 == 0;
  ws->csum_dst = fused ? d_checksum : nullptr;
  int st = step_call(ws, t, d_ids, n, d_grads, d_out, opt, stream);
  ws->csum_dst = nullptr;
  if (st || fused) return st;
  return rs_checksum(d_out, n * t->desc.dim, d_checksum, stream);
}

static int step_call(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, float* d_out, const rs_optimizer_params* opt, void* stream) {
  if (n == 0) {
    int st = rs_forward(ws, t, d_ids, n, d_out, stream);
    if (st) return st;
    return rs_backward(ws, t, d_grads, n, opt, stream);
  }
  if (n > ws->max_tokens) return fail(RS_ERR_CONFIG, "rs_step: batch exceeds workspace max_tokens");
  cudaStream_t s = S(stream);
  OptArgs o;
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  if ((st = set_smem_attrs())) return st;
  // host side, outside the graph: capacity bound (may rehash / grow rows on s),
  // bounded tables also size the device victim selection
  if ((st = t->cfg.max_keys ? table_bounded_prepare(t, n, s) : table_prepare(t, n, s, 16))) return st;
  ws->last_tile = tile_tokens_for_dim(t->desc.dim);
  if ((st = reduce_prepare(ws, t->desc.dim, n, s))) return st;
  const int mirror = t->mirror_next;
  // unbounded tables: the fast step (step_fast.cu) on its own scratch sets
  const bool fast = ws->use_fast && d_grads && ((uintptr_t)d_grads & 15u) == 0 && fast_step_supported(t);
  if (fast && (st = fast_prepare(ws))) return st;
  const int use = fast ? ws->fast.cur : ws->cur;
  auto enqueue = [&](cudaStream_t q, cudaEvent_t* ev) -> int {
    if (!fast) return step_enqueue(ws, t, d_ids, n, d_grads, d_out, o, use, mirror, q, ev);
    // the counters reach the pinned mirror from inside the step (mapped store,
    // k_fclean) when the mirror is mapped; else a copy after the step
    TableCounters* mo = t->mirror[mirror].dev_ptr;
    const int e = fast_enqueue(ws, t, d_ids, n, d_grads, d_out, &o, use, q, ev, ws->fork, mo);
    return e ? e : (mo ? RS_OK : table_mirror_copy(t, mirror, q));
  };
  // Bounded tables (evict-heavy streams: batches rarely repeat) capture a
  // step's graph only when its buffers / size come back: a one-off batch runs
  // eagerly instead of paying a capture + instantiate
  bool once = false;
  if (t->cfg.max_keys && !ws->profiling && ws->use_graphs) {
    const uint64_t sig = (uint64_t)(uintptr_t)d_ids * 0x9E3779B97F4A7C15ull ^ (uint64_t)(uintptr_t)d_grads * 31 ^
                         (uint64_t)(uintptr_t)d_out * 131 ^ n * 0xC2B2AE3D27D4EB4Full ^ (uint64_t)(uintptr_t)t;
    bool cached = false;
    for (auto& g : ws->graphs)
      cached = cached || (g.t == t && g.ids == d_ids && g.grads == d_grads && g.out == d_out && g.n == n);
    if (!cached) {
      once = std::find(ws->seen.begin(), ws->seen.end(), sig) == ws->seen.end();
      if (once) {
        if (ws->seen.size() >= 64) ws->seen.erase(ws->seen.begin());
        ws->seen.push_back(sig);
      }
    }
  }
  if (ws->profiling || !ws->use_graphs || once) {
    // profiling runs the kernels one after another (no fork) so that every
    // phase's events bracket only its own kernels
    const bool f0 = ws->fork;
    if (ws->profiling) ws->fork = false;
    st = enqueue(s, ws->profiling ? ws->prof_ev : nullptr);
    ws->fork = f0;
    if (st) return st;
    if (ws->profiling) {
      RS_CUDA(cudaEventSynchronize(ws->prof_ev[4]));
      for (int k = 0; k < 4; ++k) {
        float ms = 0;
        RS_CUDA(cudaEventElapsedTime(&ms, ws->prof_ev[k], ws->prof_ev[k + 1]));
        ws->prof_ms[k] += ms;
      }
      ws->prof_count++;
    }
  } else {
    static_assert(sizeof(OptArgs) <= sizeof(((rs_graph_entry*)0)->opt), "opt key");
    rs_graph_entry* hit = nullptr;
    for (auto& g : ws->graphs) {
      if (g.t == t && g.ids == d_ids && g.grads == d_grads && g.out == d_out && g.n == n &&
          g.csum == ws->csum_dst &&
          g.mirror == mirror && g.set == use && g.fast == fast && g.pbuf == ws->pbuf && g.tcap == t->capacity &&
          g.tgen == t->buf_gen &&
          std::memcmp(g.opt, &o, sizeof(o)) == 0) {
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
      e.csum = ws->csum_dst;
      e.n = n;
      e.mirror = mirror;
      e.set = use;
      e.fast = fast;
      e.pbuf = ws->pbuf;
      e.tcap = t->capacity;
      e.tgen = t->buf_gen;
      std::memcpy(e.opt, &o, sizeof(o));
      cudaStream_t cs = ws->cap_stream;
      RS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      const uint64_t before = launches();
      // a forked branch inside the captured graph measured slower: linear graph
      const bool fork = ws->fork;
      ws->fork = ws->fork && ws->graph_fork;
      st = enqueue(cs, nullptr);
      ws->fork = fork;
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(cs, &g);
      if (st) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
      const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, graph_flags());
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) return cuda_fail(ie, "cudaGraphInstantiate");
      e.launches = launches() - before;
      count_launch(0 - e.launches);  // capture only recorded the launches
      ws->graphs.push_back(e);
      hit = &ws->graphs.back();
    }
    hit->last_use = ++ws->graph_clock;
    RS_CUDA(cudaGraphLaunch(hit->exec, s));
    count_launch(hit->launches);
  }
  ws->last_n = n;
  ws->last_table = t;
  ws->last_exact = false;
  if (fast) {
    if ((st = fast_check_errors(ws, s))) return st;
    ws->fast.last = use;
    ws->fast.cur ^= 1;
    ws->last_fast = true;
  } else {
    ws->last_set = use;
    ws->cur ^= 1;
    ws->last_fast = false;
  }
  ws->have_forward = false;
  t->applies++;
  return table_mirror_commit(t, mirror, s);
}

int rs_sparse_update(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n,
                     const float* d_grads, const rs_optimizer_params* opt, void* stream) {
  // GradAccumulator::accumulate + apply for one window (sparse_update.cpp:45-83):
  // dedup, zero-vivify absent ids, segment-reduce fused with the update.
  if (!ws || !t) return fail(RS_ERR_CONFIG, "rs_sparse_update: null handle");
  if (n > ws->max_tokens) return fail(RS_ERR_CONFIG, "rs_sparse_update: batch exceeds max_tokens");
  cudaStream_t s = S(stream);
  OptArgs o;
  int st = opt_args(t, opt, &o, s);
  if (st) return st;
  if ((st = set_smem_attrs())) return st;
  ws->have_forward = false;
  ws->last_n = n;
  ws->last_table = t;
  if (n == 0) return RS_OK;
  ws->last_tile = tile_tokens_for_dim(t->desc.dim);
  if (!t->cfg.max_keys && (st = table_prepare(t, n, s))) return st;
  if ((st = reduce_prepare(ws, t->desc.dim, n, s))) return st;
  const int use = ws->cur;
  if ((st = forward_enqueue(ws, t, d_ids, n, nullptr, d_grads, use, s))) return st;
  if ((st = launch_finish(ws, t, use, n, d_grads, o, nullptr, s))) return st;
  if (!t->cfg.max_keys && (st = table_after_op(t, s))) return st;
  ws->last_set = use;
  ws->last_fast = false;
  ws->last_exact = false;
  ws->cur ^= 1;
  t->applies++;
  return RS_OK;
}

static const uint32_t* last_count(const rs_workspace* ws) {
  return ws->last_fast ? ws->fast.set[ws->fast.last].cnt : ws->set[ws->last_set].cnt;
}

int rs_workspace_results(rs_workspace* ws, const uint64_t** d_unique, const int32_t** d_inverse,
                         const uint32_t** d_n_unique, const int64_t** d_rows) {
  if (!ws) return fail(RS_ERR_CONFIG, "rs_workspace_results: null workspace");
  if (!ws->last_exact)
    return fail(RS_ERR_CONFIG, "rs_workspace_results: the unique ids of rs_forward / rs_step are numbered in "
                               "unspecified order; rs_dedup gives stage1_dedup's first-occurrence order");
  if (d_unique) *d_unique = ws->unique;
  if (d_inverse) *d_inverse = ws->inverse;
  if (d_n_unique) *d_n_unique = last_count(ws);
  if (d_rows) *d_rows = ws->urow64;
  return RS_OK;
}

int rs_workspace_unique(rs_workspace* ws, uint64_t* d_out, uint64_t cap, uint64_t* n_out) {
  if (!ws || !n_out) return fail(RS_ERR_CONFIG, "rs_workspace_unique: null argument");
  RS_CUDA(cudaDeviceSynchronize());
  uint32_t n = 0;
  RS_CUDA(cudaMemcpy(&n, last_count(ws), 4, cudaMemcpyDeviceToHost));
  *n_out = n;
  if (d_out) {
    if (cap < n) return fail(RS_ERR_CONFIG, "rs_workspace_unique: buffer too small");
    RS_CUDA(cudaMemcpy(d_out, ws->unique, n * 8ull, cudaMemcpyDeviceToDevice));
  }
  return RS_OK;
}

int rs_workspace_set_profiling(rs_workspace* ws, int on) {
  if (!ws) return fail(RS_ERR_CONFIG, "rs_workspace_set_profiling: null workspace");
  if (on && !ws->prof_ev[0])
    for (auto& e : ws->prof_ev) RS_CUDA(cudaEventCreate(&e));
  ws->profiling = on != 0;
  for (auto& m : ws->prof_ms) m = 0;
  ws->prof_count = 0;
  return RS_OK;
}

int rs_workspace_phase_ms(rs_workspace* ws, double* ms, uint32_t nphases, uint64_t* count) {
  if (!ws || !ms) return fail(RS_ERR_CONFIG, "rs_workspace_phase_ms: null argument");
  for (uint32_t k = 0; k < nphases && k < 8; ++k)
    ms[k] = ws->prof_count ? ws->prof_ms[k] / ws->prof_count : 0.0;
  if (count) *count = ws->prof_count;
  return RS_OK;
}

int rs_workspace_n_unique(rs_workspace* ws, uint64_t* out) {
  if (!ws || !out) return fail(RS_ERR_CONFIG, "rs_workspace_n_unique: null argument");
  RS_CUDA(cudaDeviceSynchronize());
  uint32_t n = 0;
  RS_CUDA(cudaMemcpy(&n, last_count(ws), 4, cudaMemcpyDeviceToHost));
  *out = n;
  return RS_OK;
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
    carve(k_apply_sums<V, C>), k_apply_sums<V, C><<<grid, 256, 0, s>>>(t->dev, rows, n, d_sums, o);                 \
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
