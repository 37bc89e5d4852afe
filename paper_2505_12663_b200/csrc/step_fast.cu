// step_fast.cu -- the single-GPU training step (rs_step / rs_step_checksum on
// an unbounded table): one dedup + probe kernel, then two concurrent
// branches that each own a disjoint set of ids (and so of table rows).
//
// Reference caller: run_workload (workload.cpp:506-581) with
// distributed_lookup at W = 1 (stage1_dedup + ensure + inverse expand,
// exchange_sim.cpp:117-233), then GradAccumulator::accumulate + apply
// (sparse_update.cpp:45-83).
//
//   KA  k_fa   per 256-token tile: tile-local dedup in smem, one scratch
//              insert per (tile, id) into 16-byte records {key, count, row};
//              each token's position stored at pos[slot * 64 + rank] (rank
//              = tile base from the count atomic + rank in the tile, any
//              order: KD sorts); the tile that claims an id numbers it and
//              resolves its table row right away (find-or-insert-zero,
//              grouped bucket probing); cleans the other scratch set; the
//              last block folds the table counters.
//   then, forked (both need only KA):
//   KD  k_fc   per unique id with <= 64 occurrences (G = D/4 lanes): loads
//              its row, writes it to each of its tokens (the forward
//              gather), ranks its positions in registers, sums its gradient
//              rows in token order (the reference's accumulate order:
//              bit-exact), optimizer
//   KH  k_fh   per tile: tokens of hot ids (> 64 occurrences) grouped by id;
//              each group's row to its tokens (the forward), its (tile, id)
//              partial summed in token order straight from the gradient rows
//   KF  k_fhf  per hot id: its tile partials in tile order, optimizer
//              (KH -> KF on one branch: KF updates a hot row after KH read it)
//   KS  k_fcs  rs_step_checksum only: the f64 sum of the forward rows
// Every token's row is written once and every gradient row read once; the
// pre-update rows of an id are read by the same branch that updates them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dist_sync.cuh"
#include "opt_dev.cuh"
#include "rs_host.hpp"
#include "table_dev.cuh"

namespace rs {
namespace {

using namespace odev;
using namespace tdev;

constexpr uint32_t kPosMax = 64;  // exact-order (CSR) path limit == step.cu kCsrMax
constexpr uint32_t kTT = 256;     // tokens per tile
constexpr uint32_t kHotNone = 0xFFFFFFFFu, kHotClaim = 0xFFFFFFFEu;

struct __align__(16) Rec {
  unsigned long long key;
  uint32_t cnt;  // occurrences of the id in the batch
  uint32_t row;  // table row
};

struct FSet {
  Rec* rec;         // [S + 1]; slot S holds the id equal to the empty sentinel
  uint32_t* u_slot; // slot of each unique id (the set's dirty list)
  uint32_t* cnt;    // [0] unique ids in the set
  uint64_t smask, spare;
};

struct FShared {
  uint32_t* uidx;      // [S + 1] unique index of a slot (written before read each step)
  uint32_t* hidx;      // [S + 1] hot index of a slot (kHotNone between steps)
  uint32_t* pos;       // [(S + 1) * 64] token positions per slot
  uint32_t* hot_slot;  // [max_hot]
  uint32_t* hlist;     // [max_hot * ntiles] partial index + 1 of (hot id, tile), 0 = none
  float* part;         // partial rows
  uint32_t* ctr;       // [0] hot ids [1] partials [2] error bits [3] clean blocks
  uint32_t ntiles;
  uint32_t hot_min;    // ids with more occurrences take the hot (tile partial) path, <= 64
  unsigned long long* trace;  // diagnostics timeline or null
  uint32_t* heavy;     // [max_tokens] slots of ids with > light_max occurrences (KA)
  uint32_t light_max;  // CSR ids up to this many occurrences: the light kernel; above: the heavy one
  uint64_t n_slots;    // S + 1 (checked builds)
  uint32_t max_tokens, max_hot;
};

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// Checked builds (-DRS_BOUNDS, `make EXTRA=-DRS_BOUNDS OUT=...`): every
// computed index is range-checked before use; a violation sets error bit 2
// of ctr[2] (rs_step then fails with RS_ERR_INVARIANT) and skips the access.
// compute-sanitizer is not available on this pool; this is the substitute.
#ifdef RS_BOUNDS
#define RS_IDX_OK(cond, ctr) \
  ((cond) ? true : (atomicOr((ctr) + 2, 2u), printf("step_fast bounds: %s (%s:%d)\n", #cond, __FILE__, __LINE__), false))
#else
#define RS_IDX_OK(cond, ctr) true
#endif

// Global scratch insert (linear probing on the low hash bits) into the
// 16-byte records.  first0: the start record's key read early by the caller.
__device__ __forceinline__ uint64_t rec_insert(const FSet& S, uint64_t id, uint64_t h, bool* fresh,
                                               unsigned long long first0) {
  if (id == kEmptyKey) {
    *fresh = atomicCAS(&S.rec[S.spare].key, kEmptyKey, 0ull) == kEmptyKey;
    return S.spare;
  }
  uint64_t gs = h & S.smask;
  bool use0 = true;
  for (;;) {
    const unsigned long long cur = use0 ? first0 : __ldcg(&S.rec[gs].key);
    use0 = false;
    if (cur == id) {
      *fresh = false;
      return gs;
    }
    if (cur != kEmptyKey) {
      gs = (gs + 1) & S.smask;
      continue;
    }
    const unsigned long long prev = atomicCAS(&S.rec[gs].key, kEmptyKey, (unsigned long long)id);
    if (prev == kEmptyKey) {
      *fresh = true;
      return gs;
    }
    if (prev == id) {
      *fresh = false;
      return gs;
    }
    gs = (gs + 1) & S.smask;
  }
}

// ---------------------------------------------------------------------------
// KA: dedup + positions + probe of the ids this tile claims.  blockDim == kTT.
struct FaArgs {
  const uint64_t* ids;
  uint32_t n;
  uint32_t set;  // scratch set parity of this step
  // sharded requester (send.peers != null): no table here -- the tile that
  // claims an id sends it to its owner's receive list instead of probing
  rs_dist_send send;
  FSet use, clean;
  FShared sh;
  TableDev* td;
  uint32_t* slot_of;
  uint64_t* unique;
  uint32_t* urow;
  int64_t* urow64;
  int no_table = 0;  // bounded tables: dedup + metadata only (the bounded ensure follows, then k_fpatch)
  // bounded tables, probe mode: the claiming tile probes its ids (stamp the
  // hits, list the misses, one stamp-log record per unique id at base + u)
  int probe_only = 0;
  uint32_t* missing = nullptr;
  LogArgs lg;
  // the previous step's set cleaned inside KA (no k_fclean): its slice per
  // block, the last block (ctr[3] arrivals) zeroes its count; table mode also
  // stores the counters into the host's mapped mirror from KA's epilogue
  int clean_in_ka = 0;
  TableCounters* mirror_out = nullptr;
};

// Sharded requester: the ids this tile claimed go to their owners
// (owner = hash64 % W, exchange_sim.cpp:82-85): positions from block-local
// per-owner counters and one global atomic per (block, owner), each id
// stored into the owner's ids_in[rank][j] over NVLink; the slot's record
// row becomes the received-row index owner * cap + j (the gather reads it).
// The last block publishes the counts and raises the ids flags (epoch e).
__device__ __forceinline__ void fa_send(const FaArgs& a, uint32_t nnew, const unsigned long long* fid,
                                        const uint32_t* fslot, const uint32_t* fu) {
  const rs_dist_send& S = a.send;
  __shared__ uint32_t s_ocnt[64], s_obase[64], fo[kTT], fj[kTT];
  __shared__ unsigned long long s_e;
  __shared__ bool s_last;
  const uint32_t tid = threadIdx.x;
  for (uint32_t r = tid; r < 64; r += kTT) s_ocnt[r] = 0;
  if (tid == 0) s_e = *S.epoch + 1;  // read before arriving; published by the last block
  __syncthreads();
  for (uint32_t k = tid; k < nnew; k += kTT) {
    const uint32_t o = (uint32_t)(hash64(fid[k]) % S.world);
    fo[k] = o;
    fj[k] = atomicAdd(&s_ocnt[o], 1u);
  }
  __syncthreads();
  for (uint32_t r = tid; r < S.world; r += kTT) s_obase[r] = s_ocnt[r] ? atomicAdd(&S.send_cnt[r], s_ocnt[r]) : 0u;
  __syncthreads();
  for (uint32_t k = tid; k < nnew; k += kTT) {
    const uint32_t o = fo[k], j = s_obase[o] + fj[k];
    if (!RS_IDX_OK(j < S.cap, a.sh.ctr)) continue;
    reinterpret_cast<uint64_t*>(S.peers[o] + S.off_ids)[(size_t)S.rank * S.cap + j] = fid[k];
    const uint32_t sp = o * S.cap + j;
    S.send_pos[fu[k]] = sp;
    a.urow[fu[k]] = sp;
    a.use.rec[fslot[k]].row = sp;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(S.done) : "memory");
    s_last = old == gridDim.x - 1;
    if (s_last) asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  __syncthreads();
  if (!s_last) return;
  for (uint32_t r = tid; r < S.world; r += kTT) {
    *S.cnt_ptrs[r] = S.send_cnt[r];
    S.trace_ids_sent[r] = S.send_cnt[r];
  }
  if (tid == 0) *S.trace_requested = S.n_tokens;
  __syncthreads();
  for (uint32_t r = tid; r < S.world; r += kTT) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(S.flag_ptrs[r]), "l"(s_e) : "memory");
    S.send_cnt[r] = 0;
  }
  if (tid == 0) {
    *S.epoch = s_e;
    *S.done = 0;
  }
}

__global__ void __launch_bounds__(kTT) k_fa(FaArgs a) {
  WarpTrace wt_(a.sh.trace, 0);
  constexpr uint32_t L = 2 * kTT;
  __shared__ unsigned long long lkey[L + 1];
  __shared__ uint32_t lbase[L + 1], lslot[L + 1], lnew[L + 1], lcnt[L + 1];
  __shared__ unsigned long long fid[kTT];
  __shared__ uint32_t fslot[kTT], fu[kTT];
  __shared__ uint32_t s_nnew, s_base;
  __shared__ unsigned long long s_ins, s_reuse;
  TableDev* td = a.td;
  const bool sending = a.send.peers != nullptr || a.no_table;  // (no table work in this kernel)
  const TableDesc d = sending ? TableDesc{} : td->d;
  const unsigned long long free_n0 = sending ? 0ull : td->c.free_n;
  const unsigned long long fresh0 = sending ? 0ull : td->c.fresh_next;
  const uint32_t tick_now = sending ? 0u : td->c.tick + 1;
  const uint32_t tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) {  // this step's hot-id / partial counters (KH, KF follow KA)
    a.sh.ctr[0] = 0;
    a.sh.ctr[1] = 0;
  }
  // heavy-list counts alternate with the scratch set (ctr[5 + set]): KA's
  // blocks append to this set's (zeroed by the previous step), block 0 zeroes
  // the other one for the next step
  if (blockIdx.x == 0 && tid == 0) a.sh.ctr[5 + (a.set ^ 1)] = 0;
  if (a.clean_in_ka) {  // the previous step's records back to empty (its dirty list), off every chain
    const uint32_t prev = *a.clean.cnt;
    for (uint32_t i = blockIdx.x * kTT + tid; i <= prev; i += gridDim.x * kTT) {
      const uint64_t sl = i < prev ? a.clean.u_slot[i] : a.clean.spare;
      a.clean.rec[sl] = Rec{kEmptyKey, 0u, kNoRow};
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      unsigned int* done = reinterpret_cast<unsigned int*>(a.sh.ctr + 3);
      if (atomicAdd(done, 1u) == gridDim.x - 1) {  // every block read prev: the set starts empty
        __threadfence();
        *a.clean.cnt = 0;
        *done = 0;
      }
    }
  }
  for (uint32_t i = tid; i <= L; i += kTT) {
    lkey[i] = kEmptyKey;
    lnew[i] = 0;
    lcnt[i] = 0;
  }
  if (tid == 0) {
    s_nnew = 0;
    s_ins = 0;
    s_reuse = 0;
  }
  __syncthreads();
  const uint32_t t = blockIdx.x * kTT + tid;
  const bool valid = t < a.n;
  uint64_t id = 0, h = 0;
  uint32_t p = 0, lr = 0;
  bool rep = false;
  unsigned long long first0 = kEmptyKey;
  if (valid) {
    id = a.ids[t];
    h = hash64(id);
    // the start record's key, read now: overlaps the tile-local dedup below
    if (id != kEmptyKey) first0 = __ldcg(&a.use.rec[h & a.use.smask].key);
    if (id == kEmptyKey) {
      p = L;
      rep = atomicCAS(&lkey[p], kEmptyKey, 0ull) == kEmptyKey;
    } else {
      p = (uint32_t)(h >> 40) & (L - 1);
      for (;;) {
        const unsigned long long prev = atomicCAS(&lkey[p], kEmptyKey, (unsigned long long)id);
        if (prev == kEmptyKey) {
          rep = true;
          break;
        }
        if (prev == id) break;
        p = (p + 1) & (L - 1);
      }
    }
    lr = atomicAdd(&lcnt[p], 1u);  // rank within the tile (any order: KD sorts)
  }
  __syncthreads();
  if (rep) {
    bool fresh = false;
    const uint64_t gs = rec_insert(a.use, id, h, &fresh, first0);
    const uint32_t base = atomicAdd(&a.use.rec[gs].cnt, lcnt[p]);  // the tile's base among the id's occurrences
    lbase[p] = base;
    lslot[p] = (uint32_t)gs;
    // the tile whose occurrences carry the id past light_max lists it (once) for
    // the heavy CSR kernel; past hot_min it is a hot id and that kernel skips it
    if (base <= a.sh.light_max && base + lcnt[p] > a.sh.light_max) {
      const uint32_t k = atomicAdd(&a.sh.ctr[5 + a.set], 1u);
      if (RS_IDX_OK(k < a.sh.max_tokens, a.sh.ctr)) a.sh.heavy[k] = (uint32_t)gs;
    }
    if (fresh) {
      // the probe below starts at this bucket: fetch it into L2 now (overlaps
      // the numbering barriers)
      if (!sending && id != kEmptyKey && id != kTombKey)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(d.slots + ((h >> 32) & d.nb_mask) * kBucket));
      const uint32_t k = atomicAdd(&s_nnew, 1u);
      lnew[p] = k + 1;
      fid[k] = id;
      fslot[k] = (uint32_t)gs;
    }
  }
  __syncthreads();
  if (tid == 0 && s_nnew) s_base = atomicAdd(a.use.cnt, s_nnew);
  __syncthreads();
  const uint32_t nnew = s_nnew;
  if (rep && lnew[p]) {
    const uint32_t k = lnew[p] - 1, u = s_base + k;
    const uint32_t gs = lslot[p];
    fu[k] = u;
    if (RS_IDX_OK(gs < a.sh.n_slots && u < a.sh.max_tokens, a.sh.ctr)) {
      a.sh.uidx[gs] = u;
      a.use.u_slot[u] = gs;
      a.unique[u] = id;
    }
  }
  if (valid) {
    const uint32_t gs = lslot[p];
    a.slot_of[t] = gs;
    const uint32_t rank = lbase[p] + lr;
    if (rank < kPosMax && RS_IDX_OK(gs < a.sh.n_slots, a.sh.ctr)) a.sh.pos[(size_t)gs * kPosMax + rank] = t;
  }
  __syncthreads();
  if (a.no_table) return;
  if (sending) {  // the claimed ids to their owners (positions by block-local then global counters)
    fa_send(a, nnew, fid, fslot, fu);
    return;
  }
  // the ids this tile claimed: find-or-insert-zero in the table, 8 lanes per id
  const unsigned lane = lane_id();
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  if (a.probe_only) {  // bounded tables: probe only (the evict + the insert of the misses follow)
    const unsigned long long lbase = a.lg.rec ? a.lg.ctl->tail : 0ull;
    for (uint32_t k = tid >> 3; k < nnew; k += kTT / kBucket) {
      const uint64_t key = fid[k];
      const uint32_t u = fu[k];
      uint32_t row = kNoRow, lslot = kNoLogSlot;
      const int sp = key == kEmptyKey ? 0 : (key == kTombKey ? 1 : -1);
      if (sp >= 0) {
        if (g == 0) {
          const uint32_t r = td->c.special_row[sp];
          if (r != kNoRow) {
            row = r;
            if (atomicExch(&td->c.special_tick[sp], tick_now) != tick_now) lslot = (uint32_t)(a.lg.cap + sp);
          }
        }
      } else {
        const Probe p = probe_group<true>(d.slots, d.nb_mask, key, g, gbase, gmask);
        if (p.found) {
          row = p.row == kNoRow ? wait_row(d.slots, p.slot) : p.row;
          if (g == 0 && p.tick != tick_now && atomicCAS(&d.slots[p.slot].tick, p.tick, tick_now) == p.tick)
            lslot = (uint32_t)p.slot;
        }
      }
      if (g == 0) {
        if (row == kNoRow) a.missing[atomicAdd(&td->c.missing, 1u)] = u;
        if (a.lg.rec) a.lg.rec[(lbase + u) & a.lg.mask] = LogRec{key, lslot, tick_now};
        a.use.rec[fslot[k]].row = row;
        a.urow[u] = row;
        a.urow64[u] = row == kNoRow ? -1 : (int64_t)row;
      }
    }
    // the op's records took [tail, tail + unique count): moved by the last block
    launch_epilogue(td, free_n0, fresh0, true, tick_now, nullptr, a.lg.rec ? a.lg.ctl : nullptr, 0, a.use.cnt);
    return;
  }
  for (uint32_t k = tid >> 3; k < nnew; k += kTT / kBucket) {
    const uint64_t key = fid[k];
    const uint32_t row = find_or_insert_group(td, d, key, g, gbase, gmask, tick_now, free_n0, fresh0, &s_ins,
                                              &s_reuse);
    if (g == 0) {
      a.use.rec[fslot[k]].row = row;
      a.urow[fu[k]] = row;
      a.urow64[fu[k]] = row == kNoRow ? -1 : (int64_t)row;
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (s_ins) atomicAdd(&td->c.inserted, s_ins);
    if (s_reuse) atomicAdd(&td->c.reused, s_reuse);
  }
  launch_epilogue(td, free_n0, fresh0, true, tick_now, a.mirror_out);
  // (launch_epilogue's last block has folded the counters; every block ran it)
}

// The previous step's scratch set goes back to empty records (its dirty
// list), off the critical path beside KD / KH; the last block zeroes its
// count (the next step's KA inserts into it).
__global__ void __launch_bounds__(256) k_fclean(FSet c, unsigned int* done, unsigned long long* trace,
                                                const TableDev* td, TableCounters* mirror_out) {
  WarpTrace wt_(trace, 4);
  const uint32_t prev = *c.cnt;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= prev;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t sl = i < prev ? c.u_slot[i] : c.spare;
    c.rec[sl] = Rec{kEmptyKey, 0u, kNoRow};
  }
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    *c.cnt = 0;
    *done = 0;
  }
  // the table counters (final since KA's epilogue) into the host's pinned
  // mirror (mapped memory): the sync-free capacity bookkeeping of the next
  // batches, without a copy node on the step's critical path
  if (last && mirror_out) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&td->c);
    uint32_t* dst = reinterpret_cast<uint32_t*>(mirror_out);
    for (uint32_t i = threadIdx.x; i < sizeof(TableCounters) / 4; i += blockDim.x) dst[i] = __ldcg(src + i);
    __threadfence_system();
  }
}

// ---------------------------------------------------------------------------
// KS (rs_step_checksum only): run_workload's emb_checksum (workload.cpp:
// 547-549) = the f64 sum of every gathered value.  KD / KH store each token's
// row sum (fixed lane tree); here per tile a fixed tree, then the last block
// sums the tile partials in tile order -- deterministic.
__global__ void __launch_bounds__(kTT) k_fcs(const double* __restrict__ tokcs, uint32_t n, double* out,
                                             double* part, unsigned int* ticket) {
  constexpr uint32_t NW = kTT / 32;
  __shared__ double s_cs[NW];
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t t = blockIdx.x * kTT + tid;
  double cs = t < n ? tokcs[t] : 0.0;
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
      part[blockIdx.x] = x;
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    if (__shfl_sync(kFull, last, 0)) {
      __threadfence();
      double y = 0.0;
      for (uint32_t b = lane; b < gridDim.x; b += 32) y += __ldcg(part + b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(kFull, y, o);
      if (lane == 0) {
        *out = y;
        *ticket = 0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// KD: ids with <= 64 occurrences.  G lanes per id, each owning NV float4
// chunks of the row (chunk gl + j*G).  Positions ranked within the group
// (shuffles), written sorted to smem, gradient rows summed in position order
// = the reference's accumulate order (sparse_update.cpp:49-54) -> bit-exact.
struct FcArgs {
  const TableDev* td;
  FSet use;
  FShared sh;
  const float* grads;
  float* out;        // forward rows [n x D]
  int32_t* inverse;  // [n]
  double* tokcs;     // per-token row sums (checksum) or null
  const uint32_t* urow;  // table row per unique id (KA)
  uint32_t exp;          // timing experiments (RS_FC_EXP bits, wrong results): 1 no optimizer, 2 no grads, 4 no forward
  uint32_t n_tokens;
  const uint32_t* list;    // null: every unique id; else slots (KA's heavy list) ...
  const uint32_t* list_n;  // ... and their count
  uint32_t c_min, c_max;   // ids with c_min < occurrences <= c_max
  float* const* peer_dst;  // sharded requester: sums to the owners (rows are send positions)
  uint32_t cap, rank;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// KD heavy, warp per id (D = 32 or 64; RS_FCB=1): one warp per heavy id (light_max <
// c <= 64 occurrences), EPL floats of the row per lane (float2 at D = 64:
// half the registers per row in flight of k_fc's 16 lanes x float4, so 16
// gradient rows are loaded per round trip instead of 4).  Positions ranked
// into token order, rows summed in token order -- the same sequential f32
// adds as k_fc, so the same bits -- then the forward rows and the optimizer.
template <int EPL>
__device__ __forceinline__ void ld_row(const float* p, float (&x)[EPL]) {
  if (EPL == 2) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(p));
    x[0] = v.x;
    x[EPL > 1 ? 1 : 0] = v.y;
  } else {
#pragma unroll
    for (int e = 0; e < EPL; ++e) x[e] = __ldg(p + e);
  }
}

template <int EPL, int NWB>
__global__ void __launch_bounds__(NWB * 32) k_fcb(FcArgs a, OptArgs o) {
  WarpTrace wt_(a.sh.trace, 5);
  __shared__ uint32_t s_order[NWB][kPosMax];
  const TableDesc d = a.td->d;
  const uint32_t D = d.dim;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* order = s_order[warp];
  const uint32_t nitems = *a.list_n;
  const bool peer = a.peer_dst != nullptr;
  const uint32_t e0 = lane * EPL;  // this lane's floats [e0, e0 + EPL)
  const bool mine = e0 < D;
  float* ew = d.emb;
  float* ev = d.s2;
  float* em = d.s1;
  for (uint32_t it = blockIdx.x * NWB + warp; it < nitems; it += gridDim.x * NWB) {
    const uint32_t gs = __ldg(a.list + it);
    if (!RS_IDX_OK(gs < a.sh.n_slots, a.sh.ctr)) continue;
    const uint2 cr = __ldcg(reinterpret_cast<const uint2*>(&a.use.rec[gs].cnt));
    const uint32_t c = cr.x, row = cr.y;
    const uint32_t uu = __ldcg(a.sh.uidx + gs);
    uint32_t p0 = __ldcg(a.sh.pos + (size_t)gs * kPosMax + lane);
    uint32_t p1 = __ldcg(a.sh.pos + (size_t)gs * kPosMax + 32 + lane);
    if (row == kNoRow) continue;  // table error (reported through the counters)
    if (c > a.c_max || c <= a.c_min) continue;  // (warp-uniform)
    if (!RS_IDX_OK(c <= kPosMax && (peer || row < d.row_cap), a.sh.ctr)) continue;
    // the row's state, issued before the sums
    float w[EPL], v[EPL], m[EPL];
    uint32_t st0 = 0;
#pragma unroll
    for (int e = 0; e < EPL; ++e) w[e] = v[e] = m[e] = 0.f;
    if (!peer && mine) {
      const size_t rb = (size_t)row * D + e0;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        w[e] = ew[rb + e];
        v[e] = ev[rb + e];
        if (em) m[e] = em[rb + e];
      }
    }
    if (!peer && lane == 0) st0 = d.step[row];
    if (lane >= c) p0 = kFull;
    if (32 + lane >= c) p1 = kFull;
    // rank every held position against all c positions: token order
    uint32_t r0 = 0, r1 = 0;
    const uint32_t c0 = min(c, 32u);
    for (uint32_t sl = 0; sl < c0; ++sl) {
      const uint32_t q = __shfl_sync(kFull, p0, sl);
      r0 += q < p0;
      r1 += q < p1;
    }
    for (uint32_t sl = 32; sl < c; ++sl) {
      const uint32_t q = __shfl_sync(kFull, p1, sl - 32);
      r0 += q < p0;
      r1 += q < p1;
    }
    if (lane < c && RS_IDX_OK(r0 < c && p0 < a.n_tokens, a.sh.ctr)) order[r0] = p0;
    if (32 + lane < c && RS_IDX_OK(r1 < c && p1 < a.n_tokens, a.sh.ctr)) order[r1] = p1;
    __syncwarp();
    // the forward: the pre-update row to each token
    if (!(a.exp & 4) && !peer) {
      for (uint32_t k = 0; k < c; ++k) {
        float* dst = a.out + (size_t)order[k] * D + e0;
        if (mine) {
          if (EPL == 2)
            __stcs(reinterpret_cast<float2*>(dst), make_float2(w[0], w[EPL > 1 ? 1 : 0]));
          else
#pragma unroll
            for (int e = 0; e < EPL; ++e) __stcs(dst + e, w[e]);
        }
      }
      for (uint32_t k = lane; k < c; k += 32) a.inverse[order[k]] = (int32_t)uu;
      if (a.tokcs) {  // the row sum in k_fc's tree: per float4 (x + y) + (z + w), then over the float4s
        double rs = 0.0;
#pragma unroll
        for (int e = 0; e < EPL; ++e) rs += mine ? (double)w[e] : 0.0;  // EPL 2: x + y (or z + w)
        if (EPL == 1) rs += __shfl_xor_sync(kFull, rs, 1);               // x + y
        rs += __shfl_xor_sync(kFull, rs, EPL == 1 ? 2 : 1);              // (x + y) + (z + w)
        for (uint32_t o2 = 16; o2 >= (EPL == 1 ? 4u : 2u); o2 >>= 1) rs += __shfl_xor_sync(kFull, rs, o2);
        for (uint32_t k = lane; k < c; k += 32) a.tokcs[order[k]] = rs;
      }
    }
    // the sums in token order, kB rows in flight
    float acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
    constexpr int kB = 16;
    if (!(a.exp & 2) && mine) {
      uint32_t k = 0;
      for (; k + kB <= c; k += kB) {
        float x[kB][EPL];
#pragma unroll
        for (int q = 0; q < kB; ++q) ld_row<EPL>(a.grads + (size_t)order[k + q] * D + e0, x[q]);
#pragma unroll
        for (int q = 0; q < kB; ++q)
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[e] += x[q][e];
      }
      if (k < c) {  // the tail: all its rows in flight, then the adds in order
        float x[kB][EPL];
#pragma unroll
        for (int q = 0; q < kB; ++q)
          if (k + q < c) ld_row<EPL>(a.grads + (size_t)order[k + q] * D + e0, x[q]);
#pragma unroll
        for (int q = 0; q < kB; ++q)
          if (k + q < c)
#pragma unroll
            for (int e = 0; e < EPL; ++e) acc[e] += x[q][e];
      }
    }
    __syncwarp();
    if (peer) {  // the id's sum to its owner's gradient receive buffer (NVLink store)
      const uint32_t ow = row / a.cap, jj = row - ow * a.cap;
      if (mine) {
        float* dst = a.peer_dst[ow] + ((size_t)a.rank * a.cap + jj) * D + e0;
#pragma unroll
        for (int e = 0; e < EPL; ++e) dst[e] = acc[e];
      }
      continue;
    }
    uint32_t st = 0;
    if (lane == 0) {
      st = st0 + 1;
      d.step[row] = st;
    }
    st = __shfl_sync(kFull, st, 0);
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
    if (mine) {
      const size_t rb = (size_t)row * D + e0;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        if (a.exp & 1)
          w[e] += acc[e];
        else if (o.kind == RS_OPT_ADAM)
          adam_elem(w[e], m[e], v[e], acc[e], bc1, bc2, o);
        else
          adagrad_elem(w[e], v[e], acc[e], o);
        ew[rb + e] = w[e];
        ev[rb + e] = v[e];
        if (em) em[rb + e] = m[e];
      }
    }
  }
}

#ifndef RS_FC_MINB
#define RS_FC_MINB 5
#endif
// MINB: resident blocks per SM the register budget is sized for -- the light
// kernel needs occupancy, the heavy one (few ids, long ordered sums) needs
// registers so that its B2 gradient rows are really in flight together
template <int G, int NV, int PMAX, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fc(FcArgs a, OptArgs o) {
  WarpTrace wt_(a.sh.trace, a.list ? 5 : 1);
  constexpr int PPT = (PMAX + G - 1) / G;  // positions held per thread
  __shared__ uint32_t order_s[(256 / G) * PMAX];
  const TableDesc d = a.td->d;
  const uint32_t D4 = d.dim >> 2;
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << (lane & ~(G - 1));
  const uint32_t gpb = blockDim.x / G;
  uint32_t* order = order_s + (threadIdx.x / G) * PMAX;
  const uint32_t gid = blockIdx.x * gpb + threadIdx.x / G;
  const uint32_t ngroups = gridDim.x * gpb;
  // the ids: every unique id (light kernel: c <= c_max), or KA's list of the
  // heavy ones (c_min < c <= c_max)
  const uint32_t nitems = a.list ? *a.list_n : *a.use.cnt;
  const float4* __restrict__ g4 = reinterpret_cast<const float4*>(a.grads);
  float4* rw = reinterpret_cast<float4*>(d.emb);
  float4* rv = reinterpret_cast<float4*>(d.s2);
  float4* rm = reinterpret_cast<float4*>(d.s1);
  for (uint32_t it = gid; it < nitems; it += ngroups) {
    // slot and row in one round trip (KA's claiming tile wrote both; list
    // mode: the slot's record), then the count, the positions (speculatively)
    // and the row's state together
    uint32_t gs, row, uu, c;
    if (a.list) {
      gs = __ldg(a.list + it);
      const uint2 cr = __ldcg(reinterpret_cast<const uint2*>(&a.use.rec[gs].cnt));
      c = cr.x;
      row = cr.y;
      uu = __ldcg(a.sh.uidx + gs);
    } else {
      uu = it;
      gs = __ldg(a.use.u_slot + uu);
      row = __ldg(a.urow + uu);
      c = 0;
    }
    if (row == kNoRow) continue;  // table error (reported through the counters)
    if (!RS_IDX_OK(gs < a.sh.n_slots && row < d.row_cap, a.sh.ctr)) continue;
    if (!a.list) c = __ldcg(&a.use.rec[gs].cnt);
    uint32_t p[PPT], r[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      p[j] = gl + j * G < PMAX ? __ldcg(a.sh.pos + (size_t)gs * kPosMax + gl + j * G) : kFull;
      r[j] = 0;
    }
    float4 wv[NV], vv[NV], mv[NV];
    const size_t rbase = (size_t)row * D4 + gl;
    const bool peer = a.peer_dst != nullptr;  // sharded requester: `row` is the send position
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      wv[j] = peer ? make_float4(0.f, 0.f, 0.f, 0.f) : rw[rbase + j * G];
      vv[j] = peer ? make_float4(0.f, 0.f, 0.f, 0.f) : rv[rbase + j * G];
      mv[j] = rm && !peer ? rm[rbase + j * G] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    uint32_t st0 = 0;
    if (gl == 0 && !peer) st0 = d.step[row];
    if (c > a.c_max || c <= a.c_min) continue;  // another kernel's id (group-uniform)
#pragma unroll
    for (int j = 0; j < PPT; ++j)
      if (gl + j * G >= c) p[j] = kFull;
    // rank every held position against all c positions of the id
#pragma unroll
    for (int jq = 0; jq < PPT; ++jq) {
      if ((uint32_t)(jq * G) >= c) break;
      const uint32_t lim = min((uint32_t)G, c - (uint32_t)(jq * G));
      for (uint32_t src = 0; src < lim; ++src) {
        const uint32_t q = __shfl_sync(gmask, p[jq], src, G);
#pragma unroll
        for (int j = 0; j < PPT; ++j) r[j] += q < p[j];
      }
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j)
      if (gl + j * G < c && RS_IDX_OK(r[j] < c && p[j] < a.n_tokens, a.sh.ctr)) order[r[j]] = p[j];
    __syncwarp(gmask);
    // the forward for this id: its pre-update row to each of its tokens
    // (distributed_lookup's inverse expand, exchange_sim.cpp:211-230)
    if (!(a.exp & 4) && !peer) {
      float4* o4 = reinterpret_cast<float4*>(a.out);
      for (uint32_t k = 0; k < c; ++k) {
        const size_t ob = (size_t)order[k] * D4 + gl;
#pragma unroll
        for (int j = 0; j < NV; ++j) __stcs(o4 + ob + j * G, wv[j]);
      }
      for (uint32_t k = gl; k < c; k += G) a.inverse[order[k]] = (int32_t)uu;
      if (a.tokcs) {
        double rs = 0.0;
#pragma unroll
        for (int j = 0; j < NV; ++j) rs += ((double)wv[j].x + (double)wv[j].y) + ((double)wv[j].z + (double)wv[j].w);
#pragma unroll
        for (int o2 = G / 2; o2 > 0; o2 >>= 1) rs += __shfl_xor_sync(gmask, rs, o2, G);
        for (uint32_t k = gl; k < c; k += G) a.tokcs[order[k]] = rs;
      }
    }
    float4 acc[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    // rows in flight: B2 per step of the long loop, B for the tail; a
    // register-tight build (MINB >= 4 with 64 positions) keeps B2 = B so the
    // loads are not serialized by spills
    constexpr int B = NV == 1 ? 4 : 2;
    constexpr int B2 = (MINB >= 4 && PMAX > 8) ? B : 2 * B;
    uint32_t k = (a.exp & 2) ? c : 0;
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
    __syncwarp(gmask);
    if (peer) {  // the id's sum to its owner's gradient receive buffer (NVLink store)
      const uint32_t o = row / a.cap, jj = row - o * a.cap;
      float4* dst = reinterpret_cast<float4*>(a.peer_dst[o] + ((size_t)a.rank * a.cap + jj) * d.dim);
#pragma unroll
      for (int j = 0; j < NV; ++j) dst[gl + j * G] = acc[j];
      continue;
    }
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
        if (a.exp & 1)
          wp[e] += gp[e];
        else if (o.kind == RS_OPT_ADAM)
          adam_elem(wp[e], mp[e], vp[e], gp[e], bc1, bc2, o);
        else
          adagrad_elem(wp[e], vp[e], gp[e], o);
      }
      rw[rbase + j * G] = wv[j];
      rv[rbase + j * G] = vv[j];
      if (rm) rm[rbase + j * G] = mv[j];
    }
  }
}

// ---------------------------------------------------------------------------
// KH: per tile, the tokens of hot ids grouped by id (first occurrence
// order), each group's gradient rows summed in token order straight from
// global memory by one warp; the (tile, id) partial goes to part[], its
// index to the id's tile list.
struct FhArgs {
  FSet use;
  FShared sh;
  const uint32_t* slot_of;
  uint32_t n;
  const float* grads;
  uint32_t dim;
  const float* emb;  // table rows (hot rows are not updated before KF)
  float* out;
  int32_t* inverse;
  double* tokcs;
  uint32_t exp;  // timing experiments (RS_FH_EXP bits, wrong results): 1 no forward stores, 2 no gradient sums
  // out == nullptr: no forward (sharded requester: the rows come from the owners)
};



constexpr uint32_t kRowStage = 8;  // group rows per warp staged in smem (more: read from global)

template <int VEC, int CH>
__global__ void __launch_bounds__(kTT, 4) k_fh(FhArgs a) {
  WarpTrace wt_(a.sh.trace, 2);
  constexpr uint32_t L = 2 * kTT, NW = kTT / 32;
  const uint32_t D = a.dim;
  extern __shared__ __align__(16) float srow[];  // [kRowStage * NW x D] the first groups' rows
  __shared__ uint32_t lkey[L], lfirst[L], lgroup[L];
  __shared__ uint32_t gcnt[kTT], goff[kTT], gslot[kTT], grow[kTT], gpidx[kTT];
  __shared__ uint16_t wcnt[NW * kTT];
  __shared__ uint16_t csr[kTT];
  __shared__ uint32_t wsum[32], s_ng, s_pbase, s_nhot;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t tile = blockIdx.x, t0 = tile * kTT;
  const uint32_t rows = min(kTT, a.n - t0);
  for (uint32_t i = tid; i < L; i += kTT) {
    lkey[i] = kFull;
    lfirst[i] = kFull;
  }
  for (uint32_t i = tid; i < NW * kTT; i += kTT) wcnt[i] = 0;
  const bool valid = tid < rows;
  uint32_t gs = 0, row = kNoRow;
  bool hot = false;
  if (valid) {  // the token's record (count, row) and unique index in one round trip
    gs = __ldg(a.slot_of + t0 + tid);
    const uint2 cr = __ldcg(reinterpret_cast<const uint2*>(&a.use.rec[gs].cnt));
    const uint32_t ux = __ldcg(a.sh.uidx + gs);
    hot = cr.x > a.sh.hot_min;
    row = cr.y;
    if (hot) a.inverse[t0 + tid] = (int32_t)ux;
  }
  // the hot tokens' rank in the tile (block scan of the hot flags)
  const unsigned hbal = __ballot_sync(kFull, hot);
  if (lane == 0) wsum[warp] = __popc(hbal);
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
    if (lane == 31) s_nhot = x;
  }
  __syncthreads();
  const uint32_t nhot = s_nhot;
  if (nhot == 0) return;  // no hot token in this tile (block-uniform)
  uint32_t ps = 0;
  if (hot) {
    ps = hash32(gs) & (L - 1);
    for (;;) {
      const uint32_t prev = atomicCAS(&lkey[ps], kFull, gs);
      if (prev == kFull || prev == gs) break;
      ps = (ps + 1) & (L - 1);
    }
    atomicMin(&lfirst[ps], tid);
  }
  __syncthreads();
  const bool head = hot && lfirst[ps] == tid;
  const unsigned hb = __ballot_sync(kFull, head);
  __syncthreads();  // wsum is reused
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
    if (lane == 31) s_ng = x;
  }
  __syncthreads();
  const uint32_t ng = s_ng;
  if (head) {
    const uint32_t lg = wsum[warp] + __popc(hb & lanemask_lt());
    lgroup[ps] = lg;
    gslot[lg] = gs;
    grow[lg] = row;
  }
  if (tid == 0) s_pbase = atomicAdd(&a.sh.ctr[1], ng);  // the tile's partial slots: one atomic
  __syncthreads();
  // per-warp counts of each group, then each token's place in its group (token order)
  const uint32_t mylg = hot ? lgroup[ps] : (0xFFFF0000u | lane);
  const unsigned mm = __match_any_sync(kFull, mylg);
  const uint32_t rw = __popc(mm & lanemask_lt());
  if (hot && rw == 0) wcnt[warp * kTT + mylg] = (uint16_t)__popc(mm);
  __syncthreads();
  if (tid < ng) {
    uint32_t run = 0;
    for (uint32_t w = 0; w < NW; ++w) {
      const uint32_t c = wcnt[w * kTT + tid];
      wcnt[w * kTT + tid] = (uint16_t)run;
      run += c;
    }
    gcnt[tid] = run;
    // the group's hot index (claimed by the first tile that gets here; the
    // claimer waits on nothing) and its partial slot in the id's tile list
    const uint32_t sl = gslot[tid];
    uint32_t h = __ldcg(&a.sh.hidx[sl]);
    if (h == kHotNone) {
      const uint32_t old = atomicCAS(&a.sh.hidx[sl], kHotNone, kHotClaim);
      if (old == kHotNone) {
        h = atomicAdd(&a.sh.ctr[0], 1u);
        if (RS_IDX_OK(h < a.sh.max_hot, a.sh.ctr)) a.sh.hot_slot[h] = sl;
        __threadfence();
        atomicExch(&a.sh.hidx[sl], h);
      } else {
        h = old;
      }
    }
    // bounded spin: a broken protocol reports an error instead of hanging the GPU
    for (uint32_t spin = 0; h == kHotClaim; ++spin) {
      if (spin > (1u << 22)) {
        atomicOr(&a.sh.ctr[2], 1u);
        break;
      }
      __nanosleep(32);
      h = atomicAdd(&a.sh.hidx[sl], 0u);
    }
    if (h < kHotClaim && RS_IDX_OK(h < a.sh.max_hot && tile < a.sh.ntiles && s_pbase + tid < a.n, a.sh.ctr)) {
      gpidx[tid] = s_pbase + tid;
      a.sh.hlist[(size_t)h * a.sh.ntiles + tile] = s_pbase + tid + 1;
    } else {
      gpidx[tid] = kFull;
    }
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
  if (hot) csr[goff[mylg] + wcnt[warp * kTT + mylg] + rw] = (uint16_t)tid;
  // Warp w takes a contiguous range of groups holding ~1/NW of the tile's hot
  // tokens and streams them as one list: PF gradient rows in flight across
  // group boundaries (no per-group round trip), the sums in token order per
  // group, each group's partial stored after its last token; the groups'
  // table rows are fetched up front into smem (one round trip for all) and
  // stored to each token (the forward).
  const uint32_t nhot_t = ng ? goff[ng - 1] + gcnt[ng - 1] : 0u;
  auto first_group = [&](uint32_t wq) -> uint32_t {  // groups starting before token wq * nhot / NW
    const uint64_t lim = (uint64_t)wq * nhot_t;
    uint32_t cnt = 0;
    for (uint32_t g = lane; g < ng; g += 32) cnt += (uint64_t)goff[g] * NW < lim;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o2);
    return cnt;
  };
  const uint32_t gb = warp == 0 ? 0u : first_group(warp);
  const uint32_t ge = warp == NW - 1 ? ng : first_group(warp + 1);
  if (!(a.exp & 4)) {  // the tile's first kRowStage * NW group rows -> smem, warp w fetching
     // groups w, w + NW, ...: every load issued before the first store
    float wr[kRowStage][CH][VEC];
#pragma unroll
    for (uint32_t k = 0; k < kRowStage; ++k) {
      const uint32_t gg = warp + k * NW;
      if (a.out && gg < ng && grow[gg] != kNoRow) load_vec<VEC, CH>(a.emb + (size_t)grow[gg] * D, D, wr[k], false);
    }
#pragma unroll
    for (uint32_t k = 0; k < kRowStage; ++k) {
      const uint32_t gg = warp + k * NW;
      if (a.out && gg < ng && grow[gg] != kNoRow) store_vec<VEC, CH>(srow + (size_t)gg * D, D, wr[k]);
    }
  }
  __syncthreads();
  constexpr int PF = (CH * VEC <= 4) ? 8 : (CH * VEC <= 8) ? 4 : 2;
  const uint32_t tb = gb < ng ? goff[gb] : nhot_t, te = ge < ng ? goff[ge] : nhot_t;
  uint32_t g = gb, gend = gb < ge ? goff[gb] + gcnt[gb] : 0u;
  float w[CH][VEC], acc[CH][VEC];
  zero_acc<VEC, CH>(acc);
  auto row_of = [&](uint32_t gg, float (&r)[CH][VEC]) {
    if (!a.out || grow[gg] == kNoRow) return;
    if (gg < kRowStage * NW)
      load_vec<VEC, CH>(srow + (size_t)gg * D, D, r, false);
    else
      load_vec<VEC, CH>(a.emb + (size_t)grow[gg] * D, D, r, false);
  };
  auto finish_group = [&](uint32_t gg) {
    const uint32_t pidx = gpidx[gg];
    if (pidx != kFull) store_vec<VEC, CH>(a.sh.part + (size_t)pidx * D, D, acc);
    if (a.tokcs && grow[gg] != kNoRow) {
      double rs = 0.0;
#pragma unroll
      for (int c2 = 0; c2 < CH; ++c2)
#pragma unroll
        for (int j = 0; j < VEC; ++j) rs += (double)w[c2][j];
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) rs += __shfl_xor_sync(kFull, rs, o2);
      for (uint32_t k = lane; k < gcnt[gg]; k += 32) a.tokcs[t0 + csr[goff[gg] + k]] = rs;
    }
  };
  if (gb < ge) row_of(gb, w);
  for (uint32_t i0 = tb; i0 < ((a.exp & 8) ? tb : te); i0 += PF) {
    float x[PF][CH][VEC];
#pragma unroll
    for (int q = 0; q < PF; ++q)
      if (i0 + q < te && !(a.exp & 2)) load_vec<VEC, CH>(a.grads + (size_t)(t0 + csr[i0 + q]) * D, D, x[q], false);
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const uint32_t i = i0 + q;
      if (i >= te) break;
      while (i >= gend) {  // the previous group is complete
        finish_group(g);
        zero_acc<VEC, CH>(acc);
        ++g;
        gend = goff[g] + gcnt[g];
        row_of(g, w);
      }
      if (!(a.exp & 2)) add_acc<VEC, CH>(acc, x[q]);
      if (a.out && grow[g] != kNoRow && !(a.exp & 1)) store_vec<VEC, CH>(a.out + (size_t)(t0 + csr[i]) * D, D, w);
    }
  }
  if (gb < ge && !(a.exp & 8)) finish_group(g);
}

// ---------------------------------------------------------------------------
// KF: per hot id (block of NWF warps): its partials in tile order, split over
// the warps in fixed contiguous chunks, warp sums combined in warp order
// (deterministic), then the optimizer.  Resets the id's tile list and hot
// index for the next step.
struct FfArgs {
  TableDev* td;
  FSet use;
  FShared sh;
  float* const* peer_dst;  // sharded requester: the sums to the owners (rows are send positions)
  uint32_t cap, rank;
};

template <int VEC, int CH, int NWF>
__global__ void __launch_bounds__(NWF * 32) k_fhf(FfArgs a, OptArgs o) {
  WarpTrace wt_(a.sh.trace, 3);
  extern __shared__ __align__(16) unsigned char smf[];
  uint32_t* list = reinterpret_cast<uint32_t*>(smf);                        // [ntiles]
  float* wpart = reinterpret_cast<float*>(list + ((a.sh.ntiles + 3) & ~3u));  // [NWF x D]
  __shared__ uint32_t s_w[NWF + 1];
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const TableDesc d = a.td->d;
  const uint32_t D = d.dim;
  const uint32_t nh = *reinterpret_cast<volatile uint32_t*>(&a.sh.ctr[0]);
  const uint32_t NT = a.sh.ntiles;
  for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
    if (!RS_IDX_OK(h < a.sh.max_hot, a.sh.ctr)) break;
    const uint32_t gs = a.sh.hot_slot[h];
    uint32_t* hl = a.sh.hlist + (size_t)h * NT;
    if (warp == NWF - 1 && !a.peer_dst) {  // the row's optimizer state: into L2 while the partials are summed
      const uint32_t row = __ldcg(&a.use.rec[gs].row);
      if (row != kNoRow && lane * 32u < D * 4u) {
        const char* w = reinterpret_cast<const char*>(d.emb + (size_t)row * D) + lane * 32;
        const char* v = reinterpret_cast<const char*>(d.s2 + (size_t)row * D) + lane * 32;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(w));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(v));
        if (d.s1) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(d.s1 + (size_t)row * D) + lane * 32));
      }
    }
    // compaction of the present partials, in tile order
    uint32_t m = 0;
    for (uint32_t b = 0; b < NT; b += NWF * 32) {
      const uint32_t i = b + tid;
      const uint32_t v = i < NT ? hl[i] : 0u;
      if (v) hl[i] = 0;
      const unsigned bal = __ballot_sync(kFull, v != 0);
      if (lane == 0) s_w[warp] = __popc(bal);
      __syncthreads();
      if (tid == 0) {
        uint32_t run = 0;
        for (uint32_t w = 0; w < NWF; ++w) {
          const uint32_t x = s_w[w];
          s_w[w] = run;
          run += x;
        }
        s_w[NWF] = run;
      }
      __syncthreads();
      if (v) list[m + s_w[warp] + __popc(bal & lanemask_lt())] = v - 1;
      m += s_w[NWF];
      __syncthreads();
    }
    const uint32_t per = (m + NWF - 1) / NWF;
    const uint32_t r0 = min(warp * per, m), r1 = min(r0 + per, m);
    float acc[CH][VEC];
    zero_acc<VEC, CH>(acc);
    constexpr int PF = (CH * VEC <= 4) ? 8 : (CH * VEC <= 8) ? 4 : 2;
    for (uint32_t k0 = r0; k0 < r1; k0 += PF) {
      float x[PF][CH][VEC];
#pragma unroll
      for (int q = 0; q < PF; ++q)
        if (k0 + q < r1 && RS_IDX_OK(list[k0 + q] < a.sh.max_tokens, a.sh.ctr))
          load_vec<VEC, CH>(a.sh.part + (size_t)list[k0 + q] * D, D, x[q], true);
#pragma unroll
      for (int q = 0; q < PF; ++q)
        if (k0 + q < r1) add_acc<VEC, CH>(acc, x[q]);
    }
    store_vec<VEC, CH>(wpart + (size_t)warp * D, D, acc);
    __syncthreads();
    if (warp == 0) {
      float tot[CH][VEC];
      zero_acc<VEC, CH>(tot);
      for (uint32_t w = 0; w < NWF; ++w) {
        float x[CH][VEC];
        load_vec<VEC, CH>(wpart + (size_t)w * D, D, x, false);
        add_acc<VEC, CH>(tot, x);
      }
      const uint32_t row = __ldcg(&a.use.rec[gs].row);
      if (a.peer_dst) {  // the id's sum to its owner's gradient receive buffer (NVLink store)
        const uint32_t ow = row / a.cap, jj = row - ow * a.cap;
        store_vec<VEC, CH>(a.peer_dst[ow] + ((size_t)a.rank * a.cap + jj) * D, D, tot);
      } else {
        apply_row<VEC, CH>(d, row, tot, o);
      }
      if (lane == 0) a.sh.hidx[gs] = kHotNone;
    }
    __syncthreads();
  }
}

struct Shape {
  int vec, ch;
};
Shape shape_of(uint32_t D) {
  if (D % 128 == 0 && D / 128 <= 4) return {4, (int)(D / 128)};
  if (D % 64 == 0 && D / 64 <= 2) return {2, (int)(D / 64)};
  return {1, (int)((D + 31) / 32)};
}

}  // namespace

// ---- host side ---------------------------------------------------------------
bool fast_step_supported(const rs_table* t) {
  // bounded tables too: KA without table work, then the bounded ensure (fast_enqueue); RS_FAST_BOUNDED=0: split kernels
  static const bool bounded = !getenv("RS_FAST_BOUNDED") || getenv("RS_FAST_BOUNDED")[0] != '0';
  return (bounded || !t->cfg.max_keys) && fast_dim_supported(t->desc.dim);
}

bool fast_dim_supported(uint32_t D) {
  if (D % 4) return false;
  const Shape sh = shape_of(D);
  const uint32_t D4 = D / 4;
  const bool g_ok = D4 == 4 || D4 == 8 || D4 == 16 || D4 == 32 || D4 == 64;
  const bool s_ok = (sh.vec == 4 && sh.ch <= 2) || (sh.vec == 2 && sh.ch <= 2) || (sh.vec == 1 && sh.ch <= 2);
  return g_ok && s_ok;
}

static cudaError_t fast_trace_reset(rs_workspace* ws) {
  // [kernel][block] = {start = ~0, end = 0}
  std::vector<unsigned long long> h(kTraceSlots * kTraceBlocks * 2);
  for (size_t i = 0; i < h.size(); i += 2) {
    h[i] = ~0ull;
    h[i + 1] = 0;
  }
  return cudaMemcpy(ws->fast.trace, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
}

static int fast_alloc(rs_workspace* ws) {
  rs_fast& f = ws->fast;
  if (f.ready) return RS_OK;
  const uint64_t S = ws->S, N = ws->max_tokens;
  f.ntiles = (N + kTT - 1) / kTT;
  f.hot_min = kPosMax;
  if (const char* e = getenv("RS_HOT_MIN")) f.hot_min = std::min<uint32_t>(kPosMax, std::max(1, atoi(e)));
  f.max_hot = N / (f.hot_min + 1) + 1;
  f.light_max = std::min<uint32_t>(f.hot_min, 8);  // <= the light kernel's 8 positions
  if (const char* e = getenv("RS_LIGHT_MAX")) f.light_max = std::min<uint32_t>(f.light_max, std::max(1, atoi(e)));
  auto A = [&](auto** p, size_t bytes) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 16)) == cudaSuccess;
  };
  bool ok = true;
  for (auto& x : f.set) ok = ok && A(&x.rec, (S + 1) * sizeof(Rec)) && A(&x.u_slot, N * 4) && A(&x.cnt, 16);
  ok = ok && A(&f.uidx, (S + 1) * 4) && A(&f.hidx, (S + 1) * 4) && A(&f.pos, (S + 1) * kPosMax * 4) &&
       A(&f.hot_slot, f.max_hot * 4) && A(&f.hlist, f.max_hot * f.ntiles * 4) && A(&f.ctr, 64) &&
       A(&f.tokcs, N * 8) && A(&f.heavy, N * 4);
  if (!ok) return cuda_fail(cudaGetLastError(), "fast step: cudaMalloc");
  // empty records (key ~0, count 0, row ~0): all-ones then zero counts
  for (auto& x : f.set) {
    RS_CUDA(cudaMemset(x.rec, 0xFF, (S + 1) * sizeof(Rec)));
    RS_CUDA(cudaMemset2D(reinterpret_cast<char*>(x.rec) + 8, sizeof(Rec), 0, 4, S + 1));
    RS_CUDA(cudaMemset(x.cnt, 0, 16));
  }
  RS_CUDA(cudaMemset(f.hidx, 0xFF, (S + 1) * 4));
  RS_CUDA(cudaMemset(f.hlist, 0, f.max_hot * f.ntiles * 4));
  RS_CUDA(cudaMemset(f.ctr, 0, 64));
  if (getenv("RS_TRACE") && getenv("RS_TRACE")[0] == '1') {
    RS_CUDA(cudaMalloc(&f.trace, kTraceSlots * kTraceBlocks * 2 * sizeof(unsigned long long)));
    RS_CUDA(fast_trace_reset(ws));
  }
  {  // the hot branch (KH -> KF) at the highest priority: KF's blocks go ahead of the CSR kernel's pending ones
    int lo = 0, hi = 0;
    RS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // RS_FAST_PRIO = "<hot branch><heavy CSR>", each 'h' (high) or 'n' (default)
    const char* pe = getenv("RS_FAST_PRIO");
    const bool p_hot = !pe || pe[0] != 'n', p_heavy = !pe || !pe[0] || pe[1] != 'n';
    RS_CUDA(cudaStreamCreateWithPriority(&f.aux2, cudaStreamNonBlocking, p_hot ? hi : 0));
    RS_CUDA(cudaStreamCreateWithPriority(&f.aux3, cudaStreamNonBlocking, p_heavy ? hi : 0));
  }
  RS_CUDA(cudaEventCreateWithFlags(&f.ev_fork, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&f.ev_j1, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&f.ev_j2, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&f.ev_j3, cudaEventDisableTiming));
  RS_CUDA(cudaDeviceSynchronize());
  f.ready = true;
  return RS_OK;
}

void fast_free(rs_workspace* ws) {
  rs_fast& f = ws->fast;
  for (auto& x : f.set) {
    void* ps[] = {x.rec, x.u_slot, x.cnt};
    for (void* p : ps)
      if (p) cudaFree(p);
  }
  void* ps[] = {f.uidx, f.hidx, f.pos, f.hot_slot, f.hlist, f.ctr, f.tokcs, f.trace, f.heavy};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (f.aux2) cudaStreamDestroy(f.aux2);
  if (f.aux3) cudaStreamDestroy(f.aux3);
  cudaEvent_t es[] = {f.ev_fork, f.ev_j1, f.ev_j2, f.ev_j3};
  for (auto e : es)
    if (e) cudaEventDestroy(e);
  f = rs_fast{};
}

int fast_prepare(rs_workspace* ws) { return fast_alloc(ws); }

// Checked builds: the step's device error bits (bounds violations, a hot-index
// claim that never resolved) fail the call.  No-op otherwise (no sync).
int fast_check_errors(rs_workspace* ws, cudaStream_t s) {
#ifdef RS_BOUNDS
  uint32_t bits = 0;
  RS_CUDA(cudaStreamSynchronize(s));
  RS_CUDA(cudaMemcpy(&bits, ws->fast.ctr + 2, 4, cudaMemcpyDeviceToHost));
  if (bits) return fail(RS_ERR_INVARIANT, "fast step: device error bits " + std::to_string(bits));
#else
  (void)ws;
  (void)s;
#endif
  return RS_OK;
}

static FSet fset(rs_workspace* ws, int k) {
  rs_fast_set& x = ws->fast.set[k];
  FSet s;
  s.rec = reinterpret_cast<Rec*>(x.rec);
  s.u_slot = x.u_slot;
  s.cnt = x.cnt;
  s.smask = ws->S - 1;
  s.spare = ws->S;
  return s;
}
static FShared fshared(rs_workspace* ws) {
  rs_fast& f = ws->fast;
  FShared s;
  s.uidx = f.uidx;
  s.hidx = f.hidx;
  s.pos = f.pos;
  s.hot_slot = f.hot_slot;
  s.hlist = f.hlist;
  s.part = ws->pbuf;
  s.ctr = f.ctr;
  s.ntiles = (uint32_t)f.ntiles;
  s.hot_min = f.hot_min;
  s.trace = f.trace;
  s.heavy = f.heavy;
  s.light_max = f.light_max;
  s.n_slots = ws->S + 1;
  s.max_tokens = (uint32_t)ws->max_tokens;
  s.max_hot = (uint32_t)f.max_hot;
  return s;
}

// The fast step's launches.  Single GPU: t = the table, both halves.  The
// sharded requester (dist.cu) calls the halves separately: KA with `send`
// (ids to their owners, no table), then the reduce with `peer` (sums to the
// owners' gradient buffers instead of the optimizer, no forward: the rows
// come from the owners), `td` = the receive-buffer view (only its dim and
// row bound are read).  Enqueue-only (capturable).  ev != null: eager
// profiling -- the kernels run one after another with events ev[0..4]
// around KA, KG, KD, KH+KF.
struct FastPeer {
  float* const* peer_dst;
  uint32_t cap, rank;
};
static int fast_launch(rs_workspace* ws, TableDev* td, const float* emb, uint32_t D, const uint64_t* d_ids,
                       uint64_t n, const float* d_grads, float* d_out, const OptArgs& o, int use, cudaStream_t s,
                       cudaEvent_t* ev, bool fork, TableCounters* mirror_out, const rs_dist_send* send,
                       const FastPeer* peer, bool do_ka, bool do_reduce) {
  const uint32_t ntiles = (uint32_t)((n + kTT - 1) / kTT);
  const FShared sh = fshared(ws);
  if (ev) RS_CUDA(cudaEventRecord(ev[0], s));
  FaArgs fa;
  fa.ids = d_ids;
  fa.n = (uint32_t)n;
  fa.set = (uint32_t)use;
  fa.use = fset(ws, use);
  fa.clean = fset(ws, use ^ 1);
  fa.sh = sh;
  fa.td = td;
  fa.slot_of = ws->slot_of;
  fa.unique = ws->unique;
  fa.urow = ws->urow;
  fa.urow64 = ws->urow64;
  if (send) fa.send = *send;
  // RS_CLEAN_IN_KA=1: KA cleans the previous set instead of k_fclean (the
  // single-GPU table step's counters then reach the mirror from KA's
  // epilogue) -- measured no faster at config 1 / N = 4, e2e slower; off
  static const bool clean_ka = getenv("RS_CLEAN_IN_KA") && getenv("RS_CLEAN_IN_KA")[0] == '1';
  fa.clean_in_ka = clean_ka ? 1 : 0;
  if (clean_ka && td && !send && !peer) fa.mirror_out = mirror_out;
  if (do_ka) {
    carve(k_fa), k_fa<<<std::max(ntiles, 1u), kTT, 0, s>>>(fa);  // an idle sharded rank still publishes its (empty) send
    RS_LAUNCH_CHECK("k_fa");
  }
  if (!do_reduce) return RS_OK;
  if (ev) RS_CUDA(cudaEventRecord(ev[1], s));
  rs_fast& f = ws->fast;
  cudaStream_t sd = s, sh2 = s, sd3 = s;
  if (fork && !ev) {
    RS_CUDA(cudaEventRecord(f.ev_fork, s));
    RS_CUDA(cudaStreamWaitEvent(ws->aux_stream, f.ev_fork, 0));
    RS_CUDA(cudaStreamWaitEvent(f.aux2, f.ev_fork, 0));
    RS_CUDA(cudaStreamWaitEvent(f.aux3, f.ev_fork, 0));
    sd = ws->aux_stream;
    sh2 = f.aux2;
    sd3 = f.aux3;
  }
  const Shape shp = shape_of(D);
  // hot branch first (longest chain): KH -> KF
  auto hot = [&](cudaStream_t q) -> int {
    FhArgs h;
    h.use = fa.use;
    h.sh = sh;
    h.slot_of = ws->slot_of;
    h.n = (uint32_t)n;
    h.grads = d_grads;
    h.dim = D;
    h.emb = emb;
    h.out = peer ? nullptr : d_out;
    h.inverse = ws->inverse;
    h.tokcs = ws->csum_dst && !peer ? f.tokcs : nullptr;
    static const uint32_t hexp = getenv("RS_FH_EXP") ? (uint32_t)atoi(getenv("RS_FH_EXP")) : 0u;
    h.exp = hexp;
    FfArgs ff;
    ff.td = td;
    ff.use = fa.use;
    ff.sh = sh;
    ff.peer_dst = peer ? peer->peer_dst : nullptr;
    ff.cap = peer ? peer->cap : 0u;
    ff.rank = peer ? peer->rank : 0u;
    // hot finish: a block of kf_warps warps per hot id (small blocks fit beside the CSR kernel's)
    static const int kfw = getenv("RS_KF_WARPS") ? atoi(getenv("RS_KF_WARPS")) : 8;
    const int nwf = kfw == 4 || kfw == 16 ? kfw : 8;
    const size_t fsm = ((f.ntiles + 3) & ~3ull) * 4 + (size_t)nwf * D * 4;
    const unsigned fgrid = (unsigned)std::min<uint64_t>(f.max_hot, 148 * 4);
#define RS_KF(V, C, NWV)                                                                     \
  if (nwf == NWV) {                                                                          \
    if (fsm > 48 * 1024)                                                                     \
      RS_CUDA(cudaFuncSetAttribute(k_fhf<V, C, NWV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                   (int)fsm));                                               \
    carve(k_fhf<V, C, NWV>), k_fhf<V, C, NWV><<<fgrid, NWV * 32, fsm, q>>>(ff, o);                                    \
  }
#define RS_FH(V, C)                                                                        \
  if (shp.vec == V && shp.ch == C) {                                                       \
    if ((kTT / 32) * kRowStage * D * 4 > 48 * 1024)                                         \
      RS_CUDA(cudaFuncSetAttribute(k_fh<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                   (int)((kTT / 32) * kRowStage * D * 4)));                  \
    carve(k_fh<V, C>), k_fh<V, C><<<ntiles, kTT, (kTT / 32) * kRowStage * D * 4, q>>>(h);                      \
    RS_LAUNCH_CHECK("k_fh");                                                               \
    RS_KF(V, C, 4) RS_KF(V, C, 8) RS_KF(V, C, 16)                                          \
    RS_LAUNCH_CHECK("k_fhf");                                                              \
    return RS_OK;                                                                          \
  }
    RS_FH(4, 1) RS_FH(4, 2) RS_FH(2, 1) RS_FH(2, 2) RS_FH(1, 1) RS_FH(1, 2)
#undef RS_FH
#undef RS_KF
    return fail(RS_ERR_INVARIANT, "fast step: no hot kernel for this dim");
  };
  // CSR ids: the light kernel over every unique id (c <= light_max: short
  // ordered sums, 8 lanes per id) and the heavy kernel over KA's list
  // (light_max < c <= hot_min: 16 lanes, 64 positions), on two streams
  auto csr = [&](cudaStream_t ql, cudaStream_t qh) -> int {
    FcArgs c;
    c.td = td;
    c.use = fa.use;
    c.peer_dst = peer ? peer->peer_dst : nullptr;
    c.cap = peer ? peer->cap : 0u;
    c.rank = peer ? peer->rank : 0u;
    c.sh = sh;
    c.grads = d_grads;
    c.n_tokens = (uint32_t)n;
    c.urow = ws->urow;
    static const uint32_t fexp = getenv("RS_FC_EXP") ? (uint32_t)atoi(getenv("RS_FC_EXP")) : 0u;
    c.exp = fexp;
    c.out = peer ? nullptr : d_out;
    c.inverse = ws->inverse;
    c.tokcs = ws->csum_dst && !peer ? f.tokcs : nullptr;
    const uint32_t D4 = D / 4;
    static const unsigned cap_blocks = getenv("RS_FC_GRID") ? (unsigned)atoi(getenv("RS_FC_GRID")) : 148u * 16u;
    // heavy (first: its ids start at once on their stream)
    FcArgs ch = c;
    ch.list = f.heavy;
    ch.list_n = sh.ctr + 5 + use;
    ch.c_min = f.light_max;
    ch.c_max = f.hot_min;
    const uint64_t max_heavy = n / (f.light_max + 1) + 1;
#define RS_FC(GG, NVV, PM, MB, args, q, items)                                              \
  carve(k_fc<GG, NVV, PM, MB>), k_fc<GG, NVV, PM, MB><<<grid_for(items, 256 / GG, cap_blocks), 256, 0, q>>>(args, o);
    // a grid-stride grid: the heavy ids are ~1-2% of the unique ids
    static const uint64_t hcap = getenv("RS_FCH_ITEMS") ? (uint64_t)atoll(getenv("RS_FCH_ITEMS")) : 148ull * 16;
    const uint64_t hitems = std::min<uint64_t>(max_heavy, hcap);
    static const int hminb = getenv("RS_FC_HMINB") ? atoi(getenv("RS_FC_HMINB")) : 5;  // experiment knob
    // RS_FCB=1 (D = 32 / 64): the warp-per-id heavy kernel k_fcb -- measured
    // ~1-3 us slower per step at config 1 than k_fc (its blocks delay the
    // light kernel's), kept for other shapes' experiments
    static const bool fcb = getenv("RS_FCB") && getenv("RS_FCB")[0] == '1';
    constexpr int kNWB = 4;
    if (fcb && (D4 == 8 || D4 == 16)) {
      // a grid-stride grid: the heavy ids are ~1-2 % of the unique ids
      static const unsigned gcap = getenv("RS_FCB_GRID") ? (unsigned)atoi(getenv("RS_FCB_GRID")) : 296u;
      const unsigned g = grid_for(hitems, kNWB, gcap);
      if (D4 == 16)
        carve(k_fcb<2, kNWB>), k_fcb<2, kNWB><<<g, kNWB * 32, 0, qh>>>(ch, o);
      else
        carve(k_fcb<1, kNWB>), k_fcb<1, kNWB><<<g, kNWB * 32, 0, qh>>>(ch, o);
    }
    else if (D4 == 4) { RS_FC(4, 1, 64, 5, ch, qh, hitems) }
    else if (D4 == 8) { RS_FC(8, 1, 64, 5, ch, qh, hitems) }
    else if (D4 == 16 && hminb == 2) { RS_FC(16, 1, 64, 2, ch, qh, hitems) }
    else if (D4 == 16) { RS_FC(16, 1, 64, 5, ch, qh, hitems) }
    else if (D4 == 32) { RS_FC(16, 2, 64, 4, ch, qh, hitems) }
    else { RS_FC(16, 4, 64, 3, ch, qh, hitems) }
    RS_LAUNCH_CHECK("k_fc(heavy)");
    static const int lminb = getenv("RS_FC_LMINB") ? atoi(getenv("RS_FC_LMINB")) : 4;  // experiment knob
    FcArgs cl = c;
    cl.list = nullptr;
    cl.list_n = nullptr;
    cl.c_min = 0;
    cl.c_max = f.light_max;
    if (D4 == 4) { RS_FC(4, 1, 8, 5, cl, ql, n) }
    else if (D4 == 8) { RS_FC(8, 1, 8, 5, cl, ql, n) }
    else if (D4 == 16 && lminb == 3) { RS_FC(8, 2, 8, 3, cl, ql, n) }
    else if (D4 == 16) { RS_FC(8, 2, 8, 4, cl, ql, n) }
    else if (D4 == 32) { RS_FC(8, 4, 8, 3, cl, ql, n) }
    else { RS_FC(16, 4, 8, 3, cl, ql, n) }
#undef RS_FC
    RS_LAUNCH_CHECK("k_fc(light)");
    return RS_OK;
  };
  auto checksum = [&](cudaStream_t q) -> int {
    if (!ws->csum_dst || peer) return RS_OK;
    carve(k_fcs), k_fcs<<<ntiles, kTT, 0, q>>>(f.tokcs, (uint32_t)n, ws->csum_dst, ws->csum_part, ws->csum_ticket);
    RS_LAUNCH_CHECK("k_fcs");
    return RS_OK;
  };
  // (KA cleaned the set when it ran with clean_in_ka -- here, or as the
  // sharded requester's front; the bounded step's KA did not)
  const bool cleaned = clean_ka && (do_ka || peer);
  auto clean = [&]() -> int {
    if (cleaned) return RS_OK;
    carve(k_fclean), k_fclean<<<grid_for(n + 1, 256, 148 * 2), 256, 0, s>>>(
        fa.clean, reinterpret_cast<unsigned int*>(sh.ctr + 3), sh.trace, td, mirror_out);
    RS_LAUNCH_CHECK("k_fclean");
    return RS_OK;
  };
  int st;
  if (ev) {  // eager, serial: KA (+ clean) | KD | KH + KF | KS
    if ((st = clean())) return st;
    if ((st = csr(s, s))) return st;
    RS_CUDA(cudaEventRecord(ev[2], s));
    if ((st = hot(s))) return st;
    RS_CUDA(cudaEventRecord(ev[3], s));
    if ((st = checksum(s))) return st;
    RS_CUDA(cudaEventRecord(ev[4], s));
    return RS_OK;
  }
  // RS_FAST_SKIP (timing experiments only, wrong results): 1 = no hot branch, 2 = no CSR branch
  static const int skip = getenv("RS_FAST_SKIP") ? atoi(getenv("RS_FAST_SKIP")) : 0;
  // the clean after the branches (RS_CLEAN_LAST=0: before them -- measured
  // ~2 us slower at config 1: its blocks then delay the branches' first waves)
  static const bool clean_last = !getenv("RS_CLEAN_LAST") || getenv("RS_CLEAN_LAST")[0] != '0';

  if (!clean_last && (st = clean())) return st;
  if (skip != 1 && (st = hot(sh2))) return st;
  if (skip != 2 && (st = csr(sd, sd3))) return st;
  if (clean_last && (st = clean())) return st;
  if (sd != s) {
    RS_CUDA(cudaEventRecord(f.ev_j1, sd));
    RS_CUDA(cudaStreamWaitEvent(s, f.ev_j1, 0));
    RS_CUDA(cudaEventRecord(f.ev_j2, sh2));
    RS_CUDA(cudaStreamWaitEvent(s, f.ev_j2, 0));
    RS_CUDA(cudaEventRecord(f.ev_j3, sd3));
    RS_CUDA(cudaStreamWaitEvent(s, f.ev_j3, 0));
  }
  return checksum(s);
}

// Bounded tables: the rows the bounded ensure found / inserted (urow) into
// the set's records (the reduce kernels read rec.row).
__global__ void k_fpatch(FSet use, const uint32_t* __restrict__ urow) {
  const uint32_t nu = *use.cnt;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += gridDim.x * blockDim.x)
    use.rec[use.u_slot[u]].row = urow[u];
}

int fast_enqueue(rs_workspace* ws, rs_table* t, const uint64_t* d_ids, uint64_t n, const float* d_grads,
                 float* d_out, const void* opt, int use, cudaStream_t s, cudaEvent_t* ev, bool fork,
                 TableCounters* mirror_out) {
  if (t->cfg.max_keys) {
    // bounded: KA's dedup + metadata, then the bounded ensure on its unique
    // ids (probe + stamp-log victim selection + insert of the misses,
    // table.cu / evict.cu), the rows into the records, then the reduce
    FaArgs fa;
    fa.ids = d_ids;
    fa.n = (uint32_t)n;
    fa.set = (uint32_t)use;
    fa.use = fset(ws, use);
    fa.clean = fset(ws, use ^ 1);
    fa.sh = fshared(ws);
    fa.td = t->dev;
    fa.slot_of = ws->slot_of;
    fa.unique = ws->unique;
    fa.urow = ws->urow;
    fa.urow64 = ws->urow64;
    static const bool ka_probe = !getenv("RS_BOUNDED_KA_PROBE") || getenv("RS_BOUNDED_KA_PROBE")[0] != '0';
    const uint32_t ntiles = (uint32_t)((n + kTT - 1) / kTT);
    if (ev) RS_CUDA(cudaEventRecord(ev[0], s));
    int st = RS_OK;
    if (ka_probe) {  // KA probes (stamp, log, misses), then the evict and the insert of the misses
      fa.probe_only = 1;
      fa.missing = t->d_missing;
      fa.lg = log_args(t, 1);
      RS_CUDA(cudaMemsetAsync(&t->dev->c.missing, 0, sizeof(unsigned int), s));
      carve(k_fa), k_fa<<<std::max(ntiles, 1u), kTT, 0, s>>>(fa);
      RS_LAUNCH_CHECK("k_fa(probe)");
      st = table_bounded_evict_insert(t, ws->unique, ws->fast.set[use].cnt, n, ws->urow, ws->urow64, s);
    } else {
      fa.no_table = 1;
      carve(k_fa), k_fa<<<std::max(ntiles, 1u), kTT, 0, s>>>(fa);
      RS_LAUNCH_CHECK("k_fa(no table)");
      st = table_bounded_enqueue(t, ws->unique, ws->fast.set[use].cnt, n, ws->urow, ws->urow64, nullptr,
                                 nullptr, s);
    }
    if (st) return st;
    carve(k_fpatch), k_fpatch<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(fa.use, ws->urow);
    RS_LAUNCH_CHECK("k_fpatch");
    return fast_launch(ws, t->dev, t->desc.emb, t->desc.dim, d_ids, n, d_grads, d_out,
                       *static_cast<const OptArgs*>(opt), use, s, ev, fork, mirror_out, nullptr, nullptr, false,
                       true);
  }
  return fast_launch(ws, t->dev, t->desc.emb, t->desc.dim, d_ids, n, d_grads, d_out,
                     *static_cast<const OptArgs*>(opt), use, s, ev, fork, mirror_out, nullptr, nullptr, true, true);
}

// ---- the sharded requester on the fast kernels (dist.cu) ----------------------
int fast_dist_front(rs_workspace* ws, uint32_t D, const uint64_t* d_ids, uint64_t n, int use, cudaStream_t s,
                    const rs_dist_send& send) {
  OptArgs o{};
  return fast_launch(ws, nullptr, nullptr, D, d_ids, n, nullptr, nullptr, o, use, s, nullptr, false, nullptr,
                     &send, nullptr, true, false);
}

int fast_dist_reduce(rs_workspace* ws, TableDev* view, uint32_t D, uint64_t n, const float* d_grads, int use,
                     cudaStream_t s, bool fork, float* const* peer_dst, uint32_t cap, uint32_t rank) {
  OptArgs o{};
  FastPeer p{peer_dst, cap, rank};
  return fast_launch(ws, view, nullptr, D, nullptr, n, d_grads, nullptr, o, use, s, nullptr, fork, nullptr,
                     nullptr, &p, false, true);
}

// The requester's forward: every token's row from the owners' answers in the
// receive buffer (row = its id's send position), after the emb flags.
struct FgdArgs {
  const TableDev* view;
  FSet use;
  FShared sh;
  const uint32_t* slot_of;
  uint32_t n;
  int32_t* inverse;
  float* out;
  double* csum_out;
  double* csum_part;
  unsigned int* csum_ticket;
  rs_dist_sync sync;
  unsigned long long* trace;
};

template <int LPR>
__global__ void __launch_bounds__(kTT, 4) k_fgd(FgdArgs a) {
  WarpTrace wt_(a.trace, 6);
  dist_wait(a.sync);  // the owners' rows landed
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  constexpr uint32_t NW = kTT / 32;
  const uint32_t D4 = a.view->d.dim >> 2;
  const float4* __restrict__ emb = reinterpret_cast<const float4*>(a.view->d.emb);
  float4* __restrict__ o4 = reinterpret_cast<float4*>(a.out);
  constexpr int RPI = 32 / LPR;
  constexpr int ITERS = 32 / RPI;
  constexpr int BATCH = ITERS < 4 ? ITERS : 4;  // 64 registers: co-resident with the owner kernels
  const uint32_t sub = lane / LPR, l = lane % LPR;
  const bool csum = a.csum_out != nullptr;
  double cs = 0.0;
  const uint32_t ntiles = (a.n + kTT - 1) / kTT;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // grid <= ntiles: persistent blocks
    const uint32_t t0 = tile * kTT;
    const uint32_t rows = min(kTT, a.n - t0);
    uint32_t r = 0;
    if (tid < rows) {
      const uint32_t sl = __ldg(a.slot_of + t0 + tid);
      r = __ldcg(&a.use.rec[sl].row);
      a.inverse[t0 + tid] = (int32_t)__ldcg(a.sh.uidx + sl);
    }
    const uint32_t wb = warp * 32;
    const uint32_t cnt = rows > wb ? min(32u, rows - wb) : 0u;
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
          if (tok < cnt && j < D4) v[k] = __ldcg(emb + (size_t)rr[k] * D4 + j);  // written by peers this step
        }
#pragma unroll
        for (int k = 0; k < BATCH; ++k) {
          const uint32_t tok = (b0 + k) * RPI + sub;
          if (tok < cnt && j < D4) {
            __stcs(o4 + (size_t)(t0 + wb + tok) * D4 + j, v[k]);
            if (csum) cs += ((double)v[k].x + (double)v[k].y) + ((double)v[k].z + (double)v[k].w);
          }
        }
      }
    }
  }
  if (csum) {  // fixed reduction tree, then the block partials in block order
    __shared__ double s_cs[NW];
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) cs += __shfl_xor_sync(kFull, cs, o2);
    if (lane == 0) s_cs[warp] = cs;
    __syncthreads();
    if (warp == 0) {
      double x = lane < NW ? s_cs[lane] : 0.0;
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) x += __shfl_xor_sync(kFull, x, o2);
      unsigned last = 0;
      if (lane == 0) {
        a.csum_part[blockIdx.x] = x;
        __threadfence();
        last = atomicAdd(a.csum_ticket, 1u) == gridDim.x - 1;
      }
      if (__shfl_sync(kFull, last, 0)) {
        __threadfence();
        double y = 0.0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) y += __ldcg(a.csum_part + b);
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) y += __shfl_xor_sync(kFull, y, o2);
        if (lane == 0) {
          *a.csum_out = y;
          *a.csum_ticket = 0;
        }
      }
    }
  }
}

int fast_dist_gather(rs_workspace* ws, const TableDev* view, uint32_t D, uint64_t n, float* d_out, int use,
                     cudaStream_t s, const rs_dist_sync& sync, double* csum, uint32_t grid) {
  if (n == 0) return RS_OK;
  FgdArgs g;
  g.view = view;
  g.use = fset(ws, use);
  g.sh = fshared(ws);
  g.slot_of = ws->slot_of;
  g.n = (uint32_t)n;
  g.inverse = ws->inverse;
  g.out = d_out;
  g.csum_out = csum;
  g.csum_part = ws->csum_part;
  g.csum_ticket = ws->csum_ticket;
  g.sync = sync;
  g.trace = ws->fast.trace;
  const uint32_t ntiles = (uint32_t)((n + kTT - 1) / kTT);
  const uint32_t nb = grid ? std::min(grid, ntiles) : ntiles;
  const uint32_t D4 = D / 4;
  if (D4 >= 32) carve(k_fgd<32>), k_fgd<32><<<nb, kTT, 0, s>>>(g);
  else if (D4 >= 16) carve(k_fgd<16>), k_fgd<16><<<nb, kTT, 0, s>>>(g);
  else if (D4 >= 8) carve(k_fgd<8>), k_fgd<8><<<nb, kTT, 0, s>>>(g);
  else carve(k_fgd<4>), k_fgd<4><<<nb, kTT, 0, s>>>(g);
  RS_LAUNCH_CHECK("k_fgd");
  return RS_OK;
}

}  // namespace rs

extern "C" int rs_workspace_trace(rs_workspace* ws, uint64_t* out, uint64_t cap, uint64_t* n_out) {
  using namespace rs;
  if (!ws || !n_out) return fail(RS_ERR_CONFIG, "rs_workspace_trace: null argument");
  *n_out = 0;
  if (!ws->fast.trace) return RS_OK;  // RS_TRACE=1 at the first rs_step enables it
  const uint64_t n = (uint64_t)kTraceSlots * kTraceBlocks * 2;
  *n_out = n;
  if (!out) return RS_OK;
  if (cap < n) return fail(RS_ERR_CONFIG, "rs_workspace_trace: buffer too small");
  RS_CUDA(cudaDeviceSynchronize());
  RS_CUDA(cudaMemcpy(out, ws->fast.trace, n * 8, cudaMemcpyDeviceToHost));
  RS_CUDA(fast_trace_reset(ws));
  return RS_OK;
}
