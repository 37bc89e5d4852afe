// dist.cu -- the row-sharded step over the W GPUs of one node.
//
// Reference: distributed_lookup (exchange_sim.cpp:117-233) with
// DedupMode::kTwoStage, ownership shard_of = hash64(id) % W
// (exchange_sim.cpp:82-85), and run_workload's sparse update
// (workload.cpp:519-581).  The reference simulates the two all-to-alls with
// vector copies; here every rank is a process on its own B200 and the
// exchanges are peer stores over NVLink into a symmetric "arena" each rank
// exports with CUDA IPC, issued by the kernels that produce the data:
//
//   requester  KA dedup -> KB metadata + owner partition of the unique ids,
//              ids stored straight into the owner's ids_in (k_ftable)
//   owner      wait ids -> k_flatten -> KA stage-2 dedup over the
//              source-ordered concatenation -> KB find-or-insert on the shard
//              -> k_respond: each received position's row stored straight
//              into the requester's emb_in (the embedding "all-to-all")
//   requester  wait embs -> KC gather out[t] from emb_in (local HBM)
//   backward   requester: KC + KD aggregate its grads per unique id and
//              store each row straight into the owner's grad_in; owner:
//              wait grads -> per id sum over its origins in (source,
//              position) order (stage-2 origin order) -> optimizer
//
// Signalling: per (phase, source) epoch flags in the receiver's arena,
// written with st.release.sys after fence.acq_rel.sys, polled with
// ld.acquire.sys and a bounded spin (a dead peer sets an error instead of
// hanging the GPU).  The data flow itself orders buffer reuse across steps.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "opt_dev.cuh"
#include "rs_host.hpp"
#include "dist_sync.cuh"
#include "scratch_dev.cuh"
#include "table_dev.cuh"

namespace rs {
namespace {

using namespace tdev;
using namespace sdev;
using namespace odev;

constexpr int kMaxWorld = 64;

struct ArenaHdr {
  unsigned long long sig_ids[kMaxWorld];
  unsigned long long sig_emb[kMaxWorld];
  unsigned long long sig_grad[kMaxWorld];
  unsigned long long sig_bar[kMaxWorld];
  uint32_t cnt_in[kMaxWorld];
};

// trace slots (per rank, device u64)
enum : int { kTrIdsSent = 0, kTrEmbsSent = kMaxWorld, kTrLookups = 2 * kMaxWorld,
             kTrRequested, kTrReceived, kTrError, kTrN };

struct CommDev {
  char* const* peers;  // [W] arena base of every rank (own included), device-visible
  uint32_t rank, world;
  uint32_t cap;        // ids per (source, destination) region
  uint32_t dim;
  size_t off_ids, off_emb, off_grad;  // off_grad: this epoch's gradient buffer
  unsigned long long* epoch;  // device step counter of the role (requester: bumped by KB)
  unsigned long long* trace;
  unsigned int* done;  // last-block counters [4]
  unsigned long long* tl = nullptr;  // device timeline (RS_TRACE=1, diagnostics; slots in rs_internal.cuh)
  uint32_t diag = 0;  // RS_DIAG_OWN timing experiments (wrong results): 1 rows to self only, 2 no row stores
};

__device__ __forceinline__ ArenaHdr* hdr_of(const CommDev& c, uint32_t r) {
  return reinterpret_cast<ArenaHdr*>(c.peers[r]);
}
__device__ __forceinline__ unsigned long long* flag_of(ArenaHdr* h, int phase, uint32_t src) {
  return phase == 0 ? &h->sig_ids[src] : phase == 1 ? &h->sig_emb[src] : &h->sig_grad[src];
}

// Grid-level arrival: each block's stores (peer stores included) are ordered
// before its arrival by the barrier and a gpu-scope acq_rel atomic; the last
// block to arrive therefore observes all of them, and its single system fence
// + st.release.sys flags publish them cumulatively to the peers.  Returns
// true in the last block.
__device__ __forceinline__ bool last_block_signal(const CommDev& c, int phase, unsigned int* done) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(done) : "memory");
    last = old == gridDim.x * gridDim.y - 1;
    if (last) fence_sys();
  }
  __syncthreads();
  return last;
}
__device__ __forceinline__ void raise_flags(const CommDev& c, int phase, unsigned int* done,
                                            unsigned long long e) {
  for (uint32_t r = threadIdx.x; r < c.world; r += blockDim.x)
    st_release_sys(flag_of(hdr_of(c, r), phase, c.rank), e);
  if (threadIdx.x == 0) *done = 0;
}

// Device-side barrier of the group (rs_comm_barrier): raise this rank's
// barrier flag at every peer, wait for every peer's.  The barrier epoch is
// its own device counter.
__global__ void k_barrier(CommDev c, unsigned long long* bar_epoch) {
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) {
    e = *bar_epoch + 1;
    *bar_epoch = e;
    fence_sys();
  }
  __syncthreads();
  const uint32_t r = threadIdx.x;
  if (r >= c.world) return;
  st_release_sys(&hdr_of(c, r)->sig_bar[c.rank], e);
  const unsigned long long* f = &hdr_of(c, c.rank)->sig_bar[r];
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < e) {
    if (clock64() - t0 > 40000000000ll) {
      c.trace[kTrError] = 1;
      break;
    }
    __nanosleep(100);
  }
}

// One-block wait until every source raised flag `phase` for this step.  The
// data kernels after it re-check their flags in the prologue (cheap then);
// a 1-block waiter is what keeps a concurrently running producer on the
// other stream of this GPU from being starved of SMs by spinning blocks.
__global__ void k_wait(CommDev c, int phase) {
  WarpTrace wt_(c.tl, phase == 0 ? 8 : phase == 1 ? 11 : 12);
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) {
    e = *c.epoch + (phase == 0 ? 1 : 0);  // the owner's step starts here
    if (phase == 0) *c.epoch = e;
  }
  __syncthreads();
  const uint32_t r = threadIdx.x;
  if (r < c.world) spin_flag(flag_of(hdr_of(c, c.rank), phase, r), e, c.trace + kTrError);
}

// Owner lookup: one pass over the received positions (src, j) of every
// source, 8 lanes per position: find-or-insert of the id on the shard
// (concurrent inserts of one id from several sources resolve in the table's
// slot CAS), the position appended to the row's origin list -- row-indexed
// scratch: row_cnt[row] origins so far, row_orig[row * W + k] = src * cap + j
// (the stage-2 dedup of exchange_sim.cpp:100-115, keyed by row instead of a
// second hash set), the row's first origin appends it to the touched list --
// and the row stored straight into the requester's emb_in (the embedding
// "all-to-all", one 128-bit NVLink store per lane per chunk).  Then the
// table epilogue and the rows flags.
#ifndef RS_OWN_MINB
#define RS_OWN_MINB 5  // 48 registers: the blocks carrying positions fit in one wave
#endif
struct OwnLookupArgs {
  TableDev* td;
  uint32_t* row_cnt;          // [rows] origins of each row in this op (zero between ops)
  uint32_t* row_orig;         // [rows * W] origin positions src * cap + j
  uint32_t* touched;          // [W * cap] rows with an origin in this op
  uint32_t* touched_cnt;      // their count (this op's parity)
  uint32_t* touched_clr;      // the other parity's count, zeroed here
  TableCounters* mirror_out;  // host's pinned counter mirror (mapped), or null
  bool bump;                  // no k_wait(ids) before: this kernel advances the owner epoch
};

__global__ void __launch_bounds__(256, RS_OWN_MINB) k_own_lookup(CommDev c, OwnLookupArgs a) {
  WarpTrace wt_(c.tl, 10);
  TableDev* td = a.td;
  const TableDesc d = td->d;
  const unsigned long long free_n0 = td->c.free_n;
  const unsigned long long fresh0 = td->c.fresh_next;
  const uint32_t tick_now = td->c.tick + 1;
  const ArenaHdr* h = hdr_of(c, c.rank);
  __shared__ uint32_t s_off[kMaxWorld + 1];
  __shared__ uint32_t s_w[8], s_base;
  __shared__ unsigned long long s_ins, s_reuse;
  // every source's ids landed (after k_wait: one cheap check per block; with
  // bump, the wait itself -- the last block then publishes the new epoch)
  const unsigned long long ep = *c.epoch + (a.bump ? 1 : 0);
  if (threadIdx.x < c.world) spin_flag(&h->sig_ids[threadIdx.x], ep, c.trace + kTrError);
  if (threadIdx.x == 0) {
    s_ins = 0;
    s_reuse = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the sources' position ranges in one flat index space
    uint32_t run = 0;
    for (uint32_t r = 0; r < c.world; ++r) {
      s_off[r] = run;
      run += min(*reinterpret_cast<const volatile uint32_t*>(&h->cnt_in[r]), c.cap);
    }
    s_off[c.world] = run;
    if (blockIdx.x == 0) *a.touched_clr = 0;  // the previous op's list is consumed
  }
  __syncthreads();
  const uint32_t total = s_off[c.world];
  const unsigned lane = lane_id();
  const unsigned warp = threadIdx.x >> 5;
  const unsigned g = lane & (kBucket - 1);
  const unsigned gbase = lane & ~(kBucket - 1);
  const unsigned gmask = 0xFFu << gbase;
  const uint32_t D4 = d.dim >> 2;
  const uint64_t* ids = reinterpret_cast<const uint64_t*>(c.peers[c.rank] + c.off_ids);
  constexpr unsigned kGroupsPB = 256 / kBucket;
  for (uint32_t base = blockIdx.x * kGroupsPB; base < total; base += gridDim.x * kGroupsPB) {
    const uint32_t i = base + (threadIdx.x >> 3);
    const bool valid = i < total;  // group-uniform
    uint32_t src = 0, j = 0, row = kNoRow;
    if (valid) {
      while (src + 1 < c.world && s_off[src + 1] <= i) ++src;
      j = i - s_off[src];
      const uint64_t key = ids[(size_t)src * c.cap + j];
      row = find_or_insert_group(td, d, key, g, gbase, gmask, tick_now, free_n0, fresh0, &s_ins, &s_reuse);
    }
#ifdef RS_BOUNDS
    if (valid && row != kNoRow && row >= d.row_cap) {  // checked builds
      if (g == 0) c.trace[kTrError] = 3;
      row = kNoRow;
    }
#endif
    bool first = false;
    if (valid && row != kNoRow && g == 0) {
      const uint32_t k = atomicAdd(a.row_cnt + row, 1u);
      if (k < c.world) a.row_orig[(size_t)row * c.world + k] = src * c.cap + j;
      else c.trace[kTrError] = 2;  // a source sent an id twice
      first = k == 0;
    }
    // each row's first origin appends it to the touched list (one atomic per block)
    const unsigned fm = __ballot_sync(kFull, first);
    if (lane == 0) s_w[warp] = __popc(fm);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (uint32_t w = 0; w < 8; ++w) {
        const uint32_t x = s_w[w];
        s_w[w] = run;
        run += x;
      }
      s_base = run ? atomicAdd(a.touched_cnt, run) : 0u;
    }
    __syncthreads();
    if (first) a.touched[s_base + s_w[warp] + __popc(fm & lanemask_lt())] = row;
    // the row to the requester that asked for it
    if (valid && row != kNoRow && !(c.diag & 2)) {
      const float4* e = reinterpret_cast<const float4*>(d.emb) + (size_t)row * D4;
      const uint32_t dsrc = (c.diag & 1) ? c.rank : src;
      float4* dst = reinterpret_cast<float4*>(c.peers[dsrc] + c.off_emb) + ((size_t)c.rank * c.cap + j) * D4;
      for (uint32_t q = g; q < D4; q += kBucket) dst[q] = __ldg(e + q);
    }
    __syncthreads();  // s_w / s_base of the next round
  }
  if (threadIdx.x == 0) {
    if (s_ins) atomicAdd(&td->c.inserted, s_ins);
    if (s_reuse) atomicAdd(&td->c.reused, s_reuse);
  }
  launch_epilogue(td, free_n0, fresh0, true, tick_now, a.mirror_out);
  if (blockIdx.x == 0) {  // every source's flag was observed above
    for (uint32_t r = threadIdx.x; r < c.world; r += blockDim.x) c.trace[kTrEmbsSent + r] = h->cnt_in[r];
    if (threadIdx.x == 0) c.trace[kTrReceived] = total;  // two-stage: one vector back per received id
  }
  if (last_block_signal(c, 1, c.done + 1)) {
    raise_flags(c, 1, c.done + 1, ep);
    if (threadIdx.x == 0) {
      c.trace[kTrLookups] = *reinterpret_cast<volatile uint32_t*>(a.touched_cnt);
      if (a.bump) *c.epoch = ep;  // every block read the old value before arriving
    }
  }
}

// Owner update: per touched row (G lanes, NV float4 chunks each), its <= W
// origins ranked into (source, position) order -- the stage-2 origin order
// of exchange_sim.cpp:100-115 -- the requesters' sums at those positions of
// grad_in added in that order, then the optimizer on the row
// (sparse_update.cpp:49-75 arithmetic, opt_dev.cuh).  Resets row_cnt.
struct OwnUpdateArgs {
  TableDev* td;
  uint32_t* row_cnt;
  const uint32_t* row_orig;
  const uint32_t* touched;
  const uint32_t* touched_cnt;
  const float* grad_in;  // [W * cap x D] the requesters' per-id sums (this op's parity)
};

// PPT: origin positions held per lane (W <= G * PPT); ADAM: o.kind (the
// Adagrad build carries no first-moment state or bias corrections)
template <int G, int NV, int PPT, bool ADAM>
__global__ void __launch_bounds__(256, NV <= 2 ? 4 : 2) k_own_update(CommDev c, OwnUpdateArgs a, OptArgs o) {
  WarpTrace wt_(c.tl, 14);
  __shared__ uint32_t order_s[(256 / G) * kMaxWorld];
  const TableDesc d = a.td->d;
  const uint32_t D4 = d.dim >> 2;
  const uint32_t W = c.world;
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << (lane & ~(G - 1));
  uint32_t* order = order_s + (threadIdx.x / G) * kMaxWorld;
  const uint32_t gid = blockIdx.x * (256 / G) + threadIdx.x / G;
  const uint32_t ngroups = gridDim.x * (256 / G);
  const uint32_t nu = *reinterpret_cast<const volatile uint32_t*>(a.touched_cnt);
  const float4* __restrict__ g4 = reinterpret_cast<const float4*>(a.grad_in);
  float4* rw = reinterpret_cast<float4*>(d.emb);
  float4* rv = reinterpret_cast<float4*>(d.s2);
  float4* rm = ADAM ? reinterpret_cast<float4*>(d.s1) : nullptr;
  for (uint32_t u = gid; u < nu; u += ngroups) {
    const uint32_t row = __ldcg(a.touched + u);
#ifdef RS_BOUNDS
    if (row >= d.row_cap) {  // checked builds: a bad touched row fails the step (trace error)
      if (gl == 0) c.trace[kTrError] = 3;
      continue;
    }
#endif
    // the origin count, the origin positions (speculatively, all W) and the
    // row's state in one round trip
    const uint32_t cnt = __ldcg(a.row_cnt + row);
    uint32_t p[PPT], r[PPT];
#pragma unroll
    for (int jq = 0; jq < PPT; ++jq) {
      const uint32_t k = gl + jq * G;
      p[jq] = k < W ? __ldcg(a.row_orig + (size_t)row * W + k) : kFull;
      r[jq] = 0;
    }
    const size_t rbase = (size_t)row * D4;
    float4 wv[NV], vv[NV], mv[NV];
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) {
      const uint32_t q = gl + jv * G;
      wv[jv] = vv[jv] = mv[jv] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q < D4) {
        wv[jv] = rw[rbase + q];
        vv[jv] = rv[rbase + q];
        if (rm) mv[jv] = rm[rbase + q];
      }
    }
    uint32_t st0 = 0;
    if (gl == 0) st0 = d.step[row];
    const uint32_t cc = min(cnt, W);
#pragma unroll
    for (int jq = 0; jq < PPT; ++jq)
      if (gl + jq * G >= cc) p[jq] = kFull;
    // rank every held position against all cc positions of the row
#pragma unroll
    for (int jq = 0; jq < PPT; ++jq) {
      if ((uint32_t)(jq * G) >= cc) break;
      const uint32_t lim = min((uint32_t)G, cc - (uint32_t)(jq * G));
      for (uint32_t sl = 0; sl < lim; ++sl) {
        const uint32_t qv = __shfl_sync(gmask, p[jq], sl, G);
#pragma unroll
        for (int j2 = 0; j2 < PPT; ++j2) r[j2] += qv < p[j2];
      }
    }
#pragma unroll
    for (int jq = 0; jq < PPT; ++jq)
      if (gl + jq * G < cc) order[r[jq]] = p[jq];
    __syncwarp(gmask);
    // the sums in (source, position) order, B rows in flight
    float4 acc[NV];
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) acc[jv] = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int B = NV == 1 ? 4 : 2;  // (NV = 2 at B = 4 spills at 64 registers)
    uint32_t k = 0;
#ifdef RS_BOUNDS
    {
      bool bad = false;
      for (uint32_t k2 = 0; k2 < cc; ++k2) bad |= order[k2] >= W * c.cap;
      if (bad) {
        if (gl == 0) c.trace[kTrError] = 3;
        continue;
      }
    }
#endif
    for (; k + B <= cc; k += B) {
      float4 x[B][NV];
#pragma unroll
      for (int qb = 0; qb < B; ++qb)
#pragma unroll
        for (int jv = 0; jv < NV; ++jv) {
          const uint32_t q = gl + jv * G;
          x[qb][jv] = q < D4 ? __ldcg(g4 + (size_t)order[k + qb] * D4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int qb = 0; qb < B; ++qb)
#pragma unroll
        for (int jv = 0; jv < NV; ++jv) {
          acc[jv].x += x[qb][jv].x;
          acc[jv].y += x[qb][jv].y;
          acc[jv].z += x[qb][jv].z;
          acc[jv].w += x[qb][jv].w;
        }
    }
    for (; k < cc; ++k) {
#pragma unroll
      for (int jv = 0; jv < NV; ++jv) {
        const uint32_t q = gl + jv * G;
        if (q >= D4) continue;
        const float4 x = __ldcg(g4 + (size_t)order[k] * D4 + q);
        acc[jv].x += x.x;
        acc[jv].y += x.y;
        acc[jv].z += x.z;
        acc[jv].w += x.w;
      }
    }
    __syncwarp(gmask);
    uint32_t st = 0;
    if (gl == 0) {
      a.row_cnt[row] = 0;  // the row's origin list is consumed
      st = st0 + 1;
      d.step[row] = st;
    }
    st = __shfl_sync(gmask, st, 0, G);
    double bc1 = 1.0, bc2 = 1.0;
    if (ADAM) {
      if (st < o.bc_len) {
        bc1 = o.bc[st];
        bc2 = o.bc[o.bc_len + st];
      } else {
        bc1 = 1.0 - pow(o.b1, (double)st);
        bc2 = 1.0 - pow(o.b2, (double)st);
      }
    }
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) {
      const uint32_t q = gl + jv * G;
      if (q >= D4) continue;
      float* wp = reinterpret_cast<float*>(&wv[jv]);
      float* vp = reinterpret_cast<float*>(&vv[jv]);
      float* mp = reinterpret_cast<float*>(&mv[jv]);
      const float* gp = reinterpret_cast<const float*>(&acc[jv]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (ADAM)
          adam_elem(wp[e], mp[e], vp[e], gp[e], bc1, bc2, o);
        else
          adagrad_elem(wp[e], vp[e], gp[e], o);
      }
      rw[rbase + q] = wv[jv];
      rv[rbase + q] = vv[jv];
      if (rm) rm[rbase + q] = mv[jv];
    }
  }
}

// A forward-only op's origin lists, consumed without an update (the next op
// starts from zero counts).
__global__ void k_own_reset(uint32_t* row_cnt, const uint32_t* touched, const uint32_t* touched_cnt) {
  const uint32_t nu = *touched_cnt;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += gridDim.x * blockDim.x)
    row_cnt[touched[u]] = 0;
}

// timeline stamp (RS_TRACE=1 only): the stream reached this point
__global__ void k_tl_stamp(CommDev c, int slot) { trace_mark(c.tl, slot); }

__global__ void k_signal(CommDev c, int phase) {
  WarpTrace wt_(c.tl, 7);
  if (threadIdx.x == 0) fence_sys();
  __syncthreads();
  const unsigned long long e = *c.epoch;
  for (uint32_t r = threadIdx.x; r < c.world; r += blockDim.x)
    st_release_sys(flag_of(hdr_of(c, r), phase, c.rank), e);
}

}  // namespace
}  // namespace rs

using namespace rs;

struct StepSets {
  int ru, ou, par;  // requester / owner scratch sets, gradient-buffer parity
  int fu = -1;      // requester on the fast kernels (step_fast.cu): its scratch set; -1: the split kernels
};

struct DistGraph {
  rs_table* t;
  const void *ids, *grads, *out;
  uint64_t n;
  int mirror, ru, par, fu;
  const void* pbuf;
  double* csum;
  unsigned char opt[256];
  cudaGraphExec_t exec;
  uint64_t last_use, launches;
};

struct rs_comm {
  int rank = 0, world = 1;
  bool local = false;  // rs_comm_create_local: the peers are arenas of this process
  uint64_t cap = 0;
  uint32_t dim = 0;
  char* arena = nullptr;
  size_t arena_bytes = 0, off_ids = 0, off_emb = 0, off_grad[2] = {0, 0};
  char* h_peers[kMaxWorld] = {nullptr};
  char** d_peers = nullptr;
  float** d_peer_grad[2] = {nullptr, nullptr};  // per epoch parity
  unsigned long long epoch = 0;       // host mirror of the device counter (parity)
  unsigned long long* d_epoch = nullptr;
  unsigned long long* d_bar_epoch = nullptr;
  unsigned long long** d_sig_grad_ptrs = nullptr;  // [W] &peer(r)->sig_grad[rank]
  unsigned long long** d_sig_ids_ptrs = nullptr;   // [W] &peer(r)->sig_ids[rank]
  uint32_t** d_cnt_ptrs = nullptr;                 // [W] &peer(r)->cnt_in[rank]
  const unsigned long long* own_sig_emb = nullptr;  // this arena's sig_emb[W]
  const unsigned long long* own_sig_grad = nullptr; // this arena's sig_grad[W]
  unsigned long long* trace = nullptr;
  unsigned int* done = nullptr;
  uint32_t* send_pos = nullptr;
  uint32_t* send_cnt = nullptr;
  // owner: row-indexed origin scratch (k_own_lookup / k_own_update), sized
  // for the shard's row capacity and grown with it (zero between ops)
  uint32_t* row_cnt = nullptr;    // [scr_rows]
  uint32_t* row_orig = nullptr;   // [scr_rows * W]
  uint64_t scr_rows = 0;
  uint32_t* touched[2] = {nullptr, nullptr};  // per op parity: rows with an origin
  uint32_t* touched_cnt = nullptr;            // [2]
  bool pending_reset = false;  // a forward-only op left origin counts behind
  int pending_par = 0;
  TableDev* view = nullptr;
  rs_workspace* ws_req = nullptr;
  StepSets last_sets{0, 0, 0};
  uint64_t last_n = 0;
  bool have_forward = false;
  rs_table* last_table = nullptr;
  // profiling: events at the phase boundaries of one step
  bool profiling = false;
  cudaEvent_t pev[20] = {};  // [2 * phase]: begin, [2 * phase + 1]: end
  unsigned pmask = 0;        // phases recorded in the current step
  double pms[10] = {};
  uint64_t pcount = 0;
  // CUDA graphs of rs_dist_step
  bool use_graphs = true;
  bool graph_fork = true;
  double* csum_dst = nullptr;  // rs_dist_step_checksum: sum of the gathered rows (fused in the gather)
  bool one_stream = false;          // RS_DIST_ONE_STREAM=1: both roles on the caller's stream
  cudaStream_t cap_stream = nullptr;
  cudaStream_t own_stream = nullptr;  // owner role runs here, concurrently with the requester's
  cudaStream_t gather_stream = nullptr;  // the requester's gather, concurrent with its reduce
  cudaEvent_t ev_dedup = nullptr;        // owner dedup done (reduce_after_dedup)
  bool reduce_after_dedup = false;       // RS_DIST_REDUCE_AFTER=1
  bool host_prof = false;                // RS_HOST_PROF=1
  bool lookup_spin = true;               // rs_dist_step: no k_wait(ids) (RS_DIST_LOOKUP_SPIN=0: with)
  double host_ns[5] = {0, 0, 0, 0, 0};
  uint64_t host_calls = 0;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_meta = nullptr, ev_gjoin = nullptr;
  std::vector<DistGraph> graphs;
  uint64_t graph_clock = 0;
};

// phases (rs_comm_phase_ms order) and the event pair that brackets each
enum : int { kPhReqDedup, kPhSendIds, kPhWaitIds, kPhOwnerTable, kPhRespond, kPhWaitEmbs, kPhGather,
             kPhReqReduce, kPhWaitGrads, kPhOwnerUpdate, kDistPhases };

static int prof_begin(rs_comm* c, int ph, cudaStream_t s) {
  if (c->profiling) RS_CUDA(cudaEventRecord(c->pev[2 * ph], s));
  return RS_OK;
}
static int prof_end(rs_comm* c, int ph, cudaStream_t s) {
  if (!c->profiling) return RS_OK;
  RS_CUDA(cudaEventRecord(c->pev[2 * ph + 1], s));
  c->pmask |= 1u << ph;
  return RS_OK;
}

// Each role keeps its own device step counter -- the requester's is bumped
// by KB's id send, the owner's by its first wait -- so a role never reads the
// other stream's counter before that stream advanced it.
enum Role : int { kRequester = 0, kOwner = 1 };
static unsigned long long* role_epoch(rs_comm* c, Role r) { return c->d_epoch + (r == kOwner ? 2 : 0); }

static rs_dist_sync wait_sync(rs_comm* c, const unsigned long long* flags, Role role) {
  rs_dist_sync y;
  y.wait_flags = flags;
  y.wait_n = (uint32_t)c->world;
  y.epoch = role_epoch(c, role);
  y.error = c->trace + kTrError;
  return y;
}
static rs_dist_sync signal_sync(rs_comm* c) {  // requester role
  rs_dist_sync y;
  y.epoch = role_epoch(c, kRequester);
  y.sig_flags = c->d_sig_grad_ptrs;
  y.sig_n = (uint32_t)c->world;
  y.sig_done = c->done + 2;
  y.error = c->trace + kTrError;
  return y;
}

static CommDev comm_dev(rs_comm* c, int par, Role role) {
  CommDev d;
  d.peers = c->d_peers;
  d.rank = c->rank;
  d.world = c->world;
  d.cap = (uint32_t)c->cap;
  d.dim = c->dim;
  d.off_ids = c->off_ids;
  d.off_emb = c->off_emb;
  d.off_grad = c->off_grad[par];
  d.epoch = role_epoch(c, role);
  d.trace = c->trace;
  d.done = c->done;
  d.tl = c->ws_req->fast.trace;
  static const uint32_t diag = getenv("RS_DIAG_OWN") ? (uint32_t)atoi(getenv("RS_DIAG_OWN")) : 0u;
  d.diag = diag;
  return d;
}

static cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

#define RS_TRY(x)              \
  do {                         \
    const int _st = (x);       \
    if (_st) return _st;       \
  } while (0)

// ---- the five phases of one sharded step -----------------------------------
// Enqueue-only (no host state changes, no synchronization) so that a whole
// step can be captured into a CUDA graph; ru / ou are the scratch sets of the
// requester / owner workspaces, par the gradient-buffer parity of the step.
// requester: dedup its tokens, partition the unique ids by owner and store
// them into the owners' receive lists (KA, KB metadata + send)
static int req_front(rs_comm* c, rs_table* t, const uint64_t* d_ids, uint64_t n, StepSets ss,
                     cudaStream_t s) {
  rs_workspace* wr = c->ws_req;
  const CommDev cd = comm_dev(c, ss.par, kRequester);
  const int ru = ss.ru;
  RS_TRY(prof_begin(c, kPhReqDedup, s));
  // KB (metadata) also partitions the unique ids by owner and stores them
  // into the owners' receive lists; its last block raises the ids flags
  rs_dist_send snd;
  snd.peers = c->d_peers;
  snd.off_ids = c->off_ids;
  snd.cap = (uint32_t)c->cap;
  snd.world = (uint32_t)c->world;
  snd.rank = (uint32_t)c->rank;
  snd.send_cnt = c->send_cnt;
  snd.send_pos = c->send_pos;
  snd.cnt_ptrs = c->d_cnt_ptrs;
  snd.flag_ptrs = c->d_sig_ids_ptrs;
  snd.epoch = role_epoch(c, kRequester);
  snd.done = c->done + 0;
  snd.trace_ids_sent = c->trace + kTrIdsSent;
  snd.trace_requested = c->trace + kTrRequested;
  snd.n_tokens = n;
  if (n) {
    RS_TRY(step_fdedup(wr, d_ids, n, ru, s, nullptr));
    RS_TRY(step_ftable(wr, t, ru, n, false, true, s, &snd));
  } else {  // idle rank: still clean the other scratch set (KB), send nothing, raise the flags
    RS_CUDA(cudaMemsetAsync(wr->set[ru].cnt, 0, 4, s));
    RS_TRY(step_ftable(wr, t, ru, 1, false, true, s, &snd));
    RS_CUDA(cudaMemsetAsync(wr->set[ru ^ 1].cnt, 0, 4, s));
  }
  RS_TRY(prof_end(c, kPhReqDedup, s));
  (void)cd;
  return RS_OK;
}

// owner: stage-2 dedup straight from the receive lists (KA'), then per
// owner-unique id find-or-insert on the shard (capacity prepared by the
// caller) and the row stored into every requester that asked for it (KB')
static int owner_lookup(rs_comm* c, rs_table* t, StepSets ss, cudaStream_t s,
                        TableCounters* mirror_out = nullptr, cudaEvent_t ev_dedup = nullptr,
                        bool spin = false) {
  const CommDev cd = comm_dev(c, ss.par, kOwner);
  // spin: the lookup's blocks wait for the ids themselves (the caller
  // ordered the owner stream after this rank's own id send, so they only
  // wait for remote producers); else one waiter block first
  if (!spin) {
    RS_TRY(prof_begin(c, kPhWaitIds, s));
    carve(k_wait), k_wait<<<1, kMaxWorld, 0, s>>>(cd, 0);
    RS_LAUNCH_CHECK("k_wait(ids)");
    RS_TRY(prof_end(c, kPhWaitIds, s));
  }
  if (ev_dedup) RS_CUDA(cudaEventRecord(ev_dedup, s));
  RS_TRY(prof_begin(c, kPhRespond, s));
  OwnLookupArgs a;
  a.td = t->dev;
  a.row_cnt = c->row_cnt;
  a.row_orig = c->row_orig;
  a.touched = c->touched[ss.par];
  a.touched_cnt = c->touched_cnt + ss.par;
  a.touched_clr = c->touched_cnt + (ss.par ^ 1);
  a.mirror_out = mirror_out;
  a.bump = spin;
  static const unsigned grid = getenv("RS_OWN_GRID") ? (unsigned)atoi(getenv("RS_OWN_GRID")) : 148u * RS_OWN_MINB;
  carve(k_own_lookup), k_own_lookup<<<grid, 256, 0, s>>>(cd, a);
  RS_LAUNCH_CHECK("k_own_lookup");
  return prof_end(c, kPhRespond, s);
}

// requester: wait for the rows, expand them to the tokens (KC gather)
static int req_gather(rs_comm* c, rs_table* t, uint64_t n, float* d_out, StepSets ss,
                      cudaStream_t s) {
  const CommDev cd = comm_dev(c, ss.par, kRequester);
  RS_TRY(prof_begin(c, kPhWaitEmbs, s));
  carve(k_wait), k_wait<<<1, kMaxWorld, 0, s>>>(cd, 1);
  RS_LAUNCH_CHECK("k_wait(embs)");
  RS_TRY(prof_end(c, kPhWaitEmbs, s));
  RS_TRY(prof_begin(c, kPhGather, s));
  if (n) {
    rs_dist_opts o;
    o.gather_view = c->view;
    o.sync = wait_sync(c, c->own_sig_emb, kRequester);  // the owners' rows landed
    o.csum = c->csum_dst;
    RS_TRY(step_tile(c->ws_req, t, ss.ru, n, d_out, nullptr, true, s, &o));
  }
  RS_TRY(prof_end(c, kPhGather, s));
  return RS_OK;
}

// requester: per unique id sums of its token gradients (KC + KD), each row
// stored straight into its owner's grad_in, then the gradient flags
// (partial-sum buffer prepared by the caller)
static int req_reduce(rs_comm* c, rs_table* t, const float* d_grads, uint64_t n, StepSets ss,
                      cudaStream_t s) {
  rs_workspace* wr = c->ws_req;
  const CommDev cd = comm_dev(c, ss.par, kRequester);
  RS_TRY(prof_begin(c, kPhReqReduce, s));
  if (n) {
    // one-pass KC (the split KC measured slower here; RS_DIST_SPLIT_KC=1 for experiments)
    static const bool split = getenv("RS_DIST_SPLIT_KC") && getenv("RS_DIST_SPLIT_KC")[0] == '1';
    rs_dist_opts one_pass;
    RS_TRY(step_tile(wr, t, ss.ru, n, nullptr, d_grads, false, s, split ? nullptr : &one_pass));
    rs_dist_opts o;
    o.peer_dst = c->d_peer_grad[ss.par];
    o.send_pos = c->send_pos;
    o.cap = (uint32_t)c->cap;
    o.rank = (uint32_t)c->rank;
    o.sync = signal_sync(c);  // the last finish block raises the gradient flags
    RS_TRY(step_finish(wr, t, ss.ru, n, d_grads, nullptr, nullptr, s, &o));
  } else {  // idle rank: the owners still wait for its (empty) gradients
    carve(k_signal), k_signal<<<1, 64, 0, s>>>(cd, 2);
    RS_LAUNCH_CHECK("k_signal(grads)");
  }
  RS_TRY(prof_end(c, kPhReqReduce, s));
  return RS_OK;
}

// requester, fused step: wait for the rows, then ONE pass over the tokens
// gathers the rows and segment-reduces the gradients (KC), KD stores each
// unique id's sum straight into its owner's grad_in, then the gradient flags
static int req_gather_reduce(rs_comm* c, rs_table* t, uint64_t n, float* d_out,
                             const float* d_grads, StepSets ss, cudaStream_t s) {
  rs_workspace* wr = c->ws_req;
  const CommDev cd = comm_dev(c, ss.par, kRequester);
  RS_TRY(prof_begin(c, kPhWaitEmbs, s));
  carve(k_wait), k_wait<<<1, kMaxWorld, 0, s>>>(cd, 1);
  RS_LAUNCH_CHECK("k_wait(embs)");
  RS_TRY(prof_end(c, kPhWaitEmbs, s));
  RS_TRY(prof_begin(c, kPhGather, s));
  if (n) {
    rs_dist_opts o;
    o.gather_view = c->view;
    o.sync = wait_sync(c, c->own_sig_emb, kRequester);  // the owners' rows landed
    o.csum = c->csum_dst;
    RS_TRY(step_tile(wr, t, ss.ru, n, d_out, d_grads, true, s, &o));
    rs_dist_opts f;
    f.peer_dst = c->d_peer_grad[ss.par];
    f.send_pos = c->send_pos;
    f.cap = (uint32_t)c->cap;
    f.rank = (uint32_t)c->rank;
    f.sync = signal_sync(c);  // the last finish block raises the gradient flags
    RS_TRY(step_finish(wr, t, ss.ru, n, d_grads, nullptr, nullptr, s, &f));
  } else {
    carve(k_signal), k_signal<<<1, 64, 0, s>>>(cd, 2);
    RS_LAUNCH_CHECK("k_signal(grads)");
  }
  RS_TRY(prof_end(c, kPhGather, s));
  return RS_OK;
}

// ---- the requester on the fast kernels (step_fast.cu) -----------------------
// The single-GPU step's dedup (KA) with the id send folded into it, its
// light / heavy / hot-tile segment reduce storing each unique id's sum into
// the owner's grad_in, and a gather from the receive buffer.
static rs_dist_send dist_send(rs_comm* c, uint64_t n) {
  rs_dist_send snd;
  snd.peers = c->d_peers;
  snd.off_ids = c->off_ids;
  snd.cap = (uint32_t)c->cap;
  snd.world = (uint32_t)c->world;
  snd.rank = (uint32_t)c->rank;
  snd.send_cnt = c->send_cnt;
  snd.send_pos = c->send_pos;
  snd.cnt_ptrs = c->d_cnt_ptrs;
  snd.flag_ptrs = c->d_sig_ids_ptrs;
  snd.epoch = role_epoch(c, kRequester);
  snd.done = c->done + 0;
  snd.trace_ids_sent = c->trace + kTrIdsSent;
  snd.trace_requested = c->trace + kTrRequested;
  snd.n_tokens = n;
  return snd;
}
static int req_front_fast(rs_comm* c, const uint64_t* d_ids, uint64_t n, StepSets ss, cudaStream_t s) {
  RS_TRY(prof_begin(c, kPhReqDedup, s));
  RS_TRY(fast_dist_front(c->ws_req, c->dim, d_ids, n, ss.fu, s, dist_send(c, n)));
  return prof_end(c, kPhReqDedup, s);
}
static int req_reduce_fast(rs_comm* c, const float* d_grads, uint64_t n, StepSets ss, cudaStream_t s) {
  const CommDev cd = comm_dev(c, ss.par, kRequester);
  RS_TRY(prof_begin(c, kPhReqReduce, s));
  RS_TRY(fast_dist_reduce(c->ws_req, c->view, c->dim, n, d_grads, ss.fu, s, c->ws_req->fork,
                          c->d_peer_grad[ss.par], (uint32_t)c->cap, (uint32_t)c->rank));
  carve(k_signal), k_signal<<<1, 64, 0, s>>>(cd, 2);  // every branch joined: the sums are out
  RS_LAUNCH_CHECK("k_signal(grads)");
  return prof_end(c, kPhReqReduce, s);
}
static int req_gather_fast(rs_comm* c, uint64_t n, float* d_out, StepSets ss, cudaStream_t s) {
  // One block waits for the rows first: gather blocks spinning on the flags
  // would hold the SMs the owner's kernels need to answer them.  One block
  // per tile (RS_DIST_GATHER_GRID=G: G persistent blocks, measured slower);
  // RS_DIST_GATHER_SPIN=1: no waiter kernel, the gather's blocks wait.
  static const uint32_t grid =
      getenv("RS_DIST_GATHER_GRID") ? (uint32_t)atoi(getenv("RS_DIST_GATHER_GRID")) : 0u;
  static const bool spin = getenv("RS_DIST_GATHER_SPIN") && getenv("RS_DIST_GATHER_SPIN")[0] == '1';
  const CommDev cd = comm_dev(c, ss.par, kRequester);
  if (!spin) {
    RS_TRY(prof_begin(c, kPhWaitEmbs, s));
    carve(k_wait), k_wait<<<1, kMaxWorld, 0, s>>>(cd, 1);
    RS_LAUNCH_CHECK("k_wait(embs)");
    RS_TRY(prof_end(c, kPhWaitEmbs, s));
  }
  RS_TRY(prof_begin(c, kPhGather, s));
  RS_TRY(fast_dist_gather(c->ws_req, c->view, c->dim, n, d_out, ss.fu, s,
                          wait_sync(c, c->own_sig_emb, kRequester), c->csum_dst, grid));
  return prof_end(c, kPhGather, s);
}

// owner: per id sum over its origins in (source, position) order -- the
// stage-2 origin order -- fused with the optimizer on the shard
static int owner_update(rs_comm* c, rs_table* t, const void* ob, StepSets ss, cudaStream_t s) {
  const CommDev cd = comm_dev(c, ss.par, kOwner);
  RS_TRY(prof_begin(c, kPhWaitGrads, s));
  carve(k_wait), k_wait<<<1, kMaxWorld, 0, s>>>(cd, 2);  // every requester's sums landed
  RS_LAUNCH_CHECK("k_wait(grads)");
  RS_TRY(prof_end(c, kPhWaitGrads, s));
  RS_TRY(prof_begin(c, kPhOwnerUpdate, s));
  OwnUpdateArgs a;
  a.td = t->dev;
  a.row_cnt = c->row_cnt;
  a.row_orig = c->row_orig;
  a.touched = c->touched[ss.par];
  a.touched_cnt = c->touched_cnt + ss.par;
  a.grad_in = reinterpret_cast<const float*>(c->arena + c->off_grad[ss.par]);
  OptArgs o;
  std::memcpy(&o, ob, sizeof(o));
  const uint32_t D4 = c->dim / 4;
  // G lanes x NV float4 per row; persistent grid (resident blocks)
  static const unsigned gcap = getenv("RS_OWN_UGRID") ? (unsigned)atoi(getenv("RS_OWN_UGRID")) : 0u;
#define RS_OU(GG, NN, MB)                                                                   \
  {                                                                                         \
    const unsigned grid = gcap ? gcap : 148u * (MB);                                        \
    const bool adam = o.kind == RS_OPT_ADAM;                                                \
    if ((uint32_t)c->world <= (GG) && adam)                                                 \
      carve(k_own_update<GG, NN, 1, true>), k_own_update<GG, NN, 1, true><<<grid, 256, 0, s>>>(cd, a, o); \
    else if ((uint32_t)c->world <= (GG))                                                    \
      carve(k_own_update<GG, NN, 1, false>), k_own_update<GG, NN, 1, false><<<grid, 256, 0, s>>>(cd, a, o); \
    else if (adam)                                                                          \
      carve(k_own_update<GG, NN, kMaxWorld / (GG), true>),                                  \
          k_own_update<GG, NN, kMaxWorld / (GG), true><<<grid, 256, 0, s>>>(cd, a, o);      \
    else                                                                                    \
      carve(k_own_update<GG, NN, kMaxWorld / (GG), false>),                                 \
          k_own_update<GG, NN, kMaxWorld / (GG), false><<<grid, 256, 0, s>>>(cd, a, o);     \
  }
  // D <= 64: 4 lanes x 4 float4 per row (measured ~2 us faster at config 1
  // than 8 x 2: twice the rows in flight); RS_OWN_G4=0 for 8 x 2
  static const int g4 = getenv("RS_OWN_G4") ? atoi(getenv("RS_OWN_G4")) : 1;
  if (D4 <= 4) RS_OU(4, 1, 4)
  else if (D4 <= 16 && g4) RS_OU(4, 4, 2)
  else if (D4 <= 16) RS_OU(8, 2, 4)
  else if (D4 <= 32) RS_OU(8, 4, 2)
  else if (D4 <= 64) RS_OU(8, 8, 2)
  else return fail(RS_ERR_CONFIG, "sharded step: embedding_dim > 256 unsupported");
#undef RS_OU
  RS_LAUNCH_CHECK("k_own_update");
  if (cd.tl) {
    carve(k_tl_stamp), k_tl_stamp<<<1, 32, 0, s>>>(cd, 13);
    RS_LAUNCH_CHECK("k_tl_stamp");
  }
  return prof_end(c, kPhOwnerUpdate, s);
}

static int check_call(rs_comm* c, rs_table* t, uint64_t n, const char* who) {
  if (!c || !t) return fail(RS_ERR_CONFIG, std::string(who) + ": null handle");
  if (n > c->cap) return fail(RS_ERR_CONFIG, std::string(who) + ": batch exceeds max_tokens");
  if (t->desc.dim != c->dim) return fail(RS_ERR_CONFIG, std::string(who) + ": table dim != comm dim");
  if (t->cfg.max_keys)
    return fail(RS_ERR_CONFIG, std::string(who) + ": bounded shard tables unsupported");
  if (c->dim % 4) return fail(RS_ERR_CONFIG, std::string(who) + ": needs embedding_dim % 4 == 0");
  return step_set_smem_attrs();
}

// host side of a step, outside any graph: shapes, capacity (may rehash or
// grow the row pool on s), the partial-sum buffer
static int prepare_step(rs_comm* c, rs_table* t, uint64_t n_reduce, cudaStream_t s) {
  c->ws_req->last_tile = tile_tokens_for_dim(c->dim);
  // new keys at this owner <= ids received <= world * max_tokens (the peers'
  // batch sizes are not known here without a host round trip)
  RS_TRY(table_prepare(t, (uint64_t)c->world * c->cap, s, 8));
  if (n_reduce) RS_TRY(step_reduce_prepare(c->ws_req, c->dim, n_reduce, s));
  if (c->scr_rows < t->desc.row_cap) {  // the origin scratch follows the shard's row capacity
    RS_CUDA(cudaDeviceSynchronize());     // (graphs in flight use the old one)
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
    if (c->row_cnt) cudaFree(c->row_cnt);
    if (c->row_orig) cudaFree(c->row_orig);
    c->row_cnt = c->row_orig = nullptr;
    c->scr_rows = 0;
    const uint64_t rows = t->desc.row_cap;
    if (cudaMalloc(&c->row_cnt, rows * 4) != cudaSuccess ||
        cudaMalloc(&c->row_orig, rows * 4 * (uint64_t)c->world) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "sharded step: origin scratch");
    RS_CUDA(cudaMemset(c->row_cnt, 0, rows * 4));
    c->scr_rows = rows;
  }
  if (c->pending_reset) {  // the last forward-only op's origin counts (before this op's lookup)
    carve(k_own_reset), k_own_reset<<<grid_for((uint64_t)c->world * c->cap, 256, 148 * 4), 256, 0, s>>>(
        c->row_cnt, c->touched[c->pending_par], c->touched_cnt + c->pending_par);
    RS_LAUNCH_CHECK("k_own_reset");
    c->pending_reset = false;
  }
  return RS_OK;
}
// fast: the requester runs on the fast kernels (a step with gradients, n > 0)
static int begin_step(rs_comm* c, bool fast, StepSets* out) {
  if (fast) RS_TRY(fast_prepare(c->ws_req));
  c->epoch++;
  StepSets ss{c->ws_req->cur, 0, (int)(c->epoch & 1)};
  ss.fu = fast ? c->ws_req->fast.cur : -1;
  *out = ss;
  return RS_OK;
}
static bool fast_requester(rs_comm* c, uint64_t n, const float* d_grads) {
  return c->ws_req->use_fast && n > 0 && d_grads && ((uintptr_t)d_grads & 15u) == 0 &&
         fast_dim_supported(c->dim);
}
static void end_step(rs_comm* c, StepSets ss) {
  c->last_sets = ss;
  if (ss.fu >= 0) {
    c->ws_req->fast.last = ss.fu;
    c->ws_req->fast.cur = ss.fu ^ 1;
  } else {
    c->ws_req->cur = ss.ru ^ 1;
  }
}

// The owner role runs on its own stream, concurrently with the requester
// role on the caller's: fork returns the owner stream (ordered after
// everything enqueued so far), join orders the caller's stream after it.
static int fork_owner(rs_comm* c, cudaStream_t q, cudaStream_t* own) {
  if (c->one_stream) {
    *own = q;
    return RS_OK;
  }
  RS_CUDA(cudaEventRecord(c->ev_fork, q));
  RS_CUDA(cudaStreamWaitEvent(c->own_stream, c->ev_fork, 0));
  *own = c->own_stream;
  return RS_OK;
}
static int join_owner(rs_comm* c, cudaStream_t q, cudaStream_t own) {
  if (own == q) return RS_OK;
  RS_CUDA(cudaEventRecord(c->ev_join, own));
  RS_CUDA(cudaStreamWaitEvent(q, c->ev_join, 0));
  return RS_OK;
}

// Host-side cost of rs_dist_step by section (RS_HOST_PROF=1, diagnostics):
// 0 args, 1 capacity / prepare, 2 graph lookup, 3 cudaGraphLaunch, 4 commit;
// printed when the comm is destroyed.
struct HostClock {
  rs_comm* c;
  std::chrono::steady_clock::time_point t0;
  explicit HostClock(rs_comm* c_) : c(c_) {
    if (c->host_prof) t0 = std::chrono::steady_clock::now();
  }
  void mark(int k) {
    if (!c->host_prof) return;
    const auto t1 = std::chrono::steady_clock::now();
    c->host_ns[k] += (double)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    t0 = t1;
    if (k == 4 && ++c->host_calls % 16 == 0) {  // the last 16 calls' means, then restart
      fprintf(stderr, "rs_dist_step host us/call (rank %d, calls to %llu): args %.1f prepare %.1f lookup %.1f launch %.1f commit %.1f\n",
              c->rank, (unsigned long long)c->host_calls, c->host_ns[0] / 16e3, c->host_ns[1] / 16e3,
              c->host_ns[2] / 16e3, c->host_ns[3] / 16e3, c->host_ns[4] / 16e3);
      for (double& x : c->host_ns) x = 0;
    }
  }
};

// end of a step: collect the phase times recorded during it (one sync)
static int prof_step_done(rs_comm* c) {
  if (!c->profiling) return RS_OK;
  for (int ph = 0; ph < kDistPhases; ++ph) {
    if (!(c->pmask & (1u << ph))) continue;
    RS_CUDA(cudaEventSynchronize(c->pev[2 * ph + 1]));
    float ms = 0.f;
    RS_CUDA(cudaEventElapsedTime(&ms, c->pev[2 * ph], c->pev[2 * ph + 1]));
    c->pms[ph] += ms;
  }
  c->pmask = 0;
  c->pcount++;
  return RS_OK;
}

extern "C" {

int rs_comm_create(int rank, int world, uint64_t max_tokens, uint32_t dim, rs_comm** out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || dim < 1 ||
      max_tokens < 1 || max_tokens > (1ull << 30) / (uint64_t)world)
    return fail(RS_ERR_CONFIG, "rs_comm_create: bad rank/world/dim/max_tokens");
  rs_comm* c = new rs_comm();
  c->rank = rank;
  c->world = world;
  c->cap = max_tokens;
  c->dim = dim;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t rows = (size_t)world * max_tokens;
  c->off_ids = align(sizeof(ArenaHdr));
  c->off_emb = align(c->off_ids + rows * 8);
  c->off_grad[0] = align(c->off_emb + rows * dim * 4);
  c->off_grad[1] = align(c->off_grad[0] + rows * dim * 4);
  c->arena_bytes = align(c->off_grad[1] + rows * dim * 4);
  bool ok = cudaMalloc(&c->arena, c->arena_bytes) == cudaSuccess &&
            cudaMemset(c->arena, 0, sizeof(ArenaHdr)) == cudaSuccess &&
            cudaMalloc(&c->d_peers, kMaxWorld * sizeof(char*)) == cudaSuccess &&
            cudaMalloc(&c->d_peer_grad[0], kMaxWorld * sizeof(float*)) == cudaSuccess &&
            cudaMalloc(&c->d_peer_grad[1], kMaxWorld * sizeof(float*)) == cudaSuccess &&
            cudaMalloc(&c->trace, kTrN * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMemset(c->trace, 0, kTrN * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&c->done, 16) == cudaSuccess && cudaMemset(c->done, 0, 16) == cudaSuccess &&
            cudaMalloc(&c->send_pos, max_tokens * 4) == cudaSuccess &&
            cudaMalloc(&c->send_cnt, kMaxWorld * 4) == cudaSuccess &&
            cudaMemset(c->send_cnt, 0, kMaxWorld * 4) == cudaSuccess &&
            cudaMalloc(&c->view, sizeof(TableDev)) == cudaSuccess &&
            cudaMalloc(&c->d_epoch, 32) == cudaSuccess && cudaMemset(c->d_epoch, 0, 32) == cudaSuccess;
  if (ok) c->d_bar_epoch = c->d_epoch + 1;
  ok = ok && cudaMalloc(&c->d_sig_grad_ptrs, kMaxWorld * sizeof(void*)) == cudaSuccess &&
       cudaMalloc(&c->d_sig_ids_ptrs, kMaxWorld * sizeof(void*)) == cudaSuccess &&
       cudaMalloc(&c->d_cnt_ptrs, kMaxWorld * sizeof(void*)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    rs_comm_destroy(c);
    return fail(RS_ERR_CUDA, "rs_comm_create: cudaMalloc of the arena failed");
  }
  TableDev v;
  std::memset(&v, 0, sizeof(v));
  v.d.emb = reinterpret_cast<float*>(c->arena + c->off_emb);
  v.d.dim = dim;
  v.d.row_cap = rows;
  RS_CUDA(cudaMemcpy(c->view, &v, sizeof(v), cudaMemcpyHostToDevice));
  int st = rs_workspace_create(max_tokens, &c->ws_req);
  if (st) {
    rs_comm_destroy(c);
    return st;
  }
  if (cudaMalloc(&c->touched[0], rows * 4) != cudaSuccess || cudaMalloc(&c->touched[1], rows * 4) != cudaSuccess ||
      cudaMalloc(&c->touched_cnt, 16) != cudaSuccess || cudaMemset(c->touched_cnt, 0, 16) != cudaSuccess) {
    cudaGetLastError();
    rs_comm_destroy(c);
    return fail(RS_ERR_CUDA, "rs_comm_create: cudaMalloc of the touched-row lists failed");
  }
  if (const char* e = getenv("RS_NO_GRAPH")) c->use_graphs = e[0] == '0';
  if (const char* e = getenv("RS_DIST_GRAPH_FORK")) c->graph_fork = e[0] != '0';
  if (const char* e = getenv("RS_DIST_ONE_STREAM")) c->one_stream = e[0] == '1';
  RS_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  // stream priorities (experiment knobs): RS_DIST_PRIO = "<owner><gather>",
  // each 'h' (high), 'l' (low) or 'n' (default)
  int prio_lo = 0, prio_hi = 0;
  RS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const char* pe = getenv("RS_DIST_PRIO");
  auto prio_of = [&](char ch) { return ch == 'h' ? prio_hi : (ch == 'l' ? prio_lo : 0); };
  // default "hn": the owner role (its dedup / table / update are the step's
  // critical path) ahead of the requester's reduce for free SM slots
  const int own_prio = pe && pe[0] ? prio_of(pe[0]) : prio_hi;
  const int gat_prio = pe && pe[0] && pe[1] ? prio_of(pe[1]) : 0;
  RS_CUDA(cudaStreamCreateWithPriority(&c->own_stream, cudaStreamNonBlocking, own_prio));
  RS_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  RS_CUDA(cudaStreamCreateWithPriority(&c->gather_stream, cudaStreamNonBlocking, gat_prio));
  RS_CUDA(cudaEventCreateWithFlags(&c->ev_meta, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&c->ev_gjoin, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&c->ev_dedup, cudaEventDisableTiming));
  if (const char* e = getenv("RS_DIST_REDUCE_AFTER")) c->reduce_after_dedup = e[0] == '1';
  if (const char* e = getenv("RS_HOST_PROF")) c->host_prof = e[0] == '1';
  if (const char* e = getenv("RS_DIST_LOOKUP_SPIN")) c->lookup_spin = e[0] == '1';
  c->h_peers[rank] = c->arena;
  *out = c;
  return RS_OK;
}

int rs_comm_ipc_handle(rs_comm* c, void* handle_out /* 64 bytes */) {
  if (!c || !handle_out) return fail(RS_ERR_CONFIG, "rs_comm_ipc_handle: null argument");
  cudaIpcMemHandle_t h;
  RS_CUDA(cudaIpcGetMemHandle(&h, c->arena));
  std::memcpy(handle_out, &h, sizeof(h));
  return RS_OK;
}

}  // extern "C"

// Device copies of the peer tables once h_peers[] holds every rank's arena.
static int link_peers(rs_comm* c) {
  RS_CUDA(cudaMemcpy(c->d_peers, c->h_peers, kMaxWorld * sizeof(char*), cudaMemcpyHostToDevice));
  {
    std::vector<unsigned long long*> f(kMaxWorld, nullptr);
    for (int r = 0; r < c->world; ++r)
      f[r] = &reinterpret_cast<ArenaHdr*>(c->h_peers[r])->sig_grad[c->rank];
    RS_CUDA(cudaMemcpy(c->d_sig_grad_ptrs, f.data(), kMaxWorld * sizeof(void*), cudaMemcpyHostToDevice));
    for (int r = 0; r < c->world; ++r) f[r] = &reinterpret_cast<ArenaHdr*>(c->h_peers[r])->sig_ids[c->rank];
    RS_CUDA(cudaMemcpy(c->d_sig_ids_ptrs, f.data(), kMaxWorld * sizeof(void*), cudaMemcpyHostToDevice));
    std::vector<uint32_t*> q(kMaxWorld, nullptr);
    for (int r = 0; r < c->world; ++r) q[r] = &reinterpret_cast<ArenaHdr*>(c->h_peers[r])->cnt_in[c->rank];
    RS_CUDA(cudaMemcpy(c->d_cnt_ptrs, q.data(), kMaxWorld * sizeof(void*), cudaMemcpyHostToDevice));
    c->own_sig_emb = reinterpret_cast<ArenaHdr*>(c->arena)->sig_emb;
    c->own_sig_grad = reinterpret_cast<ArenaHdr*>(c->arena)->sig_grad;
  }
  for (int b = 0; b < 2; ++b) {
    std::vector<float*> g(kMaxWorld, nullptr);
    for (int r = 0; r < c->world; ++r) g[r] = reinterpret_cast<float*>(c->h_peers[r] + c->off_grad[b]);
    RS_CUDA(cudaMemcpy(c->d_peer_grad[b], g.data(), kMaxWorld * sizeof(float*), cudaMemcpyHostToDevice));
  }
  return RS_OK;
}

extern "C" {

int rs_comm_open(rs_comm* c, const void* handles /* world x 64 bytes, rank order */) {
  if (!c || !handles) return fail(RS_ERR_CONFIG, "rs_comm_open: null argument");
  if (c->local) return fail(RS_ERR_CONFIG, "rs_comm_open: a local group is already linked");
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
    void* p = nullptr;
    RS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->h_peers[r] = static_cast<char*>(p);
  }
  return link_peers(c);
}

// W logical ranks on the current device (one process): every rank's arena is
// a plain allocation and the peers are each other's device pointers.  The
// kernels, arena layout and flag protocol are the ones of the multi-GPU step;
// only the transport is local HBM instead of NVLink.  Drive the group with
// rs_dist_group_* (never with per-rank rs_dist_* calls on concurrent streams:
// the ranks' wait kernels would depend on each other).
int rs_comm_create_local(int world, uint64_t max_tokens, uint32_t dim, rs_comm** comms_out) {
  if (!comms_out || world < 1 || world > kMaxWorld)
    return fail(RS_ERR_CONFIG, "rs_comm_create_local: bad world / null output");
  std::vector<rs_comm*> cs(world, nullptr);
  for (int r = 0; r < world; ++r) {
    const int st = rs_comm_create(r, world, max_tokens, dim, &cs[r]);
    if (st) {
      for (auto* c : cs) rs_comm_destroy(c);
      return st;
    }
    cs[r]->local = true;
  }
  for (int r = 0; r < world; ++r) {
    for (int q = 0; q < world; ++q) cs[r]->h_peers[q] = cs[q]->arena;
    const int st = link_peers(cs[r]);
    if (st) {
      for (auto* c : cs) rs_comm_destroy(c);
      return st;
    }
  }
  for (int r = 0; r < world; ++r) comms_out[r] = cs[r];
  return RS_OK;
}

int rs_comm_destroy(rs_comm* c) {
  if (!c) return RS_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (!c->local && r != c->rank && c->h_peers[r]) cudaIpcCloseMemHandle(c->h_peers[r]);
  void* ps[] = {c->arena, c->d_peers, c->d_peer_grad[0], c->d_peer_grad[1], c->trace, c->done,
                c->send_pos, c->send_cnt, c->view, c->d_epoch, c->d_sig_grad_ptrs,
                c->d_sig_ids_ptrs, c->d_cnt_ptrs, c->row_cnt, c->row_orig, c->touched[0],
                c->touched[1], c->touched_cnt};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (auto& e : c->pev)
    if (e) cudaEventDestroy(e);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->gather_stream) cudaStreamDestroy(c->gather_stream);
  if (c->ev_meta) cudaEventDestroy(c->ev_meta);
  if (c->ev_gjoin) cudaEventDestroy(c->ev_gjoin);
  if (c->ev_dedup) cudaEventDestroy(c->ev_dedup);
  rs_workspace_destroy(c->ws_req);
  delete c;
  return RS_OK;
}

// distributed_lookup (exchange_sim.cpp:117-233, two-stage) for this rank's
// tokens against the shard it owns.  Every rank of the group must call it
// for the same step.  d_out [n x dim] = bit-exact outputs[rank].
int rs_dist_forward(rs_comm* c, rs_table* t, const uint64_t* d_ids, uint64_t n, float* d_out,
                    void* stream) {
  RS_TRY(check_call(c, t, n, "rs_dist_forward"));
  cudaStream_t s = S(stream);
  RS_TRY(prepare_step(c, t, 0, s));
  StepSets ss;
  RS_TRY(begin_step(c, false, &ss));
  cudaStream_t own;
  RS_TRY(fork_owner(c, s, &own));
  RS_TRY(req_front(c, t, d_ids, n, ss, s));
  RS_TRY(owner_lookup(c, t, ss, own));
  RS_TRY(table_after_op(t, own));
  RS_TRY(req_gather(c, t, n, d_out, ss, s));
  RS_TRY(join_owner(c, s, own));
  end_step(c, ss);
  c->last_n = n;
  c->last_table = t;
  c->have_forward = true;
  c->pending_reset = true;  // unless rs_dist_backward consumes the origins
  c->pending_par = ss.par;
  return RS_OK;
}

// Backward of the last forward: this rank's token gradients d_grads[n x dim].
int rs_dist_backward(rs_comm* c, rs_table* t, const float* d_grads, uint64_t n,
                     const rs_optimizer_params* opt, void* stream) {
  if (!c || !t) return fail(RS_ERR_CONFIG, "rs_dist_backward: null handle");
  if (!c->have_forward || c->last_table != t || c->last_n != n)
    return fail(RS_ERR_CONFIG, "rs_dist_backward: must follow rs_dist_forward on the same batch");
  cudaStream_t s = S(stream);
  alignas(16) unsigned char ob[256];
  std::memset(ob, 0, sizeof(ob));
  RS_TRY(step_opt_args(t, opt, ob, s));
  if (n) RS_TRY(step_reduce_prepare(c->ws_req, c->dim, n, s));
  cudaStream_t own;
  RS_TRY(fork_owner(c, s, &own));
  RS_TRY(req_reduce(c, t, d_grads, n, c->last_sets, s));
  RS_TRY(owner_update(c, t, ob, c->last_sets, own));
  RS_TRY(join_owner(c, s, own));
  t->applies++;
  c->have_forward = false;
  c->pending_reset = false;  // the update consumed the origins
  return prof_step_done(c);
}

// The whole step in one call, the two roles on two streams: the requester
// (dedup, ids out, segment-reduce with the sums stored at the owners, then
// the gather once the rows landed) overlaps the owner (stage 2, find-or-
// insert + answer, update once the sums landed).  Identical results to
// rs_dist_forward + rs_dist_backward (the owner answers with the rows as they
// were before this step's update).  Replayed from a CUDA graph per
// (buffers, n, parities) -- the flags' epoch lives on the device.
int rs_dist_step(rs_comm* c, rs_table* t, const uint64_t* d_ids, uint64_t n, const float* d_grads,
                 float* d_out, const rs_optimizer_params* opt, void* stream) {
  HostClock hc(c);
  RS_TRY(check_call(c, t, n, "rs_dist_step"));
  cudaStream_t s = S(stream);
  alignas(16) unsigned char ob[256];
  std::memset(ob, 0, sizeof(ob));
  RS_TRY(step_opt_args(t, opt, ob, s));
  hc.mark(0);
  RS_TRY(prepare_step(c, t, n, s));
  hc.mark(1);
  StepSets ss;
  RS_TRY(begin_step(c, fast_requester(c, n, d_grads), &ss));
  const bool fast = ss.fu >= 0;
  const int mirror = t->mirror_next;
  auto enqueue = [&](cudaStream_t q) -> int {
    if (c->one_stream && fast) {  // both roles in one stream, data-flow order
      RS_TRY(req_front_fast(c, d_ids, n, ss, q));
      RS_TRY(owner_lookup(c, t, ss, q));
      RS_TRY(table_mirror_copy(t, mirror, q));
      RS_TRY(req_reduce_fast(c, d_grads, n, ss, q));
      RS_TRY(req_gather_fast(c, n, d_out, ss, q));
      return owner_update(c, t, ob, ss, q);
    }
    if (c->one_stream) {  // both roles in one stream: fused gather + reduce pass
      RS_TRY(req_front(c, t, d_ids, n, ss, q));
      RS_TRY(owner_lookup(c, t, ss, q));
      RS_TRY(table_mirror_copy(t, mirror, q));
      RS_TRY(req_gather_reduce(c, t, n, d_out, d_grads, ss, q));
      return owner_update(c, t, ob, ss, q);
    }
    // requester on q: dedup, ids out, reduce + sums out, then the gather;
    // owner on its stream: stage 2, table + answer, then the update
    cudaStream_t own;
    // (the owner stream forks after the id send when the lookup spins)
    if (!c->lookup_spin) RS_TRY(fork_owner(c, q, &own));
    if (fast) RS_TRY(req_front_fast(c, d_ids, n, ss, q));
    else RS_TRY(req_front(c, t, d_ids, n, ss, q));
    if (c->lookup_spin) RS_TRY(fork_owner(c, q, &own));
    // the gather needs only the metadata (and the rows): it runs on its own
    // stream, concurrently with the segment-reduce of the same tokens
    RS_CUDA(cudaEventRecord(c->ev_meta, q));
    RS_CUDA(cudaStreamWaitEvent(c->gather_stream, c->ev_meta, 0));
    // the counters reach the pinned mirror from k_own_table's epilogue (mapped
    // store) instead of a copy node on the owner's critical path
    TableCounters* mo = t->mirror[mirror].dev_ptr;
    if (c->reduce_after_dedup) {
      // the requester's reduce (needed only by the owners' update) waits for
      // this rank's owner dedup: the dedup, on the critical path, then finds
      // the SMs free instead of behind the reduce's long blocks
      RS_TRY(owner_lookup(c, t, ss, own, mo, c->ev_dedup));
      RS_CUDA(cudaStreamWaitEvent(q, c->ev_dedup, 0));
      if (fast) RS_TRY(req_reduce_fast(c, d_grads, n, ss, q));
      else RS_TRY(req_reduce(c, t, d_grads, n, ss, q));
    } else {
      if (fast) RS_TRY(req_reduce_fast(c, d_grads, n, ss, q));
      else RS_TRY(req_reduce(c, t, d_grads, n, ss, q));
      RS_TRY(owner_lookup(c, t, ss, own, mo, nullptr, c->lookup_spin));
    }
    if (!mo) RS_TRY(table_mirror_copy(t, mirror, own));
    RS_TRY(owner_update(c, t, ob, ss, own));
    static const bool gather_q = getenv("RS_DIST_GATHER_ON_Q") && getenv("RS_DIST_GATHER_ON_Q")[0] == '1';
    if (fast && gather_q) {  // experiment: the gather after the reduce, on the requester's stream
      RS_TRY(req_gather_fast(c, n, d_out, ss, q));
      return join_owner(c, q, own);
    }
    if (fast) RS_TRY(req_gather_fast(c, n, d_out, ss, c->gather_stream));
    else RS_TRY(req_gather(c, t, n, d_out, ss, c->gather_stream));
    RS_CUDA(cudaEventRecord(c->ev_gjoin, c->gather_stream));
    RS_CUDA(cudaStreamWaitEvent(q, c->ev_gjoin, 0));
    return join_owner(c, q, own);
  };
  if (c->profiling || !c->use_graphs) {
    RS_TRY(enqueue(s));
  } else {
    DistGraph* hit = nullptr;
    for (auto& g : c->graphs)
      if (g.t == t && g.ids == d_ids && g.grads == d_grads && g.out == d_out && g.n == n &&
          g.mirror == mirror && g.ru == ss.ru && g.par == ss.par && g.fu == ss.fu &&
          g.pbuf == c->ws_req->pbuf && g.csum == c->csum_dst && std::memcmp(g.opt, ob, sizeof(ob)) == 0) {
        hit = &g;
        break;
      }
    if (!hit) {
      if (c->graphs.size() >= 16) {  // evict the least recently used
        auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                    [](const DistGraph& x, const DistGraph& y) {
                                      return x.last_use < y.last_use;
                                    });
        cudaGraphExecDestroy(lru->exec);
        c->graphs.erase(lru);
      }
      DistGraph e;
      e.t = t;
      e.ids = d_ids;
      e.grads = d_grads;
      e.out = d_out;
      e.n = n;
      e.mirror = mirror;
      e.ru = ss.ru;
      e.par = ss.par;
      e.fu = ss.fu;
      e.pbuf = c->ws_req->pbuf;
      e.csum = c->csum_dst;
      std::memcpy(e.opt, ob, sizeof(ob));
      // hot-id finish as a forked graph branch (RS_DIST_GRAPH_FORK=0: linear)
      const bool f0 = c->ws_req->fork;
      c->ws_req->fork = c->ws_req->fork && c->graph_fork;
      const uint64_t before = launches();
      RS_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
      const int st = enqueue(c->cap_stream);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &g);
      c->ws_req->fork = f0;
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
      c->graphs.push_back(e);
      hit = &c->graphs.back();
    }
    hit->last_use = ++c->graph_clock;
    hc.mark(2);
    RS_CUDA(cudaGraphLaunch(hit->exec, s));
    hc.mark(3);
    count_launch(hit->launches);
  }
  RS_TRY(table_mirror_commit(t, mirror, s));
  end_step(c, ss);
  t->applies++;
  c->have_forward = false;
  hc.mark(4);
  return prof_step_done(c);
}

// rs_dist_step + the f64 sum of this rank's gathered rows (run_workload's
// emb_checksum, workload.cpp:547-549) into d_checksum, summed inside the
// gather kernel (D % 4 == 0; else a separate reduction over d_out).
int rs_dist_step_checksum(rs_comm* c, rs_table* t, const uint64_t* d_ids, uint64_t n,
                          const float* d_grads, float* d_out, const rs_optimizer_params* opt,
                          double* d_checksum, void* stream) {
  if (!c || !t || !d_checksum) return fail(RS_ERR_CONFIG, "rs_dist_step_checksum: null argument");
  const bool fused = n > 0 && t->desc.dim % 4 == 0;
  c->csum_dst = fused ? d_checksum : nullptr;
  const int st = rs_dist_step(c, t, d_ids, n, d_grads, d_out, opt, stream);
  c->csum_dst = nullptr;
  if (st || fused) return st;
  return rs_checksum(d_out, n * t->desc.dim, d_checksum, stream);
}

// Device-side barrier over the group on `stream` (every rank must call it):
// work enqueued after it starts only once every rank reached it.
int rs_comm_barrier(rs_comm* c, void* stream) {
  if (!c) return fail(RS_ERR_CONFIG, "rs_comm_barrier: null comm");
  carve(k_barrier), k_barrier<<<1, kMaxWorld, 0, S(stream)>>>(comm_dev(c, 0, kRequester), c->d_bar_epoch);
  RS_LAUNCH_CHECK("k_barrier");
  return RS_OK;
}

int rs_comm_set_profiling(rs_comm* c, int on) {
  if (!c) return fail(RS_ERR_CONFIG, "rs_comm_set_profiling: null comm");
  if (on && !c->pev[0])
    for (auto& e : c->pev) RS_CUDA(cudaEventCreate(&e));
  c->profiling = on != 0;
  for (auto& m : c->pms) m = 0;
  c->pcount = 0;
  return RS_OK;
}

int rs_comm_phase_ms(rs_comm* c, double* ms, int n, uint64_t* count) {
  if (!c || !ms) return fail(RS_ERR_CONFIG, "rs_comm_phase_ms: null argument");
  for (int k = 0; k < n && k < kDistPhases; ++k) ms[k] = c->pcount ? c->pms[k] / c->pcount : 0.0;
  if (count) *count = c->pcount;
  return RS_OK;
}

// This rank's ExchangeTrace row (exchange_sim.hpp:37-59): ids_sent[dst],
// embs_sent[dst] (vectors this rank, as owner, sent to dst), lookups,
// ids_requested, ids_received.  Synchronizes.
// the device timeline of this rank's last step (RS_TRACE=1): rs_workspace_trace of the requester workspace
int rs_comm_timeline(rs_comm* c, uint64_t* out, uint64_t cap, uint64_t* n_out) {
  if (!c) return fail(RS_ERR_CONFIG, "rs_comm_timeline: null comm");
  if (getenv("RS_EPOCH_DBG")) {
    unsigned long long e[4];
    RS_CUDA(cudaMemcpy(e, c->d_epoch, 32, cudaMemcpyDeviceToHost));
    fprintf(stderr, "rank %d epochs: requester %llu owner %llu host %llu\n", c->rank, e[0], e[2], c->epoch);
  }
  return rs_workspace_trace(c->ws_req, out, cap, n_out);
}

int rs_comm_trace(rs_comm* c, uint64_t* ids_sent, uint64_t* embs_sent, uint64_t* lookups,
                  uint64_t* ids_requested, uint64_t* ids_received) {
  if (!c) return fail(RS_ERR_CONFIG, "rs_comm_trace: null comm");
  RS_CUDA(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(kTrN);
  RS_CUDA(cudaMemcpy(h.data(), c->trace, kTrN * 8, cudaMemcpyDeviceToHost));
  if (h[kTrError]) return fail(RS_ERR_INVARIANT, "sharded step: a peer did not signal (timeout)");
  for (int r = 0; r < c->world; ++r) {
    if (ids_sent) ids_sent[r] = h[kTrIdsSent + r];
    if (embs_sent) embs_sent[r] = h[kTrEmbsSent + r];
  }
  if (lookups) *lookups = h[kTrLookups];
  if (ids_requested) *ids_requested = h[kTrRequested];
  if (ids_received) *ids_received = h[kTrReceived];
  return RS_OK;
}


// ---- the group of local ranks (rs_comm_create_local) --------------------------
// Every phase of one sharded step, rank by rank, on ONE stream in data-flow
// order: when a rank's wait kernel runs, the flags it waits for were raised
// by kernels earlier in the same stream, so no kernel ever waits on a kernel
// that has not run yet.  Same kernels, arena traffic and flag protocol as the
// multi-GPU step.
struct alignas(16) OptBuf {
  unsigned char b[256] = {0};
};

static int group_check(rs_comm* const* cs, rs_table* const* ts, int world, const uint64_t* n,
                       const char* who) {
  if (!cs || !ts || !n || world < 1) return fail(RS_ERR_CONFIG, std::string(who) + ": null argument");
  for (int r = 0; r < world; ++r) {
    if (!cs[r] || !cs[r]->local || cs[r]->world != world || cs[r]->rank != r)
      return fail(RS_ERR_CONFIG, std::string(who) + ": comms must be a local group in rank order");
    RS_TRY(check_call(cs[r], ts[r], n[r], who));
  }
  return RS_OK;
}

int rs_dist_group_forward(rs_comm* const* cs, rs_table* const* ts, int world, const uint64_t* const* d_ids,
                          const uint64_t* n, float* const* d_out, void* stream) {
  RS_TRY(group_check(cs, ts, world, n, "rs_dist_group_forward"));
  cudaStream_t s = S(stream);
  std::vector<StepSets> ss(world);
  for (int r = 0; r < world; ++r) {
    RS_TRY(prepare_step(cs[r], ts[r], 0, s));
    RS_TRY(begin_step(cs[r], false, &ss[r]));
  }
  for (int r = 0; r < world; ++r) RS_TRY(req_front(cs[r], ts[r], d_ids[r], n[r], ss[r], s));
  for (int r = 0; r < world; ++r) {
    RS_TRY(owner_lookup(cs[r], ts[r], ss[r], s));
    RS_TRY(table_after_op(ts[r], s));
  }
  for (int r = 0; r < world; ++r) RS_TRY(req_gather(cs[r], ts[r], n[r], d_out[r], ss[r], s));
  for (int r = 0; r < world; ++r) {
    end_step(cs[r], ss[r]);
    cs[r]->last_n = n[r];
    cs[r]->last_table = ts[r];
    cs[r]->have_forward = true;
    cs[r]->pending_reset = true;
    cs[r]->pending_par = ss[r].par;
  }
  return RS_OK;
}

int rs_dist_group_backward(rs_comm* const* cs, rs_table* const* ts, int world, const float* const* d_grads,
                           const uint64_t* n, const rs_optimizer_params* opt, void* stream) {
  if (!cs || !ts || !n || world < 1) return fail(RS_ERR_CONFIG, "rs_dist_group_backward: null argument");
  cudaStream_t s = S(stream);
  std::vector<OptBuf> obs(world);
  for (int r = 0; r < world; ++r) {
    rs_comm* c = cs[r];
    if (!c || !c->local || !c->have_forward || c->last_table != ts[r] || c->last_n != n[r])
      return fail(RS_ERR_CONFIG, "rs_dist_group_backward: must follow rs_dist_group_forward on the same batches");
    RS_TRY(step_opt_args(ts[r], opt, obs[r].b, s));
    if (n[r]) RS_TRY(step_reduce_prepare(c->ws_req, c->dim, n[r], s));
  }
  for (int r = 0; r < world; ++r) RS_TRY(req_reduce(cs[r], ts[r], d_grads[r], n[r], cs[r]->last_sets, s));
  for (int r = 0; r < world; ++r) RS_TRY(owner_update(cs[r], ts[r], obs[r].b, cs[r]->last_sets, s));
  for (int r = 0; r < world; ++r) {
    ts[r]->applies++;
    cs[r]->have_forward = false;
    cs[r]->pending_reset = false;
  }
  return RS_OK;
}

// forward + backward of one step of the group (rs_dist_step's data flow:
// the owners answer with the rows as they were before this step's update).
int rs_dist_group_step(rs_comm* const* cs, rs_table* const* ts, int world, const uint64_t* const* d_ids,
                       const uint64_t* n, const float* const* d_grads, float* const* d_out,
                       const rs_optimizer_params* opt, void* stream) {
  RS_TRY(group_check(cs, ts, world, n, "rs_dist_group_step"));
  cudaStream_t s = S(stream);
  std::vector<OptBuf> obs(world);
  std::vector<StepSets> ss(world);
  for (int r = 0; r < world; ++r) {
    RS_TRY(step_opt_args(ts[r], opt, obs[r].b, s));
    RS_TRY(prepare_step(cs[r], ts[r], n[r], s));
    RS_TRY(begin_step(cs[r], fast_requester(cs[r], n[r], d_grads[r]), &ss[r]));
  }
  for (int r = 0; r < world; ++r) {
    if (ss[r].fu >= 0) RS_TRY(req_front_fast(cs[r], d_ids[r], n[r], ss[r], s));
    else RS_TRY(req_front(cs[r], ts[r], d_ids[r], n[r], ss[r], s));
  }
  for (int r = 0; r < world; ++r) {
    RS_TRY(owner_lookup(cs[r], ts[r], ss[r], s));
    RS_TRY(table_after_op(ts[r], s));
  }
  for (int r = 0; r < world; ++r) {
    if (ss[r].fu >= 0) RS_TRY(req_reduce_fast(cs[r], d_grads[r], n[r], ss[r], s));
    else RS_TRY(req_reduce(cs[r], ts[r], d_grads[r], n[r], ss[r], s));
  }
  for (int r = 0; r < world; ++r) {
    if (ss[r].fu >= 0) RS_TRY(req_gather_fast(cs[r], n[r], d_out[r], ss[r], s));
    else RS_TRY(req_gather(cs[r], ts[r], n[r], d_out[r], ss[r], s));
  }
  for (int r = 0; r < world; ++r) RS_TRY(owner_update(cs[r], ts[r], obs[r].b, ss[r], s));
  for (int r = 0; r < world; ++r) {
    end_step(cs[r], ss[r]);
    ts[r]->applies++;
    cs[r]->have_forward = false;
  }
  return RS_OK;
}

}  // extern "C"
