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
//   requester  KA dedup -> KB metadata -> k_send_ids: owner partition of the
//              unique ids, ids stored straight into the owner's ids_in
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
#include <cstring>
#include <vector>

#include "opt_dev.cuh"
#include "rs_host.hpp"
#include "table_dev.cuh"

namespace rs {
namespace {

constexpr int kMaxWorld = 64;

struct ArenaHdr {
  unsigned long long sig_ids[kMaxWorld];
  unsigned long long sig_emb[kMaxWorld];
  unsigned long long sig_grad[kMaxWorld];
  uint32_t cnt_in[kMaxWorld];
};

// trace slots (per rank, device u64)
enum : int { kTrIdsSent = 0, kTrEmbsSent = kMaxWorld, kTrLookups = 2 * kMaxWorld,
             kTrRequested, kTrReceived, kTrError, kTrN };

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

struct CommDev {
  char* const* peers;  // [W] arena base of every rank (own included), device-visible
  uint32_t rank, world;
  uint32_t cap;        // ids per (source, destination) region
  uint32_t dim;
  size_t off_ids, off_emb, off_grad;
  unsigned long long epoch;
  unsigned long long* trace;
  unsigned int* done;  // last-block counter
};

__device__ __forceinline__ ArenaHdr* hdr_of(const CommDev& c, uint32_t r) {
  return reinterpret_cast<ArenaHdr*>(c.peers[r]);
}

// Last block of a launch raises `sig` (phase flags) at every peer.
__device__ __forceinline__ void signal_all(const CommDev& c, int phase) {
  fence_sys();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(c.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  fence_sys();
  for (uint32_t r = threadIdx.x; r < c.world; r += blockDim.x) {
    ArenaHdr* h = hdr_of(c, r);
    unsigned long long* f = phase == 0 ? &h->sig_ids[c.rank]
                            : phase == 1 ? &h->sig_emb[c.rank]
                                         : &h->sig_grad[c.rank];
    st_release_sys(f, c.epoch);
  }
  if (threadIdx.x == 0) *c.done = 0;
}

// Requester: owner partition of the unique ids, peer stores into ids_in.
__global__ void k_send_ids(CommDev c, const uint64_t* __restrict__ unique,
                           const uint32_t* __restrict__ n_unique,
                           const uint32_t* __restrict__ u_slot, uint32_t* __restrict__ srow,
                           uint32_t* __restrict__ send_pos, uint32_t* __restrict__ send_cnt,
                           uint64_t n_tokens) {
  const uint32_t nu = *n_unique;
  const uint32_t lane = lane_id();
  for (uint32_t base = blockIdx.x * blockDim.x; base < nu; base += gridDim.x * blockDim.x) {
    const uint32_t u = base + threadIdx.x;
    const bool v = u < nu;
    uint64_t id = 0;
    uint32_t o = 0xFFFFFFFFu;
    if (v) {
      id = unique[u];
      o = (uint32_t)(hash64(id) % c.world);  // shard_of (exchange_sim.cpp:84)
    }
    const unsigned mm = __match_any_sync(0xFFFFFFFFu, v ? o : (0xFFFF0000u | lane));
    const uint32_t leader = __ffs(mm) - 1;
    uint32_t j0 = 0;
    if (v && lane == leader) j0 = atomicAdd(&send_cnt[o], (uint32_t)__popc(mm));
    j0 = __shfl_sync(0xFFFFFFFFu, j0, leader);
    if (v) {
      const uint32_t j = j0 + __popc(mm & lanemask_lt());
      uint64_t* dst = reinterpret_cast<uint64_t*>(c.peers[o] + c.off_ids);
      dst[(size_t)c.rank * c.cap + j] = id;  // NVLink store into the owner's arena
      const uint32_t sp = o * c.cap + j;
      send_pos[u] = sp;
      srow[u_slot[u]] = sp;  // the gather reads emb_in row sp
    }
  }
  fence_sys();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(c.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  fence_sys();
  for (uint32_t r = threadIdx.x; r < c.world; r += blockDim.x) {
    hdr_of(c, r)->cnt_in[c.rank] = send_cnt[r];
    c.trace[kTrIdsSent + r] = send_cnt[r];
  }
  if (threadIdx.x == 0) c.trace[kTrRequested] = n_tokens;
  fence_sys();
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < c.world; r += blockDim.x) {
    st_release_sys(&hdr_of(c, r)->sig_ids[c.rank], c.epoch);
    send_cnt[r] = 0;
  }
  if (threadIdx.x == 0) *c.done = 0;
}

// Bounded wait until every source raised flag `phase` for this epoch.
__global__ void k_wait(CommDev c, int phase) {
  ArenaHdr* h = hdr_of(c, c.rank);
  const uint32_t r = threadIdx.x;
  if (r >= c.world) return;
  const unsigned long long* f = phase == 0 ? &h->sig_ids[r] : phase == 1 ? &h->sig_emb[r]
                                                                           : &h->sig_grad[r];
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < c.epoch) {
    if (clock64() - t0 > 40000000000ll) {  // ~20 s: a peer is gone; do not hang the GPU
      c.trace[kTrError] = 1;
      break;
    }
    __nanosleep(200);
  }
}

// Owner: received lists -> one source-ordered flat list (stage-2 input).
__global__ void k_flatten(CommDev c, uint64_t* __restrict__ flat_ids,
                          uint32_t* __restrict__ flat_pos, uint32_t* __restrict__ d_n2) {
  const ArenaHdr* h = hdr_of(c, c.rank);
  const uint32_t src = blockIdx.x;
  uint32_t off = 0;
  for (uint32_t r = 0; r < src; ++r) off += h->cnt_in[r];
  const uint32_t cnt = h->cnt_in[src];
  const uint64_t* in = reinterpret_cast<const uint64_t*>(c.peers[c.rank] + c.off_ids) +
                       (size_t)src * c.cap;
  for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
    flat_ids[off + j] = in[j];
    flat_pos[off + j] = src * c.cap + j;
  }
  if (threadIdx.x == 0) {
    c.trace[kTrEmbsSent + src] = cnt;  // two-stage: one vector per received id
    if (src == c.world - 1) {
      *d_n2 = off + cnt;
      c.trace[kTrReceived] = off + cnt;
    }
  }
}

// Owner: every received position's row, stored into the requester's emb_in.
template <int LPR>
__global__ void __launch_bounds__(256) k_respond(CommDev c, const TableDev* __restrict__ td,
                                                 const uint32_t* __restrict__ slot_of,
                                                 const uint32_t* __restrict__ srow,
                                                 const uint32_t* __restrict__ flat_pos,
                                                 const uint32_t* __restrict__ d_n2,
                                                 const uint32_t* __restrict__ n_unique2) {
  const uint32_t n = *d_n2;
  const uint32_t D4 = td->d.dim >> 2;
  const float4* __restrict__ emb = reinterpret_cast<const float4*>(td->d.emb);
  const uint32_t lane = lane_id(), sub = lane / LPR, l = lane % LPR;
  constexpr int RPW = 32 / LPR;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t p0 = w * RPW; p0 < n; p0 += nw * RPW) {
    const uint64_t p = p0 + sub;
    if (p < n) {
      const uint32_t row = __ldcg(srow + __ldg(slot_of + p));
      if (row == kNoRow) continue;  // table error (reported by the counters)
      const uint32_t origin = __ldg(flat_pos + p);
      const uint32_t src = origin / c.cap, j = origin - src * c.cap;
      float4* dst = reinterpret_cast<float4*>(c.peers[src] + c.off_emb) +
                    ((size_t)c.rank * c.cap + j) * D4;
      for (uint32_t k = l; k < D4; k += LPR) dst[k] = __ldg(emb + (size_t)row * D4 + k);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c.trace[kTrLookups] = *n_unique2;
  signal_all(c, 1);
}

// Requester: raise the gradient flags after KD stored its rows at the owners.
__global__ void k_signal(CommDev c, int phase) { signal_all(c, phase); }

}  // namespace
}  // namespace rs

using namespace rs;

struct rs_comm {
  int rank = 0, world = 1;
  uint64_t cap = 0;
  uint32_t dim = 0;
  char* arena = nullptr;
  size_t arena_bytes = 0, off_ids = 0, off_emb = 0, off_grad = 0;
  char* h_peers[kMaxWorld] = {nullptr};
  char** d_peers = nullptr;
  float** d_peer_grad = nullptr;
  unsigned long long epoch = 0;
  unsigned long long* trace = nullptr;
  unsigned int* done = nullptr;
  uint32_t* send_pos = nullptr;
  uint32_t* send_cnt = nullptr;
  uint64_t* flat_ids = nullptr;
  uint32_t* flat_pos = nullptr;
  uint32_t* d_n2 = nullptr;
  TableDev* view = nullptr;
  rs_workspace* ws_req = nullptr;
  rs_workspace* ws_own = nullptr;
  int req_set = 0, own_set = 0;
  uint64_t last_n = 0;
  bool have_forward = false;
  rs_table* last_table = nullptr;
};

static CommDev comm_dev(rs_comm* c) {
  CommDev d;
  d.peers = c->d_peers;
  d.rank = c->rank;
  d.world = c->world;
  d.cap = (uint32_t)c->cap;
  d.dim = c->dim;
  d.off_ids = c->off_ids;
  d.off_emb = c->off_emb;
  d.off_grad = c->off_grad;
  d.epoch = c->epoch;
  d.trace = c->trace;
  d.done = c->done;
  return d;
}

static cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

extern "C" {

int rs_comm_create(int rank, int world, uint64_t max_tokens, uint32_t dim, rs_comm** out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || dim < 1 ||
      max_tokens < 1)
    return fail(RS_ERR_CONFIG, "rs_comm_create: bad rank/world/dim/max_tokens");
  rs_comm* c = new rs_comm();
  c->rank = rank;
  c->world = world;
  c->cap = max_tokens;
  c->dim = dim;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  c->off_ids = align(sizeof(ArenaHdr));
  c->off_emb = align(c->off_ids + (size_t)world * max_tokens * 8);
  c->off_grad = align(c->off_emb + (size_t)world * max_tokens * dim * 4);
  c->arena_bytes = align(c->off_grad + (size_t)world * max_tokens * dim * 4);
  const uint64_t nflat = (uint64_t)world * max_tokens;
  bool ok = cudaMalloc(&c->arena, c->arena_bytes) == cudaSuccess &&
            cudaMemset(c->arena, 0, sizeof(ArenaHdr)) == cudaSuccess &&
            cudaMalloc(&c->d_peers, kMaxWorld * sizeof(char*)) == cudaSuccess &&
            cudaMalloc(&c->d_peer_grad, kMaxWorld * sizeof(float*)) == cudaSuccess &&
            cudaMalloc(&c->trace, kTrN * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMemset(c->trace, 0, kTrN * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&c->done, 16) == cudaSuccess && cudaMemset(c->done, 0, 16) == cudaSuccess &&
            cudaMalloc(&c->send_pos, max_tokens * 4) == cudaSuccess &&
            cudaMalloc(&c->send_cnt, kMaxWorld * 4) == cudaSuccess &&
            cudaMemset(c->send_cnt, 0, kMaxWorld * 4) == cudaSuccess &&
            cudaMalloc(&c->flat_ids, nflat * 8) == cudaSuccess &&
            cudaMalloc(&c->flat_pos, nflat * 4) == cudaSuccess &&
            cudaMalloc(&c->d_n2, 16) == cudaSuccess && cudaMalloc(&c->view, sizeof(TableDev)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return fail(RS_ERR_CUDA, "rs_comm_create: cudaMalloc of the arena failed");
  }
  TableDev v;
  std::memset(&v, 0, sizeof(v));
  v.d.emb = reinterpret_cast<float*>(c->arena + c->off_emb);
  v.d.dim = dim;
  v.d.row_cap = nflat;
  cudaMemcpy(c->view, &v, sizeof(v), cudaMemcpyHostToDevice);
  int st = rs_workspace_create(max_tokens, &c->ws_req);
  if (!st) st = rs_workspace_create(nflat, &c->ws_own);
  if (st) return st;
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

int rs_comm_open(rs_comm* c, const void* handles /* world x 64 bytes, rank order */) {
  if (!c || !handles) return fail(RS_ERR_CONFIG, "rs_comm_open: null argument");
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
    void* p = nullptr;
    RS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->h_peers[r] = static_cast<char*>(p);
  }
  std::vector<float*> g(kMaxWorld, nullptr);
  for (int r = 0; r < c->world; ++r) g[r] = reinterpret_cast<float*>(c->h_peers[r] + c->off_grad);
  RS_CUDA(cudaMemcpy(c->d_peers, c->h_peers, kMaxWorld * sizeof(char*), cudaMemcpyHostToDevice));
  RS_CUDA(cudaMemcpy(c->d_peer_grad, g.data(), kMaxWorld * sizeof(float*), cudaMemcpyHostToDevice));
  return RS_OK;
}

int rs_comm_destroy(rs_comm* c) {
  if (!c) return RS_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (r != c->rank && c->h_peers[r]) cudaIpcCloseMemHandle(c->h_peers[r]);
  void* ps[] = {c->arena, c->d_peers, c->d_peer_grad, c->trace, c->done, c->send_pos,
                c->send_cnt, c->flat_ids, c->flat_pos, c->d_n2, c->view};
  for (void* p : ps)
    if (p) cudaFree(p);
  rs_workspace_destroy(c->ws_req);
  rs_workspace_destroy(c->ws_own);
  delete c;
  return RS_OK;
}

// Forward of the sharded step: this rank's tokens d_ids[n] against the
// shard table `t` it owns.  Every rank of the group must call it for the
// same step.  d_out [n x dim] = bit-exact distributed_lookup outputs.
int rs_dist_forward(rs_comm* c, rs_table* t, const uint64_t* d_ids, uint64_t n, float* d_out,
                    void* stream) {
  if (!c || !t) return fail(RS_ERR_CONFIG, "rs_dist_forward: null handle");
  if (n > c->cap) return fail(RS_ERR_CONFIG, "rs_dist_forward: batch exceeds max_tokens");
  if (t->desc.dim != c->dim) return fail(RS_ERR_CONFIG, "rs_dist_forward: table dim != comm dim");
  if (t->cfg.max_keys) return fail(RS_ERR_CONFIG, "rs_dist_forward: bounded shard tables unsupported");
  cudaStream_t s = S(stream);
  int st = step_set_smem_attrs();
  if (st) return st;
  c->epoch++;
  const CommDev cd = comm_dev(c);
  rs_workspace* wr = c->ws_req;
  rs_workspace* wo = c->ws_own;
  const uint64_t nflat = (uint64_t)c->world * c->cap;
  // ---- requester: dedup, metadata for the backward, ids to the owners
  wr->last_tile = tile_tokens_for_dim(c->dim);
  const int ru = wr->cur;
  if (n) {
    if ((st = step_fdedup(wr, d_ids, n, ru, s, nullptr))) return st;
    if ((st = step_ftable(wr, t, ru, n, false, true, s))) return st;
  } else {  // idle rank: still clean the other scratch set (KB) and reset its count (KC)
    RS_CUDA(cudaMemsetAsync(wr->set[ru].cnt, 0, 4, s));
    if ((st = step_ftable(wr, t, ru, 1, false, true, s))) return st;
    RS_CUDA(cudaMemsetAsync(wr->set[ru ^ 1].cnt, 0, 4, s));
  }
  k_send_ids<<<grid_for(n ? n : 1, 256, 148 * 4), 256, 0, s>>>(
      cd, wr->unique, wr->set[ru].cnt, wr->set[ru].u_slot, wr->set[ru].srow, c->send_pos,
      c->send_cnt, n);
  RS_LAUNCH_CHECK("k_send_ids");
  // ---- owner: stage-2 dedup of what it received, find-or-insert, respond
  k_wait<<<1, kMaxWorld, 0, s>>>(cd, 0);
  RS_LAUNCH_CHECK("k_wait(ids)");
  k_flatten<<<c->world, 256, 0, s>>>(cd, c->flat_ids, c->flat_pos, c->d_n2);
  RS_LAUNCH_CHECK("k_flatten");
  wo->last_tile = tile_tokens_for_dim(c->dim);
  const int ou = wo->cur;
  // new keys at this owner <= ids received <= world * max_tokens (the peers'
  // batch sizes are not known here without a host round trip)
  if ((st = table_prepare(t, nflat, s))) return st;
  if ((st = step_fdedup(wo, c->flat_ids, nflat, ou, s, c->d_n2))) return st;
  if ((st = step_ftable(wo, t, ou, nflat, true, true, s))) return st;
  {
    const uint32_t d4 = c->dim / 4;
    const unsigned grid = grid_for(nflat / 8 + 1, 8, 148 * 8);
#define RS_RESP(LPR)                                                                   \
  k_respond<LPR><<<grid, 256, 0, s>>>(cd, t->dev, wo->slot_of, wo->set[ou].srow, c->flat_pos, \
                                      c->d_n2, wo->set[ou].cnt)
    if (c->dim % 4 != 0) return fail(RS_ERR_CONFIG, "sharded step needs dim % 4 == 0");
    if (d4 >= 32)
      RS_RESP(32);
    else if (d4 >= 16)
      RS_RESP(16);
    else if (d4 >= 8)
      RS_RESP(8);
    else if (d4 >= 4)
      RS_RESP(4);
    else if (d4 >= 2)
      RS_RESP(2);
    else
      RS_RESP(1);
#undef RS_RESP
    RS_LAUNCH_CHECK("k_respond");
  }
  // clean-up bookkeeping of the owner workspace (KC normally zeroes the other count)
  RS_CUDA(cudaMemsetAsync(wo->set[ou ^ 1].cnt, 0, 4, s));
  if ((st = table_after_op(t, s))) return st;
  // ---- requester: gather from the received rows
  k_wait<<<1, kMaxWorld, 0, s>>>(cd, 1);
  RS_LAUNCH_CHECK("k_wait(embs)");
  if (n) {
    rs_dist_opts o;
    o.gather_view = c->view;
    if ((st = step_tile(wr, t, ru, n, d_out, nullptr, true, s, &o))) return st;
  }
  c->req_set = ru;
  c->own_set = ou;
  wr->cur ^= 1;
  wo->cur ^= 1;
  c->last_n = n;
  c->last_table = t;
  c->have_forward = true;
  return RS_OK;
}

// Backward of the sharded step: this rank's token gradients d_grads[n x dim].
int rs_dist_backward(rs_comm* c, rs_table* t, const float* d_grads, uint64_t n,
                     const rs_optimizer_params* opt, void* stream) {
  if (!c || !t) return fail(RS_ERR_CONFIG, "rs_dist_backward: null handle");
  if (!c->have_forward || c->last_table != t || c->last_n != n)
    return fail(RS_ERR_CONFIG, "rs_dist_backward: must follow rs_dist_forward on the same batch");
  cudaStream_t s = S(stream);
  alignas(16) unsigned char ob[256];
  int st = step_opt_args(t, opt, ob, s);
  if (st) return st;
  const CommDev cd = comm_dev(c);
  rs_workspace* wr = c->ws_req;
  rs_workspace* wo = c->ws_own;
  const uint64_t nflat = (uint64_t)c->world * c->cap;
  // ---- requester: per unique id sums, stored into the owners' grad_in
  if (n) {
    if ((st = step_reduce_prepare(wr, c->dim, n, s))) return st;
    if ((st = step_tile(wr, t, c->req_set, n, nullptr, d_grads, false, s, nullptr))) return st;
    rs_dist_opts o;
    o.peer_dst = c->d_peer_grad;
    o.send_pos = c->send_pos;
    o.cap = (uint32_t)c->cap;
    o.rank = (uint32_t)c->rank;
    if ((st = step_finish(wr, t, c->req_set, n, d_grads, nullptr, nullptr, s, &o))) return st;
  }
  k_signal<<<1, 64, 0, s>>>(cd, 2);
  RS_LAUNCH_CHECK("k_signal(grads)");
  // ---- owner: ordered sum over origins + optimizer on the shard
  k_wait<<<1, kMaxWorld, 0, s>>>(cd, 2);
  RS_LAUNCH_CHECK("k_wait(grads)");
  const float* grad_in = reinterpret_cast<const float*>(c->arena + c->off_grad);
  rs_dist_opts oo;  // owner side: at most `world` origins per id -> CSR path only
  oo.d_n = c->d_n2;
  oo.pos_map = c->flat_pos;
  oo.no_stage = true;
  if ((st = step_tile(wo, t, c->own_set, nflat, nullptr, grad_in, false, s, &oo))) return st;
  if ((st = step_finish(wo, t, c->own_set, nflat, grad_in, ob, nullptr, s, nullptr))) return st;
  t->applies++;
  c->have_forward = false;
  return RS_OK;
}

// This rank's ExchangeTrace row (exchange_sim.hpp:37-59): ids_sent[dst],
// embs_sent[dst] (vectors this rank, as owner, sent to dst), lookups,
// ids_requested, ids_received.  Synchronizes.
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

}  // extern "C"
