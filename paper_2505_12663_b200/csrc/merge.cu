// merge.cu -- automatic table merging, pooled feature lookup and per-token
// routing into the merged id spaces.
//
// Reference: plan_merge (merge_registry.cpp:69-110), MergeGroup
// encode/decode (:48-51), collection_lookup (:112-158), HashTableCollection
// (:160-176), and run_workload's per-token decode + re-encode
// (workload.cpp:431-447, 506-531).
//
//   plan            host C++ (a pure function of the feature list; same
//                   ConfigError cases and messages as the reference)
//   lookup          k_encode_tables: one id per (lookup table, token), all
//                   overflow checks up front (the call fails before any table
//                   is touched); one batched find-or-insert-zero per lookup
//                   table; k_pool: out[t] = sum over lookup tables in order
//                   (f32, from 0.0f), mean = sum * (1.0f / n), 128-bit rows
//   routing         k_route_count / k_route_scan / k_route_scatter: stable
//                   partition of the tokens by merged group (token order kept
//                   inside every group, so the per-id gradient order of the
//                   step downstream is the reference's), with the catalog
//                   decode and the group encode fused in
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "rs_host.hpp"

namespace rs {
namespace {

constexpr uint32_t kMaxRouteGroups = 32;
constexpr uint32_t kMaxCatalog = 1024;
constexpr uint32_t kRouteTile = 1024;  // tokens per block (4 rounds of 256)

enum : unsigned { kErrTop = 1u, kErrIndex = 2u, kErrOverflow = 4u };

// one id per (lookup table r, token t): out[r * n + t]
struct EncodeTab {
  uint64_t tag[16];    // index << (63 - k)
  uint32_t shift[16];  // 63 - k
};

__global__ void k_encode_tables(const uint64_t* __restrict__ raw, uint64_t n, uint32_t L, EncodeTab tab,
                                uint64_t* __restrict__ out, unsigned* __restrict__ err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * L;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(i / n);
    const uint64_t x = raw[i - (uint64_t)r * n];
    if (x >> tab.shift[r]) atomicOr(err, kErrOverflow);  // encode_tagged_id overflow
    out[i] = tab.tag[r] | x;
  }
}

struct PoolTab {
  const float* emb[16];  // embedding base of the lookup table's physical table
};

// pooled rows: one warp per token, float4 lanes (dim % 4 == 0) else scalar
__global__ void k_pool(const int64_t* __restrict__ rows, uint64_t n, uint32_t L, uint32_t D,
                       PoolTab tab, int mode, float* __restrict__ out) {
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  const float inv = 1.0f / (float)L;
  for (uint64_t t = w; t < n; t += nw) {
    if ((D & 3u) == 0) {
      const uint32_t D4 = D >> 2;
      for (uint32_t j = lane; j < D4; j += 32) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t r = 0; r < L; ++r) {
          const int64_t row = __ldg(rows + (uint64_t)r * n + t);
          // row < 0: the ensure failed (table full / row pool; reported by its
          // error counters) -- pool zeros instead of reading outside the pool
          const float4 v = row < 0 ? make_float4(0.f, 0.f, 0.f, 0.f)
                                   : __ldg(reinterpret_cast<const float4*>(tab.emb[r] + (size_t)row * D) + j);
          if (mode == RS_POOL_NONE) {
            acc = v;
          } else {
            acc.x = __fadd_rn(acc.x, v.x);
            acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z);
            acc.w = __fadd_rn(acc.w, v.w);
          }
        }
        if (mode == RS_POOL_MEAN) {
          acc.x = __fmul_rn(acc.x, inv);
          acc.y = __fmul_rn(acc.y, inv);
          acc.z = __fmul_rn(acc.z, inv);
          acc.w = __fmul_rn(acc.w, inv);
        }
        reinterpret_cast<float4*>(out + t * D)[j] = acc;
      }
    } else {
      for (uint32_t j = lane; j < D; j += 32) {
        float acc = 0.f;
        for (uint32_t r = 0; r < L; ++r) {
          const int64_t row = __ldg(rows + (uint64_t)r * n + t);
          const float v = row < 0 ? 0.f : __ldg(tab.emb[r] + (size_t)row * D + j);
          acc = mode == RS_POOL_NONE ? v : __fadd_rn(acc, v);
        }
        if (mode == RS_POOL_MEAN) acc = __fmul_rn(acc, inv);
        out[t * D + j] = acc;
      }
    }
  }
}

// ---- routing ------------------------------------------------------------
struct RouteMaps {
  const uint32_t* group_of;   // [n_catalog + 1]
  const uint64_t* tag_of;     // [n_catalog + 1] member_index << (63 - k_group)
  const uint32_t* shift_of;   // [n_catalog + 1] 63 - k_group
  uint32_t cat_shift;         // 63 - catalog k
  uint32_t n_catalog;
  uint32_t n_groups;
};

__device__ __forceinline__ uint32_t route_one(const RouteMaps& m, uint64_t x, uint64_t* gid,
                                              unsigned* err) {
  if (x >> 63) {  // decode_tagged_id: top bit must be zero
    atomicOr(err, kErrTop);
    *gid = 0;
    return 0;
  }
  const uint32_t ord = (uint32_t)(x >> m.cat_shift);
  if (ord > m.n_catalog) {
    atomicOr(err, kErrIndex);
    *gid = 0;
    return 0;
  }
  const uint64_t raw = x & ((1ull << m.cat_shift) - 1);
  const uint32_t sh = __ldg(m.shift_of + ord);
  if (raw >> sh) atomicOr(err, kErrOverflow);
  *gid = __ldg(m.tag_of + ord) | raw;
  return __ldg(m.group_of + ord);
}

// per block: count of tokens per group
__global__ void __launch_bounds__(256) k_route_count(const uint64_t* __restrict__ tagged, uint64_t n,
                                                     RouteMaps m, uint32_t* __restrict__ counts,
                                                     unsigned* __restrict__ err) {
  __shared__ uint32_t c[kMaxRouteGroups];
  if (threadIdx.x < kMaxRouteGroups) c[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRouteTile;
  for (uint32_t k = 0; k < kRouteTile / 256; ++k) {
    const uint64_t t = base + k * 256 + threadIdx.x;
    if (t < n) {
      uint64_t gid;
      atomicAdd(&c[route_one(m, tagged[t], &gid, err)], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < m.n_groups) counts[(uint64_t)blockIdx.x * m.n_groups + threadIdx.x] = c[threadIdx.x];
}

// exclusive scan over blocks per group (one block of 1024 threads; group
// after group; offsets are group-major: group g starts after all tokens of
// groups < g)
__global__ void __launch_bounds__(1024) k_route_scan(uint32_t* __restrict__ counts, uint32_t nblocks,
                                                     uint32_t G, uint64_t* __restrict__ group_counts) {
  __shared__ uint32_t wsum[32];
  __shared__ uint64_t s_start;
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  if (t == 0) s_start = 0;
  __syncthreads();
  for (uint32_t g = 0; g < G; ++g) {
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < nblocks; b0 += 1024) {
      const uint32_t b = b0 + t;
      const uint32_t v = b < nblocks ? counts[(uint64_t)b * G + g] : 0u;
      uint32_t x = v;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        const uint32_t wv = wsum[lane];
        uint32_t z = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, z, o);
          if (lane >= (uint32_t)o) z += y;
        }
        wsum[lane] = z - wv;  // exclusive warp offsets
      }
      __syncthreads();
      const uint32_t excl = carry + wsum[warp] + x - v;
      if (b < nblocks) counts[(uint64_t)b * G + g] = (uint32_t)s_start + excl;
      const uint32_t tot = __shfl_sync(0xFFFFFFFFu, wsum[31] + x, 31);  // block total (warp 31's view)
      __syncthreads();
      if (warp == 31) wsum[0] = tot;  // broadcast the chunk total
      __syncthreads();
      carry += wsum[0];
      __syncthreads();
    }
    if (t == 0) {
      group_counts[g] = carry;
      s_start += carry;
    }
    __syncthreads();
  }
}

// stable scatter: rounds of 256 tokens in order, warp ballots per group
__global__ void __launch_bounds__(256) k_route_scatter(const uint64_t* __restrict__ tagged, uint64_t n,
                                                       RouteMaps m, const uint32_t* __restrict__ offs,
                                                       uint64_t* __restrict__ gids,
                                                       uint32_t* __restrict__ pos,
                                                       unsigned* __restrict__ err) {
  __shared__ uint32_t run[kMaxRouteGroups];
  __shared__ uint32_t wcnt[8][kMaxRouteGroups];
  const uint32_t G = m.n_groups, warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  if (threadIdx.x < G) run[threadIdx.x] = offs[(uint64_t)blockIdx.x * G + threadIdx.x];
  const uint64_t base = (uint64_t)blockIdx.x * kRouteTile;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (uint32_t k = 0; k < kRouteTile / 256; ++k) {
    const uint64_t t = base + k * 256 + threadIdx.x;
    const bool v = t < n;
    uint64_t gid = 0;
    uint32_t g = 0xFFFFFFFFu;
    if (v) g = route_one(m, tagged[t], &gid, err);
    __syncthreads();  // run[] of the previous round is final
    uint32_t mine = 0;
    for (uint32_t h = 0; h < G; ++h) {
      const unsigned b = __ballot_sync(0xFFFFFFFFu, g == h);
      if (lane == 0) wcnt[warp][h] = __popc(b);
      if (g == h) mine = __popc(b & lt);
    }
    __syncthreads();
    if (v) {
      uint32_t before = run[g];
      for (uint32_t w2 = 0; w2 < warp; ++w2) before += wcnt[w2][g];
      gids[before + mine] = gid;
      pos[before + mine] = (uint32_t)t;
    }
    __syncthreads();
    if (threadIdx.x < G) {
      uint32_t add = 0;
      for (uint32_t w2 = 0; w2 < 8; ++w2) add += wcnt[w2][threadIdx.x];
      run[threadIdx.x] += add;
    }
  }
}

}  // namespace
}  // namespace rs

using namespace rs;

struct rs_merge_plan {
  struct Group {
    uint32_t dim = 0, k_bits = 0;
    std::vector<std::string> members;
    std::unordered_map<std::string, uint32_t> index_of;
  };
  std::vector<Group> groups;
  std::unordered_map<std::string, uint32_t> group_of;
};

struct rs_collection {
  rs_merge_plan plan;
  std::vector<rs_table*> tables;
  uint64_t* keys = nullptr;
  int64_t* rows = nullptr;
  uint64_t cap = 0;  // entries of keys / rows
  unsigned* err = nullptr;
};

struct rs_router {
  RouteMaps m{};
  uint32_t* d_group_of = nullptr;
  uint64_t* d_tag_of = nullptr;
  uint32_t* d_shift_of = nullptr;
  uint32_t* counts = nullptr;
  uint64_t counts_cap = 0;
  unsigned* err = nullptr;
  uint64_t* d_group_counts = nullptr;
};

static std::string feat_name(const rs_feature_config& f) {
  return f.feature_name ? std::string(f.feature_name) : std::string();
}

extern "C" {

// plan_merge (merge_registry.cpp:69-110): groups by embedding dim, member
// and group order by first appearance, k = bit_width(m).
int rs_plan_merge(const rs_feature_config* configs, uint32_t n, rs_merge_plan** out) {
  if (!out || (n && !configs)) return fail(RS_ERR_CONFIG, "rs_plan_merge: null argument");
  auto* p = new rs_merge_plan();
  std::unordered_set<std::string> seen;
  std::unordered_map<uint32_t, uint32_t> group_of_dim;
  auto bad = [&](const std::string& msg) {
    delete p;
    return fail(RS_ERR_CONFIG, msg);
  };
  for (uint32_t i = 0; i < n; ++i) {
    const rs_feature_config& f = configs[i];
    const std::string name = feat_name(f);
    if (name.empty()) return bad("feature with empty name");
    if (!seen.insert(name).second) return bad("duplicate feature name: " + name);
    if (f.embedding_dim == 0) return bad("feature " + name + ": embedding_dim must be >= 1");
    if (f.n_lookup_tables == 0) return bad("feature " + name + ": lookup_tables must be non-empty");
    for (uint32_t j = 0; j < f.n_lookup_tables; ++j) {
      const std::string t = f.lookup_tables[j] ? f.lookup_tables[j] : "";
      auto known = p->group_of.find(t);
      if (known != p->group_of.end()) {
        if (p->groups[known->second].dim != f.embedding_dim)
          return bad("logical table " + t + " referenced with conflicting embedding dims");
        continue;
      }
      auto it = group_of_dim.try_emplace(f.embedding_dim, (uint32_t)p->groups.size());
      if (it.second) {
        rs_merge_plan::Group g;
        g.dim = f.embedding_dim;
        p->groups.push_back(std::move(g));
      }
      rs_merge_plan::Group& g = p->groups[it.first->second];
      g.members.push_back(t);
      g.index_of[t] = (uint32_t)g.members.size();
      p->group_of[t] = it.first->second;
    }
  }
  for (auto& g : p->groups) {
    uint32_t m = (uint32_t)g.members.size(), k = 0;
    while (m) {
      ++k;
      m >>= 1;
    }
    g.k_bits = k;
  }
  *out = p;
  return RS_OK;
}

int rs_merge_plan_destroy(rs_merge_plan* p) {
  delete p;
  return RS_OK;
}

uint32_t rs_merge_plan_groups(const rs_merge_plan* p) { return p ? (uint32_t)p->groups.size() : 0; }

int rs_merge_plan_group(const rs_merge_plan* p, uint32_t g, uint32_t* dim, uint32_t* k_bits,
                        uint32_t* n_members) {
  if (!p || g >= p->groups.size()) return fail(RS_ERR_RANGE, "rs_merge_plan_group: no such group");
  if (dim) *dim = p->groups[g].dim;
  if (k_bits) *k_bits = p->groups[g].k_bits;
  if (n_members) *n_members = (uint32_t)p->groups[g].members.size();
  return RS_OK;
}

const char* rs_merge_plan_member(const rs_merge_plan* p, uint32_t g, uint32_t index) {
  if (!p || g >= p->groups.size() || index < 1 || index > p->groups[g].members.size()) return nullptr;
  return p->groups[g].members[index - 1].c_str();
}

int rs_merge_plan_find(const rs_merge_plan* p, const char* table, uint32_t* group, uint32_t* index) {
  if (!p || !table) return fail(RS_ERR_CONFIG, "rs_merge_plan_find: null argument");
  auto it = p->group_of.find(table);
  if (it == p->group_of.end()) return fail(RS_ERR_CONFIG, std::string("unknown logical table: ") + table);
  if (group) *group = it->second;
  if (index) *index = p->groups[it->second].index_of.at(table);
  return RS_OK;
}

// HashTableCollection (merge_registry.cpp:160-175): one physical table per
// group, the prototype config with the group's embedding dim.
int rs_collection_create(const rs_merge_plan* p, const rs_table_config* prototype,
                         rs_collection** out) {
  if (!p || !prototype || !out) return fail(RS_ERR_CONFIG, "rs_collection_create: null argument");
  auto* c = new rs_collection();
  c->plan = *p;
  for (const auto& g : p->groups) {
    rs_table_config cfg = *prototype;
    cfg.embedding_dim = g.dim;
    rs_table* t = nullptr;
    const int st = rs_table_create(&cfg, &t);
    if (st) {
      rs_collection_destroy(c);
      return st;
    }
    c->tables.push_back(t);
  }
  if (cudaMalloc(&c->err, 16) != cudaSuccess) {
    rs_collection_destroy(c);
    return cuda_fail(cudaGetLastError(), "rs_collection_create");
  }
  *out = c;
  return RS_OK;
}

int rs_collection_destroy(rs_collection* c) {
  if (!c) return RS_OK;
  for (rs_table* t : c->tables) rs_table_destroy(t);
  if (c->keys) cudaFree(c->keys);
  if (c->rows) cudaFree(c->rows);
  if (c->err) cudaFree(c->err);
  delete c;
  return RS_OK;
}

rs_table* rs_collection_table(rs_collection* c, uint32_t group) {
  return (c && group < c->tables.size()) ? c->tables[group] : nullptr;
}

// collection_lookup (merge_registry.cpp:112-158) for one feature over the
// raw ids d_raw[n]: d_out [n x feature dim].  Synchronizes (the id range
// check happens before any table is touched).
int rs_collection_lookup(rs_collection* c, const rs_feature_config* f, const uint64_t* d_raw,
                         uint64_t n, float* d_out, void* stream) {
  if (!c || !f) return fail(RS_ERR_CONFIG, "rs_collection_lookup: null argument");
  const std::string name = feat_name(*f);
  if (f->pooling > RS_POOL_MEAN) return fail(RS_ERR_CONFIG, "feature " + name + ": unknown pooling");
  if (f->pooling == RS_POOL_NONE && f->n_lookup_tables != 1)
    return fail(RS_ERR_CONFIG, "feature " + name + ": pooling=none requires exactly one lookup table");
  const uint32_t L = f->n_lookup_tables;
  if (L == 0 || L > 16) return fail(RS_ERR_CONFIG, "feature " + name + ": 1..16 lookup tables supported");
  EncodeTab et{};
  PoolTab pt{};
  std::vector<uint32_t> grp(L);
  for (uint32_t r = 0; r < L; ++r) {
    uint32_t g = 0, idx = 0;
    const int st = rs_merge_plan_find(&c->plan, f->lookup_tables[r], &g, &idx);
    if (st) return st;
    const auto& G = c->plan.groups[g];
    if (G.dim != f->embedding_dim)
      return fail(RS_ERR_CONFIG, "feature " + name + ": embedding_dim differs from its tables'");
    et.shift[r] = 63 - G.k_bits;
    et.tag[r] = (uint64_t)idx << et.shift[r];
    grp[r] = g;
  }
  if (n == 0) return RS_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (c->cap < n * L) {
    if (c->keys) cudaFree(c->keys);
    if (c->rows) cudaFree(c->rows);
    c->keys = nullptr;
    c->rows = nullptr;
    c->cap = 0;
    RS_CUDA(cudaMalloc(&c->keys, n * L * 8));
    RS_CUDA(cudaMalloc(&c->rows, n * L * 8));
    c->cap = n * L;
  }
  RS_CUDA(cudaMemsetAsync(c->err, 0, 4, s));
  k_encode_tables<<<grid_for(n * L, 256, 148 * 8), 256, 0, s>>>(d_raw, n, L, et, c->keys, c->err);
  RS_LAUNCH_CHECK("k_encode_tables");
  unsigned h = 0;
  RS_CUDA(cudaMemcpyAsync(&h, c->err, 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaStreamSynchronize(s));
  if (h) return fail(RS_ERR_RANGE, "encode_tagged_id: raw id exceeds payload width");
  for (uint32_t r = 0; r < L; ++r) {
    const int st = table_ensure_any(c->tables[grp[r]], c->keys + (uint64_t)r * n, nullptr, n, nullptr,
                                    c->rows + (uint64_t)r * n, nullptr, nullptr, s);
    if (st) return st;
  }
  // rows are stable across the ensures (the pool never moves rows), but the
  // pool base may have grown: read the descriptors now
  for (uint32_t r = 0; r < L; ++r) pt.emb[r] = c->tables[grp[r]]->desc.emb;
  k_pool<<<grid_for(n, 8, 148 * 16), 256, 0, s>>>(c->rows, n, L, f->embedding_dim, pt, (int)f->pooling,
                                                  d_out);
  RS_LAUNCH_CHECK("k_pool");
  return RS_OK;
}

// ---- routing (workload.cpp:431-447, 506-531) -------------------------------
int rs_router_create(const rs_merge_plan* p, const char* const* catalog_names, uint32_t n_catalog,
                     rs_router** out) {
  if (!p || !out || (n_catalog && !catalog_names))
    return fail(RS_ERR_CONFIG, "rs_router_create: null argument");
  if (n_catalog > kMaxCatalog) return fail(RS_ERR_CONFIG, "rs_router_create: catalog too large");
  if (p->groups.empty() || p->groups.size() > kMaxRouteGroups)
    return fail(RS_ERR_CONFIG, "rs_router_create: 1..32 merge groups supported");
  std::vector<uint32_t> group_of(n_catalog + 1, 0), shift_of(n_catalog + 1, 63 - p->groups[0].k_bits);
  std::vector<uint64_t> tag_of(n_catalog + 1, 0);  // ordinal 0: identity of group 0 (index 0)
  for (uint32_t o = 1; o <= n_catalog; ++o) {
    uint32_t g = 0, idx = 0;
    const int st = rs_merge_plan_find(p, catalog_names[o - 1], &g, &idx);
    if (st) return st;
    group_of[o] = g;
    shift_of[o] = 63 - p->groups[g].k_bits;
    tag_of[o] = (uint64_t)idx << shift_of[o];
  }
  uint32_t k = 0;
  for (uint32_t m = n_catalog; m; m >>= 1) ++k;
  auto* r = new rs_router();
  r->m.cat_shift = 63 - std::max<uint32_t>(1, k);  // catalog_from: k = max(1, bit_width)
  r->m.n_catalog = n_catalog;
  r->m.n_groups = (uint32_t)p->groups.size();
  bool ok = cudaMalloc(&r->d_group_of, (n_catalog + 1) * 4) == cudaSuccess &&
            cudaMalloc(&r->d_tag_of, (n_catalog + 1) * 8) == cudaSuccess &&
            cudaMalloc(&r->d_shift_of, (n_catalog + 1) * 4) == cudaSuccess &&
            cudaMalloc(&r->err, 16) == cudaSuccess &&
            cudaMalloc(&r->d_group_counts, kMaxRouteGroups * 8) == cudaSuccess &&
            cudaMemcpy(r->d_group_of, group_of.data(), (n_catalog + 1) * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(r->d_tag_of, tag_of.data(), (n_catalog + 1) * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(r->d_shift_of, shift_of.data(), (n_catalog + 1) * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    rs_router_destroy(r);
    return cuda_fail(cudaGetLastError(), "rs_router_create");
  }
  r->m.group_of = r->d_group_of;
  r->m.tag_of = r->d_tag_of;
  r->m.shift_of = r->d_shift_of;
  *out = r;
  return RS_OK;
}

int rs_router_destroy(rs_router* r) {
  if (!r) return RS_OK;
  void* ps[] = {r->d_group_of, r->d_tag_of, r->d_shift_of, r->counts, r->err, r->d_group_counts};
  for (void* q : ps)
    if (q) cudaFree(q);
  delete r;
  return RS_OK;
}

// Stable partition of catalog-tagged tokens by merged group, each id
// re-encoded into its group's space: d_gids[n] / d_pos[n] hold group 0's
// tokens (token order) then group 1's, ...; h_counts[G] (optional,
// synchronizes and reports decode / encode range errors) the group sizes.
int rs_route_tagged(rs_router* r, const uint64_t* d_tagged, uint64_t n, uint64_t* d_gids,
                    uint32_t* d_pos, uint64_t* h_counts, void* stream) {
  if (!r) return fail(RS_ERR_CONFIG, "rs_route_tagged: null router");
  if (n > 0xFFFFFFFFull) return fail(RS_ERR_CONFIG, "rs_route_tagged: n must fit 32 bits");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t G = r->m.n_groups;
  const uint32_t nb = (uint32_t)std::max<uint64_t>(1, (n + kRouteTile - 1) / kRouteTile);
  if (r->counts_cap < (uint64_t)nb * G) {
    if (r->counts) cudaFree(r->counts);
    r->counts = nullptr;
    RS_CUDA(cudaMalloc(&r->counts, (uint64_t)nb * G * 4));
    r->counts_cap = (uint64_t)nb * G;
  }
  RS_CUDA(cudaMemsetAsync(r->err, 0, 4, s));
  k_route_count<<<nb, 256, 0, s>>>(d_tagged, n, r->m, r->counts, r->err);
  RS_LAUNCH_CHECK("k_route_count");
  k_route_scan<<<1, 1024, 0, s>>>(r->counts, nb, G, r->d_group_counts);
  RS_LAUNCH_CHECK("k_route_scan");
  k_route_scatter<<<nb, 256, 0, s>>>(d_tagged, n, r->m, r->counts, d_gids, d_pos, r->err);
  RS_LAUNCH_CHECK("k_route_scatter");
  if (h_counts) {
    unsigned e = 0;
    RS_CUDA(cudaMemcpyAsync(h_counts, r->d_group_counts, G * 8, cudaMemcpyDeviceToHost, s));
    RS_CUDA(cudaMemcpyAsync(&e, r->err, 4, cudaMemcpyDeviceToHost, s));
    RS_CUDA(cudaStreamSynchronize(s));
    if (e & kErrTop) return fail(RS_ERR_RANGE, "decode_tagged_id: top bit must be zero");
    if (e & kErrIndex) return fail(RS_ERR_RANGE, "decode_tagged_id: table index out of range");
    if (e & kErrOverflow) return fail(RS_ERR_RANGE, "encode_tagged_id: raw id exceeds payload width");
  }
  return RS_OK;
}

}  // extern "C"
