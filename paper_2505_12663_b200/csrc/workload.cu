// workload.cu -- synthetic inputs of the benchmark configs, identical to the
// reference generator (workload.hpp:36-49 Rng, workload.cpp:103-152
// TruncatedLognormal/ZipfSampler, :280-307 generate_workload, :348-355
// pseudo_sparse_grad).  std::mt19937_64 is fully specified by the standard,
// and every float mapping is explicit, so the same seed gives the same ids
// on any host.  Host side only, except rs_pseudo_grads (device kernel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <random>
#include <vector>
#include <string>
#include <cstdio>
#include <sstream>
#include <fstream>

#include "rs_internal.cuh"

namespace rs {
namespace {

struct Rng {
  std::mt19937_64 e;
  explicit Rng(uint64_t seed) : e(seed) {}
  double unit() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
  double unit_pos() { return static_cast<double>((e() >> 11) + 1) * 0x1.0p-53; }
};

double normal_cdf(double z) { return 0.5 * std::erfc(-z / std::sqrt(2.0)); }
double trunc_mean(double mu, double sigma, double upper) {
  const double lu = std::log(upper);
  return std::exp(mu + sigma * sigma / 2.0) * normal_cdf((lu - mu - sigma * sigma) / sigma) /
         normal_cdf((lu - mu) / sigma);
}

__global__ void k_pseudo_grads(const uint64_t* __restrict__ sample_of, uint64_t n, uint64_t step,
                               uint32_t dim, float* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * dim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = i / dim, e = i % dim;
    const uint64_t base =
        hash64(sample_of[t] * 0x9e3779b97f4a7c15ULL + step * 0xbf58476d1ce4e5b9ULL + 1);
    const double u = static_cast<double>(hash64(base + e) >> 11) * 0x1.0p-53;
    out[i] = static_cast<float>((u - 0.5) * 0.1);
  }
}

// one gradient row per sample (the formula of k_pseudo_grads)
__global__ void k_sample_rows(uint64_t n_seq, uint64_t first, uint64_t step, uint32_t dim,
                              float* __restrict__ rows) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_seq * dim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i / dim, e = i - s * dim;
    const uint64_t base = hash64((first + s) * 0x9e3779b97f4a7c15ULL + step * 0xbf58476d1ce4e5b9ULL + 1);
    const double u = static_cast<double>(hash64(base + e) >> 11) * 0x1.0p-53;
    rows[i] = static_cast<float>((u - 0.5) * 0.1);
  }
}

// exclusive prefix of the sequence lengths (one block)
__global__ void __launch_bounds__(1024) k_seq_offsets(const uint64_t* __restrict__ lengths, uint64_t n_seq,
                                                      uint64_t* __restrict__ offs) {
  __shared__ uint64_t part[1024];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < n_seq; b0 += 1024) {
    const uint64_t i = b0 + threadIdx.x;
    const uint64_t v = i < n_seq ? lengths[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const uint64_t y = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < n_seq) offs[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) offs[n_seq] = carry;
}

// Block s: sample s's gradient row (pseudo_sparse_grad of sample first + s)
// in smem, then copied to each of its tokens [offs[s], offs[s+1]) with
// 128-bit streaming stores.  One kernel per batch, no intermediate rows.
__global__ void __launch_bounds__(256) k_jagged_grads(const uint64_t* __restrict__ offs, uint64_t first,
                                                      uint64_t step, uint32_t dim, float* __restrict__ out) {
  extern __shared__ float4 srow4[];
  float* srow = reinterpret_cast<float*>(srow4);
  const uint32_t s = blockIdx.x;
  const uint64_t base = hash64((first + s) * 0x9e3779b97f4a7c15ULL + step * 0xbf58476d1ce4e5b9ULL + 1);
  for (uint32_t e = threadIdx.x; e < dim; e += blockDim.x) {
    const double u = static_cast<double>(hash64(base + e) >> 11) * 0x1.0p-53;
    srow[e] = static_cast<float>((u - 0.5) * 0.1);
  }
  __syncthreads();
  const uint64_t a = offs[s], b = offs[s + 1];
  const uint32_t d4 = dim >> 2;
  const uint64_t total = (b - a) * d4;
  float4* dst = reinterpret_cast<float4*>(out) + a * d4;
  for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) __stcs(dst + i, srow4[i % d4]);
}

// Chunked variant: block i handles work item (sample s, token range
// [t0, t1)) -- long samples are split so the blocks are balanced.
struct GradChunk {
  uint32_t s;
  uint32_t t0, t1;
};
__global__ void __launch_bounds__(256) k_jagged_grads_chunks(const GradChunk* __restrict__ work, uint64_t first,
                                                             uint64_t step, uint32_t dim, float* __restrict__ out) {
  extern __shared__ float4 srow4c[];
  float* srow = reinterpret_cast<float*>(srow4c);
  const GradChunk w = work[blockIdx.x];
  const uint64_t base = hash64((first + w.s) * 0x9e3779b97f4a7c15ULL + step * 0xbf58476d1ce4e5b9ULL + 1);
  for (uint32_t e = threadIdx.x; e < dim; e += blockDim.x) {
    const double u = static_cast<double>(hash64(base + e) >> 11) * 0x1.0p-53;
    srow[e] = static_cast<float>((u - 0.5) * 0.1);
  }
  __syncthreads();
  const uint32_t d4 = dim >> 2;
  float4* dst = reinterpret_cast<float4*>(out) + (uint64_t)w.t0 * d4;
  const uint32_t ntok = w.t1 - w.t0;
  if (d4 <= blockDim.x && blockDim.x % d4 == 0) {
    // fixed column per thread: one smem read, then only streaming stores
    const uint32_t c = threadIdx.x % d4, rstep = blockDim.x / d4;
    const float4 v = srow4c[c];
    for (uint32_t r = threadIdx.x / d4; r < ntok; r += rstep) __stcs(dst + (uint64_t)r * d4 + c, v);
  } else {
    const uint64_t total = (uint64_t)ntok * d4;
    for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) __stcs(dst + i, srow4c[i % d4]);
  }
}

// sample index of every token: block s fills [offs[s], offs[s+1])
__global__ void k_fill_sample(const uint64_t* __restrict__ offs, uint32_t* __restrict__ sample_of) {
  const uint32_t s = blockIdx.x;
  const uint64_t a = offs[s], b = offs[s + 1];
  for (uint64_t t = a + threadIdx.x; t < b; t += blockDim.x) sample_of[t] = s;
}

// per token: its sample's row, 128-bit copies, 4 independent chunks per
// thread (loads in flight for the bandwidth)
__global__ void __launch_bounds__(256) k_broadcast_rows(const uint32_t* __restrict__ sample_of,
                                                        const float* __restrict__ rows, uint32_t dim,
                                                        uint32_t n_tokens, float* __restrict__ out) {
  const uint32_t d4 = dim >> 2;
  const uint32_t total = n_tokens * d4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += 4 * stride) {
    float4 v[4];
    uint32_t idx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      idx[k] = i0 + k * stride;
      if (idx[k] < total) {
        const uint32_t t = idx[k] / d4, c = idx[k] - t * d4;
        v[k] = __ldg(reinterpret_cast<const float4*>(rows + (size_t)__ldg(sample_of + t) * dim) + c);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (idx[k] < total) __stcs(reinterpret_cast<float4*>(out) + idx[k], v[k]);
  }
}

// deterministic f64 sum of x[0, n): per-block partials (4 loads in flight per
// thread); the last block to finish combines them in a fixed tree order
__global__ void __launch_bounds__(256) k_sum_partials(const float* __restrict__ x, uint64_t n,
                                                      double* __restrict__ part, unsigned int* __restrict__ done,
                                                      double* __restrict__ out) {
  __shared__ double w[256];
  __shared__ bool last;
  double acc = 0.0;
  const uint64_t n4 = n >> 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      v[k] = i0 + k * stride < n4 ? __ldg(reinterpret_cast<const float4*>(x) + i0 + k * stride)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += (double)v[k].x + (double)v[k].y + (double)v[k].z + (double)v[k].w;
  }
  if (blockIdx.x == 0)
    for (uint64_t i = (n4 << 2) + threadIdx.x; i < n; i += blockDim.x) acc += (double)x[i];
  w[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < (unsigned)o) w[threadIdx.x] += w[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = w[0];
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a2 = 0.0;
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) a2 += __ldcg(part + b);
  w[threadIdx.x] = a2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < (unsigned)o) w[threadIdx.x] += w[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = w[0];
    *done = 0;
  }
}

}  // namespace
int generate(uint64_t seed, uint64_t num_sequences, double mean_len, uint64_t max_len, double sigma,
             double zipf, uint32_t tables, const uint64_t* vocab, uint64_t* lengths, uint64_t* ids,
             uint64_t max_tokens, uint64_t* n_tokens, double* labels);
}  // namespace rs

extern "C" {

int rs_workload_generate(uint64_t seed, uint64_t num_sequences, double mean_len, uint64_t max_len,
                         double sigma, double zipf, uint32_t tables, const uint64_t* vocab,
                         uint64_t* lengths, uint64_t* ids, uint64_t max_tokens,
                         uint64_t* n_tokens) {
  return rs::generate(seed, num_sequences, mean_len, max_len, sigma, zipf, tables, vocab, lengths, ids,
                      max_tokens, n_tokens, nullptr);
}

}  // extern "C"

namespace rs {
int generate(uint64_t seed, uint64_t num_sequences, double mean_len, uint64_t max_len, double sigma,
             double zipf, uint32_t tables, const uint64_t* vocab, uint64_t* lengths, uint64_t* ids,
             uint64_t max_tokens, uint64_t* n_tokens, double* labels) {
  if (!(sigma > 0) || max_len < 2 || !(mean_len > 1.0) || mean_len >= (double)max_len ||
      tables == 0 || zipf < 0)
    return fail(RS_ERR_CONFIG, "workload: bad length/zipf config");
  double lo = -20.0, hi = std::log((double)max_len) + 10.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (trunc_mean(mid, sigma, (double)max_len) < mean_len)
      lo = mid;
    else
      hi = mid;
  }
  const double mu = 0.5 * (lo + hi);
  std::vector<std::vector<double>> cdf(tables);
  for (uint32_t t = 0; t < tables; ++t) {
    if (vocab[t] < 1) return fail(RS_ERR_CONFIG, "zipf vocab must be >= 1");
    cdf[t].resize(vocab[t]);
    double total = 0;
    for (uint64_t r = 0; r < vocab[t]; ++r) {
      total += std::pow(static_cast<double>(r + 1), -zipf);
      cdf[t][r] = total;
    }
    for (double& c : cdf[t]) c /= total;
    cdf[t].back() = 1.0;
  }
  uint32_t kb = 0;
  for (uint64_t x = tables; x; x >>= 1) ++kb;
  kb = std::max<uint32_t>(kb, 1);
  Rng rng(seed);
  uint64_t tok = 0;
  for (uint64_t sid = 1; sid <= num_sequences; ++sid) {
    uint64_t len;
    for (;;) {
      const double u1 = rng.unit_pos();
      const double u2 = rng.unit();
      const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
      const double x = std::exp(mu + sigma * z);
      if (x > static_cast<double>(max_len)) continue;
      const auto nn = static_cast<uint64_t>(std::llround(x));
      len = std::max<uint64_t>(1, std::min(nn, max_len));
      break;
    }
    const double label = rng.unit();
    if (labels) labels[sid - 1] = label;
    lengths[sid - 1] = len;
    for (uint64_t t = 0; t < len; ++t) {
      const uint32_t ord = static_cast<uint32_t>(1 + t % tables);
      const double u = rng.unit();
      const auto it = std::upper_bound(cdf[ord - 1].begin(), cdf[ord - 1].end(), u);
      const uint64_t raw =
          std::min<uint64_t>(it - cdf[ord - 1].begin(), cdf[ord - 1].size() - 1);
      if (tok >= max_tokens) return fail(RS_ERR_CONFIG, "workload: max_tokens too small");
      ids[tok++] = (static_cast<uint64_t>(ord) << (63 - kb)) | raw;
    }
  }
  *n_tokens = tok;
  return RS_OK;
}
}  // namespace rs

extern "C" {

// generate_workload_file (workload.cpp:280-315): the reference's text format
// -- a "# recsparse-workload v1" header, then one line per sequence:
// sample id, TAB, label (%.4f), TAB, the catalog-tagged ids space-separated.
int rs_workload_write(const char* path, uint64_t seed, uint64_t num_sequences, double mean_len,
                      uint64_t max_len, double sigma, double zipf, uint32_t tables, const uint64_t* vocab) {
  using namespace rs;
  if (!path) return fail(RS_ERR_CONFIG, "rs_workload_write: null path");
  std::vector<uint64_t> lengths(num_sequences);
  std::vector<double> labels(num_sequences);
  std::vector<uint64_t> ids(std::max<uint64_t>(1, num_sequences * max_len));
  uint64_t n = 0;
  int st = generate(seed, num_sequences, mean_len, max_len, sigma, zipf, tables, vocab, lengths.data(),
                    ids.data(), ids.size(), &n, labels.data());
  if (st) return st;
  FILE* f = std::fopen(path, "w");
  if (!f) return fail(RS_ERR_IO, std::string("cannot open workload file for writing: ") + path);
  bool ok = std::fprintf(f, "# recsparse-workload v1 seed=%llu sequences=%llu tables=%u\n",
                         (unsigned long long)seed, (unsigned long long)num_sequences, tables) > 0;
  uint64_t tok = 0;
  for (uint64_t s = 0; ok && s < num_sequences; ++s) {
    ok = std::fprintf(f, "%llu\t%.4f\t", (unsigned long long)(s + 1), labels[s]) > 0;
    for (uint64_t t = 0; ok && t < lengths[s]; ++t)
      ok = std::fprintf(f, t ? " %llu" : "%llu", (unsigned long long)ids[tok++]) > 0;
    ok = ok && std::fputc('\n', f) != EOF;
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(RS_ERR_IO, std::string("write failed: ") + path);
  return RS_OK;
}

// read_workload_file (workload.cpp:317-339): blank and '#' lines skipped;
// each record is "sample_id label id id ..."; a record without an id or
// without both leading fields is an IoError naming path:line.  Pass zero
// capacities to get the counts only.
int rs_workload_read(const char* path, uint64_t cap_seq, uint64_t cap_tok, uint64_t* sample_ids,
                     double* labels, uint64_t* lengths, uint64_t* ids, uint64_t* n_seq, uint64_t* n_tok) {
  using namespace rs;
  if (!path || !n_seq || !n_tok) return fail(RS_ERR_CONFIG, "rs_workload_read: null argument");
  std::ifstream is(path);
  if (!is) return fail(RS_ERR_IO, std::string("cannot open workload file: ") + path);
  std::string line;
  uint64_t lineno = 0, s = 0, tok = 0;
  const bool fill = cap_seq && cap_tok;
  while (std::getline(is, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    uint64_t sid = 0;
    double label = 0;
    if (!(ls >> sid >> label))
      return fail(RS_ERR_IO, std::string(path) + ":" + std::to_string(lineno) + ": bad record");
    uint64_t id, len = 0;
    while (ls >> id) {
      if (fill && tok < cap_tok) ids[tok] = id;
      ++tok;
      ++len;
    }
    if (len == 0) return fail(RS_ERR_IO, std::string(path) + ":" + std::to_string(lineno) + ": empty sequence");
    if (fill && s < cap_seq) {
      if (sample_ids) sample_ids[s] = sid;
      if (labels) labels[s] = label;
      if (lengths) lengths[s] = len;
    }
    ++s;
  }
  *n_seq = s;
  *n_tok = tok;
  if (fill && (s > cap_seq || tok > cap_tok)) return fail(RS_ERR_CONFIG, "rs_workload_read: buffers too small");
  return RS_OK;
}

int rs_pseudo_grads(const uint64_t* d_sample_of_token, uint64_t n, uint64_t step, uint32_t dim,
                    float* d_out, void* stream) {
  using namespace rs;
  if (n == 0) return RS_OK;
  k_pseudo_grads<<<grid_for(n * dim, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      d_sample_of_token, n, step, dim, d_out);
  RS_LAUNCH_CHECK("k_pseudo_grads");
  return RS_OK;
}

// The same gradients for a jagged batch given by its sequence lengths: one
// row per sample (sample ids first_sample_id + s), broadcast to its tokens.
int rs_pseudo_grads_jagged(const uint64_t* d_lengths, uint64_t n_seq, uint64_t first_sample_id,
                           uint64_t step, uint32_t dim, uint64_t n_tokens, float* d_out,
                           void* stream) {
  using namespace rs;
  if (n_tokens == 0 || n_seq == 0) return RS_OK;
  if (dim % 4) return fail(RS_ERR_CONFIG, "rs_pseudo_grads_jagged: dim % 4 != 0");
  cudaStream_t s = (cudaStream_t)stream;
  if (n_tokens * (uint64_t)dim >= (1ull << 32) || n_seq >= (1ull << 32))
    return fail(RS_ERR_CONFIG, "rs_pseudo_grads_jagged: batch too large");
  // per-device scratch kept across calls (one caller stream per device at a
  // time; grows only)
  struct Scratch {
    uint64_t* offs = nullptr;
    float* rows = nullptr;
    uint32_t* sample_of = nullptr;
    uint64_t cap_seq = 0, cap_rows = 0, cap_tok = 0;
  };
  constexpr int kMaxDev = 64;
  static Scratch scr[kMaxDev];
  int dev = 0;
  RS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) return fail(RS_ERR_CONFIG, "rs_pseudo_grads_jagged: device ordinal out of range");
  Scratch& x = scr[dev];
  if (x.cap_tok < n_tokens) {
    if (x.sample_of) RS_CUDA(cudaFree(x.sample_of));
    RS_CUDA(cudaMalloc(&x.sample_of, n_tokens * 4));
    x.cap_tok = n_tokens;
  }
  if (x.cap_seq < n_seq + 1) {
    if (x.offs) RS_CUDA(cudaFree(x.offs));
    RS_CUDA(cudaMalloc(&x.offs, (n_seq + 1) * 8));
    x.cap_seq = n_seq + 1;
  }
  if (x.cap_rows < n_seq * dim) {
    if (x.rows) RS_CUDA(cudaFree(x.rows));
    RS_CUDA(cudaMalloc(&x.rows, n_seq * dim * 4));
    x.cap_rows = n_seq * dim;
  }
  uint64_t* offs = x.offs;
  float* rows = x.rows;
  uint32_t* sample_of = x.sample_of;
  k_seq_offsets<<<1, 1024, 0, s>>>(d_lengths, n_seq, offs);
  RS_LAUNCH_CHECK("k_seq_offsets");
  k_sample_rows<<<grid_for(n_seq * dim, 256, 148 * 8), 256, 0, s>>>(n_seq, first_sample_id, step, dim, rows);
  RS_LAUNCH_CHECK("k_sample_rows");
  k_fill_sample<<<(unsigned)n_seq, 256, 0, s>>>(offs, sample_of);
  RS_LAUNCH_CHECK("k_fill_sample");
  k_broadcast_rows<<<grid_for(n_tokens * dim / 16, 256, 148 * 8), 256, 0, s>>>(sample_of, rows, dim,
                                                                            (uint32_t)n_tokens, d_out);
  RS_LAUNCH_CHECK("k_broadcast_rows");
  return RS_OK;
}

// The same from the batch's token offsets (offs[n_seq + 1], device): one
// kernel, one block per sample.
int rs_pseudo_grads_offsets(const uint64_t* d_offsets, uint64_t n_seq, uint64_t first_sample_id,
                            uint64_t step, uint32_t dim, float* d_out, void* stream) {
  using namespace rs;
  if (n_seq == 0) return RS_OK;
  if (dim % 4 || dim > 4096) return fail(RS_ERR_CONFIG, "rs_pseudo_grads_offsets: dim % 4 != 0 or > 4096");
  k_jagged_grads<<<(unsigned)n_seq, 256, dim * 4, (cudaStream_t)stream>>>(d_offsets, first_sample_id, step, dim,
                                                                          d_out);
  RS_LAUNCH_CHECK("k_jagged_grads");
  return RS_OK;
}

// From a host-built work list of (sample, token range) chunks (device copy):
// balanced blocks, one kernel.
int rs_pseudo_grads_chunks(const void* d_work, uint32_t n_chunks, uint64_t first_sample_id, uint64_t step,
                           uint32_t dim, float* d_out, void* stream) {
  using namespace rs;
  if (n_chunks == 0) return RS_OK;
  if (dim % 4 || dim > 4096) return fail(RS_ERR_CONFIG, "rs_pseudo_grads_chunks: dim % 4 != 0 or > 4096");
  k_jagged_grads_chunks<<<n_chunks, 256, dim * 4, (cudaStream_t)stream>>>(
      static_cast<const GradChunk*>(d_work), first_sample_id, step, dim, d_out);
  RS_LAUNCH_CHECK("k_jagged_grads_chunks");
  return RS_OK;
}

// run_workload's emb_checksum (workload.cpp:547-549) of a step's outputs, in
// f64, deterministic (fixed block partition and order).
int rs_checksum(const float* d_x, uint64_t n, double* d_out, void* stream) {
  using namespace rs;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned nb = 148 * 4;
  // per-device partials, kept across calls (one stream per device at a time)
  constexpr int kMaxDev = 64;
  static double* part[kMaxDev] = {};
  static unsigned int* done[kMaxDev] = {};
  int dev = 0;
  RS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) return fail(RS_ERR_CONFIG, "rs_checksum: device ordinal out of range");
  if (!part[dev]) {
    RS_CUDA(cudaMalloc(&part[dev], nb * 8));
    RS_CUDA(cudaMalloc(&done[dev], 4));
    RS_CUDA(cudaMemset(done[dev], 0, 4));
  }
  k_sum_partials<<<nb, 256, 0, s>>>(d_x, n, part[dev], done[dev], d_out);
  RS_LAUNCH_CHECK("k_sum_partials");
  return RS_OK;
}

}  // extern "C"

namespace rs {
namespace {
// encode_tagged_id (merge_registry.cpp:23-33): (index << (63-k)) | raw; raw
// ids wider than the payload set a per-launch overflow flag.
__global__ void k_encode(const uint64_t* __restrict__ raw, uint64_t n, uint32_t shift,
                         uint64_t tag, uint64_t* __restrict__ out, unsigned int* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = raw[i];
    if (x >> shift) atomicOr(bad, 1u);
    out[i] = tag | x;
  }
}
}  // namespace
}  // namespace rs

extern "C" int rs_encode_ids(const uint64_t* d_raw, uint64_t n, uint32_t k_bits,
                             uint32_t table_index, uint32_t index_limit, uint64_t* d_out,
                             void* stream) {
  using namespace rs;
  if (table_index > index_limit)
    return fail(RS_ERR_RANGE, "encode_tagged_id: table index out of range");
  if (k_bits < 1 || k_bits > 62) return fail(RS_ERR_CONFIG, "encode_tagged_id: bad k_bits");
  if (n == 0) return RS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned int* bad = nullptr;
  RS_CUDA(cudaMallocAsync(&bad, 4, s));
  RS_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  const uint32_t shift = 63 - k_bits;
  k_encode<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(d_raw, n, shift,
                                                      (uint64_t)table_index << shift, d_out, bad);
  RS_LAUNCH_CHECK("k_encode");
  unsigned int h = 0;
  RS_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaStreamSynchronize(s));
  RS_CUDA(cudaFree(bad));
  if (h) return fail(RS_ERR_RANGE, "encode_tagged_id: raw id exceeds payload width");
  return RS_OK;
}
