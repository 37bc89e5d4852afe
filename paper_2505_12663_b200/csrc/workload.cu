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

}  // namespace
}  // namespace rs

extern "C" {

int rs_workload_generate(uint64_t seed, uint64_t num_sequences, double mean_len, uint64_t max_len,
                         double sigma, double zipf, uint32_t tables, const uint64_t* vocab,
                         uint64_t* lengths, uint64_t* ids, uint64_t max_tokens,
                         uint64_t* n_tokens) {
  using namespace rs;
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
    (void)rng.unit();  // label
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

int rs_pseudo_grads(const uint64_t* d_sample_of_token, uint64_t n, uint64_t step, uint32_t dim,
                    float* d_out, void* stream) {
  using namespace rs;
  if (n == 0) return RS_OK;
  k_pseudo_grads<<<grid_for(n * dim, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      d_sample_of_token, n, step, dim, d_out);
  RS_LAUNCH_CHECK("k_pseudo_grads");
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
