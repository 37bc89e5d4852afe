// feed.cu -- one run_workload step fed from host memory (the end-to-end path).
//
// Reference: run_workload's step body (workload.cpp:506-581): the batch's
// token ids arrive from the data loader; the per-token gradients are
// pseudo_sparse_grad(sample id, step) (workload.cpp:348-355, a pure hash --
// generated on the device here); distributed_lookup + accumulate + apply;
// the step's stats accumulate emb_checksum += sum of the outputs
// (workload.cpp:547-549).  rs_feeder_step does exactly that from pinned host
// buffers with everything asynchronous: the H2D copies of step k+1 run on a
// copy stream while step k computes (two device buffer sets, reuse ordered by
// events), and only the 8-byte checksum travels back.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstdio>
#include <chrono>

#include <algorithm>

#include "rs_host.hpp"

using namespace rs;

static constexpr uint64_t kChunkTok = 512;  // tokens per block of the gradient kernel

struct rs_feeder {
  uint64_t max_tokens = 0, max_seqs = 0;
  double wait_us = 0;  // RS_HOST_PROF: host time blocked on the staging buffer
  uint32_t dim = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t in_free[2] = {}, landed[2] = {};
  uint64_t* ids[2] = {};
  uint64_t* offs[2] = {};       // device token offsets of the batch
  uint64_t* h_offs[2] = {};     // pinned host staging of the offsets
  uint32_t* chunks[2] = {};     // device work list of the gradient kernel
  uint32_t* h_chunks[2] = {};   // pinned staging: (sample, t0, t1) triples
  uint32_t n_chunks[2] = {0, 0};
  float* grads[2] = {};
  float* out[2] = {};
  double* sum[2] = {};
  uint64_t k = 0;
};

extern "C" {

int rs_feeder_create(uint64_t max_tokens, uint64_t max_seqs, uint32_t dim, rs_feeder** out) {
  if (!out || !max_tokens || !max_seqs || !dim) return fail(RS_ERR_CONFIG, "rs_feeder_create: bad arguments");
  auto* f = new rs_feeder();
  f->max_tokens = max_tokens;
  f->max_seqs = max_seqs;
  f->dim = dim;
  bool ok = cudaStreamCreateWithFlags(&f->copy, cudaStreamNonBlocking) == cudaSuccess;
  for (int b = 0; b < 2 && ok; ++b) {
    ok = cudaEventCreateWithFlags(&f->in_free[b], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&f->landed[b], cudaEventDisableTiming) == cudaSuccess &&
         cudaMalloc(&f->ids[b], max_tokens * 8) == cudaSuccess &&
         cudaMalloc(&f->offs[b], (max_seqs + 1) * 8) == cudaSuccess &&
         cudaMallocHost(&f->h_offs[b], (max_seqs + 1) * 8) == cudaSuccess &&
         cudaMalloc(&f->chunks[b], (max_seqs + max_tokens / kChunkTok + 1) * 12) == cudaSuccess &&
         cudaMallocHost(&f->h_chunks[b], (max_seqs + max_tokens / kChunkTok + 1) * 12) == cudaSuccess &&
         cudaMalloc(&f->grads[b], max_tokens * dim * 4) == cudaSuccess &&
         cudaMalloc(&f->out[b], max_tokens * dim * 4) == cudaSuccess &&
         cudaMalloc(&f->sum[b], 8) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    rs_feeder_destroy(f);
    return fail(RS_ERR_CUDA, "rs_feeder_create: allocation failed");
  }
  *out = f;
  return RS_OK;
}

int rs_feeder_destroy(rs_feeder* f) {
  if (!f) return RS_OK;
  cudaDeviceSynchronize();
  for (int b = 0; b < 2; ++b) {
    if (f->in_free[b]) cudaEventDestroy(f->in_free[b]);
    if (f->landed[b]) cudaEventDestroy(f->landed[b]);
    void* ps[] = {f->ids[b], f->offs[b], f->grads[b], f->out[b], f->sum[b], f->chunks[b]};
    for (void* p : ps)
      if (p) cudaFree(p);
    if (f->h_offs[b]) cudaFreeHost(f->h_offs[b]);
    if (f->h_chunks[b]) cudaFreeHost(f->h_chunks[b]);
  }
  if (f->copy) cudaStreamDestroy(f->copy);
  delete f;
  return RS_OK;
}

// Device buffers of the current set (the gathered rows of the last step).
float* rs_feeder_out(rs_feeder* f, int which) { return f ? f->out[which & 1] : nullptr; }

static int feeder_stage(rs_feeder* f, const uint64_t* h_ids, uint64_t n, const uint64_t* h_lengths,
                        uint64_t n_seq, uint64_t first_sample_id, uint64_t step, cudaStream_t s, int* set) {
  if (n > f->max_tokens || n_seq > f->max_seqs)
    return fail(RS_ERR_CONFIG, "rs_feeder_step: batch exceeds the feeder's capacity");
  const int b = (int)(f->k & 1);
  if (f->k < 2) RS_CUDA(cudaEventRecord(f->in_free[b], s));  // first use: free now
  RS_CUDA(cudaStreamWaitEvent(f->copy, f->in_free[b], 0));
  // the loader's lengths -> token offsets (host, a few thousand adds); the
  // staging buffer of this set is free once its previous copy completed
  {
    static const bool prof = getenv("RS_HOST_PROF") && getenv("RS_HOST_PROF")[0] == '1';
    const auto w0 = std::chrono::steady_clock::now();
    RS_CUDA(cudaEventSynchronize(f->landed[b]));
    if (prof) f->wait_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w0).count();
  }
  {  // validate before touching the pinned staging buffers
    uint64_t tot = 0, chunks = 0;
    for (uint64_t i = 0; i < n_seq; ++i) {
      tot += h_lengths[i];
      chunks += (h_lengths[i] + kChunkTok - 1) / kChunkTok;
    }
    if (tot != n) return fail(RS_ERR_CONFIG, "rs_feeder_step: sum of lengths != number of ids");
    if (chunks > f->max_seqs + f->max_tokens / kChunkTok + 1) return fail(RS_ERR_CONFIG, "rs_feeder_step: batch exceeds the feeder's capacity");
  }
  uint64_t run = 0;
  uint32_t nc = 0;
  for (uint64_t i = 0; i < n_seq; ++i) {
    f->h_offs[b][i] = run;
    // balanced work list of the gradient kernel: <= kChunkTok tokens per block
    for (uint64_t t0 = run; t0 < run + h_lengths[i]; t0 += kChunkTok) {
      f->h_chunks[b][3 * nc] = (uint32_t)i;
      f->h_chunks[b][3 * nc + 1] = (uint32_t)t0;
      f->h_chunks[b][3 * nc + 2] = (uint32_t)std::min<uint64_t>(t0 + kChunkTok, run + h_lengths[i]);
      ++nc;
    }
    run += h_lengths[i];
  }
  f->h_offs[b][n_seq] = run;
  f->n_chunks[b] = nc;
  if (run != n) return fail(RS_ERR_CONFIG, "rs_feeder_step: sum of lengths != number of ids");
  RS_CUDA(cudaMemcpyAsync(f->ids[b], h_ids, n * 8, cudaMemcpyHostToDevice, f->copy));
  RS_CUDA(cudaMemcpyAsync(f->chunks[b], f->h_chunks[b], (size_t)nc * 12, cudaMemcpyHostToDevice, f->copy));
  // the batch's gradients are data of the batch: generated on the copy stream
  // too, so they overlap the previous step instead of preceding this one
  int st = rs_pseudo_grads_chunks(f->chunks[b], nc, first_sample_id, step, f->dim, f->grads[b], f->copy);
  if (st) return st;
  RS_CUDA(cudaEventRecord(f->landed[b], f->copy));
  RS_CUDA(cudaStreamWaitEvent(s, f->landed[b], 0));
  *set = b;
  return RS_OK;
}

// Where the step's checksum goes: straight into h_checksum when it is mapped
// pinned memory (UVA: cudaMallocHost / pinned torch tensors) -- the kernel's
// 8-byte store crosses PCIe, no copy on the stream -- else the device slot
// of the buffer set, copied back by feeder_finish.
static double* checksum_dst(rs_feeder* f, int b, double* h_checksum, bool* direct) {
  *direct = false;
  if (!h_checksum) return f->sum[b];
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, h_checksum) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
      pa.devicePointer) {
    *direct = true;
    return static_cast<double*>(pa.devicePointer);
  }
  (void)cudaGetLastError();
  return f->sum[b];
}

static int feeder_finish(rs_feeder* f, int b, uint64_t n, double* h_checksum, cudaStream_t s,
                         bool summed, double* dst, bool direct) {
  int st = summed ? RS_OK : rs_checksum(f->out[b], n * f->dim, dst, s);
  if (st) return st;
  RS_CUDA(cudaEventRecord(f->in_free[b], s));
  if (h_checksum && !direct) RS_CUDA(cudaMemcpyAsync(h_checksum, dst, 8, cudaMemcpyDeviceToHost, s));
  f->k++;
  return RS_OK;
}

// One training step from host memory on a single shard (rs_step).  h_ids /
// h_lengths / h_checksum should be pinned; nothing synchronizes.
int rs_feeder_step(rs_feeder* f, rs_workspace* ws, rs_table* t, const uint64_t* h_ids, uint64_t n,
                   const uint64_t* h_lengths, uint64_t n_seq, uint64_t first_sample_id, uint64_t step,
                   const rs_optimizer_params* opt, double* h_checksum, void* stream) {
  if (!f || !ws || !t) return fail(RS_ERR_CONFIG, "rs_feeder_step: null handle");
  if (t->desc.dim != f->dim) return fail(RS_ERR_CONFIG, "rs_feeder_step: table dim != feeder dim");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  static const bool prof = getenv("RS_HOST_PROF") && getenv("RS_HOST_PROF")[0] == '1';
  static double acc[4] = {0, 0, 0, 0};
  static uint64_t calls = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  const auto t0 = now();
  int b = 0;
  int st = feeder_stage(f, h_ids, n, h_lengths, n_seq, first_sample_id, step, s, &b);
  const auto t1 = now();
  bool direct = false;
  double* dst = checksum_dst(f, b, h_checksum, &direct);
  if (!st) st = rs_step_checksum(ws, t, f->ids[b], n, f->grads[b], f->out[b], opt, dst, stream);
  const auto t2 = now();
  if (!st) st = feeder_finish(f, b, n, h_checksum, s, true, dst, direct);
  if (prof) {  // host time by section (diagnostics): stage (incl. the staging-buffer wait), step, finish
    const auto t3 = now();
    acc[0] += us(t0, t1);
    acc[1] += us(t1, t2);
    acc[2] += us(t2, t3);
    if (++calls % 16 == 0) {
      fprintf(stderr, "rs_feeder_step host us/call: stage %.1f (of which waiting %.1f) step %.1f finish %.1f\n",
              acc[0] / 16, f->wait_us / 16, acc[1] / 16, acc[2] / 16);
      f->wait_us = 0;
      acc[0] = acc[1] = acc[2] = 0;
    }
  }
  return st;
}

// The same for this rank of a row-sharded table (rs_dist_step).
int rs_feeder_dist_step(rs_feeder* f, rs_comm* c, rs_table* shard, const uint64_t* h_ids, uint64_t n,
                        const uint64_t* h_lengths, uint64_t n_seq, uint64_t first_sample_id, uint64_t step,
                        const rs_optimizer_params* opt, double* h_checksum, void* stream) {
  if (!f || !c || !shard) return fail(RS_ERR_CONFIG, "rs_feeder_dist_step: null handle");
  if (shard->desc.dim != f->dim) return fail(RS_ERR_CONFIG, "rs_feeder_dist_step: table dim != feeder dim");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int b = 0;
  int st = feeder_stage(f, h_ids, n, h_lengths, n_seq, first_sample_id, step, s, &b);
  bool direct = false;
  double* dst = checksum_dst(f, b, h_checksum, &direct);
  if (!st) st = rs_dist_step_checksum(c, shard, f->ids[b], n, f->grads[b], f->out[b], opt, dst, stream);
  if (!st) st = feeder_finish(f, b, n, h_checksum, s, true, dst, direct);
  return st;
}

}  // extern "C"
