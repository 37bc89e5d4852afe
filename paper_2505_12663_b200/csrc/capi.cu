// capi.cpp -- meta entry points of the C-ABI (status strings, last error,
// launch accounting, id encoding).  No exceptions cross the boundary.
#include <cuda_runtime.h>

#include <atomic>
#include <string>

#include "rs_internal.cuh"

namespace rs {
namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return RS_ERR_CUDA;
}
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }
bool debug_sync() {
  static const bool on = [] {
    const char* e = getenv("RS_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
}  // namespace rs

extern "C" {

int rs_abi_version(void) { return RS_ABI_VERSION; }

const char* rs_status_string(int status) {
  switch (status) {
    case RS_OK: return "ok";
    case RS_ERR_CONFIG: return "config error";
    case RS_ERR_INVARIANT: return "invariant violated";
    case RS_ERR_IO: return "io error";
    case RS_ERR_CUDA: return "cuda error";
    case RS_ERR_CAPACITY: return "capacity exceeded";
    case RS_ERR_RANGE: return "id encoding out of range";
  }
  return "unknown status";
}

const char* rs_last_error(void) { return rs::g_last_error.c_str(); }

uint64_t rs_kernel_launches(void) { return rs::launches(); }

// Device buffers and copies for C / C++ callers without a CUDA runtime of
// their own (the C++ shim, include/recsparse_gpu): synchronous, legacy stream.
int rs_buffer_alloc(uint64_t bytes, void** out) {
  if (!out) return rs::fail(RS_ERR_CONFIG, "rs_buffer_alloc: null out");
  *out = nullptr;
  RS_CUDA(cudaMalloc(out, bytes ? bytes : 16));
  return RS_OK;
}
int rs_buffer_free(void* d) {
  if (d) RS_CUDA(cudaFree(d));
  return RS_OK;
}
int rs_copy_to_device(void* d, const void* h, uint64_t bytes) {
  if (bytes) RS_CUDA(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  return RS_OK;
}
int rs_copy_to_host(void* h, const void* d, uint64_t bytes) {
  if (bytes) RS_CUDA(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost));
  return RS_OK;
}

}  // extern "C"
