// rs_internal.cuh -- shared device/host definitions of librsgpu (sm_100a).
//
// Layout decisions:
//  * key structure: 16-byte slots {u64 key, u32 row, u32 tick} in 8-slot
//    buckets (one 128-byte line).  A group of 8 lanes probes one bucket per
//    step -- the paper's grouped parallel probing (Eq. 5)
//    with G = 8 mapped onto lanes; bucket sequence b_t = b0 + t*S, S odd.
//  * embedding structure: SoA row pool (emb, opt_m, opt_v, step), rows never
//    move when the key structure expands (embed_table.cpp:267-285).
#pragma once
#include <cstdlib>
#include <unordered_set>
#include <mutex>

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/rsgpu.h"

namespace rs {

constexpr uint64_t kEmptyKey = ~0ull;      // slot never used
constexpr uint64_t kTombKey = ~0ull - 1;   // deleted slot (embed_table.hpp:47)
constexpr uint32_t kNoRow = 0xFFFFFFFFu;
constexpr int kBucket = 8;                 // slots per bucket == lanes per probe group
constexpr int kTile = 512;                 // tokens per reduce tile (dedup + reduce agree)
constexpr int kScanItems = 4;              // tokens per thread in scan kernels
constexpr int kScanThreads = 256;
constexpr int kScanTile = kScanItems * kScanThreads;

// MurmurHash3 fmix64 (hash.hpp:26-33).
__host__ __device__ __forceinline__ uint64_t hash64(uint64_t key) {
  key ^= key >> 33;
  key *= 0xff51afd7ed558ccdULL;
  key ^= key >> 33;
  key *= 0xc4ceb9fe1a85ec53ULL;
  key ^= key >> 33;
  return key;
}

struct __align__(16) Slot {
  unsigned long long key;
  uint32_t row;
  uint32_t tick;
};

// Device-resident table descriptor.  The pointer section is written by the
// host (cudaMemcpyAsync, stream ordered) when the key structure expands or the
// row pool grows; the counter section is updated only by kernels.  Kernels
// read pointers from here, so captured CUDA graphs survive reallocation.
struct TableDesc {
  Slot* slots;
  uint64_t nb_mask;    // buckets - 1 (buckets is a power of two >= 2)
  float* emb;          // [row_cap x dim]
  float* s1;           // Adam m (or null)
  float* s2;           // Adam v / Adagrad accumulator (or null)
  uint32_t* step;      // per-row optimizer step
  uint32_t* free_stack;
  uint64_t row_cap;
  uint32_t dim;
  uint32_t opt;
};

struct TableCounters {
  unsigned long long occupied;
  unsigned long long tombstones;
  unsigned long long fresh_next;   // rows carved from the pool so far
  unsigned long long free_n;       // rows on the LIFO free stack
  unsigned long long alloc_ctr;    // per-launch allocation tickets
  unsigned long long inserted;     // per-launch new keys
  unsigned long long reused;       // per-launch tombstones reused
  unsigned long long removed;      // per-launch removals
  unsigned int blocks_done;
  unsigned int error;              // sticky error bits (kErr*)
  unsigned int tick;               // batch tick (one per batch op)
  unsigned int special_row[2];     // rows of the keys equal to kEmptyKey / kTombKey
  unsigned int special_tick[2];
  unsigned int missing;            // per-launch count of missing keys (probe mode)
  unsigned int returned;           // per-launch rows handed back (lost duplicate inserts)
};

struct TableDev {
  TableDesc d;
  TableCounters c;
};

// Bounded tables: the stamp log (evict.cu).  Every batch op of the bounded
// ensure writes one record per key at log position base + (key index): the
// entry it stamped (or inserted) with the op's tick, or a placeholder (slot
// kNoLogSlot).  Ops are stream-ordered, so the log is tick-ordered; a record
// is live while its slot still holds that key with that tick.
constexpr uint32_t kNoLogSlot = 0xFFFFFFFFu;
struct LogRec {
  unsigned long long key;
  uint32_t slot;  // slot index, capacity + {0, 1} for the sentinel keys, or kNoLogSlot
  uint32_t tick;
};
struct LogCtl {
  unsigned long long tail, head;  // positions (monotone; index = pos & mask)
  unsigned long long op_base;     // base of the last probe op (the insert pass writes there too)
  unsigned long long sorted_end;  // [0, sorted_end): rebuilt, (tick, key)-sorted
};
struct LogArgs {
  LogRec* rec = nullptr;  // null: no log
  LogCtl* ctl = nullptr;
  uint64_t mask = 0;
  uint64_t cap = 0;       // table key slots (the sentinels' virtual slots follow)
  int probe = 0;          // 1: this launch opens the op (base = tail, advances tail)
};

enum : unsigned int {
  kErrRowPool = 1u,    // ran out of pre-sized rows (host bound violated)
  kErrTableFull = 2u,  // probe walked every bucket without a usable slot
  kErrCapacity = 4u,   // bounded table cannot hold the batch
};

// ---- PTX helpers ----------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
// Uniform shared-memory carveout for every kernel of the step (host side).
// Kernels whose launch configurations ask for different L1 / shared splits
// cannot share an SM: a block of the second waits until the SM drained the
// first's.  The step runs several latency-bound kernels side by side (the
// fast step's branches, the sharded step's owner and requester roles).
// RS_CARVEOUT=<percent> gives all of them the same split (experiment knob:
// measured no faster than the driver's per-kernel choice at 50 / 75, slower
// at 25 / 100 -- the default, -1, leaves the driver's choice).
inline void carve_ptr(const void* k) {
  static const int v = getenv("RS_CARVEOUT") ? atoi(getenv("RS_CARVEOUT")) : -1;
  if (v < 0) return;
  static std::mutex mu;
  static std::unordered_set<const void*> done;
  std::lock_guard<std::mutex> g(mu);
  if (done.insert(k).second) {
    (void)cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, v);
    (void)cudaGetLastError();
  }
}
template <typename... A>
inline void carve(void (*k)(A...)) {
  carve_ptr(reinterpret_cast<const void*>(k));
}

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while its same-stream predecessor drains; pdl_wait() (first statement of
// such a kernel, before any global access) blocks until the predecessor grid
// completed and its writes are visible.  Both are no-ops for plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- host-side error plumbing --------------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(uint64_t n = 1);
uint64_t launches();
bool debug_sync();  // RS_DEBUG_SYNC=1: synchronize after every launch (debugging only)

#define RS_CUDA(call)                                       \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess) return ::rs::cuda_fail(_e, #call); \
  } while (0)

#define RS_LAUNCH_CHECK(name)                               \
  do {                                                      \
    ::rs::count_launch();                                   \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e == cudaSuccess && ::rs::debug_sync()) _e = cudaDeviceSynchronize(); \
    if (_e != cudaSuccess) return ::rs::cuda_fail(_e, name); \
  } while (0)

// <<<g, b, smem, s>>> with the programmatic-serialization attribute when pdl
// (the kernel must start with pdl_wait()).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*k)(KArgs...), unsigned g, unsigned b, size_t smem,
                              cudaStream_t s, Args... args) {
  carve(k);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(b);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap = 148u * 32u) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// Device-side timeline (rs_workspace_trace, diagnostics): per (kernel, block)
// the first warp start and the last warp end (%globaltimer, ns).
constexpr uint32_t kTraceBlocks = 4096;
// slots: 0-5 the fast step's kernels (step_fast.cu), 6-15 the sharded
// step's requester gather / signal and owner kernels (dist.cu)
constexpr uint32_t kTraceSlots = 16;
// phase mark of a block (thread 0): kernel slot kid, end time = now
__device__ __forceinline__ void trace_mark(unsigned long long* base, uint32_t kid) {
  if (base && threadIdx.x == 0 && blockIdx.x < kTraceBlocks) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned long long* p = base + ((size_t)kid * kTraceBlocks + blockIdx.x) * 2;
    atomicMin(p, t);
    atomicMax(p + 1, t);
  }
}
struct WarpTrace {
  unsigned long long* p = nullptr;
  __device__ __forceinline__ WarpTrace(unsigned long long* base, uint32_t kid) {
    if (base && (threadIdx.x & 31) == 0 && blockIdx.x < kTraceBlocks) {
      p = base + ((size_t)kid * kTraceBlocks + blockIdx.x) * 2;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMin(p, t);
    }
  }
  __device__ __forceinline__ ~WarpTrace() {
    if (p) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(p + 1, t);
    }
  }
};

}  // namespace rs
