// scratch_dev.cuh -- the per-call dedup scratch (rs_scratch, rs_host.hpp):
// open-addressed id -> slot map with per-slot counters, shared by the step
// kernels (step.cu) and the sharded owner kernels (dist.cu).
#pragma once

#include "rs_host.hpp"

namespace rs {
namespace sdev {

// Device view of one scratch set (see rs_scratch in rs_host.hpp).
struct SetDev {
  unsigned long long* skey;
  uint32_t* sfirstx;  // exact dedup: ~first position; fast step: occurrence count
  uint32_t* sntile;   // tiles containing the id
  uint32_t* suidx;    // unique index of the slot
  uint32_t* srow;     // table row of the slot
  uint32_t* u_slot;   // slot of each unique id (= the set's dirty list)
  uint32_t* cnt;      // [0] number of unique ids in the set
  uint64_t smask;     // capacity - 1
  uint64_t spare;     // slot of the id equal to the empty sentinel
};

// ---------------------------------------------------------------------------
// Scratch cleaning: reset the slots listed by a set's dirty list.
__device__ __forceinline__ void clean_set(const SetDev& c, uint64_t gtid, uint64_t gthreads) {
  const uint32_t prev = *c.cnt;
  for (uint64_t i = gtid; i <= prev; i += gthreads) {
    const uint64_t s = i < prev ? c.u_slot[i] : c.spare;
    c.skey[s] = kEmptyKey;
    c.sfirstx[s] = 0;
    c.sntile[s] = 0;
  }
}

// Probe the global scratch for `id` (linear probing on the low hash bits),
// claiming an empty slot.  Returns the slot; *fresh = slot newly claimed.
// first0: the key at slot h & smask if the caller already read it (an
// early, possibly stale read -- keys never change within a step, so a
// matching or foreign key is final and an empty one is re-checked by the CAS).
__device__ __forceinline__ uint64_t scratch_insert(const SetDev& S, uint64_t id, uint64_t h,
                                                   bool* fresh, const unsigned long long* first0 = nullptr) {
  if (id == kEmptyKey) {
    *fresh = atomicCAS(&S.skey[S.spare], kEmptyKey, 0ull) == kEmptyKey;
    return S.spare;
  }
  uint64_t gs = h & S.smask;
  bool use0 = first0 != nullptr;
  for (;;) {
    // plain L2 read first: ids repeated across tiles find their slot without
    // an atomic (hot ids would otherwise serialize every tile on one address)
    const unsigned long long cur = use0 ? *first0 : __ldcg(&S.skey[gs]);
    use0 = false;
    if (cur == id) {
      *fresh = false;
      return gs;
    }
    if (cur != kEmptyKey) {
      gs = (gs + 1) & S.smask;
      continue;
    }
    const unsigned long long prev = atomicCAS(&S.skey[gs], kEmptyKey, (unsigned long long)id);
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

inline SetDev set_dev(const rs_workspace* ws, int k) {
  const rs_scratch& x = ws->set[k];
  SetDev s;
  s.skey = x.skey;
  s.sfirstx = x.sfirstx;
  s.sntile = x.sntile;
  s.suidx = x.suidx;
  s.srow = x.srow;
  s.u_slot = x.u_slot;
  s.cnt = x.cnt;
  s.smask = ws->S - 1;
  s.spare = ws->S;
  return s;
}

}  // namespace sdev
}  // namespace rs
