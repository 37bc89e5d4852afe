// opt_dev.cuh -- the sparse optimizers and lane-distributed row vectors.
//
// FP64 math with explicit round-to-nearest intrinsics so nvcc cannot contract
// into FMA (the reference is compiled -ffp-contract=off):
//   Adam     sparse_update.cpp:22-37 (bias corrections from a host-libm table)
//   Adagrad  frozen restatement (oracle.c:or_adagrad_row)
// A row of D floats is held by a warp as acc[c][j], element (c*32+lane)*VEC+j.
#pragma once

#include "rs_internal.cuh"

namespace rs {
namespace odev {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// Optimizers: FP64 math with explicit round-to-nearest intrinsics so nvcc
// cannot contract into FMA (the reference is compiled -ffp-contract=off).
struct OptArgs {
  uint32_t kind;
  double lr, b1, b2, eps, omb1, omb2;
  const double* bc;  // [2 x bc_len]: 1 - b1^k, 1 - b2^k (host libm)
  uint64_t bc_len;
};

__device__ __forceinline__ void adagrad_elem(float& w, float& a, float gf, const OptArgs& o) {
  const double g = (double)gf;
  const double an = __dadd_rn((double)a, __dmul_rn(g, g));
  a = __double2float_rn(an);
  w = __double2float_rn(
      __dsub_rn((double)w, __ddiv_rn(__dmul_rn(o.lr, g), __dadd_rn(__dsqrt_rn(an), o.eps))));
}
__device__ __forceinline__ void adam_elem(float& w, float& m, float& v, float gf, double bc1,
                                          double bc2, const OptArgs& o) {
  const double g = (double)gf;
  const double me = __dadd_rn(__dmul_rn(o.b1, (double)m), __dmul_rn(o.omb1, g));
  const double ve = __dadd_rn(__dmul_rn(o.b2, (double)v), __dmul_rn(__dmul_rn(o.omb2, g), g));
  m = __double2float_rn(me);
  v = __double2float_rn(ve);
  const double mh = __ddiv_rn(me, bc1);
  const double vh = __ddiv_rn(ve, bc2);
  w = __double2float_rn(
      __dsub_rn((double)w, __ddiv_rn(__dmul_rn(o.lr, mh), __dadd_rn(__dsqrt_rn(vh), o.eps))));
}

// Applies one optimizer step to `row` with the lane-distributed gradient
// acc[c][j] for elements e = (c*32 + lane)*VEC + j.  Called by a full warp.
template <int VEC, int CH>
__device__ __forceinline__ void load_vec(const float* __restrict__ src, uint32_t D,
                                         float (&x)[CH][VEC], bool coherent);
template <int VEC, int CH>
__device__ __forceinline__ void store_vec(float* __restrict__ dst, uint32_t D,
                                          const float (&x)[CH][VEC]);

// Applies one optimizer step to `row` with the lane-distributed gradient
// acc[c][j] for elements e = (c*32 + lane)*VEC + j.  Called by a full warp.
// Row loads are issued before the step counter so their latencies overlap.
template <int VEC, int CH>
__device__ __forceinline__ void apply_row(const TableDesc& d, uint32_t row,
                                          const float (&acc)[CH][VEC], const OptArgs& o) {
  const unsigned lane = lane_id();
  const uint32_t D = d.dim;
  if (row == kNoRow) return;
  float* w = d.emb + (size_t)row * D;
  float* m = d.s1 ? d.s1 + (size_t)row * D : nullptr;
  float* v = d.s2 + (size_t)row * D;
  float wv[CH][VEC], mv[CH][VEC], vv[CH][VEC];
  load_vec<VEC, CH>(w, D, wv, false);
  load_vec<VEC, CH>(v, D, vv, false);
  if (m) load_vec<VEC, CH>(m, D, mv, false);
  uint32_t step = 0;
  if (lane == 0) {
    step = d.step[row] + 1;
    d.step[row] = step;
  }
  step = __shfl_sync(kFull, step, 0);
  double bc1 = 1.0, bc2 = 1.0;
  if (o.kind == RS_OPT_ADAM) {
    if (step < o.bc_len) {
      bc1 = o.bc[step];
      bc2 = o.bc[o.bc_len + step];
    } else {
      bc1 = 1.0 - pow(o.b1, (double)step);
      bc2 = 1.0 - pow(o.b2, (double)step);
    }
  }
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      if (VEC == 1 && (uint32_t)(c * 32 + lane) >= D) continue;
      if (o.kind == RS_OPT_ADAM)
        adam_elem(wv[c][j], mv[c][j], vv[c][j], acc[c][j], bc1, bc2, o);
      else
        adagrad_elem(wv[c][j], vv[c][j], acc[c][j], o);
    }
  store_vec<VEC, CH>(w, D, wv);
  store_vec<VEC, CH>(v, D, vv);
  if (m) store_vec<VEC, CH>(m, D, mv);
}

template <int VEC, int CH>
__device__ __forceinline__ void load_vec(const float* __restrict__ src, uint32_t D,
                                         float (&x)[CH][VEC], bool coherent) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const uint32_t e0 = ((uint32_t)c * 32 + lane) * VEC;
    if (VEC == 4) {
      float4 t = coherent ? __ldcg(reinterpret_cast<const float4*>(src + e0))
                          : *reinterpret_cast<const float4*>(src + e0);
      x[c][0] = t.x; x[c][1] = t.y; x[c][2] = t.z; x[c][3] = t.w;
    } else if (VEC == 2) {
      float2 t = coherent ? __ldcg(reinterpret_cast<const float2*>(src + e0))
                          : *reinterpret_cast<const float2*>(src + e0);
      x[c][0] = t.x; x[c][1] = t.y;
    } else {
      x[c][0] = e0 < D ? (coherent ? __ldcg(src + e0) : src[e0]) : 0.f;
    }
  }
}

template <int VEC, int CH>
__device__ __forceinline__ void store_vec(float* __restrict__ dst, uint32_t D,
                                          const float (&x)[CH][VEC]) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const uint32_t e0 = ((uint32_t)c * 32 + lane) * VEC;
    if (VEC == 4) {
      *reinterpret_cast<float4*>(dst + e0) = make_float4(x[c][0], x[c][1], x[c][2], x[c][3]);
    } else if (VEC == 2) {
      *reinterpret_cast<float2*>(dst + e0) = make_float2(x[c][0], x[c][1]);
    } else if (e0 < D) {
      dst[e0] = x[c][0];
    }
  }
}


template <int VEC, int CH>
__device__ __forceinline__ void zero_acc(float (&x)[CH][VEC]) {
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < VEC; ++j) x[c][j] = 0.f;
}
template <int VEC, int CH>
__device__ __forceinline__ void add_acc(float (&x)[CH][VEC], const float (&y)[CH][VEC]) {
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < VEC; ++j) x[c][j] += y[c][j];
}

}  // namespace odev
}  // namespace rs
