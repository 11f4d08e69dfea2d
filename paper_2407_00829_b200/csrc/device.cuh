// device.cuh -- device-side helpers shared by the kernels of libsable.so
// (PTX wrappers, 16-byte vector types, the unit descriptor loader).
#pragma once

#include "sable_internal.cuh"

namespace sable {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

// 16-byte vectors of the value type: N elements per column vector.
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using V = float4;
  static constexpr int N = 4;
  static __device__ __forceinline__ float get(const float4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  static __device__ __forceinline__ float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int N = 2;
  static __device__ __forceinline__ double get(const double2& v, int i) {
    return i == 0 ? v.x : v.y;
  }
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
};

// Arrival counter of a split row range: releases this warp's scratch writes
// (ordered before it by __syncwarp) and acquires the other pieces'.
__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Predicated streaming 16-byte load (ld.global.cs: evict-first).  Volatile
// so that a unit's loads are issued in program order, all before the first
// multiply-add that waits on them; with the predicate off, v keeps its old
// value.
__device__ __forceinline__ void ld_cs_if(float4& v, const float4* p, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.cs.v4.f32 {%0, %1, %2, %3}, [%4];\n}"
      : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
      : "l"(p), "r"((int)pred));
}
__device__ __forceinline__ void ld_cs_if(double2& v, const double2* p, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
      "@q ld.global.cs.v2.f64 {%0, %1}, [%2];\n}"
      : "+d"(v.x), "+d"(v.y)
      : "l"(p), "r"((int)pred));
}

// Bulk L2 prefetch (cp.async.bulk.prefetch.L2, SASS UBLKPF) of the
// 16-byte-aligned cover of [p, p + bytes).
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + (uintptr_t)bytes + 15) & ~uintptr_t(15);
  if (bytes > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
                 : "memory");
}

// A unit descriptor (32 B, read by every lane: one broadcast request).
__device__ __forceinline__ Unit load_unit(const Unit* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 a = __ldg(q), b = __ldg(q + 1);
  Unit u;
  u.voff16 = a.x;
  u.row0 = a.y;
  u.wq = a.z;
  u.xq0 = a.w;
  u.e0 = b.x;
  u.e1 = b.y;
  u.xg = b.z;
  u.nr = (uint8_t)(b.w & 0xff);
  u.llpr = (uint8_t)((b.w >> 8) & 0xff);
  u.piece = (uint16_t)((uint32_t)b.w >> 16);
  return u;
}

// KV consecutive values of x (row-major ncols x KV) as one load where the
// width allows.
template <typename T, int KV>
__device__ __forceinline__ void ldg_kv(const T* __restrict__ p, T (&o)[KV]) {
  if constexpr (KV == 1) {
    o[0] = __ldg(p);
  } else if constexpr (sizeof(T) * KV >= 16) {
    using V = typename Vec<T>::V;
    constexpr int N = Vec<T>::N;
#pragma unroll
    for (int h = 0; h < KV / N; ++h) {
      const V v = __ldg(reinterpret_cast<const V*>(p) + h);
#pragma unroll
      for (int i = 0; i < N; ++i) o[h * N + i] = Vec<T>::get(v, i);
    }
  } else {  // float x 2
    const float2 v = __ldg(reinterpret_cast<const float2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
}

}  // namespace dev
}  // namespace sable
