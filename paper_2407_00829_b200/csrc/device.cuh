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
  static __device__ __forceinline__ float4 one() { return make_float4(1.f, 1.f, 1.f, 1.f); }
};
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int N = 2;
  static __device__ __forceinline__ double get(const double2& v, int i) {
    return i == 0 ? v.x : v.y;
  }
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double2 one() { return make_double2(1.0, 1.0); }
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

// ---- shared memory, mbarriers and bulk copies (TMA engine, non-tensor)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Arrive once and expect `bytes` of bulk-copy transactions on the barrier.
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Order this thread's (and, after __syncwarp, its warp's) generic-proxy
// shared-memory accesses before later async-proxy (bulk copy) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Bulk copy global -> shared (cp.async.bulk, SASS UBLKCP), completion as
// transaction bytes on `bar`; src, dst 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes,
                                              uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ Unit unpack_unit(const int4& a, const int4& b) {
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

// Loads of data read by many units (x maps and x) and of the plan's metadata
// (unit descriptors, batch bounds, remainder row pointers): non-coherent, with
// an L2 evict_last policy so the streamed panel values and remainder entries
// (evict_first) do not push them out of L2, within one SpMV and between the
// steps of an iterated one (measured: C4 0.0854 -> 0.0826 ms with L2 flushed
// before every SpMV, C3 0.0612 -> 0.0595 ms).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

#ifndef SABLE_META_EL
#define SABLE_META_EL 1  // A/B builds: 0 = metadata loads with the default L2 policy
#endif

__device__ __forceinline__ int4 ldg_meta(const int4* p) {
#if SABLE_META_EL
  int4 v;
  asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "l"(policy_evict_last()));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ int32_t ldg_meta(const int32_t* p) {
#if SABLE_META_EL
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
#else
  return __ldg(p);
#endif
}

// A unit descriptor (32 B, read by every lane: one broadcast request).
__device__ __forceinline__ Unit load_unit(const Unit* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  return unpack_unit(ldg_meta(q), ldg_meta(q + 1));
}

// A unit descriptor staged in shared memory.
__device__ __forceinline__ Unit load_unit_smem(const void* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  return unpack_unit(q[0], q[1]);
}

__device__ __forceinline__ XMap ldg_xmap(const XMap* p) {
  int2 v;
  asm("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
      : "=r"(v.x), "=r"(v.y)
      : "l"(p), "l"(policy_evict_last()));
  return XMap{v.x, v.y};
}

// KV consecutive values of x (row-major ncols x KV) as one load where the
// width allows.
template <typename T, int KV>
__device__ __forceinline__ void ldg_kv(const T* __restrict__ p, T (&o)[KV]) {
  if constexpr (KV == 1) {
    if constexpr (sizeof(T) == 4) {
      float v;
      asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(policy_evict_last()));
      o[0] = v;
    } else {
      double v;
      asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy_evict_last()));
      o[0] = v;
    }
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
