// unit.cu -- the SpMV executor: y = A x over the VBR-C split in ONE launch
// (north_star (2)).
//
// y_i = sum_j A_ij x_j, evaluated per row as
//   y_r = sum over the dense tiles of r's block row  T(r, c) x_c      (dense)
//       + sum over r's remainder entries               v x_j          (CSR)
// -- the paper's "regular loops that operate over the entire block
// (including some zeros)" and the CSR dispatch of low-delta
// blocks, re-designed as one data-driven sm_100a kernel
// instead of generated per-block C.
//
// One warp per batch of consecutive units (plan.cu).  A unit is <= 32 rows of
// one block row:
//   dense part  the rows of the block row's row-major panel (all its dense
//               tiles side by side, rows padded to 16 bytes) with LPR lanes
//               per row (a power of two fitted to the panel width by the
//               planner: lanes across columns for wide panels, several rows
//               per warp for narrow ones -- the "shape classes" of north_star
//               s4).  Every lane streams 16-byte vectors of its rows
//               (ld.global.cs: evict-first, the values are read once), loads
//               the x values of its columns once (through the panel's x map:
//               one int32 per column vector) and reuses them for all its
//               rows, and accumulates its rows in registers; the LPR lanes of
//               a row meet in a fixed shuffle tree that leaves row r's sum in
//               a known lane.
//   remainder   the rows' CSR entries in waves of 128 (4 coalesced loads per
//               lane, the next wave's loads issued before this wave's
//               gather), x gathered through the read-only path, the products
//               staged in shared memory; lane r sums row r's products in
//               entry order (a row with more than 32 products in a wave is
//               summed by the whole warp with a fixed tree).
//   y           lane r writes y_r = dense_r + rem_r once: no atomics, no
//               read-modify-write, no second launch.  Rows split over several
//               units (very long remainder rows) meet in scratch and the last
//               piece to arrive sums the pieces in piece order.
// Every row's summation order is fixed by the matrix alone (the plan depends
// on the block row, never on the shard count or on timing), so y is bitwise
// reproducible and identical for every P.
#include "sable_internal.cuh"

namespace sable {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kUnitThreads = kUnitWarps * 32;
#ifndef SABLE_UNIT_MINW
#define SABLE_UNIT_MINW 32  // A/B builds: resident warps per SM asked of ptxas (64 regs)
#endif
constexpr int kUnitMinBlocks = SABLE_UNIT_MINW / kUnitWarps;

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

__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

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

// Predicated streaming 16-byte load (ld.global.cs: evict-first).  Volatile
// so that a unit's loads are issued in program order, all before the first
// multiply-add that waits on them; with the predicate off, v keeps its old
// value (the callers never read a row past nr).
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

// Bulk L2 prefetch (UBLKPF) of the 16-byte-aligned cover of [p, p + bytes).
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + (uintptr_t)bytes + 15) & ~uintptr_t(15);
  if (bytes > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
                 : "memory");
}

// Lane 0: pull a unit's data (dense rows, x map, remainder row pointers,
// columns and values) into L2 while the previous unit computes, so the
// unit's own loads wait on L2 rather than HBM.
template <typename T>
__device__ __forceinline__ void prefetch_unit(const UPlan<T>& P, const Unit& U) {
  if (U.wq > 0) {
    l2_prefetch(reinterpret_cast<const uint4*>(P.pv) + U.voff16, (int64_t)U.nr * U.wq * 16);
    l2_prefetch(P.xq + U.xq0, (int64_t)U.wq * 4);
  }
  if (U.e1 > U.e0) {
    l2_prefetch(P.rptr + U.row0, (int64_t)(U.nr + 1) * 4);
    l2_prefetch(P.ridx + U.e0, (int64_t)(U.e1 - U.e0) * 4);
    l2_prefetch(P.rval + U.e0, (int64_t)(U.e1 - U.e0) * sizeof(T));
  }
}

// x of the N columns of panel column vector q (x map entry m).
template <typename T>
__device__ __forceinline__ void load_xv(const UPlan<T>& P, int m, const T* __restrict__ x,
                                        T (&xv)[Vec<T>::N]) {
  constexpr int N = Vec<T>::N;
  if (m >= 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) xv[i] = __ldg(x + min(m + i, P.nm1));
  } else {
    const int4 c = __ldg(P.xside + ~m);
    xv[0] = __ldg(x + c.x);
    xv[1] = __ldg(x + c.y);
    if constexpr (N == 4) {
      xv[2] = __ldg(x + c.z);
      xv[3] = __ldg(x + c.w);
    }
  }
}

// Fold K accumulators over the LPR lanes of a row subgroup: halving steps
// for the top log2(K) bits of the lane's column index, then plain xor steps.
// Afterwards lane (sub, ql) holds the total of its accumulator ql / (LPR/K).
// Every step adds own + partner (commutative, so both lanes of a pair hold
// the same value): one fixed binary tree per (LPR, K).
template <int O, int M, typename T, int K>
__device__ __forceinline__ void fold_lanes(T (&acc)[K], int lane) {
  if constexpr (O >= 1) {
    if constexpr (M > 1) {
      const bool up = (lane & O) != 0;
#pragma unroll
      for (int i = 0; i < M / 2; ++i) {
        const T send = up ? acc[i] : acc[i + M / 2];
        const T keep = up ? acc[i + M / 2] : acc[i];
        acc[i] = keep + __shfl_xor_sync(kFull, send, O);
      }
      fold_lanes<O / 2, M / 2>(acc, lane);
    } else {
      acc[0] += __shfl_xor_sync(kFull, acc[0], O);
      fold_lanes<O / 2, 1>(acc, lane);
    }
  }
}

// Dense part of a unit with LPR lanes per row: returns row `lane`'s sum
// (valid for lane < nr).  Lane (sub, ql) takes rows sub, sub + SUB, ... (at
// most K = min(LPR, 8)) and column vectors ql, ql + LPR, ...; row sub + SUB*k
// ends in lane sub * LPR + k * (LPR / K).
template <typename T, int LPR>
__device__ __forceinline__ T dense_rows(const UPlan<T>& P, const Unit& U,
                                        const T* __restrict__ x, int lane) {
  using V = typename Vec<T>::V;
  constexpr int N = Vec<T>::N;
  constexpr int SUB = 32 / LPR;
  constexpr int K = LPR < 8 ? LPR : 8;
  const int sub = lane / LPR, ql = lane % LPR;
  const int wq = U.wq, nr = U.nr;
  const V* vp = reinterpret_cast<const V*>(P.pv) + U.voff16 + sub * wq;
  const int* xm = P.xq + U.xq0;
  T acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = T(0);
  const int64_t rstep = (int64_t)SUB * wq;
  V v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = Vec<T>::zero();
#pragma unroll 1
  for (int q = ql; q < wq; q += LPR) {
    // the rows' values first (independent of x; rows past nr are not loaded
    // and their accumulators are never read), then x of the lane's columns,
    // then the multiply-adds in column order
    const V* p = vp + q;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      ld_cs_if(v[k], p, sub + SUB * k < nr);
      p += rstep;
    }
    T xv[N];
    load_xv<T>(P, __ldg(xm + q), x, xv);
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i) acc[k] = fma(Vec<T>::get(v[k], i), xv[i], acc[k]);
  }
  fold_lanes<LPR / 2, K>(acc, lane);
  const int src = (lane % SUB) * LPR + (lane / SUB) * (LPR / K);
  return __shfl_sync(kFull, acc[0], src & 31);
}

// Remainder part in waves of kRemWave entries (kRemKB coalesced loads per
// lane): gathers x, stages the products and sums row `lane`'s entries in
// [e0, e1) in entry order (valid for lane < nr), issuing wave w + 1's loads
// before wave w's gather.
constexpr int kRemKB = 4;
constexpr int kRemWave = 32 * kRemKB;

template <typename T>
struct RemWave {
  int32_t c[kRemKB];
  T v[kRemKB];
};

template <typename T>
__device__ __forceinline__ void rem_load(const UPlan<T>& P, int c0, int e1, int lane,
                                         RemWave<T>& w) {
  const int n = e1 - c0;
#pragma unroll
  for (int k = 0; k < kRemKB; ++k) {
    const int e = k * 32 + lane;
    w.c[k] = 0;
    w.v[k] = T(0);
    if (e < n) {
      w.c[k] = __ldcs(P.ridx + c0 + e);
      w.v[k] = __ldcs(P.rval + c0 + e);
    }
  }
}

template <typename T>
__device__ __forceinline__ T rem_rows(const UPlan<T>& P, const Unit& U, const T* __restrict__ x,
                                      T* buf, int lane) {
  int lo = 0, hi = 0;
  if (lane < U.nr) {
    lo = max(__ldg(P.rptr + U.row0 + lane), U.e0);
    hi = min(__ldg(P.rptr + U.row0 + lane + 1), U.e1);
  }
  RemWave<T> w;
  rem_load(P, U.e0, U.e1, lane, w);
  T s = T(0);
#pragma unroll 1
  for (int c0 = U.e0; c0 < U.e1; c0 += kRemWave) {
    const int n = min(kRemWave, U.e1 - c0);
    T pr[kRemKB];
#pragma unroll
    for (int k = 0; k < kRemKB; ++k) pr[k] = (k * 32 + lane < n) ? w.v[k] * __ldg(x + w.c[k]) : T(0);
    if (c0 + kRemWave < U.e1) rem_load(P, c0 + kRemWave, U.e1, lane, w);
#pragma unroll
    for (int k = 0; k < kRemKB; ++k)
      if (k * 32 + lane < n) buf[k * 32 + lane] = pr[k];
    __syncwarp();
    const int a = max(lo, c0) - c0, b = min(hi, c0 + n) - c0;
    const bool longr = b - a > 32;
    if (!longr)
      for (int e = a; e < b; ++e) s += buf[e];
    unsigned lm = __ballot_sync(kFull, longr);
    while (lm) {
      const int q = __ffs(lm) - 1;
      lm &= lm - 1;
      const int a2 = __shfl_sync(kFull, a, q), b2 = __shfl_sync(kFull, b, q);
      T t = T(0);
      for (int e = a2 + lane; e < b2; e += 32) t += buf[e];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
      if (lane == q) s += t;
    }
    __syncwarp();
  }
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kUnitThreads, kUnitMinBlocks)
    unit_kernel(const __grid_constant__ UPlan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  __shared__ __align__(16) T buf_s[kUnitWarps][kRemWave];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kUnitWarps + warp;
  if (b >= P.n_batches) return;
  const int u0 = __ldg(P.batch + b), u1 = __ldg(P.batch + b + 1);
  if (lane == 0 && P.pf) l2_prefetch(P.units + u0, (int64_t)(u1 - u0) * sizeof(Unit));
  Unit Un = load_unit(P.units + u0);
  for (int u = u0; u < u1; ++u) {
    const Unit U = Un;
    if (u + 1 < u1) Un = load_unit(P.units + u + 1);
    T s = T(0);
    if (U.wq > 0) {
      switch (U.llpr) {
        case 0: s = dense_rows<T, 1>(P, U, x, lane); break;
        case 1: s = dense_rows<T, 2>(P, U, x, lane); break;
        case 2: s = dense_rows<T, 4>(P, U, x, lane); break;
        case 3: s = dense_rows<T, 8>(P, U, x, lane); break;
        case 4: s = dense_rows<T, 16>(P, U, x, lane); break;
        default: s = dense_rows<T, 32>(P, U, x, lane); break;
      }
    }
    if (lane == 0 && P.pf && u + 1 < u1) prefetch_unit(P, Un);
    if (U.e1 > U.e0) s += rem_rows<T>(P, U, x, buf_s[warp], lane);
    if (U.xg < 0) {
      if (lane < U.nr) y[U.row0 + lane] = s;
    } else {
      const int4 gv = __ldg(reinterpret_cast<const int4*>(P.xg + U.xg));
      const int64_t slot = (int64_t)(((uint64_t)(uint32_t)gv.y << 32) | (uint32_t)gv.x);
      const int counter = gv.z, np = gv.w;
      T* sp = P.scratch + slot;
      if (lane < U.nr) __stcg(sp + U.piece * 32 + lane, s);
      __syncwarp();  // the warp's partials before lane 0's release
      int last = 0;
      if (lane == 0) last = (atom_add_acq_rel(P.counters + counter, 1) + 1 == np);
      last = __shfl_sync(kFull, last, 0);
      if (last) {
        if (lane < U.nr) {
          T t = __ldcg(sp + lane);
          for (int q = 1; q < np; ++q) t += __ldcg(sp + q * 32 + lane);
          y[U.row0 + lane] = t;
        }
        if (lane == 0) P.counters[counter] = 0;  // ready for the next launch
      }
    }
  }
}

// ------------------------------------------------------------------------
// The staged executor (default): every warp pipelines its batch of units
// through two shared-memory stages.  Lane 0 pulls unit u + 1's data -- dense
// rows, x map, remainder row pointers, columns and values, each the
// 16-byte-aligned cover of its range -- with cp.async.bulk copies completing
// on the stage's mbarrier while the warp computes unit u from the other
// stage, so the HBM latency of a unit is hidden behind the previous one and
// no register holds a value in flight.  Per unit, only x (L2-resident) is
// read from global memory.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

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

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Where a unit's regions sit in its stage (bytes), and the element offset of
// each range's first element inside its 16-byte-aligned cover.
struct StageMap {
  uint32_t o_xm, o_rp, o_ix, o_rv, total;
  uint32_t d_xm, d_rp, d_ix, d_rv;
};

template <typename T>
__device__ __forceinline__ StageMap stage_map(const UPlan<T>& P, const Unit& U) {
  StageMap m{};
  uint32_t off = U.wq > 0 ? (uint32_t)U.nr * (uint32_t)U.wq * 16u : 0u;
  auto region = [&](const void* p, uint32_t bytes, uint32_t esz, uint32_t& o, uint32_t& d) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t c = bytes ? (uint32_t)(((a + bytes + 15) & ~uintptr_t(15)) - (a & ~uintptr_t(15))) : 0u;
    o = off;
    d = (uint32_t)(a & 15) / esz;
    off += c;
  };
  if (U.wq > 0) region(P.xq + U.xq0, (uint32_t)U.wq * 4u, 4u, m.o_xm, m.d_xm);
  const uint32_t ne = (uint32_t)(U.e1 - U.e0);
  if (ne > 0) {
    region(P.rptr + U.row0, ((uint32_t)U.nr + 1u) * 4u, 4u, m.o_rp, m.d_rp);
    region(P.ridx + U.e0, ne * 4u, 4u, m.o_ix, m.d_ix);
    region(P.rval + U.e0, ne * (uint32_t)sizeof(T), (uint32_t)sizeof(T), m.o_rv, m.d_rv);
  }
  m.total = off;
  return m;
}

// Lane 0: start the bulk copies of a unit's data into a stage.
template <typename T>
__device__ __forceinline__ void issue_unit(const UPlan<T>& P, const Unit& U, unsigned char* stage,
                                           uint32_t bar, uint64_t pol) {
  const StageMap m = stage_map(P, U);
  mbar_expect_tx(bar, m.total);
  const uint32_t s0 = smem_u32(stage);
  auto cp = [&](const void* p, uint32_t bytes, uint32_t o) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uint32_t c = (uint32_t)(((reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15)) - a);
    bulk_g2s(s0 + o, reinterpret_cast<const void*>(a), c, bar, pol);
  };
  if (U.wq > 0) {
    cp(reinterpret_cast<const uint4*>(P.pv) + U.voff16, (uint32_t)U.nr * (uint32_t)U.wq * 16u, 0u);
    cp(P.xq + U.xq0, (uint32_t)U.wq * 4u, m.o_xm);
  }
  const uint32_t ne = (uint32_t)(U.e1 - U.e0);
  if (ne > 0) {
    cp(P.rptr + U.row0, ((uint32_t)U.nr + 1u) * 4u, m.o_rp);
    cp(P.ridx + U.e0, ne * 4u, m.o_ix);
    cp(P.rval + U.e0, ne * (uint32_t)sizeof(T), m.o_rv);
  }
}

// Dense part from a stage (same lane mapping and tree as dense_rows).
template <typename T, int LPR>
__device__ __forceinline__ T dense_staged(const UPlan<T>& P, const Unit& U, const StageMap& m,
                                          const unsigned char* stage, const T* __restrict__ x,
                                          int lane) {
  using V = typename Vec<T>::V;
  constexpr int N = Vec<T>::N;
  constexpr int SUB = 32 / LPR;
  constexpr int K = LPR < 8 ? LPR : 8;
  const int sub = lane / LPR, ql = lane % LPR;
  const int wq = U.wq, nr = U.nr;
  const V* vs = reinterpret_cast<const V*>(stage) + sub * wq;
  const int* xm = reinterpret_cast<const int*>(stage + m.o_xm) + m.d_xm;
  T acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = T(0);
#pragma unroll 1
  for (int q = ql; q < wq; q += LPR) {
    T xv[N];
    load_xv<T>(P, xm[q], x, xv);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (sub + SUB * k < nr) {
        const V v = vs[q + k * SUB * wq];
#pragma unroll
        for (int i = 0; i < N; ++i) acc[k] = fma(Vec<T>::get(v, i), xv[i], acc[k]);
      }
    }
  }
  fold_lanes<LPR / 2, K>(acc, lane);
  const int src = (lane % SUB) * LPR + (lane / SUB) * (LPR / K);
  return __shfl_sync(kFull, acc[0], src & 31);
}

// Remainder part from a stage: the products of a wave (8 per lane) go to
// `buf`, lane r sums row r's in entry order (long rows: the whole warp, a
// fixed tree).
constexpr int kSRemKB = 8;
constexpr int kSRemWave = 32 * kSRemKB;

template <typename T>
__device__ __forceinline__ T rem_staged(const UPlan<T>& P, const Unit& U, const StageMap& m,
                                        const unsigned char* stage, const T* __restrict__ x,
                                        T* buf, int lane) {
  const int ne = U.e1 - U.e0;
  const int* rp = reinterpret_cast<const int*>(stage + m.o_rp) + m.d_rp;
  const int* ix = reinterpret_cast<const int*>(stage + m.o_ix) + m.d_ix;
  const T* rv = reinterpret_cast<const T*>(stage + m.o_rv) + m.d_rv;
  int lo = 0, hi = 0;
  if (lane < U.nr) {
    lo = max(rp[lane] - U.e0, 0);
    hi = min(rp[lane + 1] - U.e0, ne);
  }
  T s = T(0);
#pragma unroll 1
  for (int c0 = 0; c0 < ne; c0 += kSRemWave) {
    const int n = min(kSRemWave, ne - c0);
    T xg[kSRemKB];
#pragma unroll
    for (int k = 0; k < kSRemKB; ++k) {
      const int e = k * 32 + lane;
      xg[k] = e < n ? __ldg(x + ix[c0 + e]) : T(0);
    }
#pragma unroll
    for (int k = 0; k < kSRemKB; ++k) {
      const int e = k * 32 + lane;
      if (e < n) buf[e] = rv[c0 + e] * xg[k];
    }
    __syncwarp();
    const int a = max(lo, c0) - c0, b = min(hi, c0 + n) - c0;
    const bool longr = b - a > 32;
    if (!longr)
      for (int e = a; e < b; ++e) s += buf[e];
    unsigned lm = __ballot_sync(kFull, longr);
    while (lm) {
      const int q = __ffs(lm) - 1;
      lm &= lm - 1;
      const int a2 = __shfl_sync(kFull, a, q), b2 = __shfl_sync(kFull, b, q);
      T t = T(0);
      for (int e = a2 + lane; e < b2; e += 32) t += buf[e];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
      if (lane == q) s += t;
    }
    __syncwarp();
  }
  return s;
}

// y of a unit's rows (or its partials into the combine group).
template <typename T>
__device__ __forceinline__ void finish_unit(const UPlan<T>& P, const Unit& U, T s,
                                            T* __restrict__ y, int lane) {
  if (U.xg < 0) {
    if (lane < U.nr) y[U.row0 + lane] = s;
    return;
  }
  const int4 gv = __ldg(reinterpret_cast<const int4*>(P.xg + U.xg));
  const int64_t slot = (int64_t)(((uint64_t)(uint32_t)gv.y << 32) | (uint32_t)gv.x);
  const int counter = gv.z, np = gv.w;
  T* sp = P.scratch + slot;
  if (lane < U.nr) __stcg(sp + U.piece * 32 + lane, s);
  __syncwarp();  // the warp's partials before lane 0's release
  int last = 0;
  if (lane == 0) last = (atom_add_acq_rel(P.counters + counter, 1) + 1 == np);
  last = __shfl_sync(kFull, last, 0);
  if (last) {
    if (lane < U.nr) {
      T t = __ldcg(sp + lane);
      for (int q = 1; q < np; ++q) t += __ldcg(sp + q * 32 + lane);
      y[U.row0 + lane] = t;
    }
    if (lane == 0) P.counters[counter] = 0;  // ready for the next launch
  }
}

// Shared memory of one warp: 2 mbarriers (16 B), two stages, the products.
template <typename T>
__host__ __device__ constexpr uint32_t staged_warp_bytes(uint32_t stage) {
  return 16u + 2u * stage + (uint32_t)(kSRemWave * sizeof(T));
}

template <typename T>
__global__ void __launch_bounds__(kUnitThreads, kUnitMinBlocks)
    unit_staged_kernel(const __grid_constant__ UPlan<T> P, const T* __restrict__ x,
                       T* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kUnitWarps + warp;
  if (b >= P.n_batches) return;
  unsigned char* ws = smem + (size_t)warp * staged_warp_bytes<T>(P.stage);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws);
  unsigned char* stg[2] = {ws + 16, ws + 16 + P.stage};
  T* buf = reinterpret_cast<T*>(ws + 16 + 2 * P.stage);
  const int u0 = __ldg(P.batch + b), u1 = __ldg(P.batch + b + 1);
  uint64_t pol = 0;
  Unit U = load_unit(P.units + u0);
  Unit Un = U;
  if (u0 + 1 < u1) Un = load_unit(P.units + u0 + 1);
  if (lane == 0) {
    mbar_init(smem_u32(bar), 1);
    mbar_init(smem_u32(bar + 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pol = policy_evict_first();
    issue_unit(P, U, stg[0], smem_u32(bar), pol);
  }
  __syncwarp();
  for (int u = u0; u < u1; ++u) {
    const int s = (u - u0) & 1;
    const uint32_t par = (uint32_t)((u - u0) >> 1) & 1u;
    // unit u + 1's data into the other stage (freed at the end of u - 1)
    if (lane == 0 && u + 1 < u1) issue_unit(P, Un, stg[s ^ 1], smem_u32(bar + (s ^ 1)), pol);
    Unit Unn = Un;
    if (u + 2 < u1) Unn = load_unit(P.units + u + 2);
    const StageMap m = stage_map(P, U);
    mbar_wait(smem_u32(bar + s), par);
    const unsigned char* st = stg[s];
    T acc = T(0);
    if (U.wq > 0) {
      switch (U.llpr) {
        case 0: acc = dense_staged<T, 1>(P, U, m, st, x, lane); break;
        case 1: acc = dense_staged<T, 2>(P, U, m, st, x, lane); break;
        case 2: acc = dense_staged<T, 4>(P, U, m, st, x, lane); break;
        case 3: acc = dense_staged<T, 8>(P, U, m, st, x, lane); break;
        case 4: acc = dense_staged<T, 16>(P, U, m, st, x, lane); break;
        default: acc = dense_staged<T, 32>(P, U, m, st, x, lane); break;
      }
    }
    if (U.e1 > U.e0) acc += rem_staged<T>(P, U, m, st, x, buf, lane);
    finish_unit(P, U, acc, y, lane);
    __syncwarp();  // stage s is free for unit u + 2
    U = Un;
    Un = Unn;
  }
}

}  // namespace

template <typename T>
cudaError_t launch_units(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  if (h->n_ubatch == 0) return cudaSuccess;
  UPlan<T> P;
  P.units = h->units;
  P.batch = h->ubatch;
  P.xq = h->xq;
  P.xside = h->xside;
  P.pv = static_cast<const T*>(h->pv);
  P.rptr = h->rem_ptr;
  P.ridx = h->rem_idx;
  P.rval = static_cast<const T*>(h->rem_val);
  P.xg = h->uxg;
  P.scratch = static_cast<T*>(h->uscratch);
  P.counters = h->ucounters;
  P.n_batches = h->n_ubatch;
  P.nm1 = (int32_t)(h->ncols - 1);
  P.pf = h->cfg.xpf;
  P.stage = (uint32_t)h->ustage;
  const int64_t blocks = (h->n_ubatch + kUnitWarps - 1) / kUnitWarps;
  if (h->cfg.ustaged) {
    const size_t smem = (size_t)kUnitWarps * staged_warp_bytes<T>(P.stage);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    e = set_smem_attr(reinterpret_cast<const void*>(unit_staged_kernel<T>), dev, smem);
    if (e) return e;
    unit_staged_kernel<T><<<(unsigned)blocks, kUnitThreads, smem, st>>>(
        P, static_cast<const T*>(x), static_cast<T*>(y));
    return cudaGetLastError();
  }
  unit_kernel<T><<<(unsigned)blocks, kUnitThreads, 0, st>>>(P, static_cast<const T*>(x),
                                                            static_cast<T*>(y));
  return cudaGetLastError();
}

template cudaError_t launch_units<float>(const sable_handle*, const void*, void*, cudaStream_t);
template cudaError_t launch_units<double>(const sable_handle*, const void*, void*, cudaStream_t);

}  // namespace sable
