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
#ifndef SABLE_UNIT_MINB
#define SABLE_UNIT_MINB 1  // A/B builds: resident CTAs per SM asked of ptxas
#endif

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
#pragma unroll 1
  for (int q = ql; q < wq; q += LPR) {
    // the rows' values first (independent of x), then x of the lane's
    // columns, then the multiply-adds in column order
    V v[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[k] = (sub + SUB * k < nr) ? __ldcs(vp + q + k * SUB * wq) : Vec<T>::zero();
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
__global__ void __launch_bounds__(kUnitThreads, SABLE_UNIT_MINB)
    unit_kernel(const __grid_constant__ UPlan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  __shared__ __align__(16) T buf_s[kUnitWarps][kRemWave];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kUnitWarps + warp;
  if (b >= P.n_batches) return;
  const int u0 = __ldg(P.batch + b), u1 = __ldg(P.batch + b + 1);
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
  const int64_t blocks = (h->n_ubatch + kUnitWarps - 1) / kUnitWarps;
  unit_kernel<T><<<(unsigned)blocks, kUnitThreads, 0, st>>>(P, static_cast<const T*>(x),
                                                            static_cast<T*>(y));
  return cudaGetLastError();
}

template cudaError_t launch_units<float>(const sable_handle*, const void*, void*, cudaStream_t);
template cudaError_t launch_units<double>(const sable_handle*, const void*, void*, cudaStream_t);

}  // namespace sable
