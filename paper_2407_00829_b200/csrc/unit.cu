// unit.cu -- the SpMV executor: y = A x over the VBR-C split in ONE launch
// (north_star (2)), and its multi-vector form Y = A X
// for KV = 2, 4, 8 right-hand sides on the same plan.
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
//               units (very long remainder rows, very wide panels) meet in
//               scratch and the last piece to arrive sums the pieces in piece
//               order.
// With SABLE_XPREFETCH=1 (off by default: measured slower), lane 0 pulls the
// data of a warp batch's later units into L2 with bulk prefetches
// (cp.async.bulk.prefetch.L2) at the batch start.  x, the x maps and the
// plan's metadata are loaded with an L2 evict_last policy, the panel values
// and remainder entries evict-first.  With the fused exchange epilogue
// (comm.cu) every finished y row is also stored into the peers' x_next.
// Every row's summation order is
// fixed by the matrix alone (the plan depends on the block row, never on the
// shard count or on timing), so y is bitwise reproducible and identical for
// every P.
#include <algorithm>

#include "device.cuh"

namespace sable {

namespace {

using namespace dev;

constexpr int kUnitThreads = kUnitWarps * 32;
#ifndef SABLE_UNIT_MINW
#define SABLE_UNIT_MINW 32  // A/B builds: resident warps per SM asked of ptxas (64 regs)
#endif
constexpr int kUnitMinBlocks = SABLE_UNIT_MINW / kUnitWarps;

// Lane 0: pull a warp batch's data past its first unit into L2 with five
// bulk prefetches -- the units of a batch are consecutive, so their panel
// rows, x maps, remainder row pointers, columns and values are contiguous
// ranges from the first unit's to the last unit's -- so the later units'
// loads wait on L2 rather than HBM.
template <typename T>
__device__ __forceinline__ void prefetch_span(const UPlan<T>& P, const Unit& A, const Unit& B) {
  const int64_t v0 = A.wq > 0 ? A.voff16 : B.voff16;
  const int64_t v1 = B.wq > 0 ? (int64_t)B.voff16 + (int64_t)B.nr * B.wq : (int64_t)A.voff16;
  if (v1 > v0) l2_prefetch(reinterpret_cast<const uint4*>(P.pv) + v0, (v1 - v0) * 16);
  const int64_t q0 = A.wq > 0 ? A.xq0 : B.xq0;
  const int64_t q1 = B.wq > 0 ? (int64_t)B.xq0 + B.wq : (int64_t)A.xq0;
  if (q1 > q0) l2_prefetch(P.xq + q0, (q1 - q0) * (int64_t)sizeof(XMap));
  l2_prefetch(P.rptr + A.row0, ((int64_t)B.row0 + B.nr + 1 - A.row0) * 4);
  if (B.e1 > A.e0) {
    l2_prefetch(P.ridx + A.e0, (int64_t)(B.e1 - A.e0) * 4);
    l2_prefetch(P.rval + A.e0, (int64_t)(B.e1 - A.e0) * sizeof(T));
  }
}

// x (row-major ncols x KV) of the N columns of one panel column vector,
// x map entry m (sable_internal.cuh XMap: c >= 0 -- columns c + i, the ones
// from i = k on shifted by d, all inside [0, ncols) by construction; c < 0 --
// the side entry ~c lists the N columns).
template <typename T, int KV>
__device__ __forceinline__ void load_xv(const UPlan<T>& P, XMap m, const T* __restrict__ x,
                                        T (&xv)[Vec<T>::N][KV]) {
  constexpr int N = Vec<T>::N;
  if (m.c >= 0) {
    const int k = m.kd & 3, d = m.kd >> 2;  // k = 0: d = 0
#pragma unroll
    for (int i = 0; i < N; ++i) {
      SABLE_DCHECK(m.c + i + (i >= k ? d : 0) >= 0 && m.c + i + (i >= k ? d : 0) < P.ncols);
      ldg_kv<T, KV>(x + (int64_t)(m.c + i + (i >= k ? d : 0)) * KV, xv[i]);
    }
  } else {
    SABLE_DCHECK(~m.c < P.n_xside);
    const int4 c = __ldg(P.xside + ~m.c);
    SABLE_DCHECK(c.x >= 0 && c.x < P.ncols && c.y >= 0 && c.y < P.ncols);
    SABLE_DCHECK(N == 2 || (c.z >= 0 && c.z < P.ncols && c.w >= 0 && c.w < P.ncols));
    ldg_kv<T, KV>(x + (int64_t)c.x * KV, xv[0]);
    ldg_kv<T, KV>(x + (int64_t)c.y * KV, xv[1]);
    if constexpr (N == 4) {
      ldg_kv<T, KV>(x + (int64_t)c.z * KV, xv[2]);
      ldg_kv<T, KV>(x + (int64_t)c.w * KV, xv[3]);
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

// Dense part of a unit with LPR lanes per row: out[j] = row `lane`'s sum
// for vector j (valid for lane < nr).  Lane (sub, ql) takes column vectors
// ql, ql + LPR, ... of rows sub, sub + SUB, ...: K = min(LPR, 8) / KV of them
// per row pass (KV = 1: one pass), and row sub + SUB * (p * K + k) ends in
// lane sub * LPR + k * (LPR / K) after pass p's fold.
template <typename T, int LPR, int KV>
__device__ __forceinline__ void dense_rows(const UPlan<T>& P, const Unit& U,
                                           const T* __restrict__ x, int lane, T (&out)[KV]) {
  using V = typename Vec<T>::V;
  constexpr int N = Vec<T>::N;
  constexpr int SUB = 32 / LPR;
  constexpr int K8 = LPR < 8 ? LPR : 8;
  constexpr int K = K8 / KV > 0 ? K8 / KV : 1;
  constexpr int RP = K8 / K;  // row passes
  const int sub = lane / LPR, ql = lane % LPR;
  const int wq = U.wq, nr = U.nr;
  const V* vp = reinterpret_cast<const V*>(P.pv) + U.voff16 + sub * wq;
  const XMap* xm = P.xq + U.xq0;
  const int64_t rstep = (int64_t)SUB * wq;
#pragma unroll 1
  for (int rp = 0; rp < RP; ++rp) {
    if (SUB * rp * K >= nr) break;  // no lane has a row in this pass
    const int rb = sub + SUB * rp * K;
    T acc[KV][K];
#pragma unroll
    for (int j = 0; j < KV; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k) acc[j][k] = T(0);
    V v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = Vec<T>::zero();
#pragma unroll 1
    for (int q = ql; q < wq; q += LPR) {
      // the rows' values first (independent of x; rows past nr are not
      // loaded and their accumulators are never read), then x of the lane's
      // columns, then the multiply-adds in column order
      const V* p = vp + q + rp * K * rstep;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ld_cs_if(v[k], p, rb + SUB * k < nr);
        p += rstep;
      }
      T xv[N][KV];
      load_xv<T, KV>(P, ldg_xmap(xm + q), x, xv);
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j < KV; ++j)
            acc[j][k] = fma(Vec<T>::get(v[k], i), xv[i][j], acc[j][k]);
    }
#pragma unroll
    for (int j = 0; j < KV; ++j) fold_lanes<LPR / 2, K>(acc[j], lane);
    const int kk = lane / SUB - rp * K;
    const int src = (lane % SUB) * LPR + kk * (LPR / K);
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      const T t = __shfl_sync(kFull, acc[j][0], src & 31);
      if (kk >= 0 && kk < K) out[j] = t;
    }
  }
}

// Remainder part in waves of kRemWave entries (kRemKB coalesced loads per
// lane, the next wave's issued before this wave's gather): the products are
// staged in shared memory and lane r sums row r's in entry order; a row with
// more than 32 products in a wave is summed by the whole warp with a fixed
// tree.
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

template <typename T, int KV>
__device__ __forceinline__ void rem_rows(const UPlan<T>& P, const Unit& U,
                                         const T* __restrict__ x, T* buf, int lane, int lo,
                                         int hi, T (&s)[KV]) {
  RemWave<T> w;
  rem_load(P, U.e0, U.e1, lane, w);
#pragma unroll 1
  for (int c0 = U.e0; c0 < U.e1; c0 += kRemWave) {
    const int n = min(kRemWave, U.e1 - c0);
    T pr[kRemKB][KV];
#pragma unroll
    for (int k = 0; k < kRemKB; ++k) {
      T xg[KV];
#pragma unroll
      for (int j = 0; j < KV; ++j) xg[j] = T(0);
      if (k * 32 + lane < n) {
        SABLE_DCHECK(w.c[k] >= 0 && w.c[k] < P.ncols);
        ldg_kv<T, KV>(x + (int64_t)w.c[k] * KV, xg);
      }
#pragma unroll
      for (int j = 0; j < KV; ++j) pr[k][j] = w.v[k] * xg[j];
    }
    if (c0 + kRemWave < U.e1) rem_load(P, c0 + kRemWave, U.e1, lane, w);
#pragma unroll
    for (int k = 0; k < kRemKB; ++k)
      if (k * 32 + lane < n)
#pragma unroll
        for (int j = 0; j < KV; ++j) buf[(k * 32 + lane) * KV + j] = pr[k][j];
    __syncwarp();
    const int a = max(lo, c0) - c0, b = min(hi, c0 + n) - c0;
    const bool longr = b - a > 32;
    if (!longr)
      for (int e = a; e < b; ++e)
#pragma unroll
        for (int j = 0; j < KV; ++j) s[j] += buf[e * KV + j];
    unsigned lm = __ballot_sync(kFull, longr);
    while (lm) {
      const int q = __ffs(lm) - 1;
      lm &= lm - 1;
      const int a2 = __shfl_sync(kFull, a, q), b2 = __shfl_sync(kFull, b, q);
#pragma unroll
      for (int j = 0; j < KV; ++j) {
        T t = T(0);
        for (int e = a2 + lane; e < b2; e += 32) t += buf[e * KV + j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
        if (lane == q) s[j] += t;
      }
    }
    __syncwarp();
  }
}

// y of a unit's rows (row-major nloc x KV), or its partials into the
// combine group (the last piece to arrive sums the pieces in order).
template <typename T, int KV>
__device__ __forceinline__ void finish_unit(const UPlan<T>& P, const Unit& U, const T (&s)[KV],
                                            T* __restrict__ y, int lane) {
  if (U.xg < 0) {
    SABLE_DCHECK(U.row0 >= 0 && U.row0 + U.nr <= P.nloc);
    if (lane < U.nr) {
#pragma unroll
      for (int j = 0; j < KV; ++j) y[(int64_t)(U.row0 + lane) * KV + j] = s[j];
      if constexpr (KV == 1)  // fused exchange: the same row of every peer's x_next
        for (int q = 0; q < P.npeer; ++q) P.peer[q][U.row0 + lane] = s[0];
    }
    return;
  }
  const int4 gv = __ldg(reinterpret_cast<const int4*>(P.xg + U.xg));
  const int64_t slot = (int64_t)(((uint64_t)(uint32_t)gv.y << 32) | (uint32_t)gv.x);
  const int counter = gv.z, np = gv.w;
  SABLE_DCHECK(U.xg < P.n_uxg && counter >= 0 && counter < P.n_uxg && U.piece < np &&
               slot >= 0 && (slot + (int64_t)np * 32) * KV <= P.scratch_elems);
  T* sp = P.scratch + slot * KV;
  if (lane < U.nr)
#pragma unroll
    for (int j = 0; j < KV; ++j) __stcg(sp + (U.piece * 32 + lane) * KV + j, s[j]);
  __syncwarp();  // the warp's partials before lane 0's release
  int last = 0;
  if (lane == 0) last = (atom_add_acq_rel(P.counters + counter, 1) + 1 == np);
  last = __shfl_sync(kFull, last, 0);
  if (last) {
    if (lane < U.nr) {
#pragma unroll
      for (int j = 0; j < KV; ++j) {
        T t = __ldcg(sp + lane * KV + j);
        for (int q = 1; q < np; ++q) t += __ldcg(sp + (q * 32 + lane) * KV + j);
        y[(int64_t)(U.row0 + lane) * KV + j] = t;
        if constexpr (KV == 1)
          for (int q = 0; q < P.npeer; ++q) P.peer[q][U.row0 + lane] = t;
      }
    }
    if (lane == 0) P.counters[counter] = 0;  // ready for the next launch
  }
}

template <typename T, int KV>
__global__ void __launch_bounds__(kUnitThreads, kUnitMinBlocks)
    unit_kernel(const __grid_constant__ UPlan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  __shared__ __align__(16) T buf_s[kUnitWarps][kRemWave * KV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = P.b0 + (int64_t)blockIdx.x * kUnitWarps + warp;
  if (b >= P.n_batches) return;
  // the batch bounds and its first unit: loads that depend only on b
  const int u0 = ldg_meta(P.batch + b), u1 = ldg_meta(P.batch + b + 1);
  Unit Un = load_unit(P.bhead + b);
  if ((P.pf & 1) && u1 - u0 > 1) {
    // the batch's data past its first unit -- contiguous ranges of the
    // panels, x maps, remainder pointers, columns and values -- into L2
    const Unit Ul = load_unit(P.units + u1 - 1);
    if (lane == 0) prefetch_span<T>(P, Un, Ul);
  }
  SABLE_DCHECK(u0 >= 0 && u0 <= u1 && u1 <= P.n_units);
  for (int u = u0; u < u1; ++u) {
    const Unit U = Un;
    if (u + 1 < u1) Un = load_unit(P.units + u + 1);
    SABLE_DCHECK(U.nr >= 1 && U.nr <= 32 && U.llpr <= 5 && U.row0 >= 0 && U.row0 + U.nr <= P.nloc);
    SABLE_DCHECK(U.wq == 0 || (U.wq > 0 && U.voff16 >= 0 &&
                               (int64_t)U.voff16 + (int64_t)U.nr * U.wq <= P.pv_vecs &&
                               U.xq0 >= 0 && (int64_t)U.xq0 + U.wq <= P.n_xq));
    SABLE_DCHECK(U.e0 >= 0 && U.e0 <= U.e1 && U.e1 <= P.rem_nnz);
    T s[KV];
#pragma unroll
    for (int j = 0; j < KV; ++j) s[j] = T(0);
    // the remainder's row bounds, in flight during the dense part
    const int ne = U.e1 - U.e0;
    int lo = 0, hi = 0;
    if (ne > 0 && lane < U.nr) {
      lo = max(ldg_meta(P.rptr + U.row0 + lane), U.e0);
      hi = min(ldg_meta(P.rptr + U.row0 + lane + 1), U.e1);
    }
    if (U.wq > 0) {
      switch (U.llpr) {
        case 0: dense_rows<T, 1, KV>(P, U, x, lane, s); break;
        case 1: dense_rows<T, 2, KV>(P, U, x, lane, s); break;
        case 2: dense_rows<T, 4, KV>(P, U, x, lane, s); break;
        case 3: dense_rows<T, 8, KV>(P, U, x, lane, s); break;
        case 4: dense_rows<T, 16, KV>(P, U, x, lane, s); break;
        default: dense_rows<T, 32, KV>(P, U, x, lane, s); break;
      }
    }
    if (ne > 0) rem_rows<T, KV>(P, U, x, buf_s[warp], lane, lo, hi, s);
    finish_unit<T, KV>(P, U, s, y, lane);
  }
}

template <typename T>
UPlan<T> make_plan(const sable_handle* h, void* scratch) {
  UPlan<T> P;
  P.units = h->units;
  P.batch = h->ubatch;
  P.bhead = h->ubhead;
  P.xq = h->xq;
  P.xside = h->xside;
  P.pv = static_cast<const T*>(h->pv);
  P.rptr = h->rem_ptr;
  P.ridx = h->rem_idx;
  P.rval = static_cast<const T*>(h->rem_val);
  P.xg = h->uxg;
  P.scratch = static_cast<T*>(scratch);
  P.counters = h->ucounters;
  P.b0 = 0;
  P.n_batches = h->n_ubatch;
  P.pf = h->cfg.pf;
  P.npeer = 0;
  for (int q = 0; q < kMaxPeers; ++q) P.peer[q] = nullptr;
  plan_extents<T>(P, h, 0);
  return P;
}

// One launch over warp batches [b0, b1).
template <typename T, int KV>
cudaError_t launch_kv(const sable_handle* h, const void* x, void* y, void* scratch,
                      cudaStream_t st, int64_t b0 = 0, int64_t b1 = -1,
                      void* const* peers = nullptr, int npeer = 0) {
  if (b1 < 0) b1 = h->n_ubatch;
  if (b1 <= b0) return cudaSuccess;
  if (npeer < 0 || npeer > kMaxPeers || (npeer > 0 && KV != 1)) return cudaErrorInvalidValue;
  UPlan<T> P = make_plan<T>(h, scratch);
  P.npeer = npeer;
  for (int q = 0; q < npeer; ++q) P.peer[q] = static_cast<T*>(peers[q]);
  P.scratch_elems = h->uscratch_slots * (scratch == h->uscratch ? 1 : KV);
  P.b0 = b0;
  P.n_batches = b1;
  const int64_t blocks = (b1 - b0 + kUnitWarps - 1) / kUnitWarps;
  unit_kernel<T, KV><<<(unsigned)blocks, kUnitThreads, 0, st>>>(P, static_cast<const T*>(x),
                                                                 static_cast<T*>(y));
  return cudaGetLastError();
}

}  // namespace

int32_t exec_grid(const sable_handle* h) {
  return h ? (int32_t)((h->n_ubatch + kUnitWarps - 1) / kUnitWarps) : 0;
}

// y = A x (one launch).
cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  return h->dtype == SABLE_F64 ? launch_kv<double, 1>(h, x, y, h->uscratch, st)
                               : launch_kv<float, 1>(h, x, y, h->uscratch, st);
}

// y = A x with the fused exchange epilogue: every y row is also stored at the
// same local row of the npeer peer buffers (comm.cu).
cudaError_t run_spmv_fused(const sable_handle* h, const void* x, void* y, void* const* peers,
                           int npeer, cudaStream_t st) {
  return h->dtype == SABLE_F64
             ? launch_kv<double, 1>(h, x, y, h->uscratch, st, 0, -1, peers, npeer)
             : launch_kv<float, 1>(h, x, y, h->uscratch, st, 0, -1, peers, npeer);
}

// y rows of exchange slice s only (its warp batches; comm.cu).
cudaError_t run_spmv_slice(const sable_handle* h, const void* x, void* y, int s,
                           cudaStream_t st) {
  const int64_t b0 = h->slice_batch[s], b1 = h->slice_batch[s + 1];
  return h->dtype == SABLE_F64 ? launch_kv<double, 1>(h, x, y, h->uscratch, st, b0, b1)
                               : launch_kv<float, 1>(h, x, y, h->uscratch, st, b0, b1);
}

// Y = A X for k in {1, 2, 4, 8} right-hand sides (X row-major ncols x k, Y
// row-major local rows x k); scratch holds k partials per combine slot.
cudaError_t run_spmm(const sable_handle* h, const void* X, void* Y, int32_t k, void* scratch,
                     cudaStream_t st) {
  const bool f64 = h->dtype == SABLE_F64;
  switch (k) {
    case 1: return f64 ? launch_kv<double, 1>(h, X, Y, scratch, st) : launch_kv<float, 1>(h, X, Y, scratch, st);
    case 2: return f64 ? launch_kv<double, 2>(h, X, Y, scratch, st) : launch_kv<float, 2>(h, X, Y, scratch, st);
    case 4: return f64 ? launch_kv<double, 4>(h, X, Y, scratch, st) : launch_kv<float, 4>(h, X, Y, scratch, st);
    case 8: return f64 ? launch_kv<double, 8>(h, X, Y, scratch, st) : launch_kv<float, 8>(h, X, Y, scratch, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sable
