// exec.cu -- the SpMV executor: y = A x over the VBR-C split (north_star (2)).
//
// y_i = sum_j A_ij x_j, evaluated as
//   y_r = sum over the dense tiles of r's block row  T(r, c) x_c      (dense)
//       + sum over r's remainder entries               v x_j          (CSR)
// -- the paper's "regular loops that operate over the entire block
// (including some zeros)" plus the CSR dispatch of low-delta
// blocks, re-designed as one data-driven sm_100a kernel
// instead of generated per-block C.
//
// One warp owns one work item = a piece of a row group (<= 32 rows of one
// block row; a piece covers some panel columns and/or a range of the group's
// remainder entries):
//   1. x staging: the panel columns' x values are gathered once into shared
//      memory (xs), coalesced per tile.
//   2. dense slab: lane l works on row l % nr and column phase l / nr
//      (Q = 32 / nr phases), so each warp load reads Q*nr consecutive values
//      of the column-major slab; 8 independent loads per lane are in flight
//      (streaming, evict-first); rows accumulate in registers and the phases
//      are folded with warp shuffles -- no atomics.
//   3. remainder: windows of kWin entries are multiplied with gathered x into
//      shared memory; lane r then sums the window part of row r in order.
//   4. y: a single-piece group writes y directly; a split group writes its
//      partials to scratch and the last piece to arrive (atomic counter) sums
//      them in piece order, so y is deterministic and independent of timing.
#include "sable_internal.cuh"

namespace sable {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kUnroll = 8;

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
  return __ldcs(p);  // read once: cache-streaming (evict-first)
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32)
    spmv_kernel(Plan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  __shared__ T xs_s[kWarps][kXCap];
  __shared__ T buf_s[kWarps][kWin];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t it = (int64_t)blockIdx.x * kWarps + warp;
  if (it >= P.n_items) return;
  T* xs = xs_s[warp];
  T* buf = buf_s[warp];
  const Item I = P.items[it];
  const Group G = P.groups[I.g];
  const int nr = G.nr;

  // ---- dense slab: panel columns [cb, ce) -------------------------------
  T acc = T(0);
  if (I.ce > I.cb) {
    const int cb = I.cb, ce = I.ce;
    for (int tb = G.t0; tb < G.t1; tb += 32) {
      TileDesc d{0, 0, 0};
      if (tb + lane < G.t1) d = P.tiles[tb + lane];
      const int nt = min(32, G.t1 - tb);
      for (int k = 0; k < nt; ++k) {
        const int c0 = __shfl_sync(kFull, d.c0, k);
        const int w = __shfl_sync(kFull, d.w, k);
        const int cs = __shfl_sync(kFull, d.cs, k);
        const int lo = max(cs, cb), hi = min(cs + w, ce);
        for (int c = lo + lane; c < hi; c += 32) xs[c - cb] = __ldg(x + c0 + (c - cs));
      }
    }
    __syncwarp();
    const int Q = 32 / nr;
    const int active = Q * nr;
    const int ph = lane / nr;
    if (lane < active) {
      const int n = ce - cb;
      const T* vp = P.tval + G.voff + (int64_t)cb * nr + lane;
      int c = ph;
      for (; c + (kUnroll - 1) * Q < n; c += kUnroll * Q) {
        T v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(vp + (int64_t)u * active);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) acc = fma(v[u], xs[c + u * Q], acc);
        vp += (int64_t)kUnroll * active;
      }
      for (; c < n; c += Q) {
        acc = fma(ld_stream(vp), xs[c], acc);
        vp += active;
      }
    }
    for (int off = 1; off < Q; off <<= 1) {
      const T o = __shfl_down_sync(kFull, acc, off * nr);
      if (lane < active && ph + off < Q) acc += o;
    }
  }

  // ---- remainder entries [eb, ee) -----------------------------------------
  T racc = T(0);
  if (I.ee > I.eb) {
    int32_t plo = 0, phi = 0;
    if (lane < nr) {
      plo = P.rem_ptr[G.row0 + lane];
      phi = P.rem_ptr[G.row0 + lane + 1];
    }
    for (int64_t ws = I.eb; ws < I.ee; ws += kWin) {
      int32_t col[kWin / 32];
      T val[kWin / 32];
#pragma unroll
      for (int k = 0; k < kWin / 32; ++k) {
        const int64_t e = ws + k * 32 + lane;
        col[k] = 0;
        val[k] = T(0);
        if (e < I.ee) {
          col[k] = ld_stream(P.rem_idx + e);
          val[k] = ld_stream(P.rem_val + e);
        }
      }
#pragma unroll
      for (int k = 0; k < kWin / 32; ++k) buf[k * 32 + lane] = val[k] * __ldg(x + col[k]);
      __syncwarp();
      if (lane < nr) {
        const int64_t lo = max((int64_t)plo, ws);
        const int64_t hi = min(min((int64_t)phi, ws + kWin), I.ee);
        for (int64_t e = lo; e < hi; ++e) racc += buf[e - ws];
      }
      __syncwarp();
    }
  }
  const T tot = acc + racc;

  // ---- y ------------------------------------------------------------------
  if (G.npieces == 1) {
    if (lane < nr) y[G.row0 + lane] = tot;
    return;
  }
  T* sp = P.scratch + G.slot;
  if (lane < nr) sp[I.p * 32 + lane] = tot;
  __threadfence();
  __syncwarp();
  int last = 0;
  if (lane == 0) last = (atomicAdd(P.counters + I.g, 1) == G.npieces - 1);
  last = __shfl_sync(kFull, last, 0);
  if (last) {
    __threadfence();
    if (lane < nr) {
      T s = __ldcg(sp + lane);
      for (int q = 1; q < G.npieces; ++q) s += __ldcg(sp + q * 32 + lane);
      y[G.row0 + lane] = s;
    }
    if (lane == 0) P.counters[I.g] = 0;  // ready for the next launch
  }
}

template <typename T>
cudaError_t launch_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  if (h->n_items == 0) return cudaSuccess;
  Plan<T> P;
  P.items = h->items;
  P.groups = h->groups;
  P.tiles = h->tiles;
  P.tval = static_cast<const T*>(h->tval);
  P.rem_ptr = h->rem_ptr;
  P.rem_idx = h->rem_idx;
  P.rem_val = static_cast<const T*>(h->rem_val);
  P.scratch = static_cast<T*>(h->scratch);
  P.counters = h->counters;
  P.n_items = h->n_items;
  const int64_t grid = (h->n_items + kWarps - 1) / kWarps;
  spmv_kernel<T><<<(unsigned)grid, kWarps * 32, 0, st>>>(P, static_cast<const T*>(x),
                                                        static_cast<T*>(y));
  return cudaGetLastError();
}

cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  return h->dtype == SABLE_F64 ? launch_spmv<double>(h, x, y, st)
                               : launch_spmv<float>(h, x, y, st);
}

}  // namespace sable
