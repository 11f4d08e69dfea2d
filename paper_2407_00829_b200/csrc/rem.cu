// rem.cu -- the CSR remainder executor (north_star (2): "warp-per-row for the
// CSR remainder"; the paper dispatches its low-delta blocks to a CSR SpMV,
// PAPER.md:129).
//
// Runs FIRST on the stream and writes every local row: y_r = the sum of r's
// remainder entries v * x_j (0 if none); the dense-tile executor then adds
// its part to the rows of block rows with tiles.  (a + b == b + a in IEEE
// arithmetic, so y is the same as with the dense part first.)
//
// A warp takes a packet of whole consecutive rows (<= kPacketEntries
// entries): its lanes load the packet's columns and values (coalesced, 8 per
// lane in flight), gather x, and leave the products in the warp's shared
// buffer; then lane l sums the products of rows l, l + 32, ... in entry
// order and writes them.  A row longer than kPieceLen is cut into pieces of
// kPieceLen entries, one warp each, summed by a fixed tree; the last piece
// to arrive adds the pieces in order.  The summation order of a row depends
// on the row alone, so y is the same for every shard count.
#include "sable_internal.cuh"

namespace sable {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRemThreads = 256;

__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

constexpr int kWarpsR = kRemThreads / 32;
#ifndef SABLE_REM_KB
#define SABLE_REM_KB 8
#endif
constexpr int kB = SABLE_REM_KB;  // loads per lane in flight (A/B builds: -DSABLE_REM_KB=N)

#ifndef SABLE_REM_MINB
#define SABLE_REM_MINB 1  // A/B builds: -DSABLE_REM_MINB=N asks for N resident blocks per SM
#endif

template <typename T>
__global__ void __launch_bounds__(kRemThreads, SABLE_REM_MINB)
    rem_kernel(RemPlan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  __shared__ T prod_s[kWarpsR][kPacketEntries];
  __shared__ int32_t ptr_s[kWarpsR][kPacketRows + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t wid = (int64_t)blockIdx.x * kWarpsR + warp; wid < P.n_packets;
       wid += (int64_t)gridDim.x * kWarpsR) {
  const RemPacket pk = P.packets[wid];
  __syncwarp();  // the previous packet's shared buffers are free
  if (pk.r1 >= 0) {
    // whole rows [r0, r1): products of their entries, then lane-per-row sums
    T* prod = prod_s[warp];
    int32_t* pt = ptr_s[warp];
    const int n = pk.e1 - pk.e0, nrow = pk.r1 - pk.r0;
    // the packet's row pointers, loaded with the first wave of entry loads
    for (int i = lane; i <= nrow; i += 32) pt[i] = __ldg(P.ptr + pk.r0 + i) - pk.e0;
    for (int w = 0; w < n; w += 32 * kB) {
      int32_t c[kB];
      T v[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int e = w + k * 32 + lane;
        c[k] = 0;
        v[k] = T(0);
        if (e < n) {
          c[k] = __ldcs(P.idx + pk.e0 + e);
          v[k] = __ldcs(P.val + pk.e0 + e);
        }
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int e = w + k * 32 + lane;
        if (e < n) prod[e] = v[k] * __ldg(x + c[k]);
      }
    }
    __syncwarp();
    // lane l sums rows l, l + 32, ...; a row longer than 32 entries is summed
    // by the whole warp (strided, then a fixed shuffle tree), so a packet's
    // time does not hang on its longest row
    for (int r0 = pk.r0; r0 < pk.r1; r0 += 32) {
      const int r = r0 + lane;
      int lo = 0, hi = 0;
      if (r < pk.r1) {
        lo = pt[r - pk.r0];
        hi = pt[r - pk.r0 + 1];
      }
      const bool longr = hi - lo > 32;
      T s = T(0);
      if (!longr)
        for (int e = lo; e < hi; ++e) s += prod[e];
      unsigned lm = __ballot_sync(kFull, longr);
      while (lm) {
        const int q = __ffs(lm) - 1;
        lm &= lm - 1;
        const int l2 = __shfl_sync(kFull, lo, q), h2 = __shfl_sync(kFull, hi, q);
        T t = T(0);
        for (int e = l2 + lane; e < h2; e += 32) t += prod[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
        if (lane == q) s = t;
      }
      if (r < pk.r1) y[r] = s;
    }
  } else {
    // one piece of a long row
    const int piece = -1 - pk.r1;
    const int n = pk.e1 - pk.e0;
    T a0 = T(0), a1 = T(0);
    for (int w = 0; w < n; w += 32 * kB) {
      int32_t c[kB];
      T v[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int e = w + k * 32 + lane;
        c[k] = 0;
        v[k] = T(0);
        if (e < n) {
          c[k] = __ldcs(P.idx + pk.e0 + e);
          v[k] = __ldcs(P.val + pk.e0 + e);
        }
      }
#pragma unroll
      for (int k = 0; k < kB; k += 2) {
        a0 = fma(v[k], __ldg(x + c[k]), a0);
        a1 = fma(v[k + 1], __ldg(x + c[k + 1]), a1);
      }
    }
    T acc = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    T* sp = P.scratch + pk.slot;
    if (lane == 0) __stcg(sp + piece, acc);
    __syncwarp();
    int last = 0;
    if (lane == 0) last = (atom_add_acq_rel(P.counters + pk.counter, 1) + 1 == pk.npieces);
    last = __shfl_sync(kFull, last, 0);
    if (last && lane == 0) {
      T sum = __ldcg(sp);
      for (int q = 1; q < pk.npieces; ++q) sum += __ldcg(sp + q);
      y[pk.r0] = sum;
      P.counters[pk.counter] = 0;  // ready for the next launch
    }
  }
  }
}

}  // namespace

template <typename T>
cudaError_t launch_rem(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  if (h->rp.n_packets == 0) return cudaSuccess;
  RemPlan<T> P;
  P.packets = h->rp.packets;
  P.ptr = h->rem_ptr;
  P.idx = h->rem_idx;
  P.val = static_cast<const T*>(h->rem_val);
  P.scratch = static_cast<T*>(h->rp.scratch);
  P.counters = h->rp.counters;
  P.n_packets = h->rp.n_packets;
  // one warp per packet, or (SABLE_REM_GRID = blocks > 0) a persistent grid
  // whose warps stride over the packets
  int64_t blocks = (h->rp.n_packets + kWarpsR - 1) / kWarpsR;
  if (h->cfg.rem_grid > 0) blocks = std::min<int64_t>(blocks, h->cfg.rem_grid);
  rem_kernel<T><<<(unsigned)blocks, kRemThreads, 0, st>>>(P, static_cast<const T*>(x),
                                                         static_cast<T*>(y));
  return cudaGetLastError();
}

template cudaError_t launch_rem<float>(const sable_handle*, const void*, void*, cudaStream_t);
template cudaError_t launch_rem<double>(const sable_handle*, const void*, void*, cudaStream_t);

}  // namespace sable
