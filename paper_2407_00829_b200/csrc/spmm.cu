// spmm.cu -- multi-vector products Y = A X: k right-hand
// sides in one pass over the inspected matrix, so the tile stream and the
// remainder are read once for all k vectors instead of k times -- the
// "user-defined operation" generality of PAPER.md:268, 482 over the same
// VBR-C split.  Y[:, j] = A X[:, j] is y_i = sum_j A_ij x_j
// for every column.
//
// X is row-major ncols x k (the k values of one matrix column contiguous),
// Y row-major nloc x k.  The executors mirror exec.cu / rem.cu (the dense
// CTA ring of arch 1 and the packet remainder), with k accumulators per lane
// and one vector load of k x values per matrix column.  Sums run in a fixed
// order per row (deterministic), not the SpMV's order.
#include <algorithm>

#include "sable_internal.cuh"

namespace sable {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void issue_chunk(const unsigned char* stream, const ChunkRef& c,
                                            unsigned char* stage, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"((uint32_t)c.bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(stage)),
      "l"(stream + c.off), "r"((uint32_t)c.bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// k consecutive x values of one matrix column
template <typename T, int K>
__device__ __forceinline__ void load_xk(const T* __restrict__ p, T (&v)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) v[j] = __ldg(p + j);
}

struct MmPlan {
  const unsigned char* stream;
  const ChunkRef* cref;
  const int32_t* task;
  const XgInfo* xgi;
  int32_t* counters;
  int32_t nstage, stage_bytes;
};

// One bundle (see exec.cu process_bundle) with K right-hand sides.
template <typename T, int K>
__device__ __forceinline__ void bundle_k(const MmPlan& P, T* __restrict__ scratch,
                                         const unsigned char* stage, int b,
                                         const T* __restrict__ X, T* __restrict__ Y, int lane) {
  const ChunkHdr& H = *reinterpret_cast<const ChunkHdr*>(stage);
  const SItem* items = reinterpret_cast<const SItem*>(stage + H.o_item);
  const uint32_t* lmap = reinterpret_cast<const uint32_t*>(stage + H.o_lane);
  const XRun* runs = reinterpret_cast<const XRun*>(stage + H.o_gath);
  const T* val = reinterpret_cast<const T*>(stage + H.o_val);
  const uint32_t m = lmap[b * 32 + lane];
  const bool valid = (m & kLaneValid) != 0;
  const int r = (m >> 8) & 31, ph = (m >> 13) & 31, lq = (m >> 18) & 7, Q = 1 << lq;
  SItem I{};
  if (valid) I = items[m & 255];
  const int nr = I.nr;
  T acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = T(0);
  if (valid && ph < I.ncol) {
    int k = I.xb;
    XRun R = runs[k];
    while (R.cend <= ph) R = runs[++k];
    const T* vp = val + I.v + ph * nr + r;
    const int step = Q * nr;
    int c = ph;
    for (;;) {
      const int n = (min((int)R.cend, (int)I.ncol) - c + Q - 1) >> lq;
      const T* xp = X + (int64_t)(R.off + c) * K;
      for (int i = 0; i < n; ++i) {
        T xv[K];
        load_xk<T, K>(xp, xv);
        const T v = *vp;
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = fma(v, xv[j], acc[j]);
        vp += step;
        xp += (int64_t)Q * K;
      }
      c += n << lq;
      if (c >= I.ncol) break;
      do R = runs[++k];
      while (R.cend <= c);
    }
  }
  // fold the phases (binary tree fixed by Q and nr)
  const int lqmax = __reduce_max_sync(kFull, (unsigned)(valid ? lq : 0));
  for (int l = 0; l < lqmax; ++l) {
    const int d = (1 << l) * nr;
    const bool take = valid && ((ph >> l) & 1) == 0 && ph + (1 << l) < Q;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const T o = __shfl_sync(kFull, acc[j], min(lane + d, 31));
      if (take) acc[j] += o;
    }
  }
  if (valid && ph == 0 && !(I.flags & IF_XG)) {
#pragma unroll
    for (int j = 0; j < K; ++j) Y[(int64_t)(I.row0 + r) * K + j] += acc[j];
  }
  if (__any_sync(kFull, valid && (I.flags & IF_XG))) {
    const int nr0 = __shfl_sync(kFull, nr, 0), row0 = __shfl_sync(kFull, I.row0, 0);
    const XgInfo xi = P.xgi[(int64_t)H.i0 + (lmap[b * 32] & 255)];
    T* sp = scratch + xi.slot * K;
    if (valid && ph == 0) {
#pragma unroll
      for (int j = 0; j < K; ++j) __stcg(sp + (xi.p * 32 + r) * K + j, acc[j]);
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) last = (atom_add_acq_rel(P.counters + xi.g, 1) + 1 == xi.npieces);
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      if (lane < nr0) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          T sum = __ldcg(sp + lane * K + j);
          for (int q = 1; q < xi.npieces; ++q) sum += __ldcg(sp + (q * 32 + lane) * K + j);
          Y[(int64_t)(row0 + lane) * K + j] += sum;
        }
      }
      if (lane == 0) P.counters[xi.g] = 0;
    }
  }
}

constexpr int kMmThreads = (kCons + 1) * 32;

// The dense-tile executor for K vectors: arch 1's CTA ring (producer warp +
// kCons consumer warps grabbing bundles).
template <typename T, int K>
__global__ void __launch_bounds__(kMmThreads)
    spmm_cta_kernel(MmPlan P, T* __restrict__ scratch, const T* __restrict__ X,
                    T* __restrict__ Y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t kb = P.task[blockIdx.x], ke = P.task[blockIdx.x + 1];
  const int n = (int)(ke - kb);
  if (n <= 0) return;
  const int NS = P.nstage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  int* next = reinterpret_cast<int*>(empty + kMaxStages);
  unsigned char* stages = smem + 256;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(empty + s), kCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kCons) {
    int s = 0, pass = 0;
    for (int it = 0; it < n; ++it) {
      unsigned char* stage = stages + (size_t)s * P.stage_bytes;
      ChunkRef ref;
      if (pass > 0) {
        mbar_wait(smem_u32(empty + s), (uint32_t)((pass - 1) & 1));
        ref = reinterpret_cast<const ChunkHdr*>(stage)->next;
      } else {
        ref = P.cref[kb + it];
      }
      __syncwarp();
      if (lane == 0) {
        next[s] = 0;
        issue_chunk(P.stream, ref, stage, smem_u32(full + s));
      }
      if (++s == NS) { s = 0; ++pass; }
    }
    return;
  }
  int s = 0, pass = 0;
  for (int it = 0; it < n; ++it) {
    const unsigned char* stage = stages + (size_t)s * P.stage_bytes;
    mbar_wait(smem_u32(full + s), (uint32_t)(pass & 1));
    const int nb = reinterpret_cast<const ChunkHdr*>(stage)->nb;
    for (;;) {
      int b = 0;
      if (lane == 0) b = atomicAdd(next + s, 1);
      b = __shfl_sync(kFull, b, 0);
      if (b >= nb) break;
      bundle_k<T, K>(P, scratch, stage, b, X, Y, lane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + s));
    if (++s == NS) { s = 0; ++pass; }
  }
}

constexpr int kRemMmThreads = 128;
constexpr int kWarpsMm = kRemMmThreads / 32;

// The remainder for K vectors: a warp per packet of whole rows stages the
// packet's (column, value) pairs in shared memory, then lane l sums rows
// l, l + 32, ... in entry order for all K vectors; pieces of long rows are
// summed by the whole warp and combined in order by the last to arrive.
template <typename T, int K>
__global__ void __launch_bounds__(kRemMmThreads)
    rem_mm_kernel(const RemPacket* __restrict__ packets, int64_t n_packets,
                  const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                  const T* __restrict__ valr, T* __restrict__ scratch, int32_t* counters,
                  const T* __restrict__ X, T* __restrict__ Y) {
  __shared__ int32_t col_s[kWarpsMm][kPacketEntries];
  __shared__ T val_s[kWarpsMm][kPacketEntries];
  __shared__ int32_t ptr_s[kWarpsMm][kPacketRows + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * kWarpsMm + warp;
  if (wid >= n_packets) return;
  const RemPacket pk = packets[wid];
  if (pk.r1 >= 0) {
    const int ne = pk.e1 - pk.e0, nrow = pk.r1 - pk.r0;
    for (int i = lane; i <= nrow; i += 32) ptr_s[warp][i] = __ldg(ptr + pk.r0 + i) - pk.e0;
    for (int e = lane; e < ne; e += 32) {
      col_s[warp][e] = __ldcs(idx + pk.e0 + e);
      val_s[warp][e] = __ldcs(valr + pk.e0 + e);
    }
    __syncwarp();
    for (int r = pk.r0 + lane; r < pk.r1; r += 32) {
      T s[K];
#pragma unroll
      for (int j = 0; j < K; ++j) s[j] = T(0);
      const int lo = ptr_s[warp][r - pk.r0], hi = ptr_s[warp][r - pk.r0 + 1];
      for (int e = lo; e < hi; ++e) {
        T xv[K];
        load_xk<T, K>(X + (int64_t)col_s[warp][e] * K, xv);
        const T v = val_s[warp][e];
#pragma unroll
        for (int j = 0; j < K; ++j) s[j] = fma(v, xv[j], s[j]);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) Y[(int64_t)r * K + j] = s[j];
    }
  } else {
    const int piece = -1 - pk.r1;
    T a[K];
#pragma unroll
    for (int j = 0; j < K; ++j) a[j] = T(0);
    for (int e = pk.e0 + lane; e < pk.e1; e += 32) {
      T xv[K];
      load_xk<T, K>(X + (int64_t)__ldcs(idx + e) * K, xv);
      const T v = __ldcs(valr + e);
#pragma unroll
      for (int j = 0; j < K; ++j) a[j] = fma(v, xv[j], a[j]);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a[j] += __shfl_xor_sync(kFull, a[j], o);
    }
    T* sp = scratch + (int64_t)pk.slot * K;
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < K; ++j) __stcg(sp + piece * K + j, a[j]);
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) last = (atom_add_acq_rel(counters + pk.counter, 1) + 1 == pk.npieces);
    last = __shfl_sync(kFull, last, 0);
    if (last && lane < K) {
      T sum = __ldcg(sp + lane);
      for (int q = 1; q < pk.npieces; ++q) sum += __ldcg(sp + q * K + lane);
      Y[(int64_t)pk.r0 * K + lane] = sum;
    }
    if (last && lane == 0) counters[pk.counter] = 0;
  }
}

template <typename T, int K>
cudaError_t launch_k(sable_handle* h, const void* X, void* Y, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (h->rp.n_packets > 0) {
    const int64_t blocks = (h->rp.n_packets + kWarpsMm - 1) / kWarpsMm;
    rem_mm_kernel<T, K><<<(unsigned)blocks, kRemMmThreads, 0, st>>>(
        h->rp.packets, h->rp.n_packets, h->rem_ptr, h->rem_idx, static_cast<const T*>(h->rem_val),
        static_cast<T*>(h->mm_rscratch), h->rp.counters, static_cast<const T*>(X),
        static_cast<T*>(Y));
    e = cudaGetLastError();
    if (e) return e;
  }
  if (h->n_chunks == 0) return cudaSuccess;
  MmPlan P;
  P.stream = h->stream;
  P.cref = h->cref;
  P.task = h->task;
  P.xgi = h->xgi;
  P.counters = h->counters;
  P.nstage = h->cfg.nstage;
  P.stage_bytes = h->cfg.stage_bytes;
  const size_t smem = 256 + (size_t)P.nstage * P.stage_bytes;
  e = cudaFuncSetAttribute(spmm_cta_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
  if (e) return e;
  spmm_cta_kernel<T, K><<<(unsigned)h->cfg.n_tasks, kMmThreads, smem, st>>>(
      P, static_cast<T*>(h->mm_scratch), static_cast<const T*>(X), static_cast<T*>(Y));
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_t(sable_handle* h, int k, const void* X, void* Y, cudaStream_t st) {
  switch (k) {
    case 1: return launch_k<T, 1>(h, X, Y, st);
    case 2: return launch_k<T, 2>(h, X, Y, st);
    case 4: return launch_k<T, 4>(h, X, Y, st);
    case 8: return launch_k<T, 8>(h, X, Y, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

}  // namespace sable

using namespace sable;

extern "C" sable_status sable_spmm(sable_handle* h, const void* X, void* Y, int32_t k,
                                   void* cuda_stream) {
  if (!h || !X || !Y) {
    set_error("sable_spmm: NULL argument");
    return SABLE_E_INVALID_ARG;
  }
  if (k != 1 && k != 2 && k != 4 && k != 8) {
    set_error("sable_spmm: k must be 1, 2, 4 or 8");
    return SABLE_E_UNSUPPORTED;
  }
  if (h->cfg.arch == 0 && h->n_chunks > 0) {
    set_error("sable_spmm: needs the CTA-ring executor plan (SABLE_ARCH=1, the default)");
    return SABLE_E_UNSUPPORTED;
  }
  const size_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // k-wide scratch for split groups / long-row pieces: allocated once, for k = 8
  if (!h->mm_scratch) {
    cudaError_t e = cudaMalloc(&h->mm_scratch, sv * 8 * (size_t)std::max<int64_t>(h->scratch_elems, 1));
    if (!e) e = cudaMalloc(&h->mm_rscratch, sv * 8 * (size_t)std::max<int64_t>(h->rp.n_pieces, 1));
    if (e) {
      set_error(cuda_msg(e, "sable_spmm scratch"));
      return e == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA;
    }
  }
  const cudaError_t e = h->dtype == SABLE_F64 ? launch_t<double>(h, k, X, Y, st)
                                              : launch_t<float>(h, k, X, Y, st);
  if (e) {
    set_error(cuda_msg(e, "sable_spmm"));
    return SABLE_E_CUDA;
  }
  return SABLE_OK;
}
