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
// The input is one byte stream of self-describing chunks (built by the
// inspector).  Every warp owns a task: a contiguous range of chunks of about
// equal bytes.  Lane 0 streams the task's chunks through a private ring of
// shared-memory stages, ONE 1-D bulk copy per chunk (cp.async.bulk, L2
// evict-first, completion on the stage's mbarrier); a chunk's header names
// the chunk nstage ahead, so no warp ever waits on a descriptor and no warp
// waits on another.  While chunk k is computed, the x lines chunk k + 1 will
// read are prefetched into L1 (one prefetch per 128-byte line of each run of
// consecutive global columns).  Chunk k is computed bundle by bundle: a
// bundle maps the 32 lanes onto the rows of several items -- lane = (item,
// row r, phase ph of Q) -- chosen by the planner so that the lanes' work is
// even; a lane sums columns ph, ph + Q, ... of its row of the column-major
// slab from shared memory times x read through L1 (x of column c is
// x[off + c] of the run holding c); the phases fold with shuffles; the row
// is written once.  Pieces of
// a group larger than a stage are summed left to right in registers (or, if
// two tasks share the group, in global scratch by the last piece to arrive).
// No atomics on y; every row's summation order depends on the matrix alone,
// so y is bitwise reproducible and identical for every shard count.
#include "sable_internal.cuh"

namespace sable {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = kWarps * 32;

// A/B builds: -DSABLE_INNER_UNROLL=N unrolls a lane's column loop N times
#if defined(SABLE_INNER_UNROLL) && SABLE_INNER_UNROLL > 0
#define SABLE_STR2(x) #x
#define SABLE_STR(x) SABLE_STR2(x)
#define SABLE_INNER_PRAGMA _Pragma(SABLE_STR(unroll SABLE_INNER_UNROLL))
#else
#define SABLE_INNER_PRAGMA
#endif

// ---------------------------------------------------------------- PTX glue

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

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_unchanged() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// Arrival counter of a group split over tasks: release this warp's scratch
// writes (ordered before by __syncwarp), acquire the other tasks'.
__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------- chunks

// Lane 0: start the copy of a chunk into a stage.
__device__ __forceinline__ void issue_chunk(const unsigned char* stream, const ChunkRef& c,
                                            unsigned char* stage, uint32_t bar, uint64_t pol) {
  mbar_expect_tx(bar, (uint32_t)c.bytes);
  bulk_g2s(smem_u32(stage), stream + c.off, (uint32_t)c.bytes, bar, pol);
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Bring the x lines a staged chunk will read into L1 (one prefetch per 128-B
// line of each x run), while the previous chunk is computed.
template <typename T>
__device__ __forceinline__ void prefetch_chunk(const unsigned char* stage,
                                               const T* __restrict__ x, int lane) {
  const ChunkHdr& H = *reinterpret_cast<const ChunkHdr*>(stage);
  const XRun* xr = reinterpret_cast<const XRun*>(stage + H.o_gath);
  constexpr int kLine = 128 / (int)sizeof(T);
  for (int g = lane; g < H.ng; g += 32) {
    const XRun R = xr[g];
    const T* p = x + R.off;
    prefetch_l1(p + R.cbeg);
    for (int c = R.cbeg + kLine; c < R.cend; c += kLine) prefetch_l1(p + c);
    prefetch_l1(p + R.cend - 1);
  }
}

// One bundle of a staged chunk: lane = (item, row r, phase ph of Q) sums
// columns ph, ph + Q, ... of row r, the phases fold, the row is written (or,
// for a piece of a split group, summed in `run` / met in global scratch).
template <typename T>
__device__ __forceinline__ void process_bundle(const Plan<T>& P, const unsigned char* stage, int b,
                                               const T* __restrict__ x, T* __restrict__ y,
                                               T& run, int lane) {
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
  T acc = T(0);
  if (valid && ph < I.ncol) {
    // columns ph, ph + Q, ... of row r, run by run (x of column c is
    // x[off + c] in the run holding c), one accumulator in column order
    int k = I.xb;
    XRun R = runs[k];
    while (R.cend <= ph) R = runs[++k];
    const T* vp = val + I.v + ph * nr + r;
    const int step = Q * nr;
    int c = ph;
    for (;;) {
      const T* xp = x + R.off + c;
      const int n = (R.cend - c + Q - 1) >> lq;  // this lane's columns in the run
      SABLE_INNER_PRAGMA
      for (int i = 0; i < n; ++i) {
        acc = fma(*vp, __ldg(xp), acc);
        vp += step;
        xp += Q;
      }
      c += n << lq;
      if (c >= I.ncol) break;
      do R = runs[++k];
      while (R.cend <= c);
    }
  }
  // fold the phases: lane ph * nr + r collects ph + 1, ph + 2, ... in order
  // of a binary tree (fixed by Q and nr: deterministic)
  const int lqmax = __reduce_max_sync(kFull, (unsigned)(valid ? lq : 0));
  for (int l = 0; l < lqmax; ++l) {
    const int d = (1 << l) * nr;
    const T o = __shfl_sync(kFull, acc, min(lane + d, 31));
    if (valid && ((ph >> l) & 1) == 0 && ph + (1 << l) < Q) acc += o;
  }
  if (valid && ph == 0) {
    if (!(I.flags & IF_XG)) {
      run = (I.flags & IF_FIRST) ? acc : run + acc;
      if (I.flags & IF_LAST) y[I.row0 + r] += run;  // y holds the remainder part
    }
  }
  // a piece of a group shared with another task (alone in its bundle, so
  // lane 0 holds row 0 of it): meet in global scratch
  if (__any_sync(kFull, valid && (I.flags & IF_XG))) {
    const int nr0 = __shfl_sync(kFull, nr, 0), row0 = __shfl_sync(kFull, I.row0, 0);
    const XgInfo xi = P.xgi[(int64_t)H.i0 + (lmap[b * 32] & 255)];
    T* sp = P.scratch + xi.slot;
    if (valid && ph == 0) __stcg(sp + xi.p * 32 + r, acc);
    __syncwarp();
    int last = 0;
    if (lane == 0) last = (atom_add_acq_rel(P.counters + xi.g, 1) + 1 == xi.npieces);
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      if (lane < nr0) {
        T sum = __ldcg(sp + lane);
        for (int q = 1; q < xi.npieces; ++q) sum += __ldcg(sp + q * 32 + lane);
        y[row0 + lane] += sum;
      }
      if (lane == 0) P.counters[xi.g] = 0;  // ready for the next launch
    }
  }

}

template <typename T>
__device__ __forceinline__ void compute_chunk(const Plan<T>& P, const unsigned char* stage,
                                              const T* __restrict__ x, T* __restrict__ y,
                                              T& run, int lane) {
  const ChunkHdr& H = *reinterpret_cast<const ChunkHdr*>(stage);
#pragma unroll 1
  for (int b = 0; b < H.nb; ++b) process_bundle(P, stage, b, x, y, run, lane);
}

// ---------------------------------------------------------------- kernel

template <typename T>
__global__ void __launch_bounds__(kThreads)
    spmv_kernel(Plan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t task = (int64_t)blockIdx.x * kWarps + warp;
  if (task >= P.n_tasks) return;
  const int64_t kb = P.task[task], ke = P.task[task + 1];
  if (kb >= ke) return;
  const int NS = P.nstage;
  unsigned char* ws =
      smem + (size_t)warp * warp_smem_bytes(NS, P.stage_bytes, P.xbuf, (int)sizeof(T));
  uint64_t* full = reinterpret_cast<uint64_t*>(ws);  // [kMaxStages]
  unsigned char* stages = ws + 256;

  uint64_t pol = 0;
  if (lane == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < NS; ++s) mbar_init(smem_u32(full + s), 1);
    fence_barrier_init();
    for (int s = 0; s < NS && kb + s < ke; ++s)
      issue_chunk(P.stream, P.cref[kb + s], stages + (size_t)s * P.stage_bytes,
                  smem_u32(full + s), pol);
  }
  __syncwarp();

  // chunk k computes from stage s while chunk k + 1's x lines are being
  // prefetched into L1
  int s = 0;
  uint32_t phase = 0;
  mbar_wait(smem_u32(full + 0), 0);
  if (P.mode != 1) prefetch_chunk(stages, x, lane);
  T run = T(0);  // running sum of a split group's pieces (lanes < nr)
  for (int64_t k = kb; k < ke; ++k) {
    int sn = s + 1;
    uint32_t phn = phase;
    if (sn == NS) {
      sn = 0;
      phn ^= 1u;
    }
    unsigned char* stage = stages + (size_t)s * P.stage_bytes;
    if (k + 1 < ke) {
      unsigned char* nst = stages + (size_t)sn * P.stage_bytes;
      mbar_wait(smem_u32(full + sn), phn);
      if (P.mode != 1) prefetch_chunk(nst, x, lane);
    }
    if (P.mode != 1) compute_chunk(P, stage, x, y, run, lane);
    // refill this stage with the chunk nstage ahead (named by this header)
    __syncwarp();
    if (lane == 0) {
      const ChunkRef nx = reinterpret_cast<const ChunkHdr*>(stage)->next;
      if (nx.bytes > 0) issue_chunk(P.stream, nx, stage, smem_u32(full + s), pol);
    }
    __syncwarp();
    s = sn;
    phase = phn;
  }
}

// arch 1: one CTA = kCons consumer warps + a producer warp sharing a ring of
// stages.  The producer streams the CTA's chunks (one bulk copy each, after
// the consumers released the stage) and prefetches each landed chunk's x
// lines into L1; the consumers grab the bundles of the oldest staged chunk
// with a shared-memory counter and release the stage when it is exhausted.
constexpr int kCtaThreads = (kCons + 1) * 32;

template <typename T>
__global__ void __launch_bounds__(kCtaThreads, cta_regs_occupancy(sizeof(T)))
    spmv_cta_kernel(Plan<T> P, const T* __restrict__ x, T* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t kb = P.task[blockIdx.x], ke = P.task[blockIdx.x + 1];
  const int64_t nk = ke - kb;
  if (nk <= 0) return;
  const int NS = P.nstage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);        // [kMaxStages]
  uint64_t* empty = full + kMaxStages;                        // [kMaxStages]
  int* next = reinterpret_cast<int*>(empty + kMaxStages);     // [kMaxStages]
  unsigned char* stages = smem + 256;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(empty + s), kCons);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCons) {
    // ---- producer (stage s and ring pass `pass` kept incrementally: no
    // 64-bit division per chunk)
    const uint64_t pol = (P.xpf & 2) ? policy_evict_unchanged() : policy_evict_first();
    const int n = (int)nk;
    int s = 0, pass = 0;    // chunk it -> stage s, pass = it / NS
    int sp = 0, passp = 0;  // chunk it - 2 (x prefetch)
    for (int it = 0; it < n; ++it) {
      unsigned char* stage = stages + (size_t)s * P.stage_bytes;
      ChunkRef ref;
      if (pass > 0) {
        mbar_wait(smem_u32(empty + s), (uint32_t)((pass - 1) & 1));
        ref = reinterpret_cast<const ChunkHdr*>(stage)->next;  // chunk it, named by chunk it - NS
      } else {
        ref = P.cref[kb + it];
      }
      __syncwarp();
      if (lane == 0) {
        next[s] = 0;
        issue_chunk(P.stream, ref, stage, smem_u32(full + s), pol);
      }
      if (it >= 2 && P.mode != 1 && (P.xpf & 1)) {  // chunk it - 2 has landed: prefetch its x
        mbar_wait(smem_u32(full + sp), (uint32_t)(passp & 1));
        prefetch_chunk(stages + (size_t)sp * P.stage_bytes, x, lane);
        if (++sp == NS) { sp = 0; ++passp; }
      }
      if (++s == NS) { s = 0; ++pass; }
    }
    for (int it = n - 2 < 0 ? 0 : n - 2; it < n && P.mode != 1 && (P.xpf & 1); ++it) {
      mbar_wait(smem_u32(full + sp), (uint32_t)(passp & 1));
      prefetch_chunk(stages + (size_t)sp * P.stage_bytes, x, lane);
      if (++sp == NS) { sp = 0; ++passp; }
    }
    return;
  }
  // ---- consumers
  T run = T(0);
  int s = 0, pass = 0;
  for (int it = 0; it < (int)nk; ++it) {
    const unsigned char* stage = stages + (size_t)s * P.stage_bytes;
    mbar_wait(smem_u32(full + s), (uint32_t)(pass & 1));
    if (P.mode != 1) {
      const int nb = reinterpret_cast<const ChunkHdr*>(stage)->nb;
      for (;;) {
        int b = 0;
        if (lane == 0) b = atomicAdd(next + s, 1);
        b = __shfl_sync(kFull, b, 0);
        if (b >= nb) break;
        process_bundle(P, stage, b, x, y, run, lane);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + s));
    if (++s == NS) { s = 0; ++pass; }
  }
}

}  // namespace

int32_t exec_grid(const sable_handle* h) {
  if (h && h->cfg.arch == 2) return (int32_t)((h->n_ubatch + kUnitWarps - 1) / kUnitWarps);
  if (!h || h->n_chunks == 0) return 0;
  if (h->cfg.arch == 1) return h->cfg.n_tasks;
  return (h->cfg.n_tasks + kWarps - 1) / kWarps;
}

template <typename T>
cudaError_t launch_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  if (h->n_chunks == 0) return cudaSuccess;
  Plan<T> P;
  P.stream = h->stream;
  P.cref = h->cref;
  P.task = h->task;
  P.xgi = h->xgi;
  P.scratch = static_cast<T*>(h->scratch);
  P.counters = h->counters;
  P.n_tasks = h->cfg.n_tasks;
  P.nstage = h->cfg.nstage;
  P.stage_bytes = h->cfg.stage_bytes;
  P.xbuf = h->cfg.xbuf;
  P.mode = h->cfg.mode;
  P.xpf = h->cfg.xpf;
  if (h->cfg.arch >= 1) {
    const size_t smem = cta_smem_bytes(h->cfg, (int)sizeof(T));
    static size_t set_cta[2] = {0, 0};
    const int tc = sizeof(T) == 8 ? 1 : 0;
    if (set_cta[tc] < smem) {
      cudaError_t e = cudaFuncSetAttribute(spmv_cta_kernel<T>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      set_cta[tc] = smem;
    }
    spmv_cta_kernel<T><<<(unsigned)h->cfg.n_tasks, kCtaThreads, smem, st>>>(
        P, static_cast<const T*>(x), static_cast<T*>(y));
    return cudaGetLastError();
  }
  const size_t smem =
      (size_t)kWarps * warp_smem_bytes(P.nstage, P.stage_bytes, P.xbuf, (int)sizeof(T));
  static size_t set_bytes[2] = {0, 0};
  const int ti = sizeof(T) == 8 ? 1 : 0;
  if (set_bytes[ti] < smem) {
    cudaError_t e = cudaFuncSetAttribute(spmv_kernel<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_bytes[ti] = smem;
  }
  spmv_kernel<T><<<(unsigned)exec_grid(h), kThreads, smem, st>>>(P, static_cast<const T*>(x),
                                                                static_cast<T*>(y));
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rem(const sable_handle* h, const void* x, void* y, cudaStream_t st);

// y = A x: the remainder executor writes every local row (its remainder
// sum, or 0), then the dense-tile executor adds the dense part of the rows
// of block rows with tiles.
template <typename T>
cudaError_t launch_units(const sable_handle* h, const void* x, void* y, cudaStream_t st);

cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  if (h->cfg.arch == 2)
    return h->dtype == SABLE_F64 ? launch_units<double>(h, x, y, st)
                                 : launch_units<float>(h, x, y, st);
  // diagnostics (SABLE_EXEC_MODE): 2 = remainder executor only, 3 = dense only
  cudaError_t e = cudaSuccess;
  if (h->cfg.mode != 3)
    e = h->dtype == SABLE_F64 ? launch_rem<double>(h, x, y, st) : launch_rem<float>(h, x, y, st);
  if (e != cudaSuccess || h->cfg.mode == 2) return e;
  return h->dtype == SABLE_F64 ? launch_spmv<double>(h, x, y, st)
                               : launch_spmv<float>(h, x, y, st);
}

}  // namespace sable
