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
// Every warp owns a task: a contiguous range of chunks of about equal bytes
// (cut at row-group boundaries).  A chunk is a run of consecutive work items
// whose data are contiguous ranges of five arrays (item descriptors,
// remainder row pointers, dense values, remainder columns, remainder
// values).  Lane 0 streams the warp's chunks through a private ring of
// shared-memory stages with 1-D bulk copies (cp.async.bulk, L2 evict-first,
// completion on the stage's mbarrier; ranges precomputed by the planner);
// each stage also carries the descriptor of the chunk nstage ahead, so no
// warp waits on a descriptor load and no warp waits on another.  Per item:
//   (1) dense slab: lane l works on row l % nr and column phase l / nr of the
//       column-major slab in shared memory; items never span a run of
//       consecutive global columns, so the x of column c is x[xo + c], read
//       through L1 (the next item's x lines are prefetched into L1 while
//       this one computes) and broadcast to the lanes of a phase; rows
//       accumulate in registers and the phases fold with shuffles;
//   (2) remainder: lanes multiply the staged entries by gathered x into the
//       warp's product buffer (the next item's x prefetched likewise); lane
//       r sums row r (the whole warp for long rows);
//   (3) y: a row is written once.  Pieces of a split group are summed left to
//       right in registers; a group shared by two tasks meets in global
//       scratch, where the last piece to arrive sums all pieces in order.
// No atomics on y; every row's summation order depends on the matrix alone,
// so y is bitwise reproducible and identical for every shard count.
#include "sable_internal.cuh"

namespace sable {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = kWarps * 32;
constexpr int kLongRow = 32;  // remainder rows longer than this: whole warp

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

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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

// ---------------------------------------------------------------- staging

// Lane 0: start the copies of chunk c (and of the descriptor of chunk
// `ahead`, if >= 0, into the stage's first 64 bytes).
template <typename T>
__device__ __forceinline__ void issue_chunk(const Plan<T>& P, const Chunk& c, int64_t ahead,
                                            unsigned char* stage, uint32_t bar, uint64_t pol) {
  uint32_t tx = ahead >= 0 ? 64u : 0u;
#pragma unroll
  for (int k = 0; k < SR_N; ++k) tx += c.bytes[k];
  mbar_expect_tx(bar, tx);
  const uint32_t s0 = smem_u32(stage);
  if (ahead >= 0) bulk_g2s(s0, P.chunks + ahead, 64u, bar, pol);
  const unsigned char* base[SR_N] = {
      reinterpret_cast<const unsigned char*>(P.items),
      reinterpret_cast<const unsigned char*>(P.rem_ptr),
      reinterpret_cast<const unsigned char*>(P.tval),
      reinterpret_cast<const unsigned char*>(P.rem_idx),
      reinterpret_cast<const unsigned char*>(P.rem_val)};
#pragma unroll
  for (int k = 0; k < SR_N; ++k)
    if (c.bytes[k])
      bulk_g2s(s0 + (c.off[k] & ~15u), base[k] + (size_t)c.src16[k] * 16, c.bytes[k], bar, pol);
}

// ---------------------------------------------------------------- items

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 4- or 8-byte asynchronous global -> shared copy (LDGSTS, through L1).
template <typename T>
__device__ __forceinline__ void cp_async(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src),
               "n"((int)sizeof(T))
               : "memory");
}

template <typename T>
struct StageView {
  const Item* items;
  const int32_t* rptr;
  const T* val;
  const int32_t* ridx;
  const T* rval;
  int64_t v0;
  int32_t e0, r0, ni, ndx;
};

template <typename T>
__device__ __forceinline__ StageView<T> stage_view(unsigned char* stage, const Chunk& C) {
  StageView<T> S;
  S.items = reinterpret_cast<const Item*>(stage + C.off[SR_ITEM]);
  S.rptr = reinterpret_cast<const int32_t*>(stage + C.off[SR_RPTR]);
  S.val = reinterpret_cast<const T*>(stage + C.off[SR_VAL]);
  S.ridx = reinterpret_cast<const int32_t*>(stage + C.off[SR_RIDX]);
  S.rval = reinterpret_cast<const T*>(stage + C.off[SR_RVAL]);
  S.v0 = C.v0;
  S.e0 = C.e0;
  S.r0 = C.r0;
  S.ni = C.ni;
  S.ndx = C.ndx;
  return S;
}

// Start copying the x a staged chunk needs into an x buffer: each item's
// dense columns (contiguous: items never span a run), then one x per
// remainder entry.  Asynchronous (LDGSTS): it overlaps the previous chunk.
template <typename T>
__device__ __forceinline__ void gather_chunk(const StageView<T>& S, T* xb,
                                             const T* __restrict__ x, int lane) {
  int eend = S.e0;
  for (int j = 0; j < S.ni; ++j) {
    const Item I = S.items[j];
    for (int c = lane; c < I.ncol; c += 32) cp_async(xb + I.xb + c, x + I.xo + c);
    if (I.ne > 0) eend = max(eend, I.eb + (int)I.ne);
  }
  T* xr = xb + S.ndx;
  const int ne = eend - S.e0;
  for (int e = lane; e < ne; e += 32) cp_async(xr + e, x + S.ridx[e]);
}

// The row sums of one item (lanes < nr hold rows row0 .. row0 + nr - 1).
template <typename T>
__device__ __forceinline__ T item_rows(const StageView<T>& S, const Item& I, const T* xb,
                                       int lane) {
  const int nr = I.nr, ncol = I.ncol, ne = I.ne;
  // (1) dense slab
  T acc = T(0);
  if (ncol > 0) {
    const int Q = I.q, active = Q * nr, ph = (lane * (int)I.qm) >> 15, row = lane - ph * nr;
    if (lane < active) {
      const T* vp = S.val + (I.voff - S.v0) + ph * nr + row;
      const T* xs = xb + I.xb;
      const int stride = active;  // values between a lane's columns c and c + Q
      int c = ph;
      for (; c + 3 * Q < ncol; c += 4 * Q) {
        acc = fma(vp[0], xs[c], acc);
        acc = fma(vp[stride], xs[c + Q], acc);
        acc = fma(vp[2 * stride], xs[c + 2 * Q], acc);
        acc = fma(vp[3 * stride], xs[c + 3 * Q], acc);
        vp += 4 * stride;
      }
      for (; c < ncol; c += Q) {
        acc = fma(*vp, xs[c], acc);
        vp += stride;
      }
    }
    for (int off = 1; off < Q; off <<= 1) {
      const T o = __shfl_down_sync(kFull, acc, off * nr);
      if (lane < active && ph + off < Q) acc += o;
    }
  }
  // (2) remainder: lane r sums row r (the whole warp for long rows)
  if (ne > 0) {
    const int eo = I.eb - S.e0;
    const T* rv = S.rval + eo;
    const T* xr = xb + S.ndx + eo;
    int lo = 0, hi = 0;
    if (lane < nr) {
      const int rr = I.row0 + lane - S.r0;
      lo = max(S.rptr[rr], I.eb) - I.eb;
      hi = min(S.rptr[rr + 1], I.eb + ne) - I.eb;
      if (hi < lo) hi = lo;
    }
    T racc = T(0);
    const bool longr = (hi - lo) > kLongRow;
    unsigned lm = __ballot_sync(kFull, longr);
    if (!longr)
      for (int e = lo; e < hi; ++e) racc = fma(rv[e], xr[e], racc);
    while (lm) {
      const int r = __ffs(lm) - 1;
      lm &= lm - 1;
      const int l2 = __shfl_sync(kFull, lo, r), h2 = __shfl_sync(kFull, hi, r);
      T sum = T(0);
      for (int e = l2 + lane; e < h2; e += 32) sum = fma(rv[e], xr[e], sum);
      sum = warp_sum(sum);
      if (lane == r) racc = sum;
    }
    acc += racc;
  }
  return acc;
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
  uint64_t* full = reinterpret_cast<uint64_t*>(ws);     // [kMaxStages]
  Chunk* cdesc = reinterpret_cast<Chunk*>(ws + 64);     // [kMaxStages]
  T* xbuf = reinterpret_cast<T*>(ws + 512);             // [2][P.xbuf]
  unsigned char* stages = ws + 512 + ((2 * P.xbuf * (int)sizeof(T) + 127) & ~127);

  uint64_t pol = 0;
  if (lane == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < NS; ++s) mbar_init(smem_u32(full + s), 1);
    fence_barrier_init();
    for (int s = 0; s < NS && kb + s < ke; ++s) {
      const Chunk c = P.chunks[kb + s];
      cdesc[s] = c;
      issue_chunk(P, c, kb + s + NS < ke ? kb + s + NS : -1, stages + (size_t)s * P.stage_bytes,
                  smem_u32(full + s), pol);
    }
  }
  __syncwarp();

  // chunk k computes from stage s and x buffer b while chunk k + 1's x is
  // being gathered into buffer b ^ 1
  int s = 0, b = 0;
  uint32_t phase = 0;
  mbar_wait(smem_u32(full + 0), 0);
  StageView<T> S = stage_view<T>(stages, cdesc[0]);
  if (P.mode != 1) gather_chunk(S, xbuf, x, lane);
  cp_async_commit();
  T run = T(0);  // running sum of the current group's pieces (lanes < nr)
  for (int64_t k = kb; k < ke; ++k) {
    int sn = s + 1;
    uint32_t phn = phase;
    if (sn == NS) {
      sn = 0;
      phn ^= 1u;
    }
    StageView<T> Sn = S;
    if (k + 1 < ke) {
      mbar_wait(smem_u32(full + sn), phn);
      Sn = stage_view<T>(stages + (size_t)sn * P.stage_bytes, cdesc[sn]);
      if (P.mode != 1) gather_chunk(Sn, xbuf + (b ^ 1) * P.xbuf, x, lane);
    }
    cp_async_commit();
    cp_async_wait<1>();  // chunk k's x
    __syncwarp();
    if (P.mode != 1) {
      const T* xb = xbuf + b * P.xbuf;
      for (int j = 0; j < S.ni; ++j) {
        const Item I = S.items[j];
        const T tot = item_rows(S, I, xb, lane);
        if (!(I.flags & IF_XG)) {
          run = (I.flags & IF_FIRST) ? tot : run + tot;
          if ((I.flags & IF_LAST) && lane < I.nr) y[I.row0 + lane] = run;
        } else {
          // a group shared with another task: meet in global scratch
          const XgInfo xi = P.xgi[(int64_t)cdesc[s].i0 + j];
          T* sp = P.scratch + xi.slot;
          if (lane < I.nr) __stcg(sp + xi.p * 32 + lane, tot);
          __syncwarp();
          int last = 0;
          if (lane == 0) last = (atom_add_acq_rel(P.counters + xi.g, 1) + 1 == xi.npieces);
          last = __shfl_sync(kFull, last, 0);
          if (last) {
            if (lane < I.nr) {
              T sum = __ldcg(sp + lane);
              for (int q = 1; q < xi.npieces; ++q) sum += __ldcg(sp + q * 32 + lane);
              y[I.row0 + lane] = sum;
            }
            if (lane == 0) P.counters[xi.g] = 0;  // ready for the next launch
          }
        }
      }
    }
    // refill this stage with chunk k + NS (its descriptor rode in with chunk k)
    __syncwarp();
    if (lane == 0 && k + NS < ke) {
      unsigned char* stage = stages + (size_t)s * P.stage_bytes;
      const Chunk nd = *reinterpret_cast<const Chunk*>(stage);
      cdesc[s] = nd;
      issue_chunk(P, nd, k + 2 * NS < ke ? k + 2 * NS : -1, stage, smem_u32(full + s), pol);
    }
    __syncwarp();
    s = sn;
    phase = phn;
    S = Sn;
    b ^= 1;
  }
  cp_async_wait<0>();
}

}  // namespace

int32_t exec_grid(const sable_handle* h) {
  if (!h || h->n_chunks == 0) return 0;
  return (h->cfg.n_tasks + kWarps - 1) / kWarps;
}

template <typename T>
cudaError_t launch_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  if (h->n_chunks == 0) return cudaSuccess;
  Plan<T> P;
  P.chunks = h->chunks;
  P.task = h->task;
  P.items = h->items;
  P.xgi = h->xgi;
  P.tval = static_cast<const T*>(h->tval);
  P.rem_ptr = h->rem_ptr;
  P.rem_idx = h->rem_idx;
  P.rem_val = static_cast<const T*>(h->rem_val);
  P.scratch = static_cast<T*>(h->scratch);
  P.counters = h->counters;
  P.n_tasks = h->cfg.n_tasks;
  P.nstage = h->cfg.nstage;
  P.stage_bytes = h->cfg.stage_bytes;
  P.xbuf = h->cfg.xbuf;
  P.mode = h->cfg.mode;
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

cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st) {
  return h->dtype == SABLE_F64 ? launch_spmv<double>(h, x, y, st)
                               : launch_spmv<float>(h, x, y, st);
}

}  // namespace sable
