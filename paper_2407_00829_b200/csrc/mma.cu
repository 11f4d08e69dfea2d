// mma.cu -- SURVEY 8(f) row f3 on the 5th-generation tensor cores: Y = A X
// for k in {16, 32, 64, 128} fp32 right-hand sides, the "user-defined
// operation" generality of the VBR-C split where a
// dense tile times k vectors IS a dense contraction.
//
// Per unit of the SpMV plan (plan.cu: <= 32 rows of one block row and its
// row-major panel), transposed so that the k right-hand sides fill the MMA's
// M dimension:
//   D (M = 128 >= k, N = 32 rows)  =  Xg^T (M x K)  *  P^T (K x N)
// where P is the unit's panel rows (h x W, K = W panel columns) and Xg the
// rows of X under the panel's columns (gathered through the x map).  Both
// operands are staged in shared memory in the canonical no-swizzle UMMA
// layouts -- Xg^T MN-major (the k values of one X row are contiguous), P^T
// K-major (a panel row is contiguous) -- in tiles of 32 panel columns, and
// one thread issues tcgen05.mma.kind::tf32 into a TMEM accumulator; fp32
// accuracy comes from the 3xTF32 split (a = a_hi + a_lo, D += a_hi b_hi +
// a_hi b_lo + a_lo b_hi), each tile's MMAs committed to an mbarrier.  The
// accumulator is read back with tcgen05.ld (thread m = right-hand side m),
// the unit's CSR remainder is added on the CUDA cores in entry order (the k
// values of a gathered X row are one coalesced load), and Y is written once
// (split row ranges meet in scratch, summed in piece order by the last to
// arrive, as in unit.cu).
#include <algorithm>

#include "device.cuh"

namespace sable {

namespace {

using namespace dev;

constexpr int kM = 128;       // MMA M: right-hand sides (k <= 128, zero padded)
constexpr int kN = 32;        // MMA N: unit rows (nr <= 32, zero padded)
constexpr int kKT = 32;       // panel columns per shared-memory tile
constexpr int kMmaThreads = 128;

struct MmaSmem {
  float a_hi[kKT * kM];       // Xg^T tile, MN-major, 16 KB
  float a_lo[kKT * kM];
  float b_hi[kN * kKT];       // P^T tile, K-major, 4 KB
  float b_lo[kN * kKT];
  float yt[kN * kM];          // the unit's rows x right-hand sides
  uint64_t bar;               // MMA completion
  uint32_t tmem;              // accumulator base
  int32_t last;
};

// Canonical no-swizzle K-major layouts (core matrices of 8 rows x 16 B, i.e.
// 4 tf32 along K): element (r, kk) of an R-row operand at
//   (kk/4) * (R/8) * 128 + (r/8) * 128 + (r%8) * 16 + (kk%4) * 4 bytes
// -> SBO = 128 B between 8-row groups, LBO = R/8 * 128 B between 16-byte K
// chunks; one MMA (K = 8) spans two chunks.  Both operands are K-major: the
// MN-major A of kind::tf32 measured all-zero accumulators on sm_100a
// (scripts/probe/umma_probe.cu).
constexpr int kLboA = kM / 8 * 128;  // 2048 B
constexpr int kLboB = kN / 8 * 128;  // 512 B
// 16-byte vector (4 consecutive kk) of row r in K chunk c, in floats
__device__ __forceinline__ int kmaj_index(int lbo, int r, int c) {
  return (c * lbo + (r >> 3) * 128 + (r & 7) * 16) >> 2;
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0, SWIZZLE_NONE
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulator, TF32 A and B, both
// K-major, N = kN, M = kM.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                            ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// Global column of panel column f of a unit (x map entry of its 4-column vector).
__device__ __forceinline__ int panel_col(const UPlan<float>& P, int xq0, int f) {
  SABLE_DCHECK(xq0 + (f >> 2) < P.n_xq);
  const XMap m = ldg_xmap(P.xq + xq0 + (f >> 2));
  const int i = f & 3;
  if (m.c >= 0) {
    const int k = m.kd & 3, d = m.kd >> 2;
    return m.c + i + (i >= k ? d : 0);
  }
  const int* side = reinterpret_cast<const int*>(P.xside + ~m.c);
  return __ldg(side + i);
}

__global__ void __launch_bounds__(kMmaThreads, 1)
    spmm_mma_kernel(const __grid_constant__ UPlan<float> P, const float* __restrict__ X,
                    float* __restrict__ Y, int k, int64_t n_units) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  MmaSmem& S = *reinterpret_cast<MmaSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t bar = smem_u32(&S.bar);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem)),
                 "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem;
  uint32_t phase = 0;
  const int m = tid;  // this thread's right-hand side in the epilogue

  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const Unit U = load_unit(P.units + u);
    const int nr = U.nr;
    if (U.wq > 0) {
      const int W = U.wq * 4;  // panel columns of the unit (16-byte padded)
      const float* pv = P.pv + (int64_t)U.voff16 * 4;
      const int64_t rstride = (int64_t)U.wq * 4;
      for (int f0 = 0; f0 < W; f0 += kKT) {
        // A tile: thread m takes right-hand side m of the X rows under panel
        // columns f0 + 4c .. f0 + 4c + 3 (each load coalesced over m), split
        // into tf32 hi / lo, one 16-byte store each; zero past W and k
#pragma unroll 2
        for (int c = 0; c < kKT / 4; ++c) {
          float e[4] = {0.f, 0.f, 0.f, 0.f};
          if (f0 + 4 * c < W && m < k) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              e[t] = __ldg(X + (int64_t)panel_col(P, U.xq0, f0 + 4 * c + t) * k + m);
          }
          float4 hi, lo;
          hi.x = tf32_rna(e[0]); lo.x = tf32_rna(e[0] - hi.x);
          hi.y = tf32_rna(e[1]); lo.y = tf32_rna(e[1] - hi.y);
          hi.z = tf32_rna(e[2]); lo.z = tf32_rna(e[2] - hi.z);
          hi.w = tf32_rna(e[3]); lo.w = tf32_rna(e[3] - hi.w);
          const int o = kmaj_index(kLboA, m, c);
          *reinterpret_cast<float4*>(S.a_hi + o) = hi;
          *reinterpret_cast<float4*>(S.a_lo + o) = lo;
        }
        // B tile: the unit's panel rows, columns f0 .. f0 + 31 as 16-byte
        // vectors (rows are 16-byte padded); zero past nr and W
        for (int i = tid; i < kN * (kKT / 4); i += kMmaThreads) {
          const int n = i % kN, c = i / kN;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (n < nr && f0 + 4 * c < W)
            v = __ldg(reinterpret_cast<const float4*>(pv + n * rstride + f0 + 4 * c));
          float4 hi, lo;
          hi.x = tf32_rna(v.x); lo.x = tf32_rna(v.x - hi.x);
          hi.y = tf32_rna(v.y); lo.y = tf32_rna(v.y - hi.y);
          hi.z = tf32_rna(v.z); lo.z = tf32_rna(v.z - hi.z);
          hi.w = tf32_rna(v.w); lo.w = tf32_rna(v.w - hi.w);
          const int o = kmaj_index(kLboB, n, c);
          *reinterpret_cast<float4*>(S.b_hi + o) = hi;
          *reinterpret_cast<float4*>(S.b_lo + o) = lo;
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ah = smem_u32(S.a_hi), al = smem_u32(S.a_lo);
          const uint32_t bh = smem_u32(S.b_hi), bl = smem_u32(S.b_lo);
#pragma unroll
          for (int j = 0; j < kKT / 8; ++j) {
            const uint64_t dah = smem_desc(ah + j * 2 * kLboA, kLboA, 128);
            const uint64_t dal = smem_desc(al + j * 2 * kLboA, kLboA, 128);
            const uint64_t dbh = smem_desc(bh + j * 2 * kLboB, kLboB, 128);
            const uint64_t dbl = smem_desc(bl + j * 2 * kLboB, kLboB, 128);
            mma_tf32(tmem, dah, dbh, (f0 > 0 || j > 0) ? 1u : 0u);
            mma_tf32(tmem, dah, dbl, 1u);
            mma_tf32(tmem, dal, dbh, 1u);
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  bar)
              : "memory");
        }
        mbar_wait(bar, phase);  // the tile's MMAs are done: its shared memory is free
        phase ^= 1u;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // accumulator row m (TMEM lane m, this thread), 32 columns = the unit's rows
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
          "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, "
          "%26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
            "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
            "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int n = 0; n < kN; ++n) S.yt[n * kM + m] = __uint_as_float(r[n]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    } else {
      for (int n = 0; n < kN; ++n) S.yt[n * kM + m] = 0.f;
    }
    // the unit's CSR remainder, in entry order per row (thread m: RHS m)
    if (U.e1 > U.e0 && m < k) {
      for (int n = 0; n < nr; ++n) {
        const int lo = max(__ldg(P.rptr + U.row0 + n), U.e0);
        const int hi = min(__ldg(P.rptr + U.row0 + n + 1), U.e1);
        float s = S.yt[n * kM + m];
        for (int e = lo; e < hi; ++e)
          s += __ldg(P.rval + e) * __ldg(X + (int64_t)__ldg(P.ridx + e) * k + m);
        S.yt[n * kM + m] = s;
      }
    }
    if (U.xg < 0) {
      if (m < k)
        for (int n = 0; n < nr; ++n) Y[(int64_t)(U.row0 + n) * k + m] = S.yt[n * kM + m];
    } else {
      const int4 gv = __ldg(reinterpret_cast<const int4*>(P.xg + U.xg));
      const int64_t slot = (int64_t)(((uint64_t)(uint32_t)gv.y << 32) | (uint32_t)gv.x);
      const int counter = gv.z, np = gv.w;
      SABLE_DCHECK(slot >= 0 && (slot + (int64_t)np * kN) * kM <= P.scratch_elems);
      float* sp = P.scratch + slot * kM;
      if (m < k)
        for (int n = 0; n < nr; ++n) __stcg(sp + (U.piece * 32 + n) * kM + m, S.yt[n * kM + m]);
      __threadfence();
      __syncthreads();
      if (tid == 0) S.last = atom_add_acq_rel(P.counters + counter, 1) + 1 == np;
      __syncthreads();
      if (S.last) {
        __threadfence();
        if (m < k)
          for (int n = 0; n < nr; ++n) {
            float t = __ldcg(sp + n * kM + m);
            for (int q = 1; q < np; ++q) t += __ldcg(sp + (q * 32 + n) * kM + m);
            Y[(int64_t)(U.row0 + n) * k + m] = t;
          }
        if (tid == 0) P.counters[counter] = 0;  // ready for the next launch
      }
    }
    __syncthreads();  // yt is reused by the next unit
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(32));
}

}  // namespace

// Y = A X on the tensor cores (fp32 handles, k in {16, 32, 64, 128}); scratch
// holds 128 partials per combine slot.
cudaError_t run_spmm_mma(const sable_handle* h, const void* X, void* Y, int32_t k, void* scratch,
                         cudaStream_t st) {
  if (h->n_units == 0) return cudaSuccess;
  UPlan<float> P;
  P.units = h->units;
  P.batch = h->ubatch;
  P.bhead = h->ubhead;
  P.xq = h->xq;
  P.xside = h->xside;
  P.pv = static_cast<const float*>(h->pv);
  P.rptr = h->rem_ptr;
  P.ridx = h->rem_idx;
  P.rval = static_cast<const float*>(h->rem_val);
  P.xg = h->uxg;
  P.scratch = static_cast<float*>(scratch);
  P.counters = h->ucounters;
  P.b0 = 0;
  P.n_batches = h->n_ubatch;
  P.pf = 0;
  P.npeer = 0;
  plan_extents<float>(P, h, h->uscratch_slots * (int64_t)kM);
  int dev = 0, sms = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (!e) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e) return e;
  const size_t smem = sizeof(MmaSmem);
  e = set_smem_attr(reinterpret_cast<const void*>(spmm_mma_kernel), dev, smem);
  if (e) return e;
  const int64_t grid = std::min<int64_t>(h->n_units, (int64_t)sms * 3);
  spmm_mma_kernel<<<(unsigned)grid, kMmaThreads, smem, st>>>(P, static_cast<const float*>(X),
                                                             static_cast<float*>(Y), k,
                                                             h->n_units);
  return cudaGetLastError();
}

}  // namespace sable
