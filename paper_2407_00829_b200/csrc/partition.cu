// partition.cu -- the GPU partitioner: Alg. 1 "Matrix
// Partitioning" with the similarity of Eq. 1
// or Eq. 2, producing the row and
// column cut grid (rpntr / cpntr) of a CSR matrix on the device.
//
// Alg. 1 scans the rows and cuts before row i+1 when the similarity of rows
// i and i+1 drops below the threshold, extending a block across a run of
// empty rows up to the next non-empty one.  Unrolled, its cut set is
// position-wise independent: for p in [1, n),
//   cut(p) <=> (row p-1 non-empty and S(row p-1, row p) < t)
//              or (row p-1 empty and row p non-empty),
// plus the final cut n -- so one warp per p decides its cut, and a stream
// compaction lists them.  The columns are "the same procedure on the
// columns": the pattern is transposed on the device (radix sort) and the
// same kernel runs on it.  S uses the pattern only: u.v = #positions non-zero
// in both rows; Eq. 2 also counts u shifted by +-1 and takes the largest
// (reading R17); "S < t" is evaluated exactly as dot * t_den < t_num *
// max(nnz u, nnz v) for t = t_num / t_den (reading R19), so the grid is
// bit-exact against the oracle.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <vector>

#include "sable_internal.cuh"

namespace sable {

namespace {

constexpr unsigned kFull = 0xffffffffu;

struct PFail {
  sable_status st;
};

#define PT_CU(call)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_error(cuda_msg(e_, #call));                                                      \
      throw PFail{e_ == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA};          \
    }                                                                                      \
  } while (0)

struct Buf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  ~Buf() {
    if (p) cudaFreeAsync(p, s);
  }
  void alloc(size_t bytes, cudaStream_t st) {
    s = st;
    PT_CU(cudaMallocAsync(&p, bytes ? bytes : 16, st));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <typename F>
void cub_call(F f, cudaStream_t st) {
  size_t bytes = 0;
  PT_CU(f(nullptr, bytes));
  Buf tmp;
  tmp.alloc(bytes, st);
  PT_CU(f(tmp.p, bytes));
}

__device__ __forceinline__ int64_t lower_bound(const int32_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One warp per position p in [1, n): flag[p - 1] = cut before p.
__global__ void k_cut_flags(const int64_t* ptr, const int32_t* idx, int64_t n, uint32_t t_num,
                            uint32_t t_den, int32_t shifts, uint8_t* flag) {
  const int64_t p = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) + 1;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  const int64_t a0 = ptr[p - 1], na = ptr[p] - a0, b0 = ptr[p], nb = ptr[p + 1] - b0;
  if (na == 0) {
    if (lane == 0) flag[p - 1] = nb > 0 ? 1 : 0;
    return;
  }
  // dot products of row p-1 (shifted by 0, +1, -1) with row p
  const int32_t* A = idx + a0;
  const int32_t* B = idx + b0;
  int64_t d0 = 0, dr = 0, dl = 0;
  for (int64_t i = lane; i < na; i += 32) {
    const int64_t j = A[i];
    int64_t k = lower_bound(B, nb, j - 1);
    if (k < nb && B[k] == j - 1) { ++dl; ++k; }
    if (k < nb && B[k] == j) { ++d0; ++k; }
    if (k < nb && B[k] == j + 1) ++dr;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d0 += __shfl_xor_sync(kFull, d0, o);
    dr += __shfl_xor_sync(kFull, dr, o);
    dl += __shfl_xor_sync(kFull, dl, o);
  }
  if (lane == 0) {
    int64_t dot = d0;
    if (shifts) {
      dot = dr > dot ? dr : dot;
      dot = dl > dot ? dl : dot;
    }
    const int64_t mx = na > nb ? na : nb;
    flag[p - 1] = dot * (int64_t)t_den < (int64_t)t_num * mx ? 1 : 0;
  }
}

__global__ void k_pair_keys(const int64_t* ptr, const int32_t* idx, int64_t nrows, int64_t nnz,
                            uint64_t* key) {
  // key = column * nrows + row: sorting gives the transposed (CSC) pattern
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32)
    key[e] = (uint64_t)idx[e] * (uint64_t)nrows + (uint64_t)r;
  (void)nnz;
}

__global__ void k_unkey(const uint64_t* key, int64_t nnz, int64_t nrows, int32_t* row,
                        int32_t* colcount) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  row[e] = (int32_t)(key[e] % (uint64_t)nrows);
  atomicAdd(colcount + key[e] / (uint64_t)nrows, 1);
}

__global__ void k_widen(const int32_t* c, int64_t n, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = c[i];
}

unsigned blocks_for(int64_t n, int th) {
  const int64_t b = (n + th - 1) / th;
  return (unsigned)(b > 0 ? b : 1);
}

// The grid (0, cuts...) of one side; host output.
std::vector<int32_t> cuts_of(const int64_t* ptr, const int32_t* idx, int64_t n, uint32_t t_num,
                             uint32_t t_den, int32_t shifts, cudaStream_t st) {
  std::vector<int32_t> out{0};
  if (n > 1) {
    Buf flag, sel, cnt;
    flag.alloc(n - 1, st);
    sel.alloc(sizeof(int32_t) * (n - 1), st);
    cnt.alloc(sizeof(int64_t), st);
    k_cut_flags<<<blocks_for((n - 1) * 32, 256), 256, 0, st>>>(ptr, idx, n, t_num, t_den, shifts,
                                                               flag.as<uint8_t>());
    PT_CU(cudaGetLastError());
    thrust::counting_iterator<int32_t> pos(1);
    const uint8_t* fl = flag.as<uint8_t>();
    int32_t* so = sel.as<int32_t>();
    int64_t* nc = cnt.as<int64_t>();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, pos, fl, so, nc, n - 1, st);
    }, st);
    int64_t m = 0;
    PT_CU(cudaMemcpyAsync(&m, nc, sizeof(m), cudaMemcpyDeviceToHost, st));
    PT_CU(cudaStreamSynchronize(st));
    out.resize(1 + m);
    if (m) PT_CU(cudaMemcpyAsync(out.data() + 1, so, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st));
    PT_CU(cudaStreamSynchronize(st));
  }
  out.push_back((int32_t)n);
  return out;
}

}  // namespace

}  // namespace sable

using namespace sable;

extern "C" sable_status sable_partition_grid(int64_t nrows, int64_t ncols, int64_t nnz,
                                             const int64_t* rowptr, const int32_t* colidx,
                                             int32_t mem, uint32_t t_num, uint32_t t_den,
                                             int32_t shifts, void* cuda_stream, int32_t* rpntr,
                                             int32_t* nbrows, int32_t* cpntr, int32_t* nbcols) {
  if (nrows < 1 || ncols < 1 || nnz < 0 || !rowptr || (nnz > 0 && !colidx) || !rpntr ||
      !nbrows || !cpntr || !nbcols || t_den == 0 || (mem != SABLE_MEM_HOST && mem != SABLE_MEM_DEVICE)) {
    set_error("sable_partition_grid: bad arguments");
    return SABLE_E_INVALID_ARG;
  }
  if (nrows >= INT32_MAX || ncols >= INT32_MAX || nnz >= INT32_MAX) {
    set_error("sable_partition_grid: sizes must be < 2^31");
    return SABLE_E_UNSUPPORTED;
  }
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  try {
    Buf hp, hi;
    const int64_t* ptr = rowptr;
    const int32_t* idx = colidx;
    if (mem == SABLE_MEM_HOST) {
      hp.alloc(sizeof(int64_t) * (nrows + 1), st);
      hi.alloc(sizeof(int32_t) * nnz, st);
      PT_CU(cudaMemcpyAsync(hp.p, rowptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice, st));
      if (nnz) PT_CU(cudaMemcpyAsync(hi.p, colidx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
      ptr = hp.as<int64_t>();
      idx = hi.as<int32_t>();
    }
    // rows: Alg. 1 on A
    const std::vector<int32_t> rows = cuts_of(ptr, idx, nrows, t_num, t_den, shifts, st);
    // columns: Alg. 1 on the pattern of A^T
    Buf k1, k2, trow, ccnt, cptr;
    k1.alloc(sizeof(uint64_t) * nnz, st);
    k2.alloc(sizeof(uint64_t) * nnz, st);
    trow.alloc(sizeof(int32_t) * nnz, st);
    ccnt.alloc(sizeof(int32_t) * (ncols + 1), st);
    cptr.alloc(sizeof(int64_t) * (ncols + 1), st);
    PT_CU(cudaMemsetAsync(ccnt.p, 0, sizeof(int32_t) * (ncols + 1), st));
    if (nnz) {
      k_pair_keys<<<blocks_for(nrows * 32, 256), 256, 0, st>>>(ptr, idx, nrows, nnz, k1.as<uint64_t>());
      int bits = 1;
      const uint64_t kmax = (uint64_t)ncols * (uint64_t)nrows;
      while (bits < 64 && (kmax >> bits) != 0) ++bits;
      const uint64_t* ki = k1.as<uint64_t>();
      uint64_t* ko = k2.as<uint64_t>();
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortKeys(t, b, ki, ko, nnz, 0, bits, st);
      }, st);
      k_unkey<<<blocks_for(nnz, 256), 256, 0, st>>>(ko, nnz, nrows, trow.as<int32_t>(),
                                                    ccnt.as<int32_t>());
      PT_CU(cudaGetLastError());
    }
    {
      Buf wide;
      wide.alloc(sizeof(int64_t) * (ncols + 1), st);
      k_widen<<<blocks_for(ncols + 1, 256), 256, 0, st>>>(ccnt.as<int32_t>(), ncols + 1,
                                                          wide.as<int64_t>());
      const int64_t* wi = wide.as<int64_t>();
      int64_t* co = cptr.as<int64_t>();
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, wi, co, ncols + 1, st);
      }, st);
    }
    const std::vector<int32_t> cols =
        cuts_of(cptr.as<int64_t>(), trow.as<int32_t>(), ncols, t_num, t_den, shifts, st);
    PT_CU(cudaStreamSynchronize(st));
    std::copy(rows.begin(), rows.end(), rpntr);
    std::copy(cols.begin(), cols.end(), cpntr);
    *nbrows = (int32_t)rows.size() - 1;
    *nbcols = (int32_t)cols.size() - 1;
  } catch (const PFail& f) {
    cudaStreamSynchronize(st);
    return f.st;
  }
  return SABLE_OK;
}
