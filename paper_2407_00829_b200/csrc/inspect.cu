// inspect.cu -- the GPU inspector behind sable_vbr_create (north_star (1)).
//
// Steps (every step is a kernel or a device-wide
// CUB primitive on the caller's stream):
//   a1 validate  : the VBR / remainder invariants of sable.h; the first bad
//                  (array, index) wins (atomicMin on code<<48 | index).
//   a2 count     : non-zeros per stored VBR block (bit test, no FTZ: reading
//                  R4) and per remainder entry; every candidate cell (>= 1
//                  non-zero from either source, reading R5)
//                  is found by a radix sort of cell keys br*nbc+bc.
//   a3 classify  : dense <=> 100*cnt >= delta*h*w in int64 (
//                  readings R1, R3).
//   shard        : per-block-row weights -> sable_shard_bounds (host).
//   a4 build     : pack the local dense tiles into row-group panels (values
//                  from val, zero fill normalised to +0, remainder entries of
//                  dense cells scattered in); assemble the local CSR remainder
//                  (sparse cells' non-zeros from both sources, row-major,
//                  columns ascending: Fig. 3, reading R6).
//   a5 plan      : row groups of <= 32 rows, work pieces capped in bytes.
// The partition is bit-exact by construction (integer arithmetic and bit
// copies only).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "sable_internal.cuh"

namespace sable {

void free_handle(sable_handle* h);
template <typename T>
cudaError_t plan_units(sable_handle* h, const T* tval, int32_t nbl, int32_t b0,
                       const std::vector<int32_t>& H_rpntr, const std::vector<int32_t>& H_W,
                       const std::vector<int64_t>& br_vbase, const std::vector<int64_t>& br_wprefix,
                       const std::vector<int64_t>& br_t0, const std::vector<int32_t>& H_rp,
                       const std::vector<XTile>& H_xt, std::vector<int64_t>& br_pbase,
                       cudaStream_t st);

namespace {

// ----------------------------------------------------------------- helpers

enum : int {
  V_RPNTR = 1, V_CPNTR, V_BPNTR, V_REMPTR, V_BINDX, V_INDX, V_REMIDX, V_DUP
};
const char* kArrayName[] = {"?", "rpntr", "cpntr", "bpntr", "rem_indptr",
                            "bindx", "indx", "rem_indices", "rem (duplicate of val)"};

struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    release();
    s = st;
    return cudaMallocAsync(&p, bytes ? bytes : 16, st);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Widen {
  __host__ __device__ int64_t operator()(int32_t v) const { return v; }
};

struct Fail {
  sable_status st;
};

#define SB_CU(call)                                          \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) {                                 \
      set_error(cuda_msg(e_, #call));                        \
      throw Fail{e_ == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA}; \
    }                                                        \
  } while (0)

inline unsigned nblocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, b);
}

template <typename T>
__device__ __forceinline__ bool is_nz(T v);
template <>
__device__ __forceinline__ bool is_nz<float>(float v) {
  return (__float_as_uint(v) & 0x7fffffffu) != 0u;
}
template <>
__device__ __forceinline__ bool is_nz<double>(double v) {
  return (static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7fffffffffffffffull) != 0ull;
}

template <typename I>
__device__ __forceinline__ int64_t upper_bound(const I* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;  // first index with a[idx] > v
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void report(unsigned long long* err, int code, int64_t idx) {
  const unsigned long long v =
      ((unsigned long long)code << 48) |
      (unsigned long long)(idx < 0 ? 0 : (idx > 0xFFFFFFFFFFFFll ? 0xFFFFFFFFFFFFll : idx));
  atomicMin(err, v);
}

// ----------------------------------------------------------------- a1: validate

__global__ void k_check_grid(const int32_t* p, int32_t nb, int64_t n, int code,
                             unsigned long long* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nb) return;
  if (i == 0 && p[0] != 0) report(err, code, 0);
  if (i == nb && p[nb] != n) report(err, code, nb);
  if (i < nb && p[i + 1] <= p[i]) report(err, code, i + 1);
}

__global__ void k_check_ptr64(const int64_t* p, int64_t n, int64_t total, int code,
                              unsigned long long* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == 0 && p[0] != 0) report(err, code, 0);
  if (i == n && p[n] != total) report(err, code, n);
  if (i < n && p[i + 1] < p[i]) report(err, code, i + 1);
}

__global__ void k_check_blocks(const int32_t* rpntr, const int32_t* cpntr, const int64_t* bpntr,
                               int32_t nbr, int32_t nbc, const int32_t* bindx,
                               const int64_t* indx, int64_t nblk, int64_t val_len,
                               int32_t* blk_br, unsigned long long* err) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0 && indx[0] != 0) report(err, V_INDX, 0);
  if (k == 0 && indx[nblk] != val_len) report(err, V_INDX, nblk);
  if (k >= nblk) return;
  const int64_t a = upper_bound(bpntr, (int64_t)nbr + 1, k) - 1;
  blk_br[k] = (int32_t)a;
  const int32_t b = bindx[k];
  if (b < 0 || b >= nbc) {
    report(err, V_BINDX, k);
    return;
  }
  if (k > bpntr[a] && bindx[k - 1] >= b) report(err, V_BINDX, k);
  const int64_t area = (int64_t)(rpntr[a + 1] - rpntr[a]) * (int64_t)(cpntr[b + 1] - cpntr[b]);
  if (indx[k + 1] - indx[k] != area) report(err, V_INDX, k + 1);
}

// Warp per remainder row: column checks and the row id of every entry.
__global__ void k_rem_rows(const int64_t* ptr, const int32_t* idx, int64_t nrows, int64_t ncols,
                           int32_t* rowid, unsigned long long* err) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= nrows) return;
  const int64_t e0 = ptr[i], e1 = ptr[i + 1];
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int32_t j = idx[e];
    rowid[e] = (int32_t)i;
    if (j < 0 || j >= ncols) report(err, V_REMIDX, e);
    else if (e > e0 && idx[e - 1] >= j) report(err, V_REMIDX, e);
  }
}

// ----------------------------------------------------------------- a2: count

__global__ void k_axis_map(const int32_t* p, int32_t nb, int64_t n, int32_t* map) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) map[i] = (int32_t)(upper_bound(p, (int64_t)nb + 1, i) - 1);
}

template <typename T>
__global__ void k_count_vbr(const T* val, const int64_t* indx, int64_t nblk, int64_t* cnt) {
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= nblk) return;
  int64_t c = 0;
  for (int64_t e = indx[k] + lane; e < indx[k + 1]; e += 32) c += is_nz(val[e]) ? 1 : 0;
  for (int off = 16; off; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
  if (lane == 0) cnt[k] = c;
}

__global__ void k_vbr_keys(const int32_t* blk_br, const int32_t* bindx, const int64_t* cnt,
                           int64_t nblk, int64_t nbc, uint64_t sent, uint64_t* key,
                           int32_t* payload) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblk) return;
  key[k] = cnt[k] > 0 ? (uint64_t)blk_br[k] * (uint64_t)nbc + (uint64_t)bindx[k] : sent;
  payload[k] = (int32_t)k;
}

// Remainder entries: duplicate test against val, and the cell key.
template <typename T>
__global__ void k_rem_keys(const int32_t* rowid, const int32_t* ridx, const T* rval, int64_t R,
                           const int32_t* row2br, const int32_t* col2bc, const int32_t* rpntr,
                           const int32_t* cpntr, const int64_t* bpntr, const int32_t* bindx,
                           const int64_t* indx, const T* val, int64_t nblk, int64_t nbc,
                           uint64_t sent, uint64_t* key, int32_t* payload,
                           unsigned long long* err) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R) return;
  const int32_t i = rowid[e], j = ridx[e];
  const bool nz = is_nz(rval[e]);
  const int32_t br = row2br[i], bc = col2bc[j];
  if (nz) {
    // binary search block column bc among the stored blocks of block row br
    int64_t lo = bpntr[br], hi = bpntr[br + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (bindx[mid] < bc) lo = mid + 1; else hi = mid;
    }
    if (lo < bpntr[br + 1] && bindx[lo] == bc) {
      const int64_t h = rpntr[br + 1] - rpntr[br];
      const int64_t pos = indx[lo] + (int64_t)(j - cpntr[bc]) * h + (i - rpntr[br]);
      if (is_nz(val[pos])) report(err, V_DUP, e);
    }
  }
  key[nblk + e] = nz ? (uint64_t)br * (uint64_t)nbc + (uint64_t)bc : sent;
  payload[nblk + e] = (int32_t)(nblk + e);
}

__global__ void k_heads(const uint64_t* key, int64_t n, uint64_t sent, int32_t* flag) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  flag[s] = (key[s] != sent && (s == 0 || key[s] != key[s - 1])) ? 1 : 0;
}

__global__ void k_cells(const uint64_t* key, const int32_t* payload, const int32_t* cid,
                        int64_t n, uint64_t sent, int64_t nblk, const int64_t* cnt_vbr,
                        uint64_t* cell_key, int64_t* cell_cnt, int32_t* cell_blk,
                        int32_t* ecell) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n || key[s] == sent) return;
  const int32_t c = cid[s] - 1;
  if (s == 0 || key[s] != key[s - 1]) cell_key[c] = key[s];
  const int32_t p = payload[s];
  if (p < nblk) {
    atomicAdd((unsigned long long*)(cell_cnt + c), (unsigned long long)cnt_vbr[p]);
    cell_blk[c] = p;
  } else {
    atomicAdd((unsigned long long*)(cell_cnt + c), 1ull);
    ecell[p - nblk] = c;
  }
}

// ----------------------------------------------------------------- a3: classify

template <typename T>
__global__ void k_classify(const uint64_t* cell_key, const int64_t* cell_cnt,
                           const int32_t* cell_blk, const int64_t* cnt_vbr, int64_t n_cells,
                           int64_t nbc, const int32_t* rpntr, const int32_t* cpntr,
                           int32_t delta, int64_t min_area, int32_t n_rules,
                           const sable_delta_rule* rules, int32_t* cell_br, int32_t* cell_bc,
                           uint8_t* cell_dense, int32_t* br_ncell, int32_t* br_ndense,
                           int32_t* br_W, unsigned long long* br_area,
                           unsigned long long* br_rem, unsigned long long* br_vbrsparse) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  const int32_t br = (int32_t)(cell_key[c] / (uint64_t)nbc);
  const int32_t bc = (int32_t)(cell_key[c] % (uint64_t)nbc);
  const int64_t h = rpntr[br + 1] - rpntr[br], w = cpntr[bc + 1] - cpntr[bc];
  const int64_t cnt = cell_cnt[c];
  // PAPER.md:87-88 (readings R1, R3), under the per-shape policy (R22): the
  // first rule matching h x w gives delta, cells below min_area are sparse
  int32_t d = delta;
  for (int32_t k = 0; k < n_rules; ++k)
    if (h >= rules[k].h_min && h <= rules[k].h_max && w >= rules[k].w_min && w <= rules[k].w_max) {
      d = (int32_t)rules[k].delta_pct;
      break;
    }
  const bool dense = h * w >= min_area && 100 * cnt >= (int64_t)d * h * w;
  cell_br[c] = br;
  cell_bc[c] = bc;
  cell_dense[c] = dense ? 1 : 0;
  atomicAdd(br_ncell + br, 1);
  if (dense) {
    atomicAdd(br_ndense + br, 1);
    atomicAdd(br_W + br, (int32_t)w);
    atomicAdd(br_area + br, (unsigned long long)(h * w));
  } else {
    atomicAdd(br_rem + br, (unsigned long long)cnt);
    if (cell_blk[c] >= 0) atomicAdd(br_vbrsparse + br, (unsigned long long)cnt_vbr[cell_blk[c]]);
  }
}

// ----------------------------------------------------------------- a4: build

__global__ void k_tile_meta(const int32_t* tile_cell, int64_t nt, const int32_t* cell_br,
                            const int32_t* cell_bc, const int32_t* rpntr, const int32_t* cpntr,
                            int64_t cell_lo, int32_t* tile_br, int64_t* tile_area,
                            int32_t* tile_w, int32_t* cell_tile) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int32_t c = tile_cell[t];
  const int32_t br = cell_br[c], bc = cell_bc[c];
  const int64_t h = rpntr[br + 1] - rpntr[br], w = cpntr[bc + 1] - cpntr[bc];
  tile_br[t] = br;
  tile_area[t] = h * w;
  tile_w[t] = (int32_t)w;
  cell_tile[c - cell_lo] = (int32_t)t;
}

__global__ void k_tile_desc(const int32_t* tile_cell, int64_t nt, const int32_t* cell_bc,
                            const int32_t* tile_br, const int32_t* tile_w,
                            const int64_t* w_scan, const int64_t* br_wprefix, int32_t br_begin,
                            const int32_t* cpntr, TileDesc* desc, XTile* xt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  TileDesc d;
  d.c0 = cpntr[cell_bc[tile_cell[t]]];
  d.w = tile_w[t];
  d.cs = (int32_t)(w_scan[t] - br_wprefix[tile_br[t] - br_begin]);
  desc[t] = d;
  xt[t] = XTile{(int32_t)w_scan[t], d.c0};
  if (t == nt - 1) xt[nt] = XTile{(int32_t)(w_scan[t] + d.w), 0};  // sentinel
}

template <typename T>
__global__ void k_pack_vbr(const int32_t* tile_cell, int64_t nt, const int32_t* cell_blk,
                           const int32_t* tile_br, const TileDesc* desc, const int32_t* rpntr,
                           const int64_t* indx, const T* val, const int64_t* br_vbase,
                           const int32_t* br_W, int32_t br_begin, T* tval) {
  const int64_t t = blockIdx.x;
  if (t >= nt) return;
  const int32_t k = cell_blk[tile_cell[t]];
  if (k < 0) return;  // a remainder-only dense cell: filled by k_pack_rem
  const int32_t a = tile_br[t];
  const int64_t h = rpntr[a + 1] - rpntr[a];
  const TileDesc d = desc[t];
  const int64_t vb = br_vbase[a - br_begin], W = br_W[a - br_begin];
  const int64_t area = h * d.w;
  for (int64_t e = threadIdx.x; e < area; e += blockDim.x) {
    T v = val[indx[k] + e];
    if (!is_nz(v)) v = T(0);  // stored zero fill (+0 or -0) -> +0
    tval[panel_pos(vb, W, h, d.cs, e % h, e / h)] = v;
  }
}

template <typename T>
__global__ void k_pack_rem(const int32_t* rowid, const int32_t* ridx, const T* rval, int64_t R,
                           const int32_t* ecell, int64_t cell_lo, int64_t cell_hi,
                           const int32_t* cell_tile, const int32_t* tile_br,
                           const TileDesc* desc, const int32_t* rpntr, const int64_t* br_vbase,
                           const int32_t* br_W, int32_t br_begin, T* tval) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R) return;
  const int32_t c = ecell[e];
  if (c < cell_lo || c >= cell_hi) return;
  const int32_t t = cell_tile[c - cell_lo];
  if (t < 0) return;
  const int32_t a = tile_br[t];
  const TileDesc d = desc[t];
  const int64_t h = rpntr[a + 1] - rpntr[a];
  tval[panel_pos(br_vbase[a - br_begin], br_W[a - br_begin], h, d.cs, rowid[e] - rpntr[a],
                 ridx[e] - d.c0)] = rval[e];
}

// Flags of remainder entries that stay in the remainder (non-dense local cell).
__global__ void k_rem_keep(const int32_t* ecell, int64_t R, int64_t cell_lo, int64_t cell_hi,
                           const uint8_t* cell_dense, uint8_t* keep) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R) return;
  const int32_t c = ecell[e];
  keep[e] = (c >= cell_lo && c < cell_hi && !cell_dense[c]) ? 1 : 0;
}

__global__ void k_row_count(const int32_t* rows, int64_t n, int64_t row_begin, int32_t* cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) atomicAdd(cnt + (rows[e] - row_begin), 1);
}

// General remainder assembly (when sparse VBR blocks contribute non-zeros).
template <typename T>
__global__ void k_rem_pairs(const int32_t* rowid, const int32_t* ridx, const T* rval, int64_t n,
                            int64_t row_begin, int64_t ncols, uint64_t* key, T* v) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  key[e] = (uint64_t)(rowid[e] - row_begin) * (uint64_t)ncols + (uint64_t)ridx[e];
  v[e] = rval[e];
}

__global__ void k_sparse_vbr_flags(const int32_t* cell_blk, const uint8_t* cell_dense,
                                   int64_t cell_lo, int64_t n, uint8_t* flag) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  flag[c] = (!cell_dense[cell_lo + c] && cell_blk[cell_lo + c] >= 0) ? 1 : 0;
}

__global__ void k_sparse_vbr_cnt(const int32_t* scell, int64_t ns, const int32_t* cell_blk,
                                 const int64_t* cnt_vbr, int64_t* out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ns) out[s] = cnt_vbr[cell_blk[scell[s]]];
}

template <typename T>
__global__ void k_emit_sparse_vbr(const int32_t* scell, int64_t ns, const int64_t* pos0,
                                  const int32_t* cell_blk, const int32_t* cell_br,
                                  const int32_t* cell_bc, const int32_t* rpntr,
                                  const int32_t* cpntr, const int64_t* indx, const T* val,
                                  int64_t row_begin, int64_t ncols, int64_t base,
                                  unsigned long long* cursor, uint64_t* key, T* v) {
  const int64_t s = blockIdx.x;
  if (s >= ns) return;
  const int32_t c = scell[s];
  const int32_t k = cell_blk[c], a = cell_br[c], b = cell_bc[c];
  const int64_t h = rpntr[a + 1] - rpntr[a], w = cpntr[b + 1] - cpntr[b];
  for (int64_t e = threadIdx.x; e < h * w; e += blockDim.x) {
    const T x = val[indx[k] + e];
    if (!is_nz(x)) continue;
    const int64_t slot = base + pos0[s] + (int64_t)atomicAdd(cursor + s, 1ull);
    key[slot] = (uint64_t)(rpntr[a] + e % h - row_begin) * (uint64_t)ncols +
                (uint64_t)(cpntr[b] + e / h);
    v[slot] = x;
  }
}

__global__ void k_unpair(const uint64_t* key, int64_t n, int64_t ncols, int32_t* idx,
                         int32_t* rows) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  idx[e] = (int32_t)(key[e] % (uint64_t)ncols);
  rows[e] = (int32_t)(key[e] / (uint64_t)ncols);
}

// ----------------------------------------------------------------- CUB glue

template <typename F>
void cub_run(F f, cudaStream_t st) {
  size_t bytes = 0;
  SB_CU(f(nullptr, bytes));
  DevBuf tmp;
  SB_CU(tmp.alloc(bytes, st));
  SB_CU(f(tmp.p, bytes));
}

template <typename T>
void d2h(T* dst, const T* src, int64_t n, cudaStream_t st) {
  if (n > 0) SB_CU(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
}

template <typename T>
T* dev_alloc(int64_t n, cudaStream_t st) {
  void* p = nullptr;
  // +16 B tail: the executor's 16-byte-rounded bulk copies may read up to
  // 15 bytes past the last element of an array (never used)
  SB_CU(cudaMallocAsync(&p, sizeof(T) * (size_t)std::max<int64_t>(n, 1) + 16, st));
  SB_CU(cudaMemsetAsync(static_cast<char*>(p) + sizeof(T) * (size_t)std::max<int64_t>(n, 1), 0, 16, st));
  return static_cast<T*>(p);
}

// Inputs resident on the device: either the caller's (mem=DEVICE) or copies.
struct Inputs {
  const int32_t *rpntr, *cpntr, *bindx, *ridx;
  const int64_t *bpntr, *indx, *rptr;
  const void *val, *rval;
  DevBuf own[9];
};

void stage_inputs(const sable_vbr_desc* d, size_t sv, Inputs& in, cudaStream_t st) {
  const bool host = d->mem == SABLE_MEM_HOST;
  const bool has_rem = d->rem_indptr != nullptr;
  struct A {
    const void* src;
    size_t bytes;
    const void** dst;
  } arr[9] = {
      {d->rpntr, sizeof(int32_t) * (d->nbrows + 1), (const void**)&in.rpntr},
      {d->cpntr, sizeof(int32_t) * (d->nbcols + 1), (const void**)&in.cpntr},
      {d->bpntr, sizeof(int64_t) * (d->nbrows + 1), (const void**)&in.bpntr},
      {d->bindx, sizeof(int32_t) * d->nblocks, (const void**)&in.bindx},
      {d->indx, sizeof(int64_t) * (d->nblocks + 1), (const void**)&in.indx},
      {d->val, sv * d->val_len, (const void**)&in.val},
      {has_rem ? (const void*)d->rem_indptr : nullptr, sizeof(int64_t) * (d->nrows + 1),
       (const void**)&in.rptr},
      {d->rem_indices, sizeof(int32_t) * d->rem_nnz, (const void**)&in.ridx},
      {d->rem_val, sv * d->rem_nnz, (const void**)&in.rval},
  };
  for (int i = 0; i < 9; ++i) {
    if (!host || arr[i].src == nullptr) {
      *arr[i].dst = arr[i].src;
      continue;
    }
    SB_CU(in.own[i].alloc(arr[i].bytes, st));
    if (arr[i].bytes)
      SB_CU(cudaMemcpyAsync(in.own[i].p, arr[i].src, arr[i].bytes, cudaMemcpyHostToDevice, st));
    *arr[i].dst = in.own[i].p;
  }
}

void check_err(unsigned long long* err_d, cudaStream_t st, sable_status code) {
  unsigned long long err = 0;
  SB_CU(cudaMemcpyAsync(&err, err_d, sizeof(err), cudaMemcpyDeviceToHost, st));
  SB_CU(cudaStreamSynchronize(st));
  if (err == ~0ull) return;
  const int c = (int)(err >> 48);
  const long long idx = (long long)(err & 0xFFFFFFFFFFFFull);
  char msg[256];
  snprintf(msg, sizeof msg, "%s: invariant broken at index %lld",
           (c >= 1 && c <= 8) ? kArrayName[c] : "?", idx);
  set_error(msg);
  throw Fail{c == V_DUP ? SABLE_E_DUPLICATE : code};
}

int bits_for(uint64_t v) {  // bits to represent 0..v
  int b = 1;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

int64_t env_int(const char* name, int64_t dflt) {
  const char* s = std::getenv(name);
  return s ? std::atoll(s) : dflt;
}

// ------------------------------------------------------------------- a5: plan

// Executor configuration; SABLE_* environment variables override the
// defaults (tuning runs and tests).  Invalid overrides -> SABLE_E_INVALID_ARG.
ExecCfg exec_config() {
  ExecCfg c{};
  c.pf = (int32_t)env_int("SABLE_XPREFETCH", 0);
  c.ustage = (int32_t)env_int("SABLE_USTAGE", kUnitBytes);
  c.rem_rows = (int32_t)env_int("SABLE_UREM_ROWS", 32);
  c.batch = (int32_t)env_int("SABLE_UBATCH_UNITS", kUnitBatch);
  c.batch_bytes = (int32_t)env_int("SABLE_UBATCH_BYTES", kBatchBytes);
  c.sliced = env_int("SABLE_SLICED", 0) != 0 ? 1 : 0;
  c.lpr_mode = (int32_t)env_int("SABLE_LPR", 0);
  const int64_t arch = env_int("SABLE_ARCH", 2);
  if (arch != 2 || c.ustage < 1024 || c.ustage % 16 != 0 || c.ustage > (1 << 24) ||
      c.rem_rows < 1 || c.rem_rows > 32 || c.batch < 1 || (c.pf != 0 && c.pf != 1) ||
      c.batch_bytes < 1 || c.lpr_mode < 0 || c.lpr_mode > 1) {
    set_error("invalid SABLE_ARCH / SABLE_USTAGE / SABLE_UREM_ROWS / SABLE_UBATCH_UNITS / "
              "SABLE_UBATCH_BYTES / SABLE_XPREFETCH (arch 2 only; ustage a multiple of 16 in "
              "[1024, 2^24]; 1..32 rows; batch >= 1; batch bytes >= 1)");
    throw Fail{SABLE_E_INVALID_ARG};
  }
  return c;
}

// ------------------------------------------------------------------- inspect

template <typename T>
void inspect(const sable_vbr_desc* d, const sable_delta_policy* pol, int32_t rank, int32_t world,
             cudaStream_t st, sable_handle* h) {
  const int32_t delta = (int32_t)pol->delta_pct;
  const int TH = 256;
  const int64_t nrows = d->nrows, ncols = d->ncols, nblk = d->nblocks, R = d->rem_nnz;
  const int32_t nbr = d->nbrows, nbc = d->nbcols;
  const size_t sv = sizeof(T);

  Inputs in{};
  stage_inputs(d, sv, in, st);
  const T* val = static_cast<const T*>(in.val);
  const T* rval = static_cast<const T*>(in.rval);

  // ---- a1: validate -------------------------------------------------------
  DevBuf errb;
  SB_CU(errb.alloc(sizeof(unsigned long long), st));
  unsigned long long* err = errb.as<unsigned long long>();
  SB_CU(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), st));
  k_check_grid<<<nblocks_for(nbr + 1, TH), TH, 0, st>>>(in.rpntr, nbr, nrows, V_RPNTR, err);
  k_check_grid<<<nblocks_for(nbc + 1, TH), TH, 0, st>>>(in.cpntr, nbc, ncols, V_CPNTR, err);
  k_check_ptr64<<<nblocks_for(nbr + 1, TH), TH, 0, st>>>(in.bpntr, nbr, nblk, V_BPNTR, err);
  if (R > 0 || in.rptr)
    k_check_ptr64<<<nblocks_for(nrows + 1, TH), TH, 0, st>>>(in.rptr, nrows, R, V_REMPTR, err);
  SB_CU(cudaGetLastError());
  check_err(err, st, SABLE_E_FORMAT);

  DevBuf blk_br_b, rowid_b;
  SB_CU(blk_br_b.alloc(sizeof(int32_t) * nblk, st));
  SB_CU(rowid_b.alloc(sizeof(int32_t) * R, st));
  int32_t* blk_br = blk_br_b.as<int32_t>();
  int32_t* rowid = rowid_b.as<int32_t>();
  k_check_blocks<<<nblocks_for(std::max<int64_t>(nblk, 1), TH), TH, 0, st>>>(
      in.rpntr, in.cpntr, in.bpntr, nbr, nbc, in.bindx, in.indx, nblk, d->val_len, blk_br, err);
  if (R > 0)
    k_rem_rows<<<nblocks_for(nrows * 32, TH), TH, 0, st>>>(in.rptr, in.ridx, nrows, ncols,
                                                          rowid, err);
  SB_CU(cudaGetLastError());
  check_err(err, st, SABLE_E_FORMAT);

  // ---- a2: count ------------------------------------------------------------
  DevBuf row2br_b, col2bc_b, cntv_b;
  SB_CU(row2br_b.alloc(sizeof(int32_t) * nrows, st));
  SB_CU(col2bc_b.alloc(sizeof(int32_t) * ncols, st));
  SB_CU(cntv_b.alloc(sizeof(int64_t) * nblk, st));
  int32_t* row2br = row2br_b.as<int32_t>();
  int32_t* col2bc = col2bc_b.as<int32_t>();
  int64_t* cnt_vbr = cntv_b.as<int64_t>();
  k_axis_map<<<nblocks_for(nrows, TH), TH, 0, st>>>(in.rpntr, nbr, nrows, row2br);
  k_axis_map<<<nblocks_for(ncols, TH), TH, 0, st>>>(in.cpntr, nbc, ncols, col2bc);
  if (nblk > 0) k_count_vbr<T><<<nblocks_for(nblk * 32, TH), TH, 0, st>>>(val, in.indx, nblk, cnt_vbr);

  const int64_t ns = nblk + R;
  const uint64_t sent = (uint64_t)nbr * (uint64_t)nbc;
  const int kbits = bits_for(sent);
  DevBuf key_b, key2_b, pay_b, pay2_b;
  SB_CU(key_b.alloc(sizeof(uint64_t) * ns, st));
  SB_CU(key2_b.alloc(sizeof(uint64_t) * ns, st));
  SB_CU(pay_b.alloc(sizeof(int32_t) * ns, st));
  SB_CU(pay2_b.alloc(sizeof(int32_t) * ns, st));
  if (nblk > 0)
    k_vbr_keys<<<nblocks_for(nblk, TH), TH, 0, st>>>(blk_br, in.bindx, cnt_vbr, nblk, nbc, sent,
                                                     key_b.as<uint64_t>(), pay_b.as<int32_t>());
  if (R > 0)
    k_rem_keys<T><<<nblocks_for(R, TH), TH, 0, st>>>(
        rowid, in.ridx, rval, R, row2br, col2bc, in.rpntr, in.cpntr, in.bpntr, in.bindx,
        in.indx, val, nblk, nbc, sent, key_b.as<uint64_t>(), pay_b.as<int32_t>(), err);
  SB_CU(cudaGetLastError());
  check_err(err, st, SABLE_E_FORMAT);
  if (ns > 0) {
    const uint64_t* kin = key_b.as<uint64_t>();
    uint64_t* kout = key2_b.as<uint64_t>();
    const int32_t* pin = pay_b.as<int32_t>();
    int32_t* pout = pay2_b.as<int32_t>();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, pin, pout, ns, 0, kbits, st);
    }, st);
  }
  const uint64_t* skey = key2_b.as<uint64_t>();
  const int32_t* spay = pay2_b.as<int32_t>();
  key_b.release();
  pay_b.release();

  DevBuf flag_b, cid_b;
  SB_CU(flag_b.alloc(sizeof(int32_t) * ns, st));
  SB_CU(cid_b.alloc(sizeof(int32_t) * ns, st));
  int64_t n_cells_all = 0;
  if (ns > 0) {
    k_heads<<<nblocks_for(ns, TH), TH, 0, st>>>(skey, ns, sent, flag_b.as<int32_t>());
    const int32_t* fl = flag_b.as<int32_t>();
    int32_t* cid = cid_b.as<int32_t>();
    cub_run([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, fl, cid, ns, st); }, st);
    int32_t last = 0;
    d2h(&last, cid + (ns - 1), 1, st);
    SB_CU(cudaStreamSynchronize(st));
    n_cells_all = last;
  }
  DevBuf ckey_b, ccnt_b, cblk_b, ecell_b;
  SB_CU(ckey_b.alloc(sizeof(uint64_t) * n_cells_all, st));
  SB_CU(ccnt_b.alloc(sizeof(int64_t) * n_cells_all, st));
  SB_CU(cblk_b.alloc(sizeof(int32_t) * n_cells_all, st));
  SB_CU(ecell_b.alloc(sizeof(int32_t) * R, st));
  int64_t* cell_cnt = ccnt_b.as<int64_t>();
  int32_t* cell_blk = cblk_b.as<int32_t>();
  int32_t* ecell = ecell_b.as<int32_t>();
  SB_CU(cudaMemsetAsync(cell_cnt, 0, sizeof(int64_t) * n_cells_all, st));
  SB_CU(cudaMemsetAsync(cell_blk, 0xff, sizeof(int32_t) * n_cells_all, st));
  SB_CU(cudaMemsetAsync(ecell, 0xff, sizeof(int32_t) * R, st));
  if (ns > 0)
    k_cells<<<nblocks_for(ns, TH), TH, 0, st>>>(skey, spay, cid_b.as<int32_t>(), ns, sent, nblk,
                                                cnt_vbr, ckey_b.as<uint64_t>(), cell_cnt,
                                                cell_blk, ecell);
  key2_b.release();
  pay2_b.release();
  flag_b.release();
  cid_b.release();

  // ---- a3: classify -----------------------------------------------------------
  DevBuf cbr_b, cbc_b, cden_b, brs_b;
  SB_CU(cbr_b.alloc(sizeof(int32_t) * n_cells_all, st));
  SB_CU(cbc_b.alloc(sizeof(int32_t) * n_cells_all, st));
  SB_CU(cden_b.alloc(n_cells_all, st));
  // per block row: ncell, ndense, W (int32) | area, rem, vbrsparse (uint64)
  const size_t brs_bytes = (sizeof(int32_t) * 3 + sizeof(uint64_t) * 3) * (size_t)nbr;
  SB_CU(brs_b.alloc(brs_bytes, st));
  SB_CU(cudaMemsetAsync(brs_b.p, 0, brs_bytes, st));
  // 8-byte counters first so that every array stays naturally aligned
  unsigned long long* br_area = brs_b.as<unsigned long long>();
  unsigned long long* br_rem = br_area + nbr;
  unsigned long long* br_vsp = br_rem + nbr;
  int32_t* br_ncell = reinterpret_cast<int32_t*>(br_vsp + nbr);
  int32_t* br_ndense = br_ncell + nbr;
  int32_t* br_Wd = br_ndense + nbr;
  int32_t* cell_br = cbr_b.as<int32_t>();
  int32_t* cell_bc = cbc_b.as<int32_t>();
  uint8_t* cell_dense = cden_b.as<uint8_t>();
  DevBuf rules_b;
  SB_CU(rules_b.alloc(sizeof(sable_delta_rule) * std::max<int32_t>(pol->n_rules, 1), st));
  const sable_delta_rule* rules_d = rules_b.as<sable_delta_rule>();
  if (pol->n_rules > 0)
    SB_CU(cudaMemcpyAsync(rules_b.p, pol->rules, sizeof(sable_delta_rule) * pol->n_rules,
                          cudaMemcpyHostToDevice, st));
  if (n_cells_all > 0)
    k_classify<T><<<nblocks_for(n_cells_all, TH), TH, 0, st>>>(
        ckey_b.as<uint64_t>(), cell_cnt, cell_blk, cnt_vbr, n_cells_all, nbc, in.rpntr,
        in.cpntr, delta, pol->min_area, pol->n_rules, rules_d, cell_br, cell_bc, cell_dense,
        br_ncell, br_ndense, br_Wd, br_area, br_rem, br_vsp);
  SB_CU(cudaGetLastError());

  std::vector<int32_t> H_ncell(nbr), H_ndense(nbr), H_W(nbr), H_rpntr(nbr + 1);
  std::vector<uint64_t> H_area(nbr), H_rem(nbr), H_vsp(nbr);
  d2h(H_ncell.data(), br_ncell, nbr, st);
  d2h(H_ndense.data(), br_ndense, nbr, st);
  d2h(H_W.data(), br_Wd, nbr, st);
  d2h(H_area.data(), (const uint64_t*)br_area, nbr, st);
  d2h(H_rem.data(), (const uint64_t*)br_rem, nbr, st);
  d2h(H_vsp.data(), (const uint64_t*)br_vsp, nbr, st);
  d2h(H_rpntr.data(), in.rpntr, nbr + 1, st);
  SB_CU(cudaStreamSynchronize(st));

  // ---- shard (north_star s7) -------------------------------------------------
  std::vector<int64_t> weight(nbr);
  for (int32_t a = 0; a < nbr; ++a) weight[a] = (int64_t)(H_area[a] + H_rem[a]);
  std::vector<int32_t> bounds(world + 1);
  sable_shard_bounds(weight.data(), nbr, world, bounds.data());
  const int32_t b0 = bounds[rank], b1 = bounds[rank + 1];
  h->all_bounds_h = (int32_t*)malloc(sizeof(int32_t) * (world + 1));
  h->rpntr_h = (int32_t*)malloc(sizeof(int32_t) * (nbr + 1));
  if (!h->all_bounds_h || !h->rpntr_h) {
    set_error("host allocation failed");
    throw Fail{SABLE_E_OOM};
  }
  std::copy(bounds.begin(), bounds.end(), h->all_bounds_h);
  std::copy(H_rpntr.begin(), H_rpntr.end(), h->rpntr_h);
  h->br_begin = b0;
  h->br_end = b1;
  h->row_begin = H_rpntr[b0];
  h->row_end = H_rpntr[b1];
  const int64_t nloc = h->row_end - h->row_begin;
  const int32_t nbl = b1 - b0;

  int64_t cell_lo = 0, n_cells = 0, tile_lo = 0, n_dense = 0, n_dense_global = 0;
  int64_t vsp_local = 0, tile_elems = 0;
  std::vector<int64_t> br_vbase(nbl + 1), br_wprefix(nbl + 1), br_t0(nbl + 1);
  for (int32_t a = 0; a < nbr; ++a) {
    n_dense_global += H_ndense[a];
    if (a < b0) {
      cell_lo += H_ncell[a];
      tile_lo += H_ndense[a];
    }
  }
  for (int32_t la = 0; la < nbl; ++la) {
    const int32_t a = b0 + la;
    br_vbase[la] = tile_elems;
    br_t0[la] = n_dense;
    br_wprefix[la] = (la ? br_wprefix[la - 1] + H_W[a - 1] : 0);
    tile_elems += (int64_t)H_area[a];
    n_dense += H_ndense[a];
    n_cells += H_ncell[a];
    vsp_local += (int64_t)H_vsp[a];
  }
  br_vbase[nbl] = tile_elems;
  br_t0[nbl] = n_dense;
  br_wprefix[nbl] = nbl ? br_wprefix[nbl - 1] + H_W[b1 - 1] : 0;
  if (br_wprefix[nbl] > INT32_MAX - 1) {
    set_error("local dense tiles span more than 2^31-1 panel columns");
    throw Fail{SABLE_E_UNSUPPORTED};
  }
  const int64_t cell_hi = cell_lo + n_cells;
  h->cell_base = cell_lo;
  h->n_cells = n_cells;
  h->n_dense = n_dense;
  h->n_dense_global = n_dense_global;
  h->tile_elems = tile_elems;

  // local cells for export
  h->cell_br = dev_alloc<int32_t>(n_cells, st);
  h->cell_bc = dev_alloc<int32_t>(n_cells, st);
  h->cell_cnt = dev_alloc<int64_t>(n_cells, st);
  h->cell_dense = dev_alloc<uint8_t>(n_cells, st);
  if (n_cells > 0) {
    SB_CU(cudaMemcpyAsync(h->cell_br, cell_br + cell_lo, sizeof(int32_t) * n_cells, cudaMemcpyDeviceToDevice, st));
    SB_CU(cudaMemcpyAsync(h->cell_bc, cell_bc + cell_lo, sizeof(int32_t) * n_cells, cudaMemcpyDeviceToDevice, st));
    SB_CU(cudaMemcpyAsync(h->cell_cnt, cell_cnt + cell_lo, sizeof(int64_t) * n_cells, cudaMemcpyDeviceToDevice, st));
    SB_CU(cudaMemcpyAsync(h->cell_dense, cell_dense + cell_lo, n_cells, cudaMemcpyDeviceToDevice, st));
  }

  // ---- a4: pack the local dense tiles ---------------------------------------------
  DevBuf tcell_b, tarea_b, tw_b, wscan_b, ctile_b, wpre_b;
  SB_CU(tcell_b.alloc(sizeof(int32_t) * n_dense, st));
  SB_CU(ctile_b.alloc(sizeof(int32_t) * n_cells, st));
  int32_t* tile_cell = tcell_b.as<int32_t>();
  int32_t* cell_tile = ctile_b.as<int32_t>();
  SB_CU(cudaMemsetAsync(cell_tile, 0xff, sizeof(int32_t) * n_cells, st));
  if (n_dense > 0) {
    DevBuf nsel;
    SB_CU(nsel.alloc(sizeof(int64_t), st));
    thrust::counting_iterator<int32_t> ids((int32_t)cell_lo);
    const uint8_t* fl = cell_dense + cell_lo;
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, ids, fl, tile_cell, nsel.as<int64_t>(), n_cells, st);
    }, st);
  }
  h->tile_br = dev_alloc<int32_t>(n_dense, st);
  h->tiles = dev_alloc<TileDesc>(n_dense, st);
  DevBuf xt_b;  // plan-time map of the tiles' columns
  SB_CU(xt_b.alloc(sizeof(XTile) * (n_dense + 1), st));
  XTile* xt = xt_b.as<XTile>();
  SB_CU(cudaMemsetAsync(xt, 0, sizeof(XTile) * (n_dense + 1), st));
  h->tile_canon_off = dev_alloc<int64_t>(n_dense + 1, st);
  DevBuf vbase_b;
  SB_CU(vbase_b.alloc(sizeof(int64_t) * (nbl + 1), st));
  int64_t* d_vbase = vbase_b.as<int64_t>();
  h->br_W = dev_alloc<int32_t>(nbl + 1, st);
  SB_CU(cudaMemcpyAsync(d_vbase, br_vbase.data(), sizeof(int64_t) * (nbl + 1), cudaMemcpyHostToDevice, st));
  std::vector<int32_t> Wloc(nbl + 1, 0);
  for (int32_t la = 0; la < nbl; ++la) Wloc[la] = H_W[b0 + la];
  SB_CU(cudaMemcpyAsync(h->br_W, Wloc.data(), sizeof(int32_t) * (nbl + 1), cudaMemcpyHostToDevice, st));
  SB_CU(wpre_b.alloc(sizeof(int64_t) * (nbl + 1), st));
  SB_CU(cudaMemcpyAsync(wpre_b.p, br_wprefix.data(), sizeof(int64_t) * (nbl + 1), cudaMemcpyHostToDevice, st));
  SB_CU(tarea_b.alloc(sizeof(int64_t) * (n_dense + 1), st));
  SB_CU(tw_b.alloc(sizeof(int32_t) * (n_dense + 1), st));
  SB_CU(wscan_b.alloc(sizeof(int64_t) * (n_dense + 1), st));
  SB_CU(cudaMemsetAsync(h->tile_canon_off, 0, sizeof(int64_t), st));
  if (n_dense > 0) {
    k_tile_meta<<<nblocks_for(n_dense, TH), TH, 0, st>>>(tile_cell, n_dense, cell_br, cell_bc,
                                                         in.rpntr, in.cpntr, cell_lo, h->tile_br,
                                                         tarea_b.as<int64_t>(), tw_b.as<int32_t>(),
                                                         cell_tile);
    const int64_t* ta = tarea_b.as<int64_t>();
    int64_t* co = h->tile_canon_off + 1;
    cub_run([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, ta, co, n_dense, st); }, st);
    const int32_t* tw = tw_b.as<int32_t>();
    int64_t* ws = wscan_b.as<int64_t>();
    auto tw64 = thrust::make_transform_iterator(tw, Widen());
    cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, tw64, ws, n_dense, st); }, st);
    k_tile_desc<<<nblocks_for(n_dense, TH), TH, 0, st>>>(tile_cell, n_dense, cell_bc, h->tile_br,
                                                         tw, ws, wpre_b.as<int64_t>(), b0,
                                                         in.cpntr, h->tiles, xt);
  }
  // staging slabs of the dense tiles (row groups, column-major), repacked
  // into the executor's row-major panels by plan_units and then freed
  DevBuf tval_b;
  SB_CU(tval_b.alloc(sizeof(T) * std::max<int64_t>(tile_elems, 1), st));
  T* tval = tval_b.as<T>();
  SB_CU(cudaMemsetAsync(tval, 0, sizeof(T) * std::max<int64_t>(tile_elems, 1), st));
  if (n_dense > 0)
    k_pack_vbr<T><<<(unsigned)n_dense, 128, 0, st>>>(tile_cell, n_dense, cell_blk, h->tile_br,
                                                      h->tiles, in.rpntr, in.indx, val,
                                                      d_vbase, h->br_W, b0, tval);
  if (n_dense > 0 && R > 0)
    k_pack_rem<T><<<nblocks_for(R, TH), TH, 0, st>>>(rowid, in.ridx, rval, R, ecell, cell_lo,
                                                     cell_hi, cell_tile, h->tile_br, h->tiles,
                                                     in.rpntr, d_vbase, h->br_W, b0, tval);
  SB_CU(cudaGetLastError());

  // ---- a4: the local CSR remainder ------------------------------------------------
  int64_t n_keep = 0;
  DevBuf keep_b, kidx_b, kval_b, krow_b;
  if (R > 0) {
    SB_CU(keep_b.alloc(R, st));
    k_rem_keep<<<nblocks_for(R, TH), TH, 0, st>>>(ecell, R, cell_lo, cell_hi, cell_dense,
                                                  keep_b.as<uint8_t>());
    DevBuf nsel;
    SB_CU(nsel.alloc(sizeof(int64_t), st));
    SB_CU(kidx_b.alloc(sizeof(int32_t) * R, st));
    SB_CU(kval_b.alloc(sv * R, st));
    SB_CU(krow_b.alloc(sizeof(int32_t) * R, st));
    const uint8_t* fl = keep_b.as<uint8_t>();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, in.ridx, fl, kidx_b.as<int32_t>(), nsel.as<int64_t>(), R, st);
    }, st);
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, rval, fl, kval_b.as<T>(), nsel.as<int64_t>(), R, st);
    }, st);
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, (const int32_t*)rowid, fl, krow_b.as<int32_t>(), nsel.as<int64_t>(), R, st);
    }, st);
    d2h(&n_keep, nsel.as<int64_t>(), 1, st);
    SB_CU(cudaStreamSynchronize(st));
  }
  const int64_t n_rem = n_keep + vsp_local;
  if (n_rem > INT32_MAX - 1) {
    set_error("local remainder exceeds 2^31-1 entries");
    throw Fail{SABLE_E_UNSUPPORTED};
  }
  h->rem_nnz = n_rem;
  h->rem_idx = dev_alloc<int32_t>(n_rem, st);
  h->rem_val = dev_alloc<T>(n_rem, st);
  h->rem_ptr = dev_alloc<int32_t>(nloc + 1, st);
  DevBuf rcount_b, rrows_b;
  SB_CU(rcount_b.alloc(sizeof(int32_t) * (nloc + 1), st));
  SB_CU(cudaMemsetAsync(rcount_b.p, 0, sizeof(int32_t) * (nloc + 1), st));
  const int32_t* rows_src = nullptr;
  if (vsp_local == 0) {
    // fast path: the kept input entries are already row-major, columns ascending
    if (n_keep > 0) {
      SB_CU(cudaMemcpyAsync(h->rem_idx, kidx_b.p, sizeof(int32_t) * n_keep, cudaMemcpyDeviceToDevice, st));
      SB_CU(cudaMemcpyAsync(h->rem_val, kval_b.p, sv * n_keep, cudaMemcpyDeviceToDevice, st));
    }
    rows_src = krow_b.as<int32_t>();
  } else {
    // general path: add the non-zeros of sparse VBR blocks, sort by (i, j)
    DevBuf k1, v1, k2, v2, sflag, scell, scnt, spos, cur, nsel;
    SB_CU(k1.alloc(sizeof(uint64_t) * n_rem, st));
    SB_CU(v1.alloc(sv * n_rem, st));
    SB_CU(k2.alloc(sizeof(uint64_t) * n_rem, st));
    SB_CU(v2.alloc(sv * n_rem, st));
    if (n_keep > 0)
      k_rem_pairs<T><<<nblocks_for(n_keep, TH), TH, 0, st>>>(krow_b.as<int32_t>(), kidx_b.as<int32_t>(),
                                                             kval_b.as<T>(), n_keep, h->row_begin,
                                                             ncols, k1.as<uint64_t>(), v1.as<T>());
    SB_CU(sflag.alloc(n_cells, st));
    SB_CU(scell.alloc(sizeof(int32_t) * n_cells, st));
    SB_CU(nsel.alloc(sizeof(int64_t), st));
    k_sparse_vbr_flags<<<nblocks_for(n_cells, TH), TH, 0, st>>>(cell_blk, cell_dense, cell_lo,
                                                               n_cells, sflag.as<uint8_t>());
    thrust::counting_iterator<int32_t> ids((int32_t)cell_lo);
    const uint8_t* sfl = sflag.as<uint8_t>();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, ids, sfl, scell.as<int32_t>(), nsel.as<int64_t>(), n_cells, st);
    }, st);
    int64_t nsp = 0;
    d2h(&nsp, nsel.as<int64_t>(), 1, st);
    SB_CU(cudaStreamSynchronize(st));
    SB_CU(scnt.alloc(sizeof(int64_t) * nsp, st));
    SB_CU(spos.alloc(sizeof(int64_t) * nsp, st));
    SB_CU(cur.alloc(sizeof(unsigned long long) * nsp, st));
    SB_CU(cudaMemsetAsync(cur.p, 0, sizeof(unsigned long long) * std::max<int64_t>(nsp, 1), st));
    if (nsp > 0) {
      k_sparse_vbr_cnt<<<nblocks_for(nsp, TH), TH, 0, st>>>(scell.as<int32_t>(), nsp, cell_blk,
                                                           cnt_vbr, scnt.as<int64_t>());
      const int64_t* sc = scnt.as<int64_t>();
      int64_t* sp = spos.as<int64_t>();
      cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, sc, sp, nsp, st); }, st);
      k_emit_sparse_vbr<T><<<(unsigned)nsp, 128, 0, st>>>(
          scell.as<int32_t>(), nsp, spos.as<int64_t>(), cell_blk, cell_br, cell_bc, in.rpntr,
          in.cpntr, in.indx, val, h->row_begin, ncols, n_keep, cur.as<unsigned long long>(),
          k1.as<uint64_t>(), v1.as<T>());
    }
    const int kb = bits_for((uint64_t)std::max<int64_t>(nloc, 1) * (uint64_t)ncols);
    const uint64_t* ki = k1.as<uint64_t>();
    const T* vi = v1.as<T>();
    uint64_t* ko = k2.as<uint64_t>();
    T* vo = v2.as<T>();
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, n_rem, 0, kb, st);
    }, st);
    SB_CU(rrows_b.alloc(sizeof(int32_t) * n_rem, st));
    k_unpair<<<nblocks_for(n_rem, TH), TH, 0, st>>>(ko, n_rem, ncols, h->rem_idx, rrows_b.as<int32_t>());
    SB_CU(cudaMemcpyAsync(h->rem_val, vo, sv * n_rem, cudaMemcpyDeviceToDevice, st));
    SB_CU(cudaStreamSynchronize(st));  // k1..v2 are released at scope exit
    rows_src = rrows_b.as<int32_t>();
  }
  if (n_rem > 0) {
    const int64_t rb = vsp_local == 0 ? h->row_begin : 0;
    k_row_count<<<nblocks_for(n_rem, TH), TH, 0, st>>>(rows_src, n_rem, rb, rcount_b.as<int32_t>());
  }
  {
    const int32_t* rc = rcount_b.as<int32_t>();
    int32_t* rp = h->rem_ptr;
    cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, rc, rp, nloc + 1, st); }, st);
  }
  SB_CU(cudaGetLastError());

  // ---- a5: plan (host) ---------------------------------------------------------------
  std::vector<int32_t> H_rp(nloc + 1);
  d2h(H_rp.data(), h->rem_ptr, nloc + 1, st);
  std::vector<XTile> H_xt(n_dense + 1);
  d2h(H_xt.data(), xt, n_dense + 1, st);
  SB_CU(cudaStreamSynchronize(st));
  h->cfg = exec_config();
  std::vector<int64_t> br_pbase;
  SB_CU(plan_units<T>(h, tval, nbl, b0, H_rpntr, H_W, br_vbase, br_wprefix, br_t0, H_rp, H_xt,
                      br_pbase, st));
  h->br_pbase = dev_alloc<int64_t>(nbl + 1, st);
  SB_CU(cudaMemcpyAsync(h->br_pbase, br_pbase.data(), sizeof(int64_t) * (nbl + 1),
                        cudaMemcpyHostToDevice, st));

  // ---- bookkeeping ---------------------------------------------------------------------
  int64_t nnz = 0;
  {
    std::vector<int64_t> cc(n_cells);
    d2h(cc.data(), h->cell_cnt, n_cells, st);
    SB_CU(cudaStreamSynchronize(st));
    for (int64_t c : cc) nnz += c;
  }
  h->nnz = nnz;
  // algorithmic bytes per SpMV: tile
  // values + a 12-byte descriptor per tile + remainder (value, index) + row
  // pointers + x read once + y written once
  h->bytes_alg = tile_elems * (int64_t)sv + n_dense * 12 + n_rem * (int64_t)(sv + 4) +
                 (nloc + 1) * 4 + ncols * (int64_t)sv + nloc * (int64_t)sv;
  SB_CU(cudaStreamSynchronize(st));
}

}  // namespace

sable_status create_impl(const sable_vbr_desc* d, const sable_delta_policy* pol,
                         const sable_shard* sh, cudaStream_t st, sable_handle** out) {
  const auto t0 = std::chrono::steady_clock::now();
  sable_handle* h = new (std::nothrow) sable_handle();
  if (!h) {
    set_error("host allocation failed");
    return SABLE_E_OOM;
  }
  h->dtype = d->dtype;
  h->delta = (int32_t)pol->delta_pct;
  h->nrows = d->nrows;
  h->ncols = d->ncols;
  h->nbr = d->nbrows;
  h->nbc = d->nbcols;
  h->rank = sh ? sh->rank : 0;
  h->world = sh ? sh->world : 1;
  cudaGetDevice(&h->device);
  try {
    if (d->dtype == SABLE_F64)
      inspect<double>(d, pol, h->rank, h->world, st, h);
    else
      inspect<float>(d, pol, h->rank, h->world, st, h);
  } catch (const Fail& f) {
    cudaStreamSynchronize(st);
    free_handle(h);
    return f.st;
  }
  h->inspect_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = h;
  return SABLE_OK;
}

}  // namespace sable
