// abi.cu -- the extern "C" entry points of libsable.so (include/sable.h).
// Argument checking, error text, handle lifetime, info and the canonical
// partition export.  The arithmetic lives in inspect.cu, plan.cu and unit.cu.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>
#include <cstring>
#include <string>
#include <vector>

#include "sable_internal.cuh"

namespace sable {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

std::string cuda_msg(cudaError_t e, const char* what) {
  return std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
}

sable_status create_impl(const sable_vbr_desc* d, const sable_delta_policy* pol,
                         const sable_shard* sh, cudaStream_t st, sable_handle** out);
cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st);
cudaError_t run_spmm(const sable_handle* h, const void* X, void* Y, int32_t k, void* scratch,
                     cudaStream_t st);
cudaError_t run_spmm_mma(const sable_handle* h, const void* X, void* Y, int32_t k, void* scratch,
                         cudaStream_t st);
sable_status comm_destroy(sable_handle* h);
int32_t exec_grid(const sable_handle* h);

cudaError_t set_smem_attr(const void* func, int device, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{func, device}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

void free_handle(sable_handle* h) {
  if (!h) return;
  void* dev[] = {h->rem_ptr,  h->rem_idx,   h->rem_val,    h->pv,          h->units,
                 h->ubatch,   h->xq,        h->xside,      h->uxg,         h->uscratch,
                 h->ucounters, h->mm_scratch, h->mma_scratch, h->cell_br,  h->cell_bc,     h->cell_cnt,
                 h->cell_dense, h->tiles,   h->tile_canon_off, h->tile_br, h->br_pbase,
                 h->br_W,     h->x_dev,     h->y_dev,       h->ubhead};
  for (void* p : dev)
    if (p) cudaFree(p);
  free(h->all_bounds_h);
  free(h->rpntr_h);
  delete h;
}

namespace {

sable_status fail(sable_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

sable_status cuda_fail(cudaError_t e, const char* what) {
  set_error(cuda_msg(e, what));
  return e == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA;
}

template <typename T>
__global__ void k_unpack_tiles(const int64_t* canon_off, const TileDesc* desc,
                               const int32_t* tile_br, const int64_t* br_pbase,
                               const int32_t* br_W, int32_t br_begin, const T* pv, T* out) {
  const int64_t t = blockIdx.x;
  const int64_t off = canon_off[t], area = canon_off[t + 1] - off;
  const TileDesc d = desc[t];
  const int64_t h = area / d.w;
  const int32_t la = tile_br[t] - br_begin;
  const int64_t vec = 16 / (int64_t)sizeof(T);
  for (int64_t e = threadIdx.x; e < area; e += blockDim.x)  // canonical column-major
    out[off + e] = pv[panel_rm_pos(br_pbase[la], br_W[la], vec, d.cs, e % h, e / h)];
}

__global__ void k_not(const uint8_t* in, int64_t n, uint8_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] ? 0 : 1;
}

__global__ void k_ptr64(const int32_t* in, int64_t n, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

template <typename T>
sable_status export_tiles(const sable_handle* h, void* host_out) {
  if (h->tile_elems == 0) return SABLE_OK;
  T* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, sizeof(T) * h->tile_elems);
  if (e) return cuda_fail(e, "cudaMalloc(export tiles)");
  k_unpack_tiles<T><<<(unsigned)h->n_dense, 128>>>(h->tile_canon_off, h->tiles, h->tile_br,
                                                  h->br_pbase, h->br_W, h->br_begin,
                                                  static_cast<const T*>(h->pv), buf);
  e = cudaGetLastError();
  if (!e) e = cudaMemcpy(host_out, buf, sizeof(T) * h->tile_elems, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  return e ? cuda_fail(e, "export tiles") : SABLE_OK;
}

}  // namespace
}  // namespace sable

using namespace sable;

extern "C" {

int32_t sable_abi_version(void) { return SABLE_ABI_VERSION; }

const char* sable_last_error(void) { return g_last_error.c_str(); }

const char* sable_status_string(sable_status s) {
  switch (s) {
    case SABLE_OK: return "SABLE_OK";
    case SABLE_E_INVALID_ARG: return "SABLE_E_INVALID_ARG";
    case SABLE_E_FORMAT: return "SABLE_E_FORMAT";
    case SABLE_E_DIM: return "SABLE_E_DIM";
    case SABLE_E_DUPLICATE: return "SABLE_E_DUPLICATE";
    case SABLE_E_OOM: return "SABLE_E_OOM";
    case SABLE_E_CUDA: return "SABLE_E_CUDA";
    case SABLE_E_NCCL: return "SABLE_E_NCCL";
    case SABLE_E_UNSUPPORTED: return "SABLE_E_UNSUPPORTED";
  }
  return "SABLE_E_?";
}

sable_status sable_shard_bounds(const int64_t* weights, int32_t nbrows, int32_t world,
                                int32_t* bounds) {
  if (!bounds || world < 1 || nbrows < 0 || (nbrows > 0 && !weights))
    return fail(SABLE_E_INVALID_ARG, "sable_shard_bounds: bad arguments");
  long double total = 0;
  for (int32_t a = 0; a < nbrows; ++a) {
    if (weights[a] < 0) return fail(SABLE_E_INVALID_ARG, "sable_shard_bounds: negative weight");
    total += (long double)weights[a];
  }
  // boundary k = first a whose prefix weight (sum of weights[0..a)) reaches k*total/world
  bounds[0] = 0;
  int32_t a = 0;
  long double prefix = 0;
  for (int32_t k = 1; k < world; ++k) {
    const long double target = total * (long double)k / (long double)world;
    while (a < nbrows && prefix < target) prefix += (long double)weights[a++];
    bounds[k] = a;
  }
  bounds[world] = nbrows;
  return SABLE_OK;
}

sable_status sable_vbr_create_policy(const sable_vbr_desc* d, const sable_delta_policy* pol,
                                     const sable_shard* shard, void* cuda_stream,
                                     sable_handle** out) {
  if (out) *out = nullptr;
  if (!d || !out || !pol) return fail(SABLE_E_INVALID_ARG, "sable_vbr_create: NULL desc, policy or out");
  if (pol->delta_pct > 101) return fail(SABLE_E_INVALID_ARG, "delta_pct must be in [0, 101]");
  if (pol->min_area < 0 || pol->n_rules < 0 || pol->n_rules > 64 || (pol->n_rules > 0 && !pol->rules))
    return fail(SABLE_E_INVALID_ARG, "delta policy: min_area >= 0 and 0..64 rules");
  for (int32_t k = 0; k < pol->n_rules; ++k)
    if (pol->rules[k].delta_pct > 101)
      return fail(SABLE_E_INVALID_ARG, "delta policy: rule delta must be in [0, 101]");
  if (d->dtype != SABLE_F32 && d->dtype != SABLE_F64)
    return fail(SABLE_E_INVALID_ARG, "dtype must be SABLE_F32 or SABLE_F64");
  if (d->mem != SABLE_MEM_HOST && d->mem != SABLE_MEM_DEVICE)
    return fail(SABLE_E_INVALID_ARG, "mem must be SABLE_MEM_HOST or SABLE_MEM_DEVICE");
  if (d->nrows < 1 || d->ncols < 1 || d->nbrows < 1 || d->nbcols < 1 || d->nblocks < 0 ||
      d->val_len < 0 || d->rem_nnz < 0)
    return fail(SABLE_E_DIM, "sizes must be positive (nrows, ncols, nbrows, nbcols >= 1)");
  if (d->nrows >= (1ll << 31) - 1 || d->ncols >= (1ll << 31) - 1 ||
      d->nblocks + d->rem_nnz >= (1ll << 31) - 1)
    return fail(SABLE_E_UNSUPPORTED, "nrows, ncols and nblocks + rem_nnz must be < 2^31");
  if (d->nbrows > d->nrows || d->nbcols > d->ncols)
    return fail(SABLE_E_FORMAT, "more block rows/columns than rows/columns");
  if (!d->rpntr || !d->cpntr || !d->bpntr || !d->indx || (d->nblocks > 0 && !d->bindx) ||
      (d->val_len > 0 && !d->val))
    return fail(SABLE_E_INVALID_ARG, "NULL VBR array");
  const bool any_rem = d->rem_indptr || d->rem_indices || d->rem_val;
  if (any_rem && !d->rem_indptr) return fail(SABLE_E_INVALID_ARG, "remainder without rem_indptr");
  if (d->rem_nnz > 0 && (!d->rem_indptr || !d->rem_indices || !d->rem_val))
    return fail(SABLE_E_INVALID_ARG, "rem_nnz > 0 needs rem_indptr, rem_indices and rem_val");
  sable_shard sh{0, 1};
  if (shard) sh = *shard;
  if (sh.world < 1 || sh.rank < 0 || sh.rank >= sh.world)
    return fail(SABLE_E_INVALID_ARG, "shard: need 0 <= rank < world");
  set_error("");
  return create_impl(d, pol, &sh, static_cast<cudaStream_t>(cuda_stream), out);
}

sable_status sable_vbr_create(const sable_vbr_desc* d, uint32_t delta_pct,
                              const sable_shard* shard, void* cuda_stream, sable_handle** out) {
  const sable_delta_policy pol{delta_pct, 0, 0, nullptr};
  return sable_vbr_create_policy(d, &pol, shard, cuda_stream, out);
}

sable_status sable_spmv(sable_handle* h, const void* x, void* y, void* cuda_stream) {
  if (!h || !x || (!y && h->row_end > h->row_begin))
    return fail(SABLE_E_INVALID_ARG, "sable_spmv: NULL argument");
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_spmv: cudaSetDevice");
  const cudaError_t e = run_spmv(h, x, y, static_cast<cudaStream_t>(cuda_stream));
  return e ? cuda_fail(e, "spmv launch") : SABLE_OK;
}

sable_status sable_spmv_host(sable_handle* h, const void* x_host, void* y_host,
                             void* cuda_stream) {
  if (!h || !x_host || !y_host) return fail(SABLE_E_INVALID_ARG, "sable_spmv_host: NULL argument");
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_spmv_host: cudaSetDevice");
  const size_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  const int64_t nloc = h->row_end - h->row_begin;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = cudaSuccess;
  if (!h->x_dev) e = cudaMalloc(&h->x_dev, sv * h->ncols);
  if (!e && !h->y_dev) e = cudaMalloc(&h->y_dev, sv * std::max<int64_t>(nloc, 1));
  if (e) return cuda_fail(e, "cudaMalloc(e2e staging)");
  e = cudaMemcpyAsync(h->x_dev, x_host, sv * h->ncols, cudaMemcpyHostToDevice, st);
  if (!e) e = run_spmv(h, h->x_dev, h->y_dev, st);
  if (!e && nloc > 0) e = cudaMemcpyAsync(y_host, h->y_dev, sv * nloc, cudaMemcpyDeviceToHost, st);
  if (!e) e = cudaStreamSynchronize(st);
  return e ? cuda_fail(e, "sable_spmv_host") : SABLE_OK;
}

sable_status sable_destroy(sable_handle* h) {
  if (!h) return SABLE_OK;
  cudaDeviceSynchronize();
  comm_destroy(h);
  free_handle(h);
  return SABLE_OK;
}

sable_status sable_get_info(const sable_handle* h, sable_info* info) {
  if (!h || !info) return fail(SABLE_E_INVALID_ARG, "sable_get_info: NULL argument");
  memset(info, 0, sizeof(*info));
  info->nrows = h->nrows;
  info->ncols = h->ncols;
  info->nbrows = h->nbr;
  info->nbcols = h->nbc;
  info->br_begin = h->br_begin;
  info->br_end = h->br_end;
  info->row_begin = h->row_begin;
  info->row_end = h->row_end;
  info->nnz = h->nnz;
  info->n_cells = h->n_cells;
  info->cell_base = h->cell_base;
  info->n_dense = h->n_dense;
  info->tile_elems = h->tile_elems;
  info->rem_nnz = h->rem_nnz;
  info->n_dense_global = h->n_dense_global;
  info->bytes_alg = h->bytes_alg;
  info->dtype = h->dtype;
  info->delta = h->delta;
  info->suitable = h->n_dense_global > 0 ? 1 : 0;
  info->world = h->world;
  info->rank = h->rank;
  info->inspect_ms = h->inspect_ms;
  info->exec_grid = exec_grid(h);
  info->n_units = h->n_units;
  info->n_unit_batches = h->n_ubatch;
  info->n_combine = h->n_uxg;
  info->panel_elems = h->pv_elems;
  info->xmap_entries = h->n_xq;
  info->unit_bytes = h->cfg.ustage;
  return SABLE_OK;
}

sable_status sable_export_partition(const sable_handle* h, const sable_partition_host* o) {
  if (!h || !o) return fail(SABLE_E_INVALID_ARG, "sable_export_partition: NULL argument");
  const size_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  const int64_t nc = h->n_cells, nloc = h->row_end - h->row_begin;
  cudaError_t e = cudaDeviceSynchronize();
  if (e) return cuda_fail(e, "export sync");
#define CP(dst, src, bytes)                                                  \
  if ((dst) && (bytes) > 0) {                                                \
    e = cudaMemcpy((dst), (src), (bytes), cudaMemcpyDeviceToHost);          \
    if (e) return cuda_fail(e, "export copy " #dst);                         \
  }
  CP(o->cell_br, h->cell_br, sizeof(int32_t) * nc);
  CP(o->cell_bc, h->cell_bc, sizeof(int32_t) * nc);
  CP(o->cell_cnt, h->cell_cnt, sizeof(int64_t) * nc);
  CP(o->cell_dense, h->cell_dense, (size_t)nc);
  CP(o->tile_off, h->tile_canon_off, sizeof(int64_t) * (h->n_dense + 1));
  CP(o->rem_indices, h->rem_idx, sizeof(int32_t) * h->rem_nnz);
  CP(o->rem_val, h->rem_val, sv * h->rem_nnz);
  if (o->tile_val) {
    const sable_status s = h->dtype == SABLE_F64 ? export_tiles<double>(h, o->tile_val)
                                                 : export_tiles<float>(h, o->tile_val);
    if (s) return s;
  }
  if (o->rem_indptr) {
    int64_t* p = nullptr;
    e = cudaMalloc(&p, sizeof(int64_t) * (nloc + 1));
    if (e) return cuda_fail(e, "cudaMalloc(export indptr)");
    k_ptr64<<<(unsigned)((nloc + 1 + 255) / 256), 256>>>(h->rem_ptr, nloc + 1, p);
    e = cudaMemcpy(o->rem_indptr, p, sizeof(int64_t) * (nloc + 1), cudaMemcpyDeviceToHost);
    cudaFree(p);
    if (e) return cuda_fail(e, "export indptr");
  }
  if (o->ublocks && nc > h->n_dense) {
    uint8_t* fl = nullptr;
    int64_t* sel = nullptr;
    int64_t* nsel = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    thrust::counting_iterator<int64_t> ids(0);
    e = cudaMalloc(&fl, nc);
    if (!e) e = cudaMalloc(&sel, sizeof(int64_t) * nc);
    if (!e) e = cudaMalloc(&nsel, sizeof(int64_t));
    if (!e) {
      k_not<<<(unsigned)((nc + 255) / 256), 256>>>(h->cell_dense, nc, fl);
      e = cub::DeviceSelect::Flagged(nullptr, tb, ids, fl, sel, nsel, nc);
    }
    if (!e) e = cudaMalloc(&tmp, tb);
    if (!e) e = cub::DeviceSelect::Flagged(tmp, tb, ids, fl, sel, nsel, nc);
    if (!e)
      e = cudaMemcpy(o->ublocks, sel, sizeof(int64_t) * (nc - h->n_dense), cudaMemcpyDeviceToHost);
    cudaFree(fl);
    cudaFree(sel);
    cudaFree(nsel);
    cudaFree(tmp);
    if (e) return cuda_fail(e, "export ublocks");
  }
#undef CP
  return SABLE_OK;
}

sable_status sable_spmm(sable_handle* h, const void* X, void* Y, int32_t k, void* cuda_stream) {
  if (!h || !X || (!Y && h->row_end > h->row_begin))
    return fail(SABLE_E_INVALID_ARG, "sable_spmm: NULL argument");
  const bool cuda_cores = k == 1 || k == 2 || k == 4 || k == 8;
  const bool tensor = k == 16 || k == 32 || k == 64 || k == 128;
  if (!cuda_cores && !tensor)
    return fail(SABLE_E_UNSUPPORTED, "sable_spmm: k must be 1, 2, 4, 8, 16, 32, 64 or 128");
  if (tensor && h->dtype != SABLE_F32)
    return fail(SABLE_E_UNSUPPORTED, "sable_spmm: k >= 16 (tensor cores, 3xTF32) needs fp32");
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_spmm: cudaSetDevice");
  const size_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  // k-wide partials of split row ranges: allocated once (8 or 128 per slot)
  void** scr = tensor ? &h->mma_scratch : &h->mm_scratch;
  if (!*scr) {
    const cudaError_t e = cudaMalloc(scr, sv * (tensor ? 128 : 8) *
                                              (size_t)std::max<int64_t>(h->uscratch_slots, 1));
    if (e) {
      *scr = nullptr;
      return cuda_fail(e, "sable_spmm scratch");
    }
  }
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const cudaError_t e = tensor ? run_spmm_mma(h, X, Y, k, *scr, st) : run_spmm(h, X, Y, k, *scr, st);
  return e ? cuda_fail(e, "sable_spmm launch") : SABLE_OK;
}

}  // extern "C"
