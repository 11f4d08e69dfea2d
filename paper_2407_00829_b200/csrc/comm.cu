// comm.cu -- the multi-GPU exchange step (north_star s7:
// "each GPU holds the full x, and the y slices are all-gathered with NCCL
// over NVLink for iterated SpMV").
//
// sable_spmv_allgather writes the local y rows straight into x_next at
// [row_begin, row_end) and then all-gathers the variable-size slices with one
// ncclBroadcast per rank inside an NCCL group (an all-gatherv in place); over
// NVSwitch every rank receives (P-1)/P of x per step.
#include <nccl.h>

#include <cstring>

#include "sable_internal.cuh"

namespace sable {

cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st);

sable_status comm_destroy(sable_handle* h) {
  if (h && h->comm) {
    ncclCommDestroy(static_cast<ncclComm_t>(h->comm));
    h->comm = nullptr;
  }
  return SABLE_OK;
}

namespace {
sable_status nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return SABLE_E_NCCL;
}
}  // namespace

}  // namespace sable

using namespace sable;

extern "C" {

sable_status sable_nccl_unique_id(void* out128) {
  if (!out128) {
    set_error("sable_nccl_unique_id: NULL out");
    return SABLE_E_INVALID_ARG;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
  return SABLE_OK;
}

sable_status sable_comm_init(sable_handle* h, const void* id128) {
  if (!h || !id128) {
    set_error("sable_comm_init: NULL argument");
    return SABLE_E_INVALID_ARG;
  }
  comm_destroy(h);
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = ncclCommInitRank(&comm, h->world, id, h->rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  h->comm = comm;
  return SABLE_OK;
}

sable_status sable_spmv_allgather(sable_handle* h, const void* x_full, void* x_next_full,
                                  void* cuda_stream) {
  if (!h || !x_full || !x_next_full) {
    set_error("sable_spmv_allgather: NULL argument");
    return SABLE_E_INVALID_ARG;
  }
  if (h->nrows != h->ncols) {
    set_error("sable_spmv_allgather: the matrix must be square");
    return SABLE_E_DIM;
  }
  if (h->world > 1 && !h->comm) {
    set_error("sable_spmv_allgather: call sable_comm_init first");
    return SABLE_E_INVALID_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const size_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  char* xn = static_cast<char*>(x_next_full);
  cudaError_t e = run_spmv(h, x_full, xn + sv * h->row_begin, st);
  if (e) {
    set_error(cuda_msg(e, "spmv launch"));
    return SABLE_E_CUDA;
  }
  if (h->world == 1) return SABLE_OK;
  const ncclDataType_t dt = h->dtype == SABLE_F64 ? ncclFloat64 : ncclFloat32;
  ncclComm_t comm = static_cast<ncclComm_t>(h->comm);
  ncclResult_t r = ncclGroupStart();
  for (int32_t q = 0; q < h->world && r == ncclSuccess; ++q) {
    const int64_t b = h->rpntr_h[h->all_bounds_h[q]];
    const int64_t n = h->rpntr_h[h->all_bounds_h[q + 1]] - b;
    if (n > 0) r = ncclBroadcast(xn + sv * b, xn + sv * b, (size_t)n, dt, q, comm, st);
  }
  const ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclBroadcast");
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  return SABLE_OK;
}

sable_status sable_spmv_iterate(sable_handle* h, void* x_a, void* x_b, int32_t iters,
                                void* cuda_stream, int32_t* result_in_b) {
  if (!h || !x_a || !x_b || iters < 0) {
    set_error("sable_spmv_iterate: bad argument");
    return SABLE_E_INVALID_ARG;
  }
  void* cur = x_a;
  void* nxt = x_b;
  for (int32_t k = 0; k < iters; ++k) {
    const sable_status s = sable_spmv_allgather(h, cur, nxt, cuda_stream);
    if (s != SABLE_OK) return s;
    void* t = cur;
    cur = nxt;
    nxt = t;
  }
  if (result_in_b) *result_in_b = (cur == x_b) ? 1 : 0;
  return SABLE_OK;
}

}  // extern "C"
