// comm.cu -- the multi-GPU exchange step (north_star s7:
// "each GPU holds the full x, and the y slices are all-gathered with NCCL
// over NVLink for iterated SpMV").
//
// One step x_next = A x on a row-sharded matrix: the local y rows are written
// straight into x_next[row_begin, row_end), and every rank's rows are
// all-gathered into x_next with in-place ncclBroadcasts (an all-gatherv).
// The step is pipelined: the shard's units are cut into kSlices exchange
// slices (plan.cu: whole row ranges, about equal bytes); slice s's rows are
// broadcast on the handle's exchange stream as soon as its launch ends,
// while slice s + 1 computes, so the NVLink transfer overlaps the SpMV
// (serialized vs overlapped bound).  Every rank's slice row
// bounds are all-gathered once at sable_comm_init.
//
// Fused exchange epilogue.  Once the two ping-pong x
// buffers are registered (sable_comm_fuse: their CUDA IPC handles are
// all-gathered and every peer's buffers mapped over NVLink;
// sable_comm_set_peers: the caller supplies the peer mappings), a step is ONE
// unit-kernel launch whose epilogue stores each finished y row into its own
// x_next and into the same row of every peer's x_next (st.global through the
// peer mapping), so the transfer rides along with the SpMV row by row and no
// broadcast follows.  The step ends with a barrier (a one-word ncclAllReduce
// on the caller's stream): after it every rank's rows have landed in this
// rank's x_next, and every rank has finished reading the buffer the next
// step overwrites.
//
// sable_spmv_iterate runs `iters` steps ping-ponging two x buffers as ONE
// CUDA graph (captured once per (x_a, x_b, iters), relaunched afterwards; the
// NCCL calls are captured with the kernels) on an internal stream joined to
// the caller's stream by events.  Asynchronous NCCL errors are polled with
// ncclCommGetAsyncError before every step / iterate call and by
// sable_comm_check; a failed communicator is aborted and SABLE_E_NCCL is
// returned.
#include <nccl.h>

#include <cstring>
#include <vector>

#include "sable_internal.cuh"

namespace sable {

cudaError_t run_spmv(const sable_handle* h, const void* x, void* y, cudaStream_t st);
cudaError_t run_spmv_slice(const sable_handle* h, const void* x, void* y, int s,
                           cudaStream_t st);
cudaError_t run_spmv_fused(const sable_handle* h, const void* x, void* y, void* const* peers,
                           int npeer, cudaStream_t st);

namespace {

sable_status nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return SABLE_E_NCCL;
}

sable_status cuda_fail(cudaError_t e, const char* what) {
  set_error(cuda_msg(e, what));
  return e == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA;
}

cudaEvent_t* events(sable_handle* h) { return static_cast<cudaEvent_t*>(h->comm_events); }

void drop_graph(sable_handle* h) {
  if (h->graph_exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(h->graph_exec));
  h->graph_exec = nullptr;
  h->graph_key[0] = h->graph_key[1] = nullptr;
  h->graph_iters = -1;
}

// Poll the communicator for an asynchronous error (non-blocking).
sable_status check_async(sable_handle* h) {
  if (!h->comm) return SABLE_OK;
  ncclComm_t comm = static_cast<ncclComm_t>(h->comm);
  ncclResult_t a = ncclSuccess;
  const ncclResult_t r = ncclCommGetAsyncError(comm, &a);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
  if (a != ncclSuccess && a != ncclInProgress) {
    ncclCommAbort(comm);
    h->comm = nullptr;
    drop_graph(h);
    return nccl_fail(a, "NCCL communicator failed (aborted)");
  }
  return SABLE_OK;
}

// 0 / 1: x_next is the registered fused buffer a / b; -1: not fused.
int fused_buffer(const sable_handle* h, const void* xn) {
  if (h->fuse_n < 0) return -1;
  if (xn == h->fuse_buf[0]) return 0;
  if (xn == h->fuse_buf[1]) return 1;
  return -1;
}

void drop_fuse(sable_handle* h) {
  for (void* b : h->fuse_ipc) cudaIpcCloseMemHandle(b);
  h->fuse_ipc.clear();
  h->fuse_n = -1;
  h->fuse_buf[0] = h->fuse_buf[1] = nullptr;
  if (h->fuse_flag) cudaFree(h->fuse_flag);
  h->fuse_flag = nullptr;
}

// Enqueue one exchange step on st (capturable): slices compute on st and
// their rows are broadcast on the exchange stream, which is forked from st
// and joined back at the end.
sable_status enqueue_step(sable_handle* h, const void* x, void* xn, cudaStream_t st) {
  const size_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  char* xb = static_cast<char*>(xn);
  const int fb = fused_buffer(h, xn);
  if (fb >= 0) {
    // fused epilogue: the local rows into x_next and into every peer's
    // x_next at the same global rows, then the step barrier
    void* peers[kMaxPeers];
    for (int q = 0; q < h->fuse_n; ++q)
      peers[q] = static_cast<char*>(h->fuse_peer[fb][q]) + sv * h->row_begin;
    const cudaError_t e = run_spmv_fused(h, x, xb + sv * h->row_begin, peers, h->fuse_n, st);
    if (e) return cuda_fail(e, "fused spmv launch");
    if (h->comm) {
      ncclComm_t comm = static_cast<ncclComm_t>(h->comm);
      const ncclResult_t r = ncclAllReduce(h->fuse_flag, h->fuse_flag, 1, ncclInt32, ncclMax, comm, st);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(step barrier)");
    }
    return SABLE_OK;
  }
  if (h->world == 1) {
    // one launch; SABLE_SLICED=1 runs the slice launches of the world > 1
    // pipeline back to back instead (tests: the slices tile the rows)
    cudaError_t e = cudaSuccess;
    if (h->cfg.sliced)
      for (int s = 0; s < kSlices && !e; ++s) e = run_spmv_slice(h, x, xb + sv * h->row_begin, s, st);
    else
      e = run_spmv(h, x, xb + sv * h->row_begin, st);
    return e ? cuda_fail(e, "spmv launch") : SABLE_OK;
  }
  cudaStream_t cs = static_cast<cudaStream_t>(h->comm_stream);
  cudaEvent_t* ev = events(h);
  const ncclDataType_t dt = h->dtype == SABLE_F64 ? ncclFloat64 : ncclFloat32;
  ncclComm_t comm = static_cast<ncclComm_t>(h->comm);
  const int S = kSlices;
  for (int s = 0; s < S; ++s) {
    cudaError_t e = run_spmv_slice(h, x, xb + sv * h->row_begin, s, st);
    if (!e) e = cudaEventRecord(ev[s], st);
    if (!e) e = cudaStreamWaitEvent(cs, ev[s], 0);
    if (e) return cuda_fail(e, "exchange step");
    ncclResult_t r = ncclGroupStart();
    for (int32_t q = 0; q < h->world && r == ncclSuccess; ++q) {
      const int64_t r0 = h->all_slice_rows[(size_t)q * (S + 1) + s];
      const int64_t r1 = h->all_slice_rows[(size_t)q * (S + 1) + s + 1];
      if (r1 > r0) r = ncclBroadcast(xb + sv * r0, xb + sv * r0, (size_t)(r1 - r0), dt, q, comm, cs);
    }
    const ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclBroadcast");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  }
  cudaError_t e = cudaEventRecord(ev[S], cs);
  if (!e) e = cudaStreamWaitEvent(st, ev[S], 0);
  return e ? cuda_fail(e, "exchange join") : SABLE_OK;
}

sable_status step_args(sable_handle* h, const void* a, const void* b, const char* who) {
  if (!h || !a || !b) {
    set_error(std::string(who) + ": NULL argument");
    return SABLE_E_INVALID_ARG;
  }
  if (a == b) {
    set_error(std::string(who) + ": x and x_next must not alias");
    return SABLE_E_INVALID_ARG;
  }
  if (h->nrows != h->ncols) {
    set_error(std::string(who) + ": the matrix must be square");
    return SABLE_E_DIM;
  }
  if (h->world > 1 && !h->comm && fused_buffer(h, b) < 0) {
    set_error(std::string(who) + ": call sable_comm_init first");
    return SABLE_E_INVALID_ARG;
  }
  return SABLE_OK;
}

}  // namespace

sable_status comm_destroy(sable_handle* h) {
  if (!h) return SABLE_OK;
  drop_graph(h);
  drop_fuse(h);
  if (h->comm_events) {
    for (int s = 0; s <= kSlices; ++s) cudaEventDestroy(events(h)[s]);
    delete[] events(h);
    h->comm_events = nullptr;
  }
  if (h->comm_stream) cudaStreamDestroy(static_cast<cudaStream_t>(h->comm_stream));
  h->comm_stream = nullptr;
  if (h->comm) ncclCommDestroy(static_cast<ncclComm_t>(h->comm));
  h->comm = nullptr;
  return SABLE_OK;
}

// Streams and events of the exchange (created on first use).
sable_status comm_streams(sable_handle* h) {
  if (h->comm_stream) return SABLE_OK;
  cudaStream_t cs = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e) return cuda_fail(e, "exchange stream");
  cudaEvent_t* ev = new cudaEvent_t[kSlices + 1];
  for (int s = 0; s <= kSlices && !e; ++s) e = cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming);
  h->comm_stream = cs;
  h->comm_events = ev;
  return e ? cuda_fail(e, "exchange events") : SABLE_OK;
}

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
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_comm_init: cudaSetDevice");
  comm_destroy(h);
  sable_status s = comm_streams(h);
  if (s) return s;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = ncclCommInitRank(&comm, h->world, id, h->rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  h->comm = comm;
  // every rank's exchange slices (global row bounds), all-gathered once
  const int S1 = kSlices + 1;
  std::vector<int64_t> mine(S1);
  for (int i = 0; i < S1; ++i) mine[i] = h->row_begin + h->slice_row[i];
  h->all_slice_rows.assign((size_t)h->world * S1, 0);
  int64_t* d = nullptr;
  cudaStream_t cs = static_cast<cudaStream_t>(h->comm_stream);
  cudaError_t e = cudaMalloc(&d, sizeof(int64_t) * (size_t)h->world * S1);
  if (!e) e = cudaMemcpyAsync(d + (size_t)h->rank * S1, mine.data(), sizeof(int64_t) * S1,
                              cudaMemcpyHostToDevice, cs);
  ncclResult_t r2 = ncclSuccess;
  if (!e) r2 = ncclAllGather(d + (size_t)h->rank * S1, d, (size_t)S1, ncclInt64, comm, cs);
  if (!e && r2 == ncclSuccess)
    e = cudaMemcpyAsync(h->all_slice_rows.data(), d, sizeof(int64_t) * (size_t)h->world * S1,
                        cudaMemcpyDeviceToHost, cs);
  if (!e) e = cudaStreamSynchronize(cs);
  if (d) cudaFree(d);
  if (r2 != ncclSuccess) return nccl_fail(r2, "ncclAllGather(slice rows)");
  if (e) return cuda_fail(e, "sable_comm_init");
  // the slices must tile each rank's rows of the all-gather layout
  for (int32_t q = 0; q < h->world; ++q) {
    const int64_t* a = h->all_slice_rows.data() + (size_t)q * S1;
    const int64_t lo = h->rpntr_h[h->all_bounds_h[q]], hi = h->rpntr_h[h->all_bounds_h[q + 1]];
    bool ok = a[0] == lo && a[kSlices] == hi;
    for (int i = 0; i < kSlices && ok; ++i) ok = a[i] <= a[i + 1];
    if (!ok) {
      set_error("sable_comm_init: ranks disagree on the row layout (different matrices?)");
      return SABLE_E_INVALID_ARG;
    }
  }
  return SABLE_OK;
}

sable_status sable_comm_check(sable_handle* h) {
  if (!h) {
    set_error("sable_comm_check: NULL handle");
    return SABLE_E_INVALID_ARG;
  }
  return check_async(h);
}

sable_status sable_spmv_allgather(sable_handle* h, const void* x_full, void* x_next_full,
                                  void* cuda_stream) {
  sable_status s = step_args(h, x_full, x_next_full, "sable_spmv_allgather");
  if (s) return s;
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_spmv_allgather: cudaSetDevice");
  if ((s = check_async(h))) return s;
  return enqueue_step(h, x_full, x_next_full, static_cast<cudaStream_t>(cuda_stream));
}

sable_status sable_spmv_iterate(sable_handle* h, void* x_a, void* x_b, int32_t iters,
                                void* cuda_stream, int32_t* result_in_b) {
  if (iters < 0) {
    set_error("sable_spmv_iterate: iters < 0");
    return SABLE_E_INVALID_ARG;
  }
  sable_status s = step_args(h, x_a, x_b, "sable_spmv_iterate");
  if (s) return s;
  if (result_in_b) *result_in_b = iters % 2;
  if (iters == 0) return SABLE_OK;
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_spmv_iterate: cudaSetDevice");
  if ((s = check_async(h))) return s;
  if ((s = comm_streams(h))) return s;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // the graph runs on an internal stream (capture needs a non-legacy
  // stream), forked from and joined back to the caller's stream
  static thread_local cudaStream_t is = nullptr;
  static thread_local int is_dev = -1;
  cudaError_t e = cudaSuccess;
  if (!is || is_dev != h->device) {
    e = cudaStreamCreateWithFlags(&is, cudaStreamNonBlocking);
    if (e) return cuda_fail(e, "iterate stream");
    is_dev = h->device;
  }
  cudaEvent_t* ev = events(h);
  const bool hit = h->graph_exec && h->graph_key[0] == x_a && h->graph_key[1] == x_b &&
                   h->graph_iters == iters;
  if (!hit) {
    drop_graph(h);
    cudaGraph_t graph = nullptr;
    e = cudaStreamBeginCapture(is, cudaStreamCaptureModeThreadLocal);
    if (e) return cuda_fail(e, "iterate capture");
    void* cur = x_a;
    void* nxt = x_b;
    sable_status ss = SABLE_OK;
    for (int32_t k = 0; k < iters && !ss; ++k) {
      ss = enqueue_step(h, cur, nxt, is);
      void* t = cur;
      cur = nxt;
      nxt = t;
    }
    e = cudaStreamEndCapture(is, &graph);
    if (ss) {
      if (graph) cudaGraphDestroy(graph);
      return ss;
    }
    if (e) return cuda_fail(e, "iterate capture end");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e) return cuda_fail(e, "iterate graph instantiate");
    h->graph_exec = exec;
    h->graph_key[0] = x_a;
    h->graph_key[1] = x_b;
    h->graph_iters = iters;
  }
  e = cudaEventRecord(ev[0], st);
  if (!e) e = cudaStreamWaitEvent(is, ev[0], 0);
  if (!e) e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(h->graph_exec), is);
  if (!e) e = cudaEventRecord(ev[kSlices], is);
  if (!e) e = cudaStreamWaitEvent(st, ev[kSlices], 0);
  return e ? cuda_fail(e, "iterate launch") : SABLE_OK;
}

namespace {

// Register the fused buffers and their peer mappings on the handle.
sable_status set_peers(sable_handle* h, void* x_a, void* x_b, void* const* pa, void* const* pb,
                       int32_t n) {
  drop_graph(h);
  h->fuse_buf[0] = x_a;
  h->fuse_buf[1] = x_b;
  for (int q = 0; q < n; ++q) {
    h->fuse_peer[0][q] = pa[q];
    h->fuse_peer[1][q] = pb[q];
  }
  h->fuse_n = n;
  if (!h->fuse_flag) {
    cudaError_t e = cudaMalloc(&h->fuse_flag, sizeof(int32_t));
    if (!e) e = cudaMemset(h->fuse_flag, 0, sizeof(int32_t));
    if (e) return cuda_fail(e, "fused exchange: barrier word");
  }
  return SABLE_OK;
}

struct FuseMsg {  // what each rank publishes: IPC handles of the allocations
  cudaIpcMemHandle_t mem[2];  // holding x_a / x_b, and the buffers' offsets
  int64_t off[2];             // inside them
};

}  // namespace

sable_status sable_comm_set_peers(sable_handle* h, void* x_a, void* x_b,
                                  void* const* peers_a, void* const* peers_b, int32_t npeers) {
  if (!h || !x_a || !x_b || x_a == x_b || npeers < 0 || npeers > kMaxPeers ||
      (npeers > 0 && (!peers_a || !peers_b))) {
    set_error("sable_comm_set_peers: bad arguments (two distinct buffers, 0..7 peers)");
    return SABLE_E_INVALID_ARG;
  }
  for (int q = 0; q < npeers; ++q)
    if (!peers_a[q] || !peers_b[q] || peers_a[q] == x_a || peers_b[q] == x_b) {
      set_error("sable_comm_set_peers: NULL peer or a peer aliasing the local buffer");
      return SABLE_E_INVALID_ARG;
    }
  if (h->nrows != h->ncols) {
    set_error("sable_comm_set_peers: the matrix must be square");
    return SABLE_E_DIM;
  }
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_comm_set_peers: cudaSetDevice");
  drop_fuse(h);
  return set_peers(h, x_a, x_b, peers_a, peers_b, npeers);
}

sable_status sable_comm_unfuse(sable_handle* h) {
  if (!h) {
    set_error("sable_comm_unfuse: NULL handle");
    return SABLE_E_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_comm_unfuse: cudaSetDevice");
  drop_graph(h);
  drop_fuse(h);
  return SABLE_OK;
}

sable_status sable_comm_fuse(sable_handle* h, void* x_a, void* x_b) {
  if (!h || !x_a || !x_b || x_a == x_b) {
    set_error("sable_comm_fuse: two distinct device buffers required");
    return SABLE_E_INVALID_ARG;
  }
  if (h->nrows != h->ncols) {
    set_error("sable_comm_fuse: the matrix must be square");
    return SABLE_E_DIM;
  }
  if (h->world > 1 && !h->comm) {
    set_error("sable_comm_fuse: call sable_comm_init first");
    return SABLE_E_INVALID_ARG;
  }
  if (h->world - 1 > kMaxPeers) {
    set_error("sable_comm_fuse: at most 8 ranks");
    return SABLE_E_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  if (g.err) return cuda_fail(g.err, "sable_comm_fuse: cudaSetDevice");
  sable_status s = check_async(h);
  if (s) return s;
  drop_graph(h);
  drop_fuse(h);
  if (h->world == 1) return set_peers(h, x_a, x_b, nullptr, nullptr, 0);
  // this rank's message: the IPC handle of each buffer's allocation (the
  // driver's address range query gives its base) and the buffer's offset
  typedef int (*range_fn)(unsigned long long*, size_t*, unsigned long long);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &qr);
  if (e || !fp || qr != cudaDriverEntryPointSuccess)
    return cuda_fail(e ? e : cudaErrorUnknown, "sable_comm_fuse: cuMemGetAddressRange entry point");
  FuseMsg mine;
  void* bufs[2] = {x_a, x_b};
  for (int i = 0; i < 2; ++i) {
    unsigned long long base = 0;
    size_t size = 0;
    if (reinterpret_cast<range_fn>(fp)(&base, &size, (unsigned long long)(uintptr_t)bufs[i]) != 0) {
      set_error("sable_comm_fuse: x buffer is not a device allocation");
      return SABLE_E_INVALID_ARG;
    }
    mine.off[i] = (int64_t)((unsigned long long)(uintptr_t)bufs[i] - base);
    e = cudaIpcGetMemHandle(&mine.mem[i], reinterpret_cast<void*>((uintptr_t)base));
    if (e) return cuda_fail(e, "sable_comm_fuse: cudaIpcGetMemHandle (cudaMalloc memory required)");
  }
  // all-gather the messages
  const int W = h->world;
  std::vector<FuseMsg> all((size_t)W);
  FuseMsg* d = nullptr;
  ncclComm_t comm = static_cast<ncclComm_t>(h->comm);
  cudaStream_t cs = static_cast<cudaStream_t>(h->comm_stream);
  e = cudaMalloc(&d, sizeof(FuseMsg) * (size_t)W);
  if (!e) e = cudaMemcpyAsync(d + h->rank, &mine, sizeof(FuseMsg), cudaMemcpyHostToDevice, cs);
  ncclResult_t r = ncclSuccess;
  if (!e) r = ncclAllGather(d + h->rank, d, sizeof(FuseMsg), ncclInt8, comm, cs);
  if (!e && r == ncclSuccess)
    e = cudaMemcpyAsync(all.data(), d, sizeof(FuseMsg) * (size_t)W, cudaMemcpyDeviceToHost, cs);
  if (!e) e = cudaStreamSynchronize(cs);
  if (d) cudaFree(d);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather(IPC handles)");
  if (e) return cuda_fail(e, "sable_comm_fuse: handle exchange");
  // map every peer's two allocations (an allocation shared by both buffers
  // is opened once)
  void* pa[kMaxPeers];
  void* pb[kMaxPeers];
  int n = 0;
  for (int q = 0; q < W; ++q) {
    if (q == h->rank) continue;
    void* base[2] = {nullptr, nullptr};
    for (int i = 0; i < 2; ++i) {
      if (i == 1 && memcmp(&all[q].mem[0], &all[q].mem[1], sizeof(cudaIpcMemHandle_t)) == 0) {
        base[1] = base[0];
        continue;
      }
      e = cudaIpcOpenMemHandle(&base[i], all[q].mem[i], cudaIpcMemLazyEnablePeerAccess);
      if (e) {
        drop_fuse(h);
        return cuda_fail(e, "sable_comm_fuse: cudaIpcOpenMemHandle (one process per GPU, "
                            "peer access over NVLink required)");
      }
      h->fuse_ipc.push_back(base[i]);
    }
    pa[n] = static_cast<char*>(base[0]) + all[q].off[0];
    pb[n] = static_cast<char*>(base[1]) + all[q].off[1];
    ++n;
  }
  return set_peers(h, x_a, x_b, pa, pb, n);
}

// The all-gather layout on the host (no GPU needed): the row bounds of every
// rank's slice of y for a matrix with per-block-row weights and grid rpntr,
// row_bounds[q] = rpntr[shard bound q] (world + 1 entries).
sable_status sable_exchange_rows(const int64_t* weights, int32_t nbrows, const int32_t* rpntr,
                                 int32_t world, int64_t* row_bounds) {
  if (!rpntr || !row_bounds || world < 1) {
    set_error("sable_exchange_rows: bad arguments");
    return SABLE_E_INVALID_ARG;
  }
  std::vector<int32_t> b((size_t)world + 1);
  const sable_status s = sable_shard_bounds(weights, nbrows, world, b.data());
  if (s) return s;
  for (int32_t q = 0; q <= world; ++q) row_bounds[q] = rpntr[b[q]];
  return SABLE_OK;
}

}  // extern "C"
