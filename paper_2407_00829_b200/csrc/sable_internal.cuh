// sable_internal.cuh -- internal types of libsable.so (not part of the ABI).
//
// HBM layout of an inspected handle:
//   pv     : dense tile values of the local block rows as ROW-MAJOR panels:
//            block row a (h rows, panel width W = the sum of its dense
//            tiles' widths, tiles in bc order) owns h rows of Wp = W rounded
//            up to one 16-byte vector (zero padded); row r of the panel at
//            pv[base_a + r * Wp].  For one tile this is the tile transposed
//            from the paper's column-major storage (
//            reading R8: the internal layout is free).
//   xq     : per panel, one XMap (8 B) per 16-byte column vector: the global
//            columns of its N columns (xside for vectors spanning three or
//            more runs of global columns).
//   units  : the executor's work list (plan.cu), batches of consecutive
//            units per warp.
//   rem_*  : the CSR remainder of the local rows (int32 row pointers).
//   tiles  : export geometry of the dense tiles (TileDesc).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "sable.h"

namespace sable {

constexpr int kGroupRows = 32;  // rows per row group of the inspector's staging slabs

struct TileDesc {  // export geometry of a dense tile
  int32_t c0;  // first global column of the tile
  int32_t w;   // width
  int32_t cs;  // first column inside the block-row panel
};

// x-gather map (plan time).  The local dense tiles' columns, concatenated in
// tile order, form the "flattened panel column" space; a run is a maximal
// range of it mapping to consecutive global columns (adjacent tiles of one
// rectangle merge): flattened column f in run k -> global column c0 + (f - tp).
struct XTile {
  int32_t tp;  // first flattened panel column of the tile / run
  int32_t c0;  // its global column
};

// Executor configuration (runtime; SABLE_* environment overrides are for
// tuning and tests, validated by inspect.cu's exec_config).
struct ExecCfg {
  int32_t pf;          // 1: bulk L2 prefetch of a warp batch's later units (SABLE_XPREFETCH)
  int32_t ustage;      // cap on one unit's bytes (SABLE_USTAGE; plan.cu)
  int32_t rem_rows;    // rows per remainder-only unit (SABLE_UREM_ROWS)
  int32_t batch;       // max units per warp batch (SABLE_UBATCH_UNITS)
  int32_t batch_bytes; // bytes that close a warp batch (SABLE_UBATCH_BYTES)
  int32_t sliced;      // 1: world-1 exchange steps run the slice launches (SABLE_SLICED, tests)
  int32_t lpr_mode;    // lanes per row: 0 cover the panel in one pass, 1 largest power of two <= wq (SABLE_LPR)
};

// ---- the unit executor (unit.cu, plan.cu)
//
// A UNIT is one warp's work: a range of <= 32 consecutive rows of one block
// row with the block row's whole panel (or a column chunk of one row of a
// very wide panel, or rows without tiles) and the remainder entries [e0, e1)
// of those rows.  A unit whose rows are complete writes y once; the pieces of
// a row range split over several units meet in scratch, summed in piece
// order by the last to arrive.

struct Unit {        // 32 B
  int32_t voff16;    // first value of the unit's first row, in 16-byte vectors
  int32_t row0;      // first local row
  int32_t wq;        // dense panel width in 16-byte column vectors (0: no dense part)
  int32_t xq0;       // the block row's x map: xq[xq0 + q] for column vector q
  int32_t e0, e1;    // remainder entries of rows [row0, row0 + nr) clamped to [e0, e1)
  int32_t xg;        // -1: complete rows (write y); else its combine group
  uint8_t nr;        // rows (1..32)
  uint8_t llpr;      // log2 of the lanes per row of the dense part (0..5)
  uint16_t piece;    // piece index inside the combine group
};
static_assert(sizeof(Unit) == 32, "Unit is 32 B");

// x map of a panel, one XMap per 16-byte column vector q (panel columns
// qN .. qN + N - 1, N = 16 / sizeof(T)): c >= 0 -- column i of the vector
// reads x[c + i] for i < k and x[c + i + d] for i >= k, where k = kd & 3 and
// d = kd >> 2 (k = 0, d = 0: the vector lies in one run of consecutive
// global columns; k > 0: its first k columns end one run and the rest start
// the next, d apart); columns past the panel width hold zero values and read
// any column inside the matrix; every column an entry yields is in
// [0, ncols) (plan.cu), so the executors never clamp; c < 0 -- the vector
// spans three or more runs and its N global columns are xside[~c] (int32
// each, padded to 16 B).
struct XMap {
  int32_t c;
  int32_t kd;
};
static_assert(sizeof(XMap) == 8, "XMap is 8 B");

struct XgU {         // combine group of split units (16 B)
  int64_t slot;      // scratch base (npieces * 32 partials)
  int32_t counter;   // arrival counter
  int32_t npieces;
};
static_assert(sizeof(XgU) == 16, "XgU is 16 B");

#ifndef SABLE_UNIT_WARPS
#define SABLE_UNIT_WARPS 1  // A/B builds: warps per unit-executor CTA (1: measured r02)
#endif
constexpr int kUnitWarps = SABLE_UNIT_WARPS;
constexpr int kUnitBytes = 16384;  // default cap on one unit's data (plan.cu)
constexpr int kBatchBytes = 8192;  // default bytes that close a warp batch (plan.cu)
constexpr int kUnitBatch = 4;      // default units per warp batch
constexpr int kSlices = 8;         // exchange slices of a shard (comm.cu overlap)
constexpr int kMaxPeers = 7;       // peers of the fused exchange epilogue (world <= 8)

template <typename T>
struct UPlan {
  const Unit* units;
  const int32_t* batch;   // n_batches + 1 unit boundaries (one batch per warp)
  const Unit* bhead;      // each batch's first unit descriptor
  const XMap* xq;         // x maps of the panels
  const int4* xside;      // columns of straddling vectors
  const T* pv;
  const int32_t* rptr;    // local remainder row pointers
  const int32_t* ridx;
  const T* rval;
  const XgU* xg;
  T* scratch;
  int32_t* counters;
  int64_t b0, n_batches;  // batches [b0, n_batches) of this launch
  int32_t pf;             // 1: bulk L2 prefetch of the next unit's data
  // fused exchange epilogue (comm.cu): every finished y row
  // is also stored at the same local row of npeer peer buffers (the other
  // ranks' x_next + row_begin, reached over NVLink peer mappings)
  int32_t npeer;
  T* peer[kMaxPeers];
  // array extents, read only by the bounds-checked build (SABLE_CHECKED)
  int64_t n_units, pv_vecs, n_xq, n_xside, rem_nnz, nloc, ncols, n_uxg, scratch_elems;
};

// Bounds-checked build (build.py variant "checked", -DSABLE_CHECKED): every
// index the executors follow is checked on the device and a violation traps
// (cudaErrorLaunchFailure), the pool's stand-in for compute-sanitizer.
#ifdef SABLE_CHECKED
#define SABLE_DCHECK(cond) \
  do {                     \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define SABLE_DCHECK(cond) \
  do {                     \
  } while (0)
#endif

// Host side: fill the extents of a plan from its handle.
template <typename T>
inline void plan_extents(UPlan<T>& P, const sable_handle* h, int64_t scratch_elems);

// Position of element (r, c) of a tile whose first panel column is cs, in a
// row-major panel of width W at base pb (rows padded to 16 bytes).
__host__ __device__ __forceinline__ int64_t panel_rm_pos(int64_t pb, int64_t W, int64_t vec,
                                                         int64_t cs, int64_t r, int64_t c) {
  const int64_t Wp = (W + vec - 1) / vec * vec;
  return pb + r * Wp + cs + c;
}

// Internal position of element (r, c) in the inspector's staging slabs
// (row groups of <= 32 rows, each column-major) -- packing only.
__device__ __forceinline__ int64_t panel_pos(int64_t vbase, int64_t W, int64_t h, int64_t cs,
                                             int64_t r, int64_t c) {
  const int64_t g = r / kGroupRows;
  const int64_t nr = (h - g * kGroupRows) < kGroupRows ? (h - g * kGroupRows) : kGroupRows;
  return vbase + g * kGroupRows * W + (cs + c) * nr + (r - g * kGroupRows);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
// for at least `bytes` (thread-safe).
cudaError_t set_smem_attr(const void* func, int device, size_t bytes);

// Thread-local error text for sable_last_error().
void set_error(const std::string& msg);
std::string cuda_msg(cudaError_t e, const char* what);

// Make the handle's device current for the scope of a call (restored after).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (!err && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace sable

struct sable_handle {
  int device = 0;
  int32_t dtype = SABLE_F32;
  int32_t delta = 50;
  int64_t nrows = 0, ncols = 0;
  int32_t nbr = 0, nbc = 0;
  int32_t br_begin = 0, br_end = 0;
  int64_t row_begin = 0, row_end = 0;
  int32_t rank = 0, world = 1;
  sable::ExecCfg cfg{};

  // remainder CSR of the local rows (device)
  int32_t* rem_ptr = nullptr;
  int32_t* rem_idx = nullptr;
  void* rem_val = nullptr;
  int64_t rem_nnz = 0;

  // unit executor (device)
  void* pv = nullptr;                // row-major panels
  int64_t pv_elems = 0;
  sable::Unit* units = nullptr;
  int64_t n_units = 0;
  int32_t* ubatch = nullptr;         // n_ubatch + 1
  sable::Unit* ubhead = nullptr;     // n_ubatch: each batch's first unit (plan.cu)
  int64_t n_ubatch = 0;
  sable::XMap* xq = nullptr;
  int64_t n_xq = 0;
  int4* xside = nullptr;
  int64_t n_xside = 0;
  sable::XgU* uxg = nullptr;
  int64_t n_uxg = 0;
  int64_t uscratch_slots = 0;        // combine partial slots (sum of pieces * 32)
  void* uscratch = nullptr;
  int32_t* ucounters = nullptr;
  void* mm_scratch = nullptr;        // sable_spmm: 8 partials per slot (first use)
  void* mma_scratch = nullptr;       // sable_spmm on the tensor cores: 128 partials per slot
  std::vector<int64_t> slice_batch;  // kSlices + 1 batch boundaries (host)
  std::vector<int64_t> slice_row;    // kSlices + 1 local row boundaries (host)

  // export data (device): local cells and tile geometry
  int32_t* cell_br = nullptr;
  int32_t* cell_bc = nullptr;
  int64_t* cell_cnt = nullptr;
  uint8_t* cell_dense = nullptr;
  int64_t n_cells = 0, cell_base = 0;
  int64_t n_dense = 0;
  int64_t tile_elems = 0;
  sable::TileDesc* tiles = nullptr;
  int64_t* tile_canon_off = nullptr;  // n_dense + 1
  int32_t* tile_br = nullptr;         // block row of each tile
  int64_t* br_pbase = nullptr;        // per local block row: panel base in pv
  int32_t* br_W = nullptr;            // per local block row: panel width

  // shard bounds (block rows) of every rank, for the all-gather
  int32_t* all_bounds_h = nullptr;  // world + 1 (host)
  int32_t* rpntr_h = nullptr;       // nbr + 1 (host copy)

  // end-to-end staging
  void* x_dev = nullptr;
  void* y_dev = nullptr;

  // multi-GPU exchange (comm.cu)
  void* comm = nullptr;              // ncclComm_t
  void* comm_stream = nullptr;       // cudaStream_t of the exchange (overlap)
  void* comm_events = nullptr;       // kSlices + 1 cudaEvent_t (slice done, exchange done)
  std::vector<int64_t> all_slice_rows;  // world * (kSlices + 1) global row bounds (host)
  // fused exchange epilogue: the registered ping-pong buffers, the peers'
  // mappings of the same buffers (row 0), opened IPC bases, barrier word
  void* fuse_buf[2] = {nullptr, nullptr};
  void* fuse_peer[2][sable::kMaxPeers] = {};
  int32_t fuse_n = -1;               // -1: not registered; else peers per buffer
  std::vector<void*> fuse_ipc;       // cudaIpcOpenMemHandle bases to close
  int32_t* fuse_flag = nullptr;      // device word of the step barrier (all-reduce)
  void* graph_exec = nullptr;        // cudaGraphExec_t of sable_spmv_iterate
  const void* graph_key[2] = {nullptr, nullptr};
  int32_t graph_iters = -1;

  // info
  int64_t nnz = 0;
  int64_t n_dense_global = 0;
  int64_t bytes_alg = 0;
  double inspect_ms = 0.0;
};

namespace sable {
template <typename T>
inline void plan_extents(UPlan<T>& P, const sable_handle* h, int64_t scratch_elems) {
  P.n_units = h->n_units;
  P.pv_vecs = h->pv_elems * (int64_t)sizeof(T) / 16;
  P.n_xq = h->n_xq;
  P.n_xside = h->n_xside;
  P.rem_nnz = h->rem_nnz;
  P.nloc = h->row_end - h->row_begin;
  P.ncols = h->ncols;
  P.n_uxg = h->n_uxg;
  P.scratch_elems = scratch_elems;
}
}  // namespace sable
