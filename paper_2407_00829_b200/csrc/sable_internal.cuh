// sable_internal.cuh -- internal types of libsable.so (not part of the ABI).
//
// HBM layout of an inspected handle:
//   tval   : dense tile values of the local block rows, "row-group panels".
//            A block row a of height h owns the panel P_a = its dense tiles
//            side by side (h x W_a, W_a = sum of their widths, tiles in bc
//            order).  P_a is cut into row groups of <= 32 rows; each group's
//            nr x W_a slab is stored column-major (leading dimension nr), the
//            groups of a block row back to back.  For h <= 32 this is exactly
//            the paper's column-major tile storage.
//   stream : the executor's input, chunk after chunk; each chunk (<= one
//            stage) = header, item descriptors, bundle lane maps, x gather
//            segments, its rows' remainder pointers, its dense values, its
//            remainder columns and values -- copied with one bulk copy.
//   task   : per executor warp, a contiguous chunk range of about equal bytes.
//   tiles  : export geometry of the dense tiles (TileDesc).
//   rem_*  : the CSR remainder of the local rows (int32 row pointers).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "sable.h"

namespace sable {

constexpr int kGroupRows = 32;  // rows per row group (= warp width)
constexpr int kWarps = 4;       // warps per executor CTA
constexpr int kMaxStages = 8;   // stage ring depth cap (barrier arrays in the 256-B header)

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

// Item flags.
enum : uint8_t {
  IF_FIRST = 1,  // first piece of its row group
  IF_LAST = 2,   // last piece of its row group (write y after it)
  IF_XG = 4,     // the group's pieces are in several warp tasks (global combine)
};

// Where a chunk's stream lives (16 B).
struct ChunkRef {
  int64_t off;    // byte offset in the stream buffer (128-aligned)
  int32_t bytes;  // stream bytes (multiple of 16; 0 = no chunk)
  int32_t pad_;
};

// The executor's HBM input is one byte stream, chunk after chunk; a chunk is
// copied into a warp's stage with ONE bulk copy and describes itself:
//   [ChunkHdr | items | lane maps | x gathers | rem_ptr | values | rem cols | rem vals]
// every region 16-byte aligned, offsets relative to the chunk start.
struct ChunkHdr {
  ChunkRef next;   // the chunk nstage ahead in the same warp task (bytes 0: none)
  uint16_t o_item, o_lane, o_gath, o_rptr, o_val, o_ridx, o_rval;
  uint16_t ni;     // items
  uint16_t nb;     // bundles (32 lane maps each)
  uint16_t ng;     // x runs (XRun, o_gath)
  uint16_t ndx;    // unused (0)
  uint16_t pad16_;
  int32_t r0;      // local row whose pointer is rem_ptr element 0 of the chunk
  int32_t e0;      // first remainder entry (rem_ptr values are relative to it after -e0)
  int32_t nent;    // remainder entries
  int32_t i0;      // global index of the chunk's first item
  int32_t pad_[2];
};
static_assert(sizeof(ChunkHdr) == 64, "ChunkHdr is 64 B");

// One work item in a chunk (16 B): a whole row group (nr <= 32 rows of one
// block row: its dense slab, column-major with leading dimension nr, and its
// remainder entries), or a piece of a group larger than a stage.
struct SItem {
  uint16_t v;      // element offset of the slab in the chunk's value region
  uint16_t e;      // element offset of the entries in the chunk's entry regions
  uint16_t ne;     // remainder entries
  uint16_t ncol;   // dense columns
  int32_t row0;    // first local row of the group
  uint16_t xb;     // index of the item's first x run in the chunk's run array
  uint8_t nr;      // rows (1..32)
  uint8_t flags;   // IF_*
};
static_assert(sizeof(SItem) == 16, "SItem is 16 B");

// A bundle maps the 32 lanes of a warp onto the rows of several consecutive
// items: lane = base_i + ph * nr_i + r works on row r of item i, columns and
// entries ph, ph + Q_i, ... (Q_i = 2^lq phases, chosen by the planner to even
// out the lanes' work).  Packed lane map (4 B):
//   item (8 b) | row (5 b) << 8 | ph (5 b) << 13 | lq (3 b) << 18 | valid << 21
constexpr uint32_t kLaneValid = 1u << 21;

// One run of an item's columns over consecutive global columns: item columns
// c in [cbeg, cend) read x[off + c].  An item's runs are consecutive in the
// chunk's run array and cover its columns in order.
struct XRun {
  int32_t off;
  uint16_t cbeg, cend;
};
static_assert(sizeof(XRun) == 8, "XRun is 8 B");

// Cross-task combine data of an IF_XG item (side table by global item index).
struct XgInfo {
  int64_t slot;     // scratch base (npieces * 32 partials)
  int32_t g;        // arrival counter index
  int32_t p;        // piece index
  int32_t npieces;  // pieces of the group
  int32_t pad_;
};
static_assert(sizeof(XgInfo) == 24, "XgInfo is 24 B");

// Executor shape (runtime; the planner sizes items, chunks and tasks for it).
struct ExecCfg {
  int32_t item_bytes;   // cap on one item's streamed bytes
  int32_t stage_bytes;  // bytes of one stage (per warp), multiple of 128, <= 65536
  int32_t nstage;       // stages in each warp's ring (2..4)
  int32_t xbuf;         // x elements gathered per chunk (dense columns + remainder entries)
  int32_t ctas_per_sm;  // CTAs (kWarps warps each) per SM
  int32_t n_tasks;      // warp tasks = grid * kWarps
  int32_t mode;         // diagnostics: 0 = full; 1 = dense streams only; 2 = remainder only; 3 = dense only
  int32_t arch;         // 0: a private stage ring per warp; 1: a shared ring per CTA
  int32_t rem_grid;     // remainder executor blocks (0: one warp per packet)
  int32_t xpf;          // arch 1 producer: 1 = prefetch each landed chunk's x lines into L1
  int32_t ustaged;      // arch 2: 1 = the staged unit executor (bulk copies), 0 = direct loads
};

constexpr int kCons = 8;  // arch 1: consumer warps per CTA (+ one producer warp)

// Resident arch 1 CTAs per SM the registers allow (288 threads: 56 regs
// for fp32 -> 4, 72 for fp64 -> 3; measured r01: a 4th fp64 CTA that does not
// fit only adds a tail wave).
constexpr __host__ __device__ int cta_regs_occupancy(size_t sv) { return sv == 8 ? 3 : 4; }

// Shared memory of one arch 1 CTA: barriers (256 B) and the stages.
inline __host__ __device__ uint32_t cta_smem_bytes(const ExecCfg& c, int sv) {
  uint32_t b = 256 + (uint32_t)(c.nstage * c.stage_bytes);
  (void)sv;
  return b;
}

// Shared memory of one warp: mbarriers (256 B) and the stages.
inline __host__ __device__ uint32_t warp_smem_bytes(int nstage, int stage_bytes, int xbuf, int sv) {
  (void)xbuf;
  (void)sv;
  return 256 + (uint32_t)(nstage * stage_bytes);
}

// Device-side view used by the executor kernel.
template <typename T>
struct Plan {
  const unsigned char* stream;
  const ChunkRef* cref;   // per chunk (the prologue of each task)
  const int32_t* task;    // n_tasks + 1 chunk boundaries
  const XgInfo* xgi;
  T* scratch;
  int32_t* counters;
  int32_t n_tasks;
  int32_t nstage, stage_bytes, xbuf;
  int32_t xpf;
  int32_t mode;
};

// ---- CSR remainder executor (rem.cu)

constexpr int kPieceLen = 512;   // remainder rows longer than this are cut into warp pieces (<= kPacketEntries)
constexpr int kPacketEntries = 512;  // entries per row-range packet (whole rows)
constexpr int kPacketRows = 256;     // rows per row-range packet

// One warp's work in the remainder executor (32 B): a range of whole rows
// [r0, r1) and their entries [e0, e1), or one piece of a long row.
struct RemPacket {
  int32_t r0, r1;    // rows (piece: r0 = its row, r1 = -1 - piece index)
  int32_t e0, e1;    // entries
  int32_t npieces;   // piece: pieces of its row
  int32_t slot;      // piece: scratch base of its row's partials
  int32_t counter;   // piece: arrival counter of its row
  int32_t pad_;
};
static_assert(sizeof(RemPacket) == 32, "RemPacket is 32 B");

template <typename T>
struct RemPlan {
  const RemPacket* packets;
  const int32_t* ptr;  // local CSR row pointers
  const int32_t* idx;
  const T* val;
  T* scratch;
  int32_t* counters;
  int64_t n_packets;
};

struct RemHost {
  RemPacket* packets = nullptr;
  void* scratch = nullptr;
  int32_t* counters = nullptr;
  int64_t n_packets = 0, n_pieces = 0, n_long = 0;
};

// ---- the unit executor (unit.cu, plan.cu)
//
// Dense values of the local block rows as ROW-MAJOR panels `pv`: block row a
// (h rows, panel width W = the sum of its dense tiles' widths, tiles in bc
// order) owns rows of Wp = W rounded up to one 16-byte vector (zero padded),
// row r of the panel at pv[base_a + r * Wp].  A UNIT is one warp's work: a
// range of <= 32 consecutive rows of one block row with the block row's whole
// panel (or rows without tiles) and the remainder entries [e0, e1) of those
// rows.  A unit whose rows are complete writes y once; the pieces of a row
// range split over several units (rows with very long remainders) meet in
// scratch, summed in piece order by the last to arrive.

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

// x map of a panel, one int32 per 16-byte column vector q (panel columns
// vN .. vN + N - 1, N = 16 / sizeof(T)): c >= 0 -- the vector's columns read
// x[c], x[c + 1], ... (clamped to ncols - 1: columns past the panel width
// hold zero values); c < 0 -- the vector straddles a run boundary and its N
// global columns are xside[~c] (int32 each, N per entry, padded to 16 B).

struct XgU {         // combine group of split units (16 B)
  int64_t slot;      // scratch base (npieces * 32 partials)
  int32_t counter;   // arrival counter
  int32_t npieces;
};

#ifndef SABLE_UNIT_WARPS
#define SABLE_UNIT_WARPS 1  // A/B builds: warps per unit-executor CTA (1: measured r02)
#endif
constexpr int kUnitWarps = SABLE_UNIT_WARPS;
constexpr int kUnitStage = 4096;     // bytes of one stage of the staged executor
constexpr int kUnitBytes = 32768;    // default cap on one unit's data (direct executor)

template <typename T>
struct UPlan {
  const Unit* units;
  const int32_t* batch;   // n_batches + 1 unit boundaries (one batch per warp)
  const int32_t* xq;      // x maps of the panels
  const int4* xside;      // columns of straddling vectors
  const T* pv;
  const int32_t* rptr;    // local remainder row pointers
  const int32_t* ridx;
  const T* rval;
  const XgU* xg;
  T* scratch;
  int32_t* counters;
  int64_t n_batches;
  int32_t nm1;            // ncols - 1
  int32_t pf;             // 1: bulk L2 prefetch of the next unit's data
  uint32_t stage;         // bytes of one stage (a unit's data)
};

// Internal position of element (r, c) of a tile whose first panel column is
// cs, in a block row of height h, panel width W and panel base vbase.
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

  // executor data (device)
  void* tval = nullptr;
  int64_t tile_elems = 0;
  sable::TileDesc* tiles = nullptr;
  int64_t n_dense = 0;
  sable::XTile* xt = nullptr;        // per tile (plan time only, freed after)
  int64_t n_runs = 0;
  unsigned char* stream = nullptr;   // executor byte stream (chunk after chunk)
  int64_t stream_bytes = 0;
  sable::ChunkRef* cref = nullptr;   // per chunk
  sable::XgInfo* xgi = nullptr;      // per item
  int32_t* task = nullptr;           // warp task chunk boundaries (n_tasks + 1)
  int64_t n_groups = 0, n_items = 0, n_chunks = 0, n_bundles = 0, n_bundle_lanes = 0;
  sable::RemHost rp;                 // remainder executor plan
  sable::ExecCfg cfg{};
  int32_t* rem_ptr = nullptr;
  int32_t* rem_idx = nullptr;
  void* rem_val = nullptr;
  int64_t rem_nnz = 0;
  void* scratch = nullptr;
  int32_t* counters = nullptr;
  int64_t scratch_elems = 0;

  // unit executor (arch 2)
  void* pv = nullptr;                // row-major panels
  int64_t pv_elems = 0;
  sable::Unit* units = nullptr;
  int64_t n_units = 0;
  int32_t* ubatch = nullptr;         // n_ubatch + 1
  int64_t n_ubatch = 0;
  int32_t* xq = nullptr;
  int64_t n_xq = 0;
  int4* xside = nullptr;
  int64_t n_xside = 0;
  sable::XgU* uxg = nullptr;
  int64_t n_uxg = 0;
  void* uscratch = nullptr;
  int32_t* ucounters = nullptr;
  int32_t ustage = 0;                // bytes of a unit's stage (plan.cu)

  // export data (device): local cells and tile geometry
  int32_t* cell_br = nullptr;
  int32_t* cell_bc = nullptr;
  int64_t* cell_cnt = nullptr;
  uint8_t* cell_dense = nullptr;
  int64_t n_cells = 0, cell_base = 0;
  int64_t* tile_canon_off = nullptr;  // n_dense + 1
  int32_t* tile_br = nullptr;         // block row of each tile
  int64_t* br_vbase = nullptr;        // per local block row: panel base in tval
  int32_t* br_W = nullptr;            // per local block row: panel width

  // shard bounds (block rows) of every rank, for the all-gather
  int32_t* all_bounds_h = nullptr;  // world + 1 (host)
  int32_t* rpntr_h = nullptr;       // nbr + 1 (host copy)

  // end-to-end staging
  void* x_dev = nullptr;
  void* y_dev = nullptr;

  // multi-vector products (spmm.cu): k-wide scratch, allocated on first use
  void* mm_scratch = nullptr;
  void* mm_rscratch = nullptr;

  // NCCL
  void* comm = nullptr;

  // info
  int64_t nnz = 0;
  int64_t n_dense_global = 0;
  int64_t bytes_alg = 0;
  double inspect_ms = 0.0;
};
