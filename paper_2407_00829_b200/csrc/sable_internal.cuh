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
//   items  : one 32-byte Item per warp work unit (row group or piece of one),
//            in row order; xgi: cross-task combine data per item.
//   chunks : one 64-byte Chunk per stage load (consecutive items).
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
constexpr int kRE = 256;        // remainder entries per item (per-warp product buffer)
constexpr int kWarps = 4;       // warps per executor CTA

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

// One unit of a warp's stream (32 B): a whole row group, or a piece of a
// split group -- a range of panel columns inside one run, or a range of the
// group's remainder entries.  Items never span runs, so the x of item
// column c is x[xo + c].
struct Item {
  int64_t voff;   // first dense value (group slab column-major, ld nr)
  int32_t eb;     // first remainder entry (position in the local CSR)
  int32_t xo;     // x index of the item's first dense column
  int32_t row0;   // first local row of the group
  int16_t ncol;   // dense columns of the item (0 = remainder only)
  int16_t ne;     // remainder entries [eb, eb + ne), <= kRE
  uint16_t qm;    // floor(32768 / nr) + 1: lane / nr == (lane * qm) >> 15 for lane < 32
  int16_t xb;     // first element of the item's dense x in its chunk's x buffer
  uint8_t nr;     // rows (1..32)
  uint8_t q;      // column phases 32 / nr
  uint8_t flags;  // IF_*
  uint8_t pad_;
};
static_assert(sizeof(Item) == 32, "Item is 32 B");

// Cross-task combine data of an IF_XG item (side table, read only for those).
struct XgInfo {
  int64_t slot;     // scratch base (npieces * 32 partials)
  int32_t g;        // arrival counter index
  int16_t p;        // piece index
  int16_t pad_;
  int32_t npieces;  // pieces of the group
  int32_t pad2_;
};
static_assert(sizeof(XgInfo) == 24, "XgInfo is 24 B");

// Streamed arrays of a chunk, in stage order.
enum { SR_ITEM = 0, SR_RPTR, SR_VAL, SR_RIDX, SR_RVAL, SR_N };

// One stage load of a warp (64 B): consecutive items whose data are
// contiguous ranges of five arrays, copied with 1-D bulk copies (16-byte
// granular) into the warp's stage after a 64-byte slot that carries the
// descriptor of the chunk nstage ahead.  Offsets are precomputed by the
// planner, so issuing a chunk is five copy instructions.
struct Chunk {
  uint32_t src16[SR_N];  // first byte / 16 of each range in its array
  uint16_t bytes[SR_N];  // bytes copied (multiple of 16; 0 = none)
  uint16_t off[SR_N];    // stage offset of the first wanted element (dst = off & ~15)
  int64_t v0;            // dense value index of the chunk's first value
  int32_t e0;            // remainder entry of the chunk's first entry
  int32_t r0;            // local row whose pointer is rem_ptr element 0 of the stage
  int16_t ni;            // items
  int16_t ndx;           // dense x elements; the x buffer is [dense x | remainder x]
  int32_t i0;            // index of the chunk's first item
};
static_assert(sizeof(Chunk) == 64, "Chunk is 64 B");

// Executor shape (runtime; the planner sizes items, chunks and tasks for it).
struct ExecCfg {
  int32_t item_bytes;   // cap on one item's streamed bytes
  int32_t stage_bytes;  // bytes of one stage (per warp), multiple of 128
  int32_t nstage;       // stages in each warp's ring (2..4)
  int32_t xbuf;         // x elements gathered per chunk (dense columns + remainder entries)
  int32_t ctas_per_sm;  // CTAs (kWarps warps each) per SM
  int32_t n_tasks;      // warp tasks = grid * kWarps
  int32_t mode;         // diagnostics: 0 = full; 1 = stream only
};

constexpr int kMaxStages = 4;

// Shared memory of one warp: mbarriers + chunk descriptors (512 B), two x
// buffers [xbuf] (the chunk being computed, the next one being gathered),
// then the stages.
inline __host__ __device__ uint32_t warp_smem_bytes(int nstage, int stage_bytes, int xbuf, int sv) {
  return 512 + (uint32_t)((2 * xbuf * sv + 127) & ~127) + (uint32_t)(nstage * stage_bytes);
}

// Device-side view used by the executor kernel.
template <typename T>
struct Plan {
  const Chunk* chunks;
  const int32_t* task;  // n_tasks + 1 chunk boundaries
  const Item* items;
  const XgInfo* xgi;
  const T* tval;
  const int32_t* rem_ptr;  // local rows + 1
  const int32_t* rem_idx;
  const T* rem_val;
  T* scratch;
  int32_t* counters;
  int32_t n_tasks;
  int32_t nstage, stage_bytes, xbuf;
  int32_t mode;
};

// Internal position of element (r, c) of a tile whose first panel column is
// cs, in a block row of height h, panel width W and panel base vbase.
__device__ __forceinline__ int64_t panel_pos(int64_t vbase, int64_t W, int64_t h, int64_t cs,
                                             int64_t r, int64_t c) {
  const int64_t g = r / kGroupRows;
  const int64_t nr = (h - g * kGroupRows) < kGroupRows ? (h - g * kGroupRows) : kGroupRows;
  return vbase + g * kGroupRows * W + (cs + c) * nr + (r - g * kGroupRows);
}

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
  sable::Item* items = nullptr;
  sable::XgInfo* xgi = nullptr;      // per item
  sable::Chunk* chunks = nullptr;
  int32_t* task = nullptr;           // warp task chunk boundaries (n_tasks + 1)
  int64_t n_groups = 0, n_items = 0, n_chunks = 0;
  sable::ExecCfg cfg{};
  int32_t* rem_ptr = nullptr;
  int32_t* rem_idx = nullptr;
  void* rem_val = nullptr;
  int64_t rem_nnz = 0;
  void* scratch = nullptr;
  int32_t* counters = nullptr;
  int64_t scratch_elems = 0;

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

  // NCCL
  void* comm = nullptr;

  // info
  int64_t nnz = 0;
  int64_t n_dense_global = 0;
  int64_t bytes_alg = 0;
  double inspect_ms = 0.0;
};
