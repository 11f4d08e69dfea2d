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
//   tiles  : one TileDesc per dense tile (global column c0, width w, first
//            panel column cs).
//   groups : one Group per row group; items: one Item per work piece.
//   rem_*  : the CSR remainder of the local rows (int32 row pointers).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "sable.h"

namespace sable {

constexpr int kGroupRows = 32;  // rows per row group (= warp width)
constexpr int kXCap = 512;      // max dense panel columns per work item (xs smem)
constexpr int kWin = 128;       // remainder entries per smem window
constexpr int kWarps = 8;       // warps per executor CTA

struct TileDesc {
  int32_t c0;  // first global column of the tile
  int32_t w;   // width
  int32_t cs;  // first column inside the block-row panel
};

struct Group {
  int64_t voff;     // first value of this group's nr x W slab in tval
  int32_t row0;     // first local row
  int32_t nr;       // rows in the group (1..32)
  int32_t t0, t1;   // dense tiles of the block row
  int32_t W;        // panel width of the block row
  int32_t npieces;  // work items of this group (>= 1)
  int64_t slot;     // scratch base (npieces * 32 partials) when npieces > 1
};

struct Item {
  int64_t eb, ee;  // remainder entries [eb, ee) of the group's rows
  int32_t g;       // group
  int32_t p;       // piece index inside the group
  int32_t cb, ce;  // panel columns [cb, ce)
};

// Device-side view used by the executor kernel.
template <typename T>
struct Plan {
  const Item* items;
  const Group* groups;
  const TileDesc* tiles;
  const T* tval;
  const int32_t* rem_ptr;  // local rows + 1
  const int32_t* rem_idx;
  const T* rem_val;
  T* scratch;
  int32_t* counters;
  int64_t n_items;
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
  sable::Group* groups = nullptr;
  int64_t n_groups = 0;
  sable::Item* items = nullptr;
  int64_t n_items = 0;
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
