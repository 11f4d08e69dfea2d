/*
 * sable.h -- C-ABI of libsable.so, the B200 (sm_100a) VBR SpMV hot path of
 * SABLE (arXiv 2407.00829, "Staging Blocked Evaluation over Structured Sparse
 * Matrices").  Citations "PAPER.md:L" are lines of the paper's LaTeX source;
 * readings R1..R18 are listed in DESIGN.md ("Readings of the paper").
 *
 * The boundary (BASELINE.json north_star s3): sable_vbr_create takes the VBR
 * indirection arrays rpntr / cpntr / bpntr / bindx / indx / val (Fig. 2,
 * PAPER.md:221-228; "SABLE assumes that the sparse matrix is already stored
 * in the VBR format and takes several storage format indirection arrays as
 * input") plus the delta threshold ("delta-dense ... the
 * percentage of non-zero elements is at least delta %"), runs
 * the GPU inspector, and returns a handle; sable_spmv computes y = A x
 * with the dense tiles / CSR remainder split of VBR-C (Fig. 3,
 * PAPER.md:271-347); sable_destroy frees the handle.
 *
 * Conventions for every entry point:
 *   - plain C types and pointers only; no exceptions cross the ABI; every call
 *     returns a sable_status; the text of the last failure on the calling
 *     thread is available from sable_last_error().
 *   - "device pointer" = CUDA device memory of the current device (e.g. the
 *     data_ptr() of a torch CUDA tensor); "host pointer" = ordinary or pinned
 *     host memory.
 *   - cuda_stream is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Indices are 0-based.  Sizes are element counts unless named *_bytes.
 */
#ifndef SABLE_H_
#define SABLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SABLE_ABI_VERSION 2

typedef struct sable_handle sable_handle;

typedef enum {
  SABLE_OK = 0,
  SABLE_E_INVALID_ARG = 1, /* NULL pointer, delta > 101, bad enum, bad shard   */
  SABLE_E_FORMAT = 2,      /* a VBR / remainder invariant is broken; the last
                              error names the array and the first bad index    */
  SABLE_E_DIM = 3,         /* sizes disagree (e.g. iterate on a non-square A)  */
  SABLE_E_DUPLICATE = 4,   /* the same (i,j) non-zero in val and the remainder */
  SABLE_E_OOM = 5,         /* device or host allocation failed                 */
  SABLE_E_CUDA = 6,        /* a CUDA runtime error (text in sable_last_error)  */
  SABLE_E_NCCL = 7,        /* an NCCL error                                    */
  SABLE_E_UNSUPPORTED = 8  /* outside the supported limits (see below)         */
} sable_status;

typedef enum { SABLE_F32 = 0, SABLE_F64 = 1 } sable_dtype;
typedef enum { SABLE_MEM_HOST = 0, SABLE_MEM_DEVICE = 1 } sable_mem;

/*
 * A matrix in VBR form (Fig. 2) with an optional CSR
 * remainder (Fig. 3 indptr/indices/csr_val).
 *
 * Layout and invariants (violations -> SABLE_E_FORMAT, naming array + index):
 *   rpntr[nbrows+1] int32: 0 = rpntr[0] < rpntr[1] < ... < rpntr[nbrows] = nrows
 *                          ("starting index of each block row", Fig. 2 Rpntr)
 *   cpntr[nbcols+1] int32: the same for columns (Fig. 2 Cpntr)
 *   bpntr[nbrows+1] int64: the stored blocks of block row a are
 *                          [bpntr[a], bpntr[a+1]); bpntr[0]=0, non-decreasing,
 *                          bpntr[nbrows] = nblocks.  The paper's pair is
 *                          Bpntrb[a] = bpntr[a] (or -1 if empty), Bpntre[a] =
 *                          bpntr[a+1] (reading R9).
 *   bindx[nblocks]  int32: block column of each block, in [0, nbcols), strictly
 *                          increasing within a block row (Fig. 2 Bindx; R10)
 *   indx[nblocks+1] int64: indx[0]=0, indx[k+1]-indx[k] = h*w of block k,
 *                          indx[nblocks] = val_len ("inclusive of the length
 *                          of the Val array")
 *   val[val_len]    dtype: block k's h x w values column-major:
 *                          A(r0+r, c0+c) = val[indx[k] + c*h + r]
 *                          (reading R8).  Stored zeros
 *                          (+0 or -0) are zero fill, not non-zeros (R4).
 *   rem_indptr[nrows+1] int64, rem_indices[rem_nnz] int32, rem_val[rem_nnz]:
 *                          optional CSR remainder (all three NULL and
 *                          rem_nnz = 0 for none); columns strictly increasing
 *                          within a row.  A position that is non-zero in both
 *                          val and the remainder -> SABLE_E_DUPLICATE.
 * The matrix is the union of both sources.  The inspector's partition does not
 * depend on how the caller splits non-zeros between them (reading R5).
 * nblocks, val_len and rem_nnz are passed explicitly so that sizes are known
 * without reading device memory; they are checked against the arrays.
 * Limits (-> SABLE_E_UNSUPPORTED): nrows, ncols < 2^31; nblocks + rem_nnz
 * < 2^31; the local remainder after classification < 2^31 entries.
 */
typedef struct {
  int64_t nrows, ncols;
  int32_t nbrows, nbcols;
  int64_t nblocks;  /* = bpntr[nbrows]      */
  int64_t val_len;  /* = indx[nblocks]      */
  int64_t rem_nnz;  /* = rem_indptr[nrows]  */
  int32_t dtype;    /* sable_dtype of val, rem_val, x and y */
  int32_t mem;      /* sable_mem: where ALL arrays of this descriptor live */
  const int32_t* rpntr;
  const int32_t* cpntr;
  const int64_t* bpntr;
  const int32_t* bindx;
  const int64_t* indx;
  const void* val;
  const int64_t* rem_indptr;
  const int32_t* rem_indices;
  const void* rem_val;
} sable_vbr_desc;

/* Row sharding for multi-GPU (BASELINE.json north_star s7): the handle of
 * rank r of world P owns a contiguous block-row range chosen by
 * sable_shard_bounds over per-block-row stored-entry weights.  NULL or
 * {0, 1} = the whole matrix. */
typedef struct {
  int32_t rank, world;
} sable_shard;

typedef struct {
  int64_t nrows, ncols;
  int32_t nbrows, nbcols;
  int32_t br_begin, br_end;   /* local block rows [br_begin, br_end)          */
  int64_t row_begin, row_end; /* local rows: y has row_end - row_begin entries */
  int64_t nnz;                /* true non-zeros in the local rows             */
  int64_t n_cells;            /* local candidate cells (cnt >= 1)             */
  int64_t cell_base;          /* candidate cells in block rows < br_begin     */
  int64_t n_dense;            /* local delta-dense cells (tiles)              */
  int64_t tile_elems;         /* sum of their areas (zero fill included)      */
  int64_t rem_nnz;            /* local remainder non-zeros                    */
  int64_t n_dense_global;     /* tiles over the whole matrix                  */
  int64_t bytes_alg;          /* algorithmic bytes per sable_spmv */
  int32_t dtype;
  int32_t delta;
  int32_t suitable;           /* >= 1 dense tile in the matrix */
  int32_t world, rank;
  double inspect_ms;          /* wall time of sable_vbr_create's inspector    */
  /* the executor's plan (DESIGN.md sections 5-6) */
  int32_t exec_grid;          /* CTAs of one sable_spmv launch (one warp each) */
  int32_t unit_bytes;         /* cap on one unit's bytes                       */
  int64_t n_units;            /* warp work units (<= 32 rows of one block row) */
  int64_t n_unit_batches;     /* warp batches of consecutive units             */
  int64_t n_combine;          /* row ranges split over several units           */
  int64_t panel_elems;        /* row-major panel elements (16-byte padded rows) */
  int64_t xmap_entries;       /* x map entries (one per 16-byte column vector)  */
} sable_info;

/* Caller-allocated HOST buffers for sable_export_partition, sized from
 * sable_info of the same handle (the canonical export of DESIGN.md, equal
 * byte for byte to the oracle's, restricted to the local block rows):
 *   cell_br, cell_bc [n_cells] int32; cell_cnt [n_cells] int64;
 *   cell_dense [n_cells] uint8      -- candidate cells in (br, bc) order
 *   tile_off [n_dense+1] int64      -- dense-only offsets (reading R7)
 *   tile_val [tile_elems] dtype     -- column-major, zero-filled tiles
 *   ublocks [n_cells-n_dense] int64 -- ordinals of non-dense cells, relative
 *                                      to the first local cell (add cell_base
 *                                      for global ordinals; Fig. 3 ublocks)
 *   rem_indptr [row_end-row_begin+1] int64, rem_indices [rem_nnz] int32,
 *   rem_val [rem_nnz] dtype         -- the remainder, row-major (reading R6)
 * Any pointer may be NULL to skip that array. */
typedef struct {
  int32_t* cell_br;
  int32_t* cell_bc;
  int64_t* cell_cnt;
  uint8_t* cell_dense;
  int64_t* tile_off;
  void* tile_val;
  int64_t* ublocks;
  int64_t* rem_indptr;
  int32_t* rem_indices;
  void* rem_val;
} sable_partition_host;

/* Inspect a VBR matrix on the current CUDA device (north_star (1)): validate
 * the arrays (SPEC-style invariants above), count the non-zeros of every grid
 * cell from val and the remainder, classify each candidate cell as
 * delta-dense (100*cnt >= delta*h*w in int64, readings R1,
 * R3), pack the dense tiles, assemble the CSR remainder, and plan the
 * executor work.  delta_pct in [0, 101] (101 = nothing dense).
 * All inputs are copied; the call synchronises cuda_stream before returning,
 * so the caller may free its arrays.  The handle owns its device memory.
 * On any error *out is set to NULL and nothing is leaked. */
sable_status sable_vbr_create(const sable_vbr_desc* desc, uint32_t delta_pct,
                              const sable_shard* shard, void* cuda_stream,
                              sable_handle** out);

/* y = A x for the handle's local rows.  x: device pointer to
 * ncols dtype values (the full x); y: device pointer to row_end-row_begin
 * values, written once each (no accumulation into y).  x and y must not
 * alias.  Asynchronous on cuda_stream: no host synchronisation, no
 * allocation.  A handle must not run two calls concurrently (split-row
 * scratch).  x must be finite (reading R13). */
sable_status sable_spmv(sable_handle* h, const void* x, void* y, void* cuda_stream);

/* The same product with HOST buffers (end-to-end path): copies x host->device
 * into handle-owned memory, runs sable_spmv, copies y device->host, and
 * synchronises cuda_stream.  Pinned host memory gives full copy bandwidth. */
sable_status sable_spmv_host(sable_handle* h, const void* x_host, void* y_host,
                             void* cuda_stream);

/* ---- per-shape delta policy (reading R22) --
 * The paper decides dense vs sparse per block with a model trained on its
 * CPU's timings; here a measured B200 policy can replace
 * the single delta: a candidate cell of h x w is dense iff h*w >= min_area
 * and 100*cnt >= delta(h, w)*h*w, delta(h, w) = the delta of the FIRST rule
 * with h_min <= h <= h_max and w_min <= w <= w_max, else delta_pct.  With
 * no rules and min_area <= 1 this is sable_vbr_create's rule exactly.
 * scripts/calibrate.py measures a policy (profiles/r02_f2_policy.json). */
typedef struct {
  int32_t h_min, h_max;  /* inclusive block-height range */
  int32_t w_min, w_max;  /* inclusive block-width range  */
  uint32_t delta_pct;    /* 0..101 for cells of these shapes */
} sable_delta_rule;

typedef struct {
  uint32_t delta_pct;            /* cells matched by no rule, 0..101 */
  int64_t min_area;              /* cells with h*w < min_area are never dense (>= 0) */
  int32_t n_rules;               /* 0..64 */
  const sable_delta_rule* rules; /* host memory, n_rules records */
} sable_delta_policy;

/* sable_vbr_create under a per-shape policy (SABLE_E_INVALID_ARG for a delta
 * outside 0..101, a negative min_area or more than 64 rules). */
sable_status sable_vbr_create_policy(const sable_vbr_desc* desc, const sable_delta_policy* policy,
                                     const sable_shard* shard, void* cuda_stream,
                                     sable_handle** out);

/* Free the handle (NULL is a no-op).  Synchronises the device first. */
sable_status sable_destroy(sable_handle* h);

sable_status sable_get_info(const sable_handle* h, sable_info* info);

/* Copy the canonical partition of the local block rows to host buffers
 * (see sable_partition_host).  Synchronous. */
sable_status sable_export_partition(const sable_handle* h, const sable_partition_host* out);

/* Host-only (no GPU needed): block-row shard boundaries for `world` ranks.
 * weights[nbrows] >= 0 (stored entries streamed per block row: tile areas +
 * remainder non-zeros, reading of north_star s7 in DESIGN.md); bounds[world+1]
 * receives 0 = b0 <= b1 <= ... <= b_world = nbrows with boundary k = the
 * first a whose prefix weight reaches k * total / world. */
sable_status sable_shard_bounds(const int64_t* weights, int32_t nbrows, int32_t world,
                                int32_t* bounds);

/* ---- multi-GPU exchange (north_star s7: y slices all-gathered with NCCL) */

/* Write a fresh ncclUniqueId (128 bytes) to out; rank 0 calls this and
 * broadcasts the bytes (e.g. over torch.distributed). */
sable_status sable_nccl_unique_id(void* out128);

/* Create the handle's NCCL communicator (rank/world from the create shard),
 * its exchange stream, and all-gather every rank's exchange-slice row bounds
 * (SABLE_E_INVALID_ARG if the ranks' row layouts disagree). */
sable_status sable_comm_init(sable_handle* h, const void* id128);

/* Poll the communicator for an asynchronous NCCL error (non-blocking,
 * ncclCommGetAsyncError): SABLE_OK, or SABLE_E_NCCL after aborting a failed
 * communicator.  The exchange calls below poll before enqueueing work. */
sable_status sable_comm_check(sable_handle* h);

/* One exchange step: x_next[row_begin:row_end] = (A x)[local
 * rows], then every rank's rows are all-gathered into x_next (ncols entries)
 * on every rank with in-place ncclBroadcasts.  Pipelined: the shard's rows are
 * cut into exchange slices of whole row ranges; slice s is broadcast on the
 * handle's exchange stream while slice s + 1 computes.
 * Requires a square matrix (SABLE_E_DIM) and sable_comm_init when world > 1.
 * x_full and x_next_full are device pointers, not aliased.  Asynchronous on
 * cuda_stream (the exchange stream is forked from and joined back to it). */
sable_status sable_spmv_allgather(sable_handle* h, const void* x_full, void* x_next_full,
                                  void* cuda_stream);

/* iters exchange steps ping-ponging x_a -> x_b -> x_a ...; *result_in_b = 1
 * if the final x is in x_b.  The steps run as ONE CUDA graph (kernels and
 * NCCL calls captured once per (x_a, x_b, iters) and relaunched on later
 * calls) on an internal stream ordered after / before cuda_stream by events.
 * Asynchronous; bitwise the same as iters sable_spmv_allgather calls. */
sable_status sable_spmv_iterate(sable_handle* h, void* x_a, void* x_b, int32_t iters,
                                void* cuda_stream, int32_t* result_in_b);

/* ---- fused exchange epilogue (north_star s7) ------------
 * Iterated SpMV ping-pongs two full x buffers.  Once they
 * are registered with the handle, an exchange step whose x_next is one of
 * them is ONE kernel launch: the SpMV's epilogue stores every finished y row
 * into the local x_next and into the same row of every peer's x_next through
 * NVLink peer mappings, so no broadcast follows the SpMV; the step ends with
 * a one-word ncclAllReduce as the barrier (all rows have landed here; every
 * rank is done reading the buffer the next step overwrites).  y is bitwise
 * the same as on the NCCL path.  Steps on unregistered buffers keep using the
 * NCCL broadcast pipeline.  At most 8 ranks.
 *
 * sable_comm_fuse: x_a, x_b are device buffers (ncols values each) inside
 *   cudaMalloc allocations (CUDA IPC: not cudaMallocAsync / VMM memory), one
 *   process per GPU, after sable_comm_init; collective (every rank calls it):
 *   the allocations' IPC handles are all-gathered and every peer's buffers
 *   mapped (SABLE_E_CUDA if peer access is unavailable).  world == 1: no
 *   peers, the step is the plain SpMV.
 * sable_comm_set_peers: the caller supplies the mappings itself (peers_a[q],
 *   peers_b[q]: peer q's x_a / x_b as device pointers valid on this GPU, from
 *   its own symmetric-memory or IPC setup; host arrays of npeers <= 7
 *   pointers, copied).  With a communicator the step barrier is the
 *   all-reduce above; without one (sable_comm_init not called) the caller
 *   orders the ranks' steps itself (e.g. all ranks of a test on one stream).
 * sable_comm_unfuse: forget the registration (unmaps IPC mappings).
 * The buffers must stay allocated while registered; sable_destroy and
 * sable_comm_init unfuse. */
sable_status sable_comm_fuse(sable_handle* h, void* x_a, void* x_b);
sable_status sable_comm_set_peers(sable_handle* h, void* x_a, void* x_b,
                                  void* const* peers_a, void* const* peers_b, int32_t npeers);
sable_status sable_comm_unfuse(sable_handle* h);

/* The all-gather layout on the host (no device work): for per-block-row
 * weights (as in sable_shard_bounds) and the row grid rpntr[nbrows+1], the
 * global row bounds of every rank's slice of y, row_bounds[world+1]
 * (row_bounds[q] = rpntr[shard bound q]) -- the rows rank q broadcasts. */
sable_status sable_exchange_rows(const int64_t* weights, int32_t nbrows, const int32_t* rpntr,
                                 int32_t world, int64_t* row_bounds);

/* ---- the partitioner ------------------------------
 * Alg. 1 "Matrix Partitioning" on the device: the row
 * grid rpntr and column grid cpntr of a CSR matrix, cutting between rows
 * i and i+1 when S(row i, row i+1) < t, Eq. 1 when
 * shifts == 0, Eq. 2 (+-1 shifts, reading R17) when
 * shifts != 0; runs of empty rows extend one block; the
 * columns are the same procedure on the pattern of A^T.  Readings R19-R21
 * (DESIGN.md): strictly increasing grids, t = t_num / t_den compared exactly
 * (dot * t_den < t_num * max(nnz)), no similarity for an empty row i.
 *   rowptr[nrows+1] (int64, rowptr[0] = 0), colidx[nnz] (int32, strictly
 *   increasing within a row, < ncols): the pattern; values are not needed.
 *   mem: where rowptr/colidx live (SABLE_MEM_HOST: copied in; DEVICE: read
 *   in place, must be device memory of the current device).
 *   rpntr[nrows+1], cpntr[ncols+1]: HOST buffers (capacity for the finest
 *   grid) receiving 0 = g0 < ... < gk = n; *nbrows / *nbcols = k.
 * Synchronises cuda_stream; scratch is stream-ordered and freed on return.
 * Errors: SABLE_E_INVALID_ARG (NULL, nrows/ncols < 1, t_den == 0, bad mem),
 * SABLE_E_UNSUPPORTED (sizes >= 2^31), SABLE_E_OOM, SABLE_E_CUDA.  The
 * pattern is not validated (use sable_vbr_create's validation for that). */
sable_status sable_partition_grid(int64_t nrows, int64_t ncols, int64_t nnz,
                                  const int64_t* rowptr, const int32_t* colidx, int32_t mem,
                                  uint32_t t_num, uint32_t t_den, int32_t shifts,
                                  void* cuda_stream, int32_t* rpntr, int32_t* nbrows,
                                  int32_t* cpntr, int32_t* nbcols);

/* ---- multi-vector products ------------------------
 * Y = A X for k right-hand sides in one pass over the inspected matrix (the
 * panels and the remainder are read once for all k): Y[:, j] = A X[:, j],
 * y_i = sum_j A_ij x_j per column -- the "user-defined
 * operation" over the same VBR-C split.
 *   X: device, row-major ncols x k (the k values of matrix column c at
 *      X[c*k .. c*k+k)), dtype of the handle; Y: device, row-major
 *      (row_end - row_begin) x k, fully written; not aliased with X.
 *   k in {1, 2, 4, 8}: the SpMV's plan and kernel with k accumulators per row
 *      (CUDA cores; k = 1 is bitwise sable_spmv, k > 1 folds lanes in another
 *      fixed tree).
 *   k in {16, 32, 64, 128}, fp32 handles only: every unit's panel rows times
 *      the gathered X rows on the tensor cores (tcgen05.mma kind::tf32 into
 *      TMEM, 3xTF32 split for fp32 accuracy; csrc/mma.cu), the remainder on
 *      the CUDA cores in entry order.
 *   Other k, or k >= 16 on fp64: SABLE_E_UNSUPPORTED.  Asynchronous on
 *   cuda_stream; the first call per path allocates k-wide scratch
 *   (synchronously).  Each row's sums run in a fixed order (deterministic
 *   run to run), within the SpMV tolerance of the definition. */
sable_status sable_spmm(sable_handle* h, const void* X, void* Y, int32_t k, void* cuda_stream);

/* ---- handle images ---------------------------------
 * Compile once, run many: the inspected state of a handle
 * -- the executor's unit plan (units, batches, x maps, combine groups), the
 * row-major panels, the remainder CSR, tile geometry, local cells, scalars
 * incl. the suitability flag of sable_get_info -- as one byte
 * image ("SABLEVC3": header with an FNV-1a
 * checksum, then fixed sections 8-byte aligned).  No NCCL state: call
 * sable_comm_init again on a world > 1 handle.  The image is tied to
 * SABLE_ABI_VERSION and to the executor configuration it was planned with.
 *
 * sable_serialize: buf == NULL (cap ignored) -> *size = image bytes only;
 * otherwise writes the image to HOST buf (cap >= *size, else
 * SABLE_E_INVALID_ARG).  Synchronises the handle's device.  Serialising the
 * same handle twice, or a handle loaded from an image, gives identical bytes.
 * sable_deserialize: a new handle on the current device from an image of
 * `size` bytes in host memory (copied; buf may be freed on return).  Errors:
 * SABLE_E_FORMAT (bad magic, other library version, inconsistent sizes,
 * checksum mismatch), SABLE_E_OOM, SABLE_E_CUDA. */
sable_status sable_serialize(const sable_handle* h, void* buf, int64_t cap, int64_t* size);
sable_status sable_deserialize(const void* buf, int64_t size, void* cuda_stream,
                               sable_handle** out);

const char* sable_status_string(sable_status s);
const char* sable_last_error(void); /* thread-local; "" if none */
int32_t sable_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SABLE_H_ */
