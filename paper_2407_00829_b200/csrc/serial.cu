// serial.cu -- handle serialization: the inspected state
// of a handle as one self-checking byte image, so that a compile-once /
// run-many user skips the inspector on the next run.
// The image holds everything sable_spmv, sable_export_partition and the
// exchange steps read: the executor byte stream and its chunk/task tables,
// the remainder CSR and its packet plan, the panel values and tile geometry
// and the local cells, plus the handle's scalars and the suitability flag of
// sable_get_info.  Scratch and arrival counters are not data:
// they are re-allocated (counters zeroed) on load.  Layout (little endian):
//   ImageHeader (scalars, section count, payload FNV-1a 64)
//   sections in a fixed order, each 8-byte aligned (zero padding).
// The image is device-independent (no pointers) but tied to the ABI version,
// the struct layouts below and the executor configuration it was planned for.
#include <cstring>
#include <vector>

#include "sable_internal.cuh"

namespace sable {

void free_handle(sable_handle* h);

namespace {

constexpr char kMagic[8] = {'S', 'A', 'B', 'L', 'E', 'V', 'C', '1'};
constexpr int kSections = 21;

struct ImageHeader {
  char magic[8];
  int32_t abi_version, header_bytes;
  int32_t sizeof_chunkref, sizeof_xginfo, sizeof_remp, sizeof_tiledesc;
  int32_t dtype, delta;
  int64_t nrows, ncols;
  int32_t nbr, nbc, br_begin, br_end;
  int64_t row_begin, row_end;
  int32_t rank, world;
  int64_t tile_elems, n_dense, n_runs, stream_bytes;
  int64_t n_groups, n_items, n_chunks, n_bundles, n_bundle_lanes;
  int64_t rp_packets, rp_pieces, rp_long;
  ExecCfg cfg;
  int64_t rem_nnz, scratch_elems, n_cells, cell_base;
  int64_t nnz, n_dense_global, bytes_alg;
  double inspect_ms;
  int64_t n_sections;
  uint64_t payload_fnv;
  int64_t section_bytes[kSections];
};

struct Section {
  void* dev;    // device array (or nullptr for a host array)
  void* host;   // host array
  int64_t bytes;
};

// The fixed section list of a handle (sizes from its scalars).
std::vector<Section> sections(sable_handle* h) {
  const int64_t sv = h->dtype == SABLE_F64 ? 8 : 4;
  const int64_t nloc = h->row_end - h->row_begin;
  const int64_t nbl = (int64_t)h->br_end - h->br_begin;
  return {
      {h->stream, nullptr, h->stream_bytes},
      {h->cref, nullptr, (int64_t)sizeof(ChunkRef) * h->n_chunks},
      {h->xgi, nullptr, (int64_t)sizeof(XgInfo) * h->n_items},
      {h->task, nullptr, 4 * ((int64_t)h->cfg.n_tasks + 1)},
      {h->rp.packets, nullptr, (int64_t)sizeof(RemPacket) * h->rp.n_packets},
      {h->rem_ptr, nullptr, 4 * (nloc + 1)},
      {h->rem_idx, nullptr, 4 * h->rem_nnz},
      {h->rem_val, nullptr, sv * h->rem_nnz},
      {h->tval, nullptr, sv * h->tile_elems},
      {h->tiles, nullptr, (int64_t)sizeof(TileDesc) * h->n_dense},
      {h->tile_canon_off, nullptr, 8 * (h->n_dense + 1)},
      {h->tile_br, nullptr, 4 * h->n_dense},
      {h->br_vbase, nullptr, 8 * (nbl + 1)},
      {h->br_W, nullptr, 4 * (nbl + 1)},
      {h->cell_br, nullptr, 4 * h->n_cells},
      {h->cell_bc, nullptr, 4 * h->n_cells},
      {h->cell_cnt, nullptr, 8 * h->n_cells},
      {h->cell_dense, nullptr, h->n_cells},
      {nullptr, h->all_bounds_h, 4 * ((int64_t)h->world + 1)},
      {nullptr, h->rpntr_h, 4 * ((int64_t)h->nbr + 1)},
      {nullptr, nullptr, 0},  // reserved
  };
}

int64_t pad8(int64_t b) { return (b + 7) & ~(int64_t)7; }

uint64_t fnv1a(const unsigned char* p, int64_t n, uint64_t hsh = 1469598103934665603ull) {
  for (int64_t i = 0; i < n; ++i) {
    hsh ^= p[i];
    hsh *= 1099511628211ull;
  }
  return hsh;
}

void fill_header(const sable_handle* h, ImageHeader* H) {
  memset(H, 0, sizeof(*H));
  memcpy(H->magic, kMagic, 8);
  H->abi_version = SABLE_ABI_VERSION;
  H->header_bytes = (int32_t)sizeof(ImageHeader);
  H->sizeof_chunkref = (int32_t)sizeof(ChunkRef);
  H->sizeof_xginfo = (int32_t)sizeof(XgInfo);
  H->sizeof_remp = (int32_t)sizeof(RemPacket);
  H->sizeof_tiledesc = (int32_t)sizeof(TileDesc);
  H->dtype = h->dtype;
  H->delta = h->delta;
  H->nrows = h->nrows;
  H->ncols = h->ncols;
  H->nbr = h->nbr;
  H->nbc = h->nbc;
  H->br_begin = h->br_begin;
  H->br_end = h->br_end;
  H->row_begin = h->row_begin;
  H->row_end = h->row_end;
  H->rank = h->rank;
  H->world = h->world;
  H->tile_elems = h->tile_elems;
  H->n_dense = h->n_dense;
  H->n_runs = h->n_runs;
  H->stream_bytes = h->stream_bytes;
  H->n_groups = h->n_groups;
  H->n_items = h->n_items;
  H->n_chunks = h->n_chunks;
  H->n_bundles = h->n_bundles;
  H->n_bundle_lanes = h->n_bundle_lanes;
  H->rp_packets = h->rp.n_packets;
  H->rp_pieces = h->rp.n_pieces;
  H->rp_long = h->rp.n_long;
  H->cfg = h->cfg;
  H->rem_nnz = h->rem_nnz;
  H->scratch_elems = h->scratch_elems;
  H->n_cells = h->n_cells;
  H->cell_base = h->cell_base;
  H->nnz = h->nnz;
  H->n_dense_global = h->n_dense_global;
  H->bytes_alg = h->bytes_alg;
  H->inspect_ms = h->inspect_ms;
  H->n_sections = kSections;
}

void load_header(const ImageHeader& H, sable_handle* h) {
  h->dtype = H.dtype;
  h->delta = H.delta;
  h->nrows = H.nrows;
  h->ncols = H.ncols;
  h->nbr = H.nbr;
  h->nbc = H.nbc;
  h->br_begin = H.br_begin;
  h->br_end = H.br_end;
  h->row_begin = H.row_begin;
  h->row_end = H.row_end;
  h->rank = H.rank;
  h->world = H.world;
  h->tile_elems = H.tile_elems;
  h->n_dense = H.n_dense;
  h->n_runs = H.n_runs;
  h->stream_bytes = H.stream_bytes;
  h->n_groups = H.n_groups;
  h->n_items = H.n_items;
  h->n_chunks = H.n_chunks;
  h->n_bundles = H.n_bundles;
  h->n_bundle_lanes = H.n_bundle_lanes;
  h->rp.n_packets = H.rp_packets;
  h->rp.n_pieces = H.rp_pieces;
  h->rp.n_long = H.rp_long;
  h->cfg = H.cfg;
  h->rem_nnz = H.rem_nnz;
  h->scratch_elems = H.scratch_elems;
  h->n_cells = H.n_cells;
  h->cell_base = H.cell_base;
  h->nnz = H.nnz;
  h->n_dense_global = H.n_dense_global;
  h->bytes_alg = H.bytes_alg;
  h->inspect_ms = H.inspect_ms;
}

sable_status fail(sable_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

}  // namespace

}  // namespace sable

using namespace sable;

extern "C" sable_status sable_serialize(const sable_handle* hc, void* buf, int64_t cap,
                                        int64_t* size) {
  if (!hc || !size || (cap > 0 && !buf) || cap < 0)
    return fail(SABLE_E_INVALID_ARG, "sable_serialize: bad arguments");
  sable_handle* h = const_cast<sable_handle*>(hc);
  const std::vector<Section> S = sections(h);
  int64_t total = (int64_t)sizeof(ImageHeader);
  for (const Section& s : S) total += pad8(s.bytes);
  *size = total;
  if (!buf) return SABLE_OK;  // size query
  if (cap < total) return fail(SABLE_E_INVALID_ARG, "sable_serialize: buffer too small");
  int dev_prev = 0;
  cudaGetDevice(&dev_prev);
  cudaSetDevice(h->device);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned char* out = static_cast<unsigned char*>(buf);
  ImageHeader H;
  fill_header(h, &H);
  int64_t off = (int64_t)sizeof(ImageHeader);
  for (int i = 0; i < kSections && !e; ++i) {
    const Section& s = S[i];
    H.section_bytes[i] = s.bytes;
    if (s.bytes > 0) {
      if (s.dev)
        e = cudaMemcpy(out + off, s.dev, (size_t)s.bytes, cudaMemcpyDeviceToHost);
      else
        memcpy(out + off, s.host, (size_t)s.bytes);
    }
    memset(out + off + s.bytes, 0, (size_t)(pad8(s.bytes) - s.bytes));
    off += pad8(s.bytes);
  }
  cudaSetDevice(dev_prev);
  if (e) {
    set_error(cuda_msg(e, "sable_serialize"));
    return SABLE_E_CUDA;
  }
  H.payload_fnv = fnv1a(out + sizeof(ImageHeader), total - (int64_t)sizeof(ImageHeader));
  memcpy(out, &H, sizeof(H));
  return SABLE_OK;
}

extern "C" sable_status sable_deserialize(const void* buf, int64_t size, void* cuda_stream,
                                          sable_handle** out) {
  if (!buf || !out || size < (int64_t)sizeof(ImageHeader))
    return fail(SABLE_E_INVALID_ARG, "sable_deserialize: bad arguments");
  *out = nullptr;
  const unsigned char* in = static_cast<const unsigned char*>(buf);
  ImageHeader H;
  memcpy(&H, in, sizeof(H));
  if (memcmp(H.magic, kMagic, 8) != 0) return fail(SABLE_E_FORMAT, "sable_deserialize: not a SABLEVC1 image");
  if (H.abi_version != SABLE_ABI_VERSION || H.header_bytes != (int32_t)sizeof(ImageHeader) ||
      H.sizeof_chunkref != (int32_t)sizeof(ChunkRef) || H.sizeof_xginfo != (int32_t)sizeof(XgInfo) ||
      H.sizeof_remp != (int32_t)sizeof(RemPacket) || H.sizeof_tiledesc != (int32_t)sizeof(TileDesc) ||
      H.n_sections != kSections)
    return fail(SABLE_E_FORMAT, "sable_deserialize: image written by another library version");
  if ((H.dtype != SABLE_F32 && H.dtype != SABLE_F64) || H.world < 1 || H.rank < 0 ||
      H.rank >= H.world || H.nbr < 1 || H.br_begin < 0 || H.br_end < H.br_begin || H.br_end > H.nbr ||
      H.row_begin < 0 || H.row_end < H.row_begin || H.row_end > H.nrows)
    return fail(SABLE_E_FORMAT, "sable_deserialize: inconsistent header");
  {
    const int64_t lim = (int64_t)1 << 40;  // bounds every count so that byte sizes cannot wrap
    const int64_t cnt[] = {H.nrows, H.ncols, H.tile_elems, H.n_dense, H.stream_bytes, H.n_groups,
                           H.n_items, H.n_chunks, H.rp_packets, H.rp_pieces, H.rp_long,
                           H.rem_nnz, H.scratch_elems, H.n_cells, (int64_t)H.cfg.n_tasks,
                           (int64_t)H.nbr, (int64_t)H.world};
    for (int64_t c : cnt)
      if (c < 0 || c > lim) return fail(SABLE_E_FORMAT, "sable_deserialize: count out of range");
  }
  sable_handle* h = new (std::nothrow) sable_handle();
  if (!h) return fail(SABLE_E_OOM, "host allocation failed");
  load_header(H, h);
  cudaGetDevice(&h->device);
  // the expected section sizes follow from the scalars: check before reading
  h->all_bounds_h = (int32_t*)malloc(sizeof(int32_t) * ((size_t)H.world + 1));
  h->rpntr_h = (int32_t*)malloc(sizeof(int32_t) * ((size_t)H.nbr + 1));
  if (!h->all_bounds_h || !h->rpntr_h) {
    free_handle(h);
    return fail(SABLE_E_OOM, "host allocation failed");
  }
  std::vector<Section> S = sections(h);
  int64_t total = (int64_t)sizeof(ImageHeader);
  for (int i = 0; i < kSections; ++i) {
    if (S[i].bytes < 0 || S[i].bytes != H.section_bytes[i]) {
      free_handle(h);
      return fail(SABLE_E_FORMAT, "sable_deserialize: section " + std::to_string(i) +
                                      " size disagrees with the header");
    }
    total += pad8(S[i].bytes);
  }
  if (total != size) {
    free_handle(h);
    return fail(SABLE_E_FORMAT, "sable_deserialize: image size " + std::to_string(size) +
                                    " != " + std::to_string(total));
  }
  if (fnv1a(in + sizeof(ImageHeader), size - (int64_t)sizeof(ImageHeader)) != H.payload_fnv) {
    free_handle(h);
    return fail(SABLE_E_FORMAT, "sable_deserialize: payload checksum mismatch");
  }
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int64_t sv = H.dtype == SABLE_F64 ? 8 : 4;
  cudaError_t e = cudaSuccess;
  auto dal = [&](void** p, int64_t bytes) {
    if (!e) e = cudaMalloc(p, (size_t)std::max<int64_t>(bytes, 1) + 16);
  };
  // device arrays in section order (pointers of the fresh handle)
  void** dst[kSections] = {(void**)&h->stream, (void**)&h->cref, (void**)&h->xgi,
                           (void**)&h->task, (void**)&h->rp.packets, (void**)&h->rem_ptr,
                           (void**)&h->rem_idx, &h->rem_val, &h->tval, (void**)&h->tiles,
                           (void**)&h->tile_canon_off, (void**)&h->tile_br,
                           (void**)&h->br_vbase, (void**)&h->br_W, (void**)&h->cell_br,
                           (void**)&h->cell_bc, (void**)&h->cell_cnt, (void**)&h->cell_dense,
                           nullptr, nullptr, nullptr};
  int64_t off = (int64_t)sizeof(ImageHeader);
  for (int i = 0; i < kSections; ++i) {
    if (dst[i]) {
      dal(dst[i], S[i].bytes);
      if (!e && S[i].bytes > 0)
        e = cudaMemcpyAsync(*dst[i], in + off, (size_t)S[i].bytes, cudaMemcpyHostToDevice, st);
    } else if (i == 18) {
      memcpy(h->all_bounds_h, in + off, (size_t)S[i].bytes);
    } else if (i == 19) {
      memcpy(h->rpntr_h, in + off, (size_t)S[i].bytes);
    }
    off += pad8(S[i].bytes);
  }
  // scratch and arrival counters (the executors leave counters at zero)
  dal(&h->scratch, sv * h->scratch_elems);
  dal((void**)&h->counters, 4 * h->n_groups);
  dal(&h->rp.scratch, sv * h->rp.n_pieces);
  dal((void**)&h->rp.counters, 4 * h->rp.n_long);
  if (!e) e = cudaMemsetAsync(h->counters, 0, 4 * (size_t)std::max<int64_t>(h->n_groups, 1), st);
  if (!e) e = cudaMemsetAsync(h->rp.counters, 0, 4 * (size_t)std::max<int64_t>(h->rp.n_long, 1), st);
  if (!e) e = cudaStreamSynchronize(st);  // the host image may be released on return
  if (e) {
    set_error(cuda_msg(e, "sable_deserialize"));
    cudaStreamSynchronize(st);
    free_handle(h);
    return e == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA;
  }
  (void)sv;
  *out = h;
  return SABLE_OK;
}
