// serial.cu -- handle serialization: the inspected state
// of a handle as one self-checking byte image, so that a compile-once /
// run-many user skips the inspector on the next run.
// The image holds everything sable_spmv, sable_spmm, sable_export_partition
// and the exchange steps read: the unit plan (units, warp batches, x maps,
// combine groups), the row-major panels, the remainder CSR, the tile
// geometry and the local cells, plus the handle's scalars and the
// suitability flag of sable_get_info.  Scratch and arrival
// counters are not data: they are re-allocated (counters zeroed) on load.
// Layout (little endian):
//   ImageHeader (scalars, section count, payload FNV-1a 64)
//   sections in a fixed order, each 8-byte aligned (zero padding).
// The image is device-independent (no pointers) but tied to the ABI version
// and the struct layouts below.  Loading checks every index the kernels
// follow (unit ranges, x maps, remainder columns, combine slots, shard
// bounds), so an image that passes cannot make the kernels read out of
// bounds.
#include <algorithm>
#include <cstring>
#include <vector>

#include "sable_internal.cuh"

namespace sable {

void free_handle(sable_handle* h);
cudaError_t upload_batch_heads(sable_handle* h, const Unit* U, const int32_t* batch,
                               cudaStream_t st);  // plan.cu

namespace {

constexpr char kMagic[8] = {'S', 'A', 'B', 'L', 'E', 'V', 'C', '3'};
constexpr int kSections = 22;

struct ImageHeader {
  char magic[8];
  int32_t abi_version, header_bytes;
  int32_t sizeof_unit, sizeof_xgu, sizeof_tiledesc, sizeof_cfg;
  int32_t dtype, delta;
  int64_t nrows, ncols;
  int32_t nbr, nbc, br_begin, br_end;
  int64_t row_begin, row_end;
  int32_t rank, world;
  ExecCfg cfg;
  int64_t tile_elems, n_dense;
  int64_t n_units, n_ubatch, n_xq, n_xside, n_uxg, uscratch_slots, pv_elems;
  int64_t rem_nnz, n_cells, cell_base;
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
      {h->units, nullptr, (int64_t)sizeof(Unit) * h->n_units},
      {h->ubatch, nullptr, 4 * (h->n_ubatch + 1)},
      {h->xq, nullptr, (int64_t)sizeof(XMap) * h->n_xq},
      {h->xside, nullptr, 16 * h->n_xside},
      {h->uxg, nullptr, (int64_t)sizeof(XgU) * h->n_uxg},
      {h->pv, nullptr, sv * h->pv_elems},
      {h->rem_ptr, nullptr, 4 * (nloc + 1)},
      {h->rem_idx, nullptr, 4 * h->rem_nnz},
      {h->rem_val, nullptr, sv * h->rem_nnz},
      {h->tiles, nullptr, (int64_t)sizeof(TileDesc) * h->n_dense},
      {h->tile_canon_off, nullptr, 8 * (h->n_dense + 1)},
      {h->tile_br, nullptr, 4 * h->n_dense},
      {h->br_pbase, nullptr, 8 * (nbl + 1)},
      {h->br_W, nullptr, 4 * (nbl + 1)},
      {h->cell_br, nullptr, 4 * h->n_cells},
      {h->cell_bc, nullptr, 4 * h->n_cells},
      {h->cell_cnt, nullptr, 8 * h->n_cells},
      {h->cell_dense, nullptr, h->n_cells},
      {nullptr, h->all_bounds_h, 4 * ((int64_t)h->world + 1)},
      {nullptr, h->rpntr_h, 4 * ((int64_t)h->nbr + 1)},
      {nullptr, h->slice_batch.data(), 8 * (int64_t)h->slice_batch.size()},
      {nullptr, h->slice_row.data(), 8 * (int64_t)h->slice_row.size()},
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
  H->sizeof_unit = (int32_t)sizeof(Unit);
  H->sizeof_xgu = (int32_t)sizeof(XgU);
  H->sizeof_tiledesc = (int32_t)sizeof(TileDesc);
  H->sizeof_cfg = (int32_t)sizeof(ExecCfg);
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
  H->cfg = h->cfg;
  H->tile_elems = h->tile_elems;
  H->n_dense = h->n_dense;
  H->n_units = h->n_units;
  H->n_ubatch = h->n_ubatch;
  H->n_xq = h->n_xq;
  H->n_xside = h->n_xside;
  H->n_uxg = h->n_uxg;
  H->uscratch_slots = h->uscratch_slots;
  H->pv_elems = h->pv_elems;
  H->rem_nnz = h->rem_nnz;
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
  h->cfg = H.cfg;
  h->tile_elems = H.tile_elems;
  h->n_dense = H.n_dense;
  h->n_units = H.n_units;
  h->n_ubatch = H.n_ubatch;
  h->n_xq = H.n_xq;
  h->n_xside = H.n_xside;
  h->n_uxg = H.n_uxg;
  h->uscratch_slots = H.uscratch_slots;
  h->pv_elems = H.pv_elems;
  h->rem_nnz = H.rem_nnz;
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

template <typename T>
const T* sec(const unsigned char* in, const std::vector<int64_t>& off, int i) {
  return reinterpret_cast<const T*>(in + off[i]);
}

// Every index the kernels and the exchange follow, checked on the host image
// before anything is uploaded.  Returns "" if the image is consistent.
std::string check_image(const ImageHeader& H, const unsigned char* in,
                        const std::vector<int64_t>& off) {
  const int64_t nloc = H.row_end - H.row_begin;
  const int64_t vec = H.dtype == SABLE_F64 ? 2 : 4;
  const int64_t pv16 = H.pv_elems / vec;
  // shard bounds and block-row pointers (sable_spmv_allgather indexes them)
  const int32_t* bounds = sec<int32_t>(in, off, 18);
  const int32_t* rp = sec<int32_t>(in, off, 19);
  if (bounds[0] != 0 || bounds[H.world] != H.nbr) return "shard bounds";
  for (int32_t q = 0; q < H.world; ++q)
    if (bounds[q + 1] < bounds[q]) return "shard bounds";
  if (bounds[H.rank] != H.br_begin || bounds[H.rank + 1] != H.br_end) return "shard bounds";
  if (rp[0] != 0 || rp[H.nbr] != H.nrows) return "rpntr";
  for (int32_t a = 0; a < H.nbr; ++a)
    if (rp[a + 1] <= rp[a]) return "rpntr";
  if (rp[H.br_begin] != H.row_begin || rp[H.br_end] != H.row_end) return "local rows";
  // remainder CSR
  const int32_t* rptr = sec<int32_t>(in, off, 6);
  const int32_t* ridx = sec<int32_t>(in, off, 7);
  if (rptr[0] != 0 || rptr[nloc] != H.rem_nnz) return "rem_ptr";
  for (int64_t r = 0; r < nloc; ++r)
    if (rptr[r + 1] < rptr[r]) return "rem_ptr";
  for (int64_t e = 0; e < H.rem_nnz; ++e)
    if (ridx[e] < 0 || ridx[e] >= H.ncols) return "rem_indices";
  // x maps
  const XMap* xq = sec<XMap>(in, off, 2);
  const int32_t* xside = sec<int32_t>(in, off, 3);
  for (int64_t i = 0; i < H.n_xq; ++i) {
    const XMap m = xq[i];
    if (m.c < 0) {
      if ((int64_t)~m.c >= H.n_xside) return "x map";
      continue;
    }
    const int64_t k = m.kd & 3, d = m.kd >> 2, vec = H.dtype == SABLE_F64 ? 2 : 4;
    if (k >= vec || (k == 0 && d != 0)) return "x map";
    for (int64_t i = 0; i < vec; ++i) {  // every column the executors read
      const int64_t c = m.c + i + (i >= k ? d : 0);
      if (c < 0 || c >= H.ncols) return "x map";
    }
  }
  for (int64_t i = 0; i < 4 * H.n_xside; ++i)
    if (xside[i] < 0 || xside[i] >= H.ncols) return "x side map";
  // combine groups
  const XgU* xg = sec<XgU>(in, off, 4);
  for (int64_t g = 0; g < H.n_uxg; ++g)
    if (xg[g].counter != g || xg[g].npieces < 2 || xg[g].slot < 0 ||
        xg[g].slot + 32 * (int64_t)xg[g].npieces > H.uscratch_slots)
      return "combine groups";
  // warp batches and units
  const int32_t* batch = sec<int32_t>(in, off, 1);
  if (batch[0] != 0 || batch[H.n_ubatch] != H.n_units) return "batches";
  for (int64_t b = 0; b < H.n_ubatch; ++b)
    if (batch[b + 1] <= batch[b]) return "batches";
  const Unit* U = sec<Unit>(in, off, 0);
  for (int64_t u = 0; u < H.n_units; ++u) {
    const Unit& x = U[u];
    if (x.nr < 1 || x.nr > 32 || x.llpr > 5 || x.row0 < 0 || x.row0 + (int64_t)x.nr > nloc ||
        x.e0 < 0 || x.e1 < x.e0 || x.e1 > H.rem_nnz || x.wq < 0)
      return "unit " + std::to_string(u);
    if (x.wq > 0 && (x.voff16 < 0 || (int64_t)x.voff16 + (int64_t)x.nr * x.wq > pv16 ||
                     x.xq0 < 0 || (int64_t)x.xq0 + x.wq > H.n_xq))
      return "unit " + std::to_string(u);
    if (x.xg >= 0 && (x.xg >= H.n_uxg || x.piece >= xg[x.xg].npieces))
      return "unit " + std::to_string(u);
    if (x.xg < -1) return "unit " + std::to_string(u);
  }
  // exchange slices: batch and row boundaries, cut at unit boundaries
  const int64_t* sb = sec<int64_t>(in, off, 20);
  const int64_t* sr = sec<int64_t>(in, off, 21);
  if (sb[0] != 0 || sb[kSlices] != H.n_ubatch || sr[0] != 0 || sr[kSlices] != nloc)
    return "slices";
  for (int s = 0; s < kSlices; ++s) {
    if (sb[s + 1] < sb[s] || sr[s + 1] < sr[s]) return "slices";
    if (sb[s] < H.n_ubatch && U[batch[sb[s]]].row0 != sr[s]) return "slices";
  }
  // export geometry
  const int64_t* toff = sec<int64_t>(in, off, 10);
  if (toff[0] != 0 || toff[H.n_dense] != H.tile_elems) return "tile offsets";
  const int32_t* tbr = sec<int32_t>(in, off, 11);
  const TileDesc* td = sec<TileDesc>(in, off, 9);
  const int64_t* pbase = sec<int64_t>(in, off, 12);
  const int32_t* bW = sec<int32_t>(in, off, 13);
  for (int64_t t = 0; t < H.n_dense; ++t) {
    const int64_t area = toff[t + 1] - toff[t];
    if (tbr[t] < H.br_begin || tbr[t] >= H.br_end || td[t].w < 1 || area < 0 || area % td[t].w)
      return "tiles";
    const int64_t la = tbr[t] - H.br_begin, h = area / td[t].w;
    const int64_t Wp = ((int64_t)bW[la] + vec - 1) / vec * vec;
    if (td[t].cs < 0 || (int64_t)td[t].cs + td[t].w > bW[la] || pbase[la] < 0 ||
        pbase[la] + h * Wp > H.pv_elems)
      return "tiles";
  }
  return "";
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
  DeviceGuard g(h->device);
  cudaError_t e = g.err;
  if (!e) e = cudaDeviceSynchronize();
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
  if (memcmp(H.magic, kMagic, 8) != 0) return fail(SABLE_E_FORMAT, "sable_deserialize: not a SABLEVC3 image");
  if (H.abi_version != SABLE_ABI_VERSION || H.header_bytes != (int32_t)sizeof(ImageHeader) ||
      H.sizeof_unit != (int32_t)sizeof(Unit) || H.sizeof_xgu != (int32_t)sizeof(XgU) ||
      H.sizeof_tiledesc != (int32_t)sizeof(TileDesc) || H.sizeof_cfg != (int32_t)sizeof(ExecCfg) ||
      H.n_sections != kSections)
    return fail(SABLE_E_FORMAT, "sable_deserialize: image written by another library version");
  if ((H.dtype != SABLE_F32 && H.dtype != SABLE_F64) || H.world < 1 || H.rank < 0 ||
      H.rank >= H.world || H.nbr < 1 || H.nbc < 1 || H.br_begin < 0 || H.br_end < H.br_begin ||
      H.br_end > H.nbr || H.row_begin < 0 || H.row_end < H.row_begin || H.row_end > H.nrows ||
      H.nrows < 1 || H.ncols < 1 || H.nrows >= (1ll << 31) - 1 || H.ncols >= (1ll << 31) - 1)
    return fail(SABLE_E_FORMAT, "sable_deserialize: inconsistent header");
  if (H.cfg.pf < 0 || H.cfg.pf > 1 || H.cfg.ustage < 1024 || H.cfg.ustage % 16 != 0 ||
      H.cfg.ustage > (1 << 24) || H.cfg.rem_rows < 1 || H.cfg.rem_rows > 32 || H.cfg.batch < 1 ||
      H.cfg.batch_bytes < 1 || H.cfg.lpr_mode < 0 || H.cfg.lpr_mode > 1)
    return fail(SABLE_E_FORMAT, "sable_deserialize: executor configuration out of range");
  {
    const int64_t lim = (int64_t)1 << 40;  // bounds every count so that byte sizes cannot wrap
    const int64_t cnt[] = {H.nrows,  H.ncols,  H.tile_elems, H.n_dense, H.n_units, H.n_ubatch,
                           H.n_xq,   H.n_xside, H.n_uxg,     H.uscratch_slots, H.pv_elems,
                           H.rem_nnz, H.n_cells, (int64_t)H.nbr, (int64_t)H.world};
    for (int64_t c : cnt)
      if (c < 0 || c > lim) return fail(SABLE_E_FORMAT, "sable_deserialize: count out of range");
    if (H.rem_nnz >= (1ll << 31) || H.n_units >= (1ll << 31) || H.n_xq >= (1ll << 31))
      return fail(SABLE_E_FORMAT, "sable_deserialize: count out of range");
  }
  sable_handle* h = new (std::nothrow) sable_handle();
  if (!h) return fail(SABLE_E_OOM, "host allocation failed");
  load_header(H, h);
  cudaGetDevice(&h->device);
  // the expected section sizes follow from the scalars: check before reading
  h->all_bounds_h = (int32_t*)malloc(sizeof(int32_t) * ((size_t)H.world + 1));
  h->rpntr_h = (int32_t*)malloc(sizeof(int32_t) * ((size_t)H.nbr + 1));
  h->slice_batch.assign(kSlices + 1, 0);
  h->slice_row.assign(kSlices + 1, 0);
  if (!h->all_bounds_h || !h->rpntr_h) {
    free_handle(h);
    return fail(SABLE_E_OOM, "host allocation failed");
  }
  std::vector<Section> S = sections(h);
  std::vector<int64_t> offs(kSections);
  int64_t total = (int64_t)sizeof(ImageHeader);
  for (int i = 0; i < kSections; ++i) {
    if (S[i].bytes < 0 || S[i].bytes != H.section_bytes[i]) {
      free_handle(h);
      return fail(SABLE_E_FORMAT, "sable_deserialize: section " + std::to_string(i) +
                                      " size disagrees with the header");
    }
    offs[i] = total;
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
  const std::string bad = check_image(H, in, offs);
  if (!bad.empty()) {
    free_handle(h);
    return fail(SABLE_E_FORMAT, "sable_deserialize: inconsistent " + bad);
  }
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int64_t sv = H.dtype == SABLE_F64 ? 8 : 4;
  cudaError_t e = cudaSuccess;
  auto dal = [&](void** p, int64_t bytes) {
    if (!e) e = cudaMalloc(p, (size_t)std::max<int64_t>(bytes, 1) + 16);
  };
  // device arrays in section order (pointers of the fresh handle)
  void** dst[kSections] = {(void**)&h->units,    (void**)&h->ubatch,   (void**)&h->xq,
                           (void**)&h->xside,    (void**)&h->uxg,      &h->pv,
                           (void**)&h->rem_ptr,  (void**)&h->rem_idx,  &h->rem_val,
                           (void**)&h->tiles,    (void**)&h->tile_canon_off,
                           (void**)&h->tile_br,  (void**)&h->br_pbase, (void**)&h->br_W,
                           (void**)&h->cell_br,  (void**)&h->cell_bc,  (void**)&h->cell_cnt,
                           (void**)&h->cell_dense, nullptr,            nullptr,
                           nullptr,              nullptr};
  for (int i = 0; i < kSections; ++i) {
    if (dst[i]) {
      dal(dst[i], S[i].bytes);
      if (!e && S[i].bytes > 0)
        e = cudaMemcpyAsync(*dst[i], in + offs[i], (size_t)S[i].bytes, cudaMemcpyHostToDevice, st);
    } else if (i == 18) {
      memcpy(h->all_bounds_h, in + offs[i], (size_t)S[i].bytes);
    } else if (i == 19) {
      memcpy(h->rpntr_h, in + offs[i], (size_t)S[i].bytes);
    } else if (i == 20) {
      memcpy(h->slice_batch.data(), in + offs[i], (size_t)S[i].bytes);
    } else if (i == 21) {
      memcpy(h->slice_row.data(), in + offs[i], (size_t)S[i].bytes);
    }
  }
  // scratch and arrival counters (the executor leaves counters at zero)
  dal(&h->uscratch, sv * h->uscratch_slots);
  dal((void**)&h->ucounters, 4 * h->n_uxg);
  if (!e) e = cudaMemsetAsync(h->ucounters, 0, 4 * (size_t)std::max<int64_t>(h->n_uxg, 1), st);
  if (!e) e = cudaStreamSynchronize(st);  // the host image may be released on return
  if (!e)
    e = upload_batch_heads(h, reinterpret_cast<const Unit*>(in + offs[0]),
                           reinterpret_cast<const int32_t*>(in + offs[1]), st);
  if (e) {
    set_error(cuda_msg(e, "sable_deserialize"));
    cudaStreamSynchronize(st);
    free_handle(h);
    return e == cudaErrorMemoryAllocation ? SABLE_E_OOM : SABLE_E_CUDA;
  }
  *out = h;
  return SABLE_OK;
}
