// plan.cu -- a5 plan for the unit executor (unit.cu): row-major panels,
// x maps, units, combine groups and warp batches.
//
// Everything here depends on the local block rows alone -- each block row is
// planned by itself with fixed budgets -- so a row's units (and with them
// its summation order) are the same whatever the shard count (north_star
// s7; reading R12).  Parallelism follows the paper's block-row granularity
// (PAPER.md:747): a unit never crosses a block row that has dense tiles.
//
// Every unit's data (dense rows, x map, remainder row pointers, columns and
// values, each as its 16-byte-aligned cover) is capped at UnitBudget::stage
// bytes (32 KB by default), so units stay comparable in size and long rows
// or very wide panels are split into pieces.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <utility>
#include <vector>

#include "sable_internal.cuh"

namespace sable {

namespace {

struct PanelDesc {  // per local block row with dense tiles, for the packer
  int64_t vb;       // base of its row-group slabs in tval
  int64_t pb;       // base of its row-major panel in pv
  int32_t W, h;
};

// pv[pb + r * Wp + f] = tval[panel_pos(vb, W, h, 0, r, f)] (0 for f >= W).
template <typename T>
__global__ void k_pack_panels(const PanelDesc* pd, const T* tval, int vec, T* pv) {
  const PanelDesc d = pd[blockIdx.x];
  const int64_t Wp = (d.W + vec - 1) / vec * vec;
  const int64_t n = Wp * d.h;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t r = i / Wp, f = i % Wp;
    pv[d.pb + i] = f < d.W ? tval[panel_pos(d.vb, d.W, d.h, 0, r, f)] : T(0);
  }
}

// Upper bound of the 16-byte-aligned cover of `bytes` bytes.
constexpr int64_t cover(int64_t bytes) { return bytes > 0 ? bytes + 32 : 0; }

}  // namespace

// The first unit's descriptor of every warp batch, so a CTA starts its batch
// with loads that depend only on its batch index (unit.cu).
cudaError_t upload_batch_heads(sable_handle* h, const Unit* U, const int32_t* batch,
                               cudaStream_t st) {
  std::vector<Unit> head((size_t)std::max<int64_t>(h->n_ubatch, 1));
  for (int64_t b = 0; b < h->n_ubatch; ++b) head[(size_t)b] = U[batch[b]];
  if (h->ubhead) cudaFree(h->ubhead);
  h->ubhead = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&h->ubhead), sizeof(Unit) * head.size());
  if (!e) e = cudaMemcpyAsync(h->ubhead, head.data(), sizeof(Unit) * head.size(),
                              cudaMemcpyHostToDevice, st);
  if (!e) e = cudaStreamSynchronize(st);
  return e;
}

// Plan budgets (from the executor configuration, inspect.cu exec_config).
struct UnitBudget {
  int64_t stage;        // cap on one unit's bytes (its data's aligned covers)
  int64_t rem_rows;     // rows per remainder-only unit (<= 32)
  int64_t batch_units;  // max units per warp batch
  int64_t batch_bytes;  // a batch closes once its units hold this many bytes
};

UnitBudget unit_budget(const ExecCfg& c) {
  UnitBudget b;
  b.stage = c.ustage;
  b.rem_rows = c.rem_rows;
  b.batch_units = c.batch;
  b.batch_bytes = c.batch_bytes;
  return b;
}

// Lanes per row for a panel of wq column vectors: mode 0 -- the smallest
// power of two covering the panel in one pass; mode 1 -- the largest power of
// two not above wq (every lane busy, several passes over the columns, more
// rows per unit); both capped at 32.
int choose_llpr(int64_t wq, int mode) {
  int l = 0;
  if (mode == 1) {
    while (l < 5 && (2ll << l) <= wq) ++l;
  } else {
    while (l < 5 && (1ll << l) < wq) ++l;
  }
  return l;
}

template <typename T>
cudaError_t plan_units(sable_handle* h, const T* tval, int32_t nbl, int32_t b0,
                       const std::vector<int32_t>& H_rpntr, const std::vector<int32_t>& H_W,
                       const std::vector<int64_t>& br_vbase, const std::vector<int64_t>& br_wprefix,
                       const std::vector<int64_t>& br_t0, const std::vector<int32_t>& H_rp,
                       const std::vector<XTile>& H_xt, std::vector<int64_t>& br_pbase,
                       cudaStream_t st) {
  const int64_t sv = sizeof(T), vec = 16 / sv, ent = 4 + sv;
  const UnitBudget B = unit_budget(h->cfg);
  br_pbase.assign((size_t)nbl + 1, 0);
  const int64_t S = B.stage;
  auto rp_bytes = [](int64_t nr) { return cover((nr + 1) * 4); };
  auto rem_cap = [&](int64_t nr) {  // entries of a remainder-only unit of nr rows
    return std::max<int64_t>(1, (S - rp_bytes(nr) - 64) / ent);
  };
  std::vector<Unit> U;
  std::vector<XMap> xq;        // x map, one entry per column vector
  std::vector<int32_t> xside;  // 4 columns per straddling column vector
  std::vector<XgU> xg;
  std::vector<PanelDesc> pd;
  U.reserve(H_rp.size() / 16 + (size_t)nbl + 1);
  int64_t pb = 0, slot = 0;

  // A row range's pieces: dense chunks first, then remainder chunks.  One
  // piece writes y itself; several meet in a combine group (in piece order).
  std::vector<Unit> pieces;
  auto flush = [&]() {
    if (pieces.size() == 1) {
      pieces[0].xg = -1;
      U.push_back(pieces[0]);
    } else if (pieces.size() > 1) {
      const int32_t g = (int32_t)xg.size();
      xg.push_back(XgU{slot, g, (int32_t)pieces.size()});
      slot += (int64_t)pieces.size() * 32;
      for (size_t p = 0; p < pieces.size(); ++p) {
        pieces[p].xg = g;
        pieces[p].piece = (uint16_t)p;
        U.push_back(pieces[p]);
      }
    }
    pieces.clear();
  };
  // remainder entries [e, e1) of rows [g0, g1) in chunks of `cap`
  auto rem_pieces = [&](int32_t g0, int32_t g1, int64_t e, int64_t e1, int64_t cap) {
    for (; e < e1; e += cap) {
      Unit u{};
      u.row0 = g0;
      u.nr = (uint8_t)(g1 - g0);
      u.e0 = (int32_t)e;
      u.e1 = (int32_t)std::min(e1, e + cap);
      pieces.push_back(u);
    }
  };

  // consecutive rows without tiles: groups of <= rem_rows rows whose entries
  // fit a stage; a row longer than that is a group of its own (in pieces)
  auto emit_rem_rows = [&](int32_t r0, int32_t r1) {
    int32_t g0 = r0;
    while (g0 < r1) {
      int32_t g1 = g0 + 1;
      while (g1 < r1 && g1 - g0 < B.rem_rows &&
             (int64_t)H_rp[g1 + 1] - H_rp[g0] <= rem_cap(g1 + 1 - g0))
        ++g1;
      const int64_t e0 = H_rp[g0], e1 = H_rp[g1];
      if (e1 == e0) {
        Unit u{};
        u.row0 = g0;
        u.nr = (uint8_t)(g1 - g0);
        u.e0 = u.e1 = (int32_t)e0;
        pieces.push_back(u);
      } else {
        rem_pieces(g0, g1, e0, e1, rem_cap(g1 - g0));
      }
      flush();
      g0 = g1;
    }
  };

  int32_t pend = -1;  // first row of a pending run of rows without tiles
  for (int32_t la = 0; la < nbl; ++la) {
    const int32_t a = b0 + la;
    const int32_t hgt = H_rpntr[a + 1] - H_rpntr[a];
    const int32_t r0 = (int32_t)(H_rpntr[a] - h->row_begin);
    const int32_t W = H_W[a];
    br_pbase[la] = pb;
    if (W == 0) {
      if (pend < 0) pend = r0;
      continue;
    }
    if (pend >= 0) {
      emit_rem_rows(pend, r0);
      pend = -1;
    }
    // x runs of the block row (adjacent tiles whose panel and global columns
    // advance together merge), then its x map: per column vector q, the
    // global column of its first column when all its columns lie in one run
    // (or are padding past W, whose values are zero), else a side entry with
    // the global column of each (padding columns repeat a valid one)
    std::vector<std::pair<int32_t, int32_t>> R;  // (tp, c0)
    for (int64_t t = br_t0[la]; t < br_t0[la + 1]; ++t) {
      const int32_t tp = (int32_t)(H_xt[t].tp - br_wprefix[la]);
      const int32_t c0 = H_xt[t].c0;
      if (!R.empty() && c0 - tp == R.back().second - R.back().first) continue;
      R.push_back({tp, c0});
    }
    const int64_t wq = (W + vec - 1) / vec, Wp = wq * vec;
    const int32_t xq0 = (int32_t)xq.size();
    {
      size_t k = 0;
      auto col = [&](int64_t f, size_t& kk) {  // global column of panel column f < W
        while (kk + 1 < R.size() && R[kk + 1].first <= f) ++kk;
        return (int32_t)(R[kk].second + (f - R[kk].first));
      };
      // every column index an entry yields is in [0, ncols) (no clamp on the
      // device): padding columns past W (zero values) continue the last run
      // when that stays inside the matrix, else read columns 0, 1, ...
      const int64_t ncols = h->ncols;
      auto encode = [&](const int64_t* cc) -> bool {
        for (int64_t i = 0; i < vec; ++i)
          if (cc[i] < 0 || cc[i] >= ncols) return false;
        for (int64_t kk = 0; kk < vec; ++kk) {  // kk = 0: one run; else split before kk
          bool ok = true;
          for (int64_t i = 0; i < vec && ok; ++i)
            ok = i < kk || kk == 0 ? cc[i] == cc[0] + i : cc[i] == cc[kk] + (i - kk);
          const int64_t d = kk == 0 ? 0 : cc[kk] - (cc[0] + kk);
          if (ok && d >= -(1ll << 29) && d < (1ll << 29)) {
            xq.push_back(XMap{(int32_t)cc[0], (int32_t)(d * 4 + kk)});
            return true;
          }
        }
        return false;
      };
      for (int64_t q = 0; q < wq; ++q) {
        const int64_t f0 = q * vec;
        int64_t cc[4], last = 0;
        size_t k2 = k;
        for (int64_t i = 0; i < vec; ++i) {
          if (f0 + i < W) {
            last = col(f0 + i, k2);
            cc[i] = last;
          } else {
            cc[i] = last + (f0 + i - (W - 1));
          }
        }
        col(f0, k);  // advance the run cursor
        if (encode(cc)) continue;
        if (f0 + vec > W) {
          for (int64_t i = 0; i < vec; ++i)
            if (f0 + i >= W) cc[i] = f0 + i - W;
          if (encode(cc)) continue;
        }
        // three or more runs (or no encodable padding): the side table
        xq.push_back(XMap{~(int32_t)(xside.size() / 4), 0});
        for (int64_t i = 0; i < 4; ++i) {
          if (i < vec && f0 + i < W) last = cc[i];
          xside.push_back((int32_t)last);
        }
      }
    }
    pd.push_back(PanelDesc{br_vbase[la], pb, W, hgt});
    const int64_t vbase = pb / vec;  // panel base in 16-byte vectors
    const int64_t row_b = wq * 16;
    const int64_t xm_b = cover(wq * (int64_t)sizeof(XMap));
    if (row_b + xm_b + rp_bytes(1) + 64 + ent <= S) {
      // row groups: as many rows as the lanes' accumulators and a stage hold
      const int llpr = choose_llpr(wq, h->cfg.lpr_mode);
      const int64_t L = 1ll << llpr;
      const int64_t ru = std::min<int64_t>(32, (32 / L) * std::min<int64_t>(L, 8));
      const int64_t rs = std::max<int64_t>(1, (S - xm_b - rp_bytes(32) - 64 - ent) / row_b);
      const int64_t per = std::min(ru, rs);
      const int64_t ng = (hgt + per - 1) / per;
      int64_t g0 = 0;
      for (int64_t g = 0; g < ng; ++g) {
        const int64_t nr = hgt / ng + (g < hgt % ng ? 1 : 0);
        const int32_t a0 = r0 + (int32_t)g0, a1 = a0 + (int32_t)nr;
        Unit u{};
        u.row0 = a0;
        u.nr = (uint8_t)nr;
        u.wq = (int32_t)wq;
        u.xq0 = xq0;
        u.voff16 = (int32_t)(vbase + g0 * wq);
        u.llpr = (uint8_t)llpr;
        const int64_t e0 = H_rp[a0], e1 = H_rp[a1];
        const int64_t room = S - nr * row_b - xm_b - rp_bytes(nr) - 64;
        const int64_t k0 = std::min<int64_t>(e1 - e0, std::max<int64_t>(0, room / ent));
        u.e0 = (int32_t)e0;
        u.e1 = (int32_t)(e0 + k0);
        pieces.push_back(u);
        rem_pieces(a0, a1, e0 + k0, e1, rem_cap(nr));
        flush();
        g0 += nr;
      }
    } else {
      // a panel wider than a stage: every row in column chunks
      const int64_t cq = std::max<int64_t>(1, (S - rp_bytes(1) - 64 - 64) / 20);
      for (int32_t r = 0; r < hgt; ++r) {
        for (int64_t qa = 0; qa < wq; qa += cq) {
          const int64_t n = std::min(cq, wq - qa);
          Unit u{};
          u.row0 = r0 + r;
          u.nr = 1;
          u.wq = (int32_t)n;
          u.xq0 = xq0 + (int32_t)qa;
          u.voff16 = (int32_t)(vbase + (int64_t)r * wq + qa);
          u.llpr = (uint8_t)choose_llpr(n, h->cfg.lpr_mode);
          u.e0 = u.e1 = H_rp[r0 + r];
          pieces.push_back(u);
        }
        rem_pieces(r0 + r, r0 + r + 1, H_rp[r0 + r], H_rp[r0 + r + 1], rem_cap(1));
        flush();
      }
    }
    pb += Wp * hgt;
  }
  const int64_t nloc = (int64_t)H_rp.size() - 1;
  if (pend >= 0) emit_rem_rows(pend, (int32_t)nloc);
  br_pbase[nbl] = pb;
  if (pb / vec > INT32_MAX || (int64_t)xq.size() > INT32_MAX || (int64_t)U.size() > INT32_MAX) {
    set_error("unit plan exceeds 2^31 vectors, x map entries or units");
    return cudaErrorInvalidValue;
  }

  // exchange slices: kSlices runs of consecutive units of about equal bytes,
  // cut only where a row range starts (never inside a combine group), so a
  // slice's rows are final when its launch ends (comm.cu overlaps their
  // all-gather with the next slice); then warp batches of batch_units
  // consecutive units inside each slice
  std::vector<int64_t> ucut(1, 0);
  {
    int64_t tot = 0;
    for (const Unit& u : U) tot += (int64_t)u.nr * u.wq * 16 + (int64_t)(u.e1 - u.e0) * ent + 64;
    int64_t acc = 0;
    for (size_t i = 0; i < U.size(); ++i) {
      const int s = (int)ucut.size();  // next boundary index
      const bool starts = U[i].xg < 0 || U[i].piece == 0;
      if (s < kSlices && starts && i > 0 && acc * kSlices >= tot * s) ucut.push_back((int64_t)i);
      acc += (int64_t)U[i].nr * U[i].wq * 16 + (int64_t)(U[i].e1 - U[i].e0) * ent + 64;
    }
    while ((int)ucut.size() < kSlices + 1) ucut.push_back((int64_t)U.size());
  }
  // units per batch: at most batch_units, fewer when the shard has too few
  // units to give every resident warp slot (SMs x 32) about two batches
  int64_t bu = B.batch_units;
  {
    int nsm = 148;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess)
      nsm = 148;
    const int64_t slots = 2ll * nsm * 32;
    bu = std::max<int64_t>(1, std::min<int64_t>(bu, (int64_t)U.size() / slots));
  }
  std::vector<int32_t> batch;
  h->slice_batch.assign(kSlices + 1, 0);
  h->slice_row.assign(kSlices + 1, 0);
  for (int s = 0; s < kSlices; ++s) {
    h->slice_batch[s] = (int64_t)batch.size();
    h->slice_row[s] = ucut[s] < (int64_t)U.size() ? U[ucut[s]].row0 : nloc;
    // a batch closes at batch_units units or batch_bytes bytes, whichever
    // comes first, so batches are comparable in work and the CTA scheduler
    // balances them dynamically
    int64_t nb = 0, bb = 0;
    for (int64_t i = ucut[s]; i < ucut[s + 1]; ++i) {
      if (nb == 0) batch.push_back((int32_t)i);
      bb += (int64_t)U[i].nr * U[i].wq * 16 + (int64_t)(U[i].e1 - U[i].e0) * ent + 64;
      if (++nb >= bu || bb >= B.batch_bytes) nb = bb = 0;
    }
  }
  h->slice_batch[kSlices] = (int64_t)batch.size();
  h->slice_row[kSlices] = nloc;
  batch.push_back((int32_t)U.size());

  // upload
  cudaError_t e = cudaSuccess;
  h->n_units = (int64_t)U.size();
  h->n_ubatch = (int64_t)batch.size() - 1;
  h->n_xq = (int64_t)xq.size();
  h->n_xside = (int64_t)xside.size() / 4;
  h->n_uxg = (int64_t)xg.size();
  h->pv_elems = pb;
  h->uscratch_slots = slot;
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (e) return;
    e = cudaMalloc(dst, bytes + 16);  // +16 B: the staged executor's 16-byte covers
    if (!e && bytes) e = cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st);
  };
  up(reinterpret_cast<void**>(&h->units), U.data(), sizeof(Unit) * U.size());
  up(reinterpret_cast<void**>(&h->ubatch), batch.data(), sizeof(int32_t) * batch.size());
  up(reinterpret_cast<void**>(&h->xq), xq.data(), sizeof(XMap) * xq.size());
  up(reinterpret_cast<void**>(&h->xside), xside.data(), sizeof(int32_t) * xside.size());
  up(reinterpret_cast<void**>(&h->uxg), xg.data(), sizeof(XgU) * xg.size());
  if (!e) e = cudaMalloc(&h->uscratch, (size_t)std::max<int64_t>(slot, 1) * sv);
  if (!e) e = cudaMalloc(reinterpret_cast<void**>(&h->ucounters),
                         sizeof(int32_t) * std::max<size_t>(xg.size(), 1));
  if (!e) e = cudaMemsetAsync(h->ucounters, 0, sizeof(int32_t) * std::max<size_t>(xg.size(), 1), st);
  if (!e) e = cudaMalloc(&h->pv, (size_t)std::max<int64_t>(pb, 1) * sv + 16);
  PanelDesc* pd_d = nullptr;
  if (!e && !pd.empty()) {
    e = cudaMalloc(reinterpret_cast<void**>(&pd_d), sizeof(PanelDesc) * pd.size());
    if (!e) e = cudaMemcpyAsync(pd_d, pd.data(), sizeof(PanelDesc) * pd.size(), cudaMemcpyHostToDevice, st);
    if (!e) {
      k_pack_panels<T><<<(unsigned)pd.size(), 256, 0, st>>>(pd_d, tval,
                                                           (int)vec, static_cast<T*>(h->pv));
      e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(st);
  }
  if (pd_d) cudaFree(pd_d);
  if (!e) e = cudaStreamSynchronize(st);
  if (!e) e = upload_batch_heads(h, U.data(), batch.data(), st);
  return e;
}

#define SABLE_PLAN_INST(T)                                                                  \
  template cudaError_t plan_units<T>(                                                      \
      sable_handle*, const T*, int32_t, int32_t, const std::vector<int32_t>&,              \
      const std::vector<int32_t>&, const std::vector<int64_t>&, const std::vector<int64_t>&, \
      const std::vector<int64_t>&, const std::vector<int32_t>&, const std::vector<XTile>&,  \
      std::vector<int64_t>&, cudaStream_t);
SABLE_PLAN_INST(float)
SABLE_PLAN_INST(double)

}  // namespace sable
