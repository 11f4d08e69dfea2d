// plan.cu -- a5 plan for the unit executor (unit.cu): row-major panels,
// x runs, units, combine groups and warp batches.
//
// Everything here depends on the local block rows alone -- each block row is
// planned by itself with fixed budgets -- so a row's units (and with them
// its summation order) are the same whatever the shard count (north_star
// s7; reading R12).  Parallelism follows the paper's block-row granularity
// (PAPER.md:747): a unit never crosses a block row that has dense tiles.
#include <algorithm>
#include <climits>
#include <utility>
#include <cstdlib>
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

int64_t env_i64(const char* name, int64_t dflt) {
  const char* s = getenv(name);
  return s && *s ? atoll(s) : dflt;
}

}  // namespace

// Plan budgets (SABLE_U* environment overrides are for tuning runs only).
struct UnitBudget {
  int64_t dense_bytes;  // cap on one unit's dense values
  int64_t piece_ent;    // remainder entries per unit in a split row range
  int64_t rem_ent;      // remainder entries per remainder-only unit
  int64_t batch_bytes;  // a warp takes consecutive units up to this many bytes
  int64_t batch_units;  // ... and at most this many units
  int64_t unit_cost;    // fixed cost of a unit in lane steps (for the LPR choice)
};

UnitBudget unit_budget() {
  UnitBudget b;
  b.dense_bytes = env_i64("SABLE_UDENSE", 32768);
  b.piece_ent = env_i64("SABLE_UPIECE", 2048);
  b.rem_ent = env_i64("SABLE_UREM", 512);
  b.batch_bytes = env_i64("SABLE_UBATCH", 16384);
  b.batch_units = env_i64("SABLE_UBATCH_UNITS", 4);
  b.unit_cost = env_i64("SABLE_UCOST", 4);
  return b;
}

// Lanes per row for a panel of Wq column vectors: the smallest power of two
// covering the panel in one pass, capped at 32 -- every lane then issues all
// its rows' loads of a pass at once (the executor is latency-bound per unit,
// so fewer serial passes beat fuller lanes).  SABLE_ULPR_MODE=1 picks the
// fewest lane steps instead (A/B).
int choose_llpr(int64_t Wq, int64_t h, const UnitBudget& B) {
  if (env_i64("SABLE_ULPR_MODE", 0) == 0) {
    int l = 0;
    while (l < 5 && (1ll << l) < Wq) ++l;
    return l;
  }
  int best = 5;
  int64_t best_cost = INT64_MAX;
  for (int l = 5; l >= 0; --l) {
    const int64_t L = 1ll << l, sub = 32 / L, K = std::min<int64_t>(L, 8);
    const int64_t ru = std::min<int64_t>(32, sub * K);
    const int64_t ng = (h + ru - 1) / ru;
    int64_t cost = 0;
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t nr = h / ng + (g < h % ng ? 1 : 0);
      cost += ((Wq + L - 1) / L) * ((nr + sub - 1) / sub) + B.unit_cost;
    }
    if (cost < best_cost) {
      best_cost = cost;
      best = l;
    }
  }
  return best;
}

template <typename T>
cudaError_t plan_units(sable_handle* h, int32_t nbl, int32_t b0, const std::vector<int32_t>& H_rpntr,
                       const std::vector<int32_t>& H_W, const std::vector<int64_t>& br_vbase,
                       const std::vector<int64_t>& br_wprefix, const std::vector<int64_t>& br_t0,
                       const std::vector<int32_t>& H_rp, const std::vector<XTile>& H_xt,
                       cudaStream_t st) {
  const int64_t sv = sizeof(T), vec = 16 / sv;
  const UnitBudget B = unit_budget();
  std::vector<Unit> U;
  std::vector<int32_t> xq;       // x map, one entry per column vector
  std::vector<int32_t> xside;    // 4 columns per straddling column vector
  std::vector<XgU> xg;
  std::vector<PanelDesc> pd;
  U.reserve(H_rp.size() / 16 + (size_t)nbl + 1);
  int64_t pb = 0, slot = 0;

  // one row range [g0, g1) (local rows) with its dense part, split into
  // pieces when its remainder is longer than a piece
  auto emit = [&](int32_t g0, int32_t g1, int32_t wq, int32_t xq0, int64_t voff, int llpr) {
    const int64_t e0 = H_rp[g0], e1 = H_rp[g1];
    const int64_t cap = wq > 0 ? B.piece_ent : std::max(B.piece_ent, B.rem_ent);
    Unit u{};
    u.row0 = g0;
    u.nr = (uint8_t)(g1 - g0);
    u.wq = wq;
    u.xq0 = xq0;
    u.voff16 = (int32_t)(voff / vec);
    u.llpr = (uint8_t)llpr;
    u.xg = -1;
    if (e1 - e0 <= cap) {
      u.e0 = (int32_t)e0;
      u.e1 = (int32_t)e1;
      U.push_back(u);
      return;
    }
    const int64_t np = (e1 - e0 + cap - 1) / cap;
    const int32_t g = (int32_t)xg.size();
    xg.push_back(XgU{slot, g, (int32_t)np});
    slot += np * 32;
    for (int64_t p = 0; p < np; ++p) {
      Unit v = u;
      v.e0 = (int32_t)(e0 + p * cap);
      v.e1 = (int32_t)std::min(e1, e0 + (p + 1) * cap);
      v.xg = g;
      v.piece = (uint16_t)p;
      if (p > 0) v.wq = 0;  // the dense part rides on piece 0
      U.push_back(v);
    }
  };

  // consecutive rows without tiles: groups of <= 32 rows and <= rem_ent
  // entries; a row longer than that is a group of its own (split in pieces)
  auto emit_rem_rows = [&](int32_t r0, int32_t r1) {
    int32_t g0 = r0;
    while (g0 < r1) {
      int32_t g1 = g0 + 1;
      while (g1 < r1 && g1 - g0 < 32 && (int64_t)H_rp[g1 + 1] - H_rp[g0] <= B.rem_ent) ++g1;
      emit(g0, g1, 0, 0, 0, 0);
      g0 = g1;
    }
  };

  int32_t pend = -1;  // first row of a pending run of rows without tiles
  for (int32_t la = 0; la < nbl; ++la) {
    const int32_t a = b0 + la;
    const int32_t hgt = H_rpntr[a + 1] - H_rpntr[a];
    const int32_t r0 = (int32_t)(H_rpntr[a] - h->row_begin);
    const int32_t W = H_W[a];
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
    const int64_t Wq = (W + vec - 1) / vec, Wp = Wq * vec;
    const int32_t xq0 = (int32_t)xq.size();
    {
      size_t k = 0;
      auto col = [&](int64_t f, size_t& kk) {  // global column of panel column f < W
        while (kk + 1 < R.size() && R[kk + 1].first <= f) ++kk;
        return (int32_t)(R[kk].second + (f - R[kk].first));
      };
      for (int64_t q = 0; q < Wq; ++q) {
        const int64_t f0 = q * vec;
        const int32_t c = col(f0, k);
        const int64_t run_end = k + 1 < R.size() ? R[k + 1].first : W;
        if (f0 + vec <= run_end || run_end == W) {
          xq.push_back(c);
        } else {
          xq.push_back(~(int32_t)(xside.size() / 4));
          size_t k2 = k;
          int32_t last = c;
          for (int64_t i = 0; i < 4; ++i) {
            if (i < vec && f0 + i < W) last = col(f0 + i, k2);
            xside.push_back(last);
          }
        }
      }
    }
    pd.push_back(PanelDesc{br_vbase[la], pb, W, hgt});
    const int llpr = choose_llpr(Wq, hgt, B);
    const int64_t L = 1ll << llpr;
    const int64_t ru = std::min<int64_t>(32, (32 / L) * std::min<int64_t>(L, 8));
    const int64_t rb = std::max<int64_t>(1, B.dense_bytes / (Wp * sv));
    const int64_t per = std::min(ru, rb);
    const int64_t ng = (hgt + per - 1) / per;
    int64_t g0 = 0;
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t nr = hgt / ng + (g < hgt % ng ? 1 : 0);
      emit(r0 + (int32_t)g0, r0 + (int32_t)(g0 + nr), (int32_t)Wq, xq0, pb + g0 * Wp, llpr);
      g0 += nr;
    }
    pb += Wp * hgt;
  }
  const int64_t nloc = (int64_t)H_rp.size() - 1;
  if (pend >= 0) emit_rem_rows(pend, (int32_t)nloc);
  if (pb / vec > INT32_MAX) {
    set_error("row-major panels exceed 2^31 16-byte vectors");
    return cudaErrorInvalidValue;
  }

  // warp batches: consecutive units up to batch_bytes (at least one unit)
  std::vector<int32_t> batch;
  batch.push_back(0);
  {
    int64_t acc = 0, cnt = 0;
    for (size_t i = 0; i < U.size(); ++i) {
      const Unit& u = U[i];
      acc += (int64_t)u.wq * 16 * u.nr + (int64_t)(u.e1 - u.e0) * (sv + 4) + 64;
      ++cnt;
      if (acc >= B.batch_bytes || cnt >= B.batch_units || i + 1 == U.size()) {
        batch.push_back((int32_t)(i + 1));
        acc = 0;
        cnt = 0;
      }
    }
  }

  // upload
  cudaError_t e = cudaSuccess;
  h->n_units = (int64_t)U.size();
  h->n_ubatch = (int64_t)batch.size() - 1;
  h->n_xq = (int64_t)xq.size();
  h->n_xside = (int64_t)xside.size() / 4;
  h->n_uxg = (int64_t)xg.size();
  h->pv_elems = pb;
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (e) return;
    e = cudaMalloc(dst, bytes ? bytes : 16);
    if (!e && bytes) e = cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st);
  };
  up(reinterpret_cast<void**>(&h->units), U.data(), sizeof(Unit) * U.size());
  up(reinterpret_cast<void**>(&h->ubatch), batch.data(), sizeof(int32_t) * batch.size());
  up(reinterpret_cast<void**>(&h->xq), xq.data(), sizeof(int32_t) * xq.size());
  up(reinterpret_cast<void**>(&h->xside), xside.data(), sizeof(int32_t) * xside.size());
  up(reinterpret_cast<void**>(&h->uxg), xg.data(), sizeof(XgU) * xg.size());
  if (!e) e = cudaMalloc(&h->uscratch, (size_t)std::max<int64_t>(slot, 1) * sv);
  if (!e) e = cudaMalloc(reinterpret_cast<void**>(&h->ucounters),
                         sizeof(int32_t) * std::max<size_t>(xg.size(), 1));
  if (!e) e = cudaMemsetAsync(h->ucounters, 0, sizeof(int32_t) * std::max<size_t>(xg.size(), 1), st);
  if (!e) e = cudaMalloc(&h->pv, (size_t)std::max<int64_t>(pb, 1) * sv);
  PanelDesc* pd_d = nullptr;
  if (!e && !pd.empty()) {
    e = cudaMalloc(reinterpret_cast<void**>(&pd_d), sizeof(PanelDesc) * pd.size());
    if (!e) e = cudaMemcpyAsync(pd_d, pd.data(), sizeof(PanelDesc) * pd.size(), cudaMemcpyHostToDevice, st);
    if (!e) {
      k_pack_panels<T><<<(unsigned)pd.size(), 256, 0, st>>>(pd_d, static_cast<const T*>(h->tval),
                                                           (int)vec, static_cast<T*>(h->pv));
      e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(st);
  }
  if (pd_d) cudaFree(pd_d);
  if (!e) e = cudaStreamSynchronize(st);
  return e;
}

template cudaError_t plan_units<float>(sable_handle*, int32_t, int32_t, const std::vector<int32_t>&,
                                       const std::vector<int32_t>&, const std::vector<int64_t>&,
                                       const std::vector<int64_t>&, const std::vector<int64_t>&,
                                       const std::vector<int32_t>&, const std::vector<XTile>&,
                                       cudaStream_t);
template cudaError_t plan_units<double>(sable_handle*, int32_t, int32_t, const std::vector<int32_t>&,
                                        const std::vector<int32_t>&, const std::vector<int64_t>&,
                                        const std::vector<int64_t>&, const std::vector<int64_t>&,
                                        const std::vector<int32_t>&, const std::vector<XTile>&,
                                        cudaStream_t);

}  // namespace sable
