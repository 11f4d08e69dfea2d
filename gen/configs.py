"""Seeded synthetic workloads C1..C5 (BASELINE.json configs[0..4]).

The recipes follow SURVEY.md 8(d) (restated in DESIGN.md "Inputs"); every
parameter the config text leaves open is fixed here and marked "(inv.)".
The paper measures on SuiteSparse, which is not available;
these synthetic matrices stand in for it, with the block structure the paper
targets (variable blocks on a cut grid plus scattered non-zeros, PAPER.md:81,
99-103, 243-245) and the paper's own synthetic-matrix method of overlaying a
grid and populating blocks at random positions.

Random numbers come from counter-based Philox streams keyed by
(seed, stream id), so every array is reproducible on any host.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .encode import encode_vbr

# stream ids
PLACE, FILL, SCATTER, VALUES, XSTREAM, EXTRA = 1, 2, 3, 4, 5, 6


def rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))


def log_uniform_int(g: np.random.Generator, lo: int, hi: int, size) -> np.ndarray:
    """floor(exp(U(ln lo, ln(hi+1)))) clipped to [lo, hi]."""
    u = g.uniform(math.log(lo), math.log(hi + 1), size=size)
    return np.clip(np.floor(np.exp(u)).astype(np.int64), lo, hi)


@dataclass
class Synth:
    """A synthetic matrix: sorted duplicate-free non-zero COO, its cut grid,
    the placed rectangles, x, delta, and the GPU input split."""
    name: str
    nrows: int
    ncols: int
    dtype: type
    delta: int
    rpntr: np.ndarray
    cpntr: np.ndarray
    rects: np.ndarray  # (R, 4): r0, c0, h, w
    I: np.ndarray
    J: np.ndarray
    V: np.ndarray
    x: np.ndarray
    in_rect: np.ndarray  # bool per triple: inside a placed rectangle's cells
    iterations: int = 1
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(len(self.I))

    def vbr_input(self, split: str = "rect") -> dict:
        """VBR + remainder arrays for the C-ABI (split: rect | all_vbr | all_rem)."""
        if split == "rect":
            mask = self.in_rect
        elif split == "all_vbr":
            mask = np.ones(self.nnz, dtype=bool)
        elif split == "all_rem":
            mask = np.zeros(self.nnz, dtype=bool)
        else:
            raise ValueError(split)
        d = encode_vbr(self.nrows, self.ncols, self.rpntr, self.cpntr, self.I, self.J,
                       self.V, mask)
        d["dtype"] = self.dtype
        return d

    def rowptr(self) -> np.ndarray:
        rp = np.zeros(self.nrows + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.I, minlength=self.nrows), out=rp[1:])
        return rp


# ---------------------------------------------------------------------------
# helpers (placement, fill, scatter) -- drawing only, no method arithmetic


class _Occupancy:
    """Bucket grid for non-overlap rejection of rectangles."""

    def __init__(self, bucket: int):
        self.b = bucket
        self.cells: dict = {}

    def _keys(self, r0, c0, h, w):
        b = self.b
        for br in range(r0 // b, (r0 + h - 1) // b + 1):
            for bc in range(c0 // b, (c0 + w - 1) // b + 1):
                yield (br, bc)

    def overlaps(self, r0, c0, h, w) -> bool:
        for k in self._keys(r0, c0, h, w):
            for (a0, b0, hh, ww) in self.cells.get(k, ()):
                if r0 < a0 + hh and a0 < r0 + h and c0 < b0 + ww and b0 < c0 + w:
                    return True
        return False

    def add(self, r0, c0, h, w):
        for k in self._keys(r0, c0, h, w):
            self.cells.setdefault(k, []).append((r0, c0, h, w))


def _place_random(g, n, occ, count, draw_hw, max_tries=10_000_000):
    """Uniform top-left positions, rejected on overlap with earlier rectangles."""
    out = []
    tries = 0
    while len(out) < count:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("rectangle placement did not converge")
        h, w = draw_hw()
        r0 = int(g.integers(0, n - h + 1))
        c0 = int(g.integers(0, n - w + 1))
        if occ.overlaps(r0, c0, h, w):
            continue
        occ.add(r0, c0, h, w)
        out.append((r0, c0, h, w))
    return out


def _fill_rects(g, rects, fills):
    """round(f*h*w) (>= 1) distinct uniform positions in each rectangle."""
    Is, Js = [], []
    for (r0, c0, h, w), f in zip(rects, fills):
        area = h * w
        k = max(1, int(round(f * area)))
        k = min(k, area)
        pos = g.choice(area, size=k, replace=False) if k < area else np.arange(area)
        Is.append(r0 + pos % h)
        Js.append(c0 + pos // h)
    if not Is:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(Is).astype(np.int64), np.concatenate(Js).astype(np.int64)


def _scatter(g, nrows, ncols, count, taken_keys):
    """count uniform positions over the matrix, excluding taken ones
    (taken_keys: sorted unique int64 keys i*ncols + j)."""
    got = np.zeros(0, dtype=np.int64)
    while len(got) < count:
        need = count - len(got)
        draw = g.integers(0, nrows * ncols, size=int(need * 1.05) + 16, dtype=np.int64)
        _, first = np.unique(draw, return_index=True)
        draw = draw[np.sort(first)]  # unique, in draw order
        if len(taken_keys):
            pos = np.searchsorted(taken_keys, draw)
            pos[pos == len(taken_keys)] = 0
            draw = draw[taken_keys[pos] != draw]
        if len(got):
            draw = draw[~np.isin(draw, got)]
        got = np.concatenate([got, draw[:need]])
    return got


def _values(g, kind, size, dtype):
    """Values of the given distribution in dtype, exact zeros redrawn."""
    def draw(m):
        if kind == "u11":
            return g.uniform(-1.0, 1.0, size=m)
        if kind == "n01":
            return g.standard_normal(size=m)
        if kind == "n002":
            return 0.02 * g.standard_normal(size=m)
        if kind == "u01":  # U(0, 1]
            return 1.0 - g.random(size=m)
        raise ValueError(kind)
    v = draw(size).astype(dtype)
    z = np.flatnonzero(v == 0)
    while len(z):
        v[z] = draw(len(z)).astype(dtype)
        z = z[v[z] == 0]
    return v


def _grid_from_rects(n, rects, axis):
    """Union of rectangle boundaries on one axis, with {0, n} (reading R15)."""
    if len(rects) == 0:
        return np.array([0, n], dtype=np.int32)
    r = np.asarray(rects, dtype=np.int64)
    s = r[:, 0] if axis == 0 else r[:, 1]
    e = s + (r[:, 2] if axis == 0 else r[:, 3])
    cuts = np.unique(np.concatenate([[0, n], s, e]))
    return cuts.astype(np.int32)


def _in_rect_cells(I, J, rpntr, cpntr, rects):
    """True where triple (i,j) lies in a placed rectangle (each rectangle is a
    union of whole grid cells because its edges are grid lines)."""
    nbc = len(cpntr) - 1
    if len(rects) == 0:
        return np.zeros(len(I), dtype=bool)
    keys = []
    for (r0, c0, h, w) in rects:
        a0 = np.searchsorted(rpntr, r0)
        a1 = np.searchsorted(rpntr, r0 + h)
        b0 = np.searchsorted(cpntr, c0)
        b1 = np.searchsorted(cpntr, c0 + w)
        aa, bb = np.meshgrid(np.arange(a0, a1, dtype=np.int64),
                             np.arange(b0, b1, dtype=np.int64), indexing="ij")
        keys.append((aa * nbc + bb).ravel())
    keys = np.unique(np.concatenate(keys))
    br = np.searchsorted(rpntr, I, side="right") - 1
    bc = np.searchsorted(cpntr, J, side="right") - 1
    k = br.astype(np.int64) * nbc + bc
    pos = np.searchsorted(keys, k)
    pos[pos == len(keys)] = 0
    return keys[pos] == k


def _finish(name, n, dtype, delta, rects, I, J, V, x, rpntr=None, cpntr=None,
            iterations=1, meta=None):
    """Sort by (i,j), build the grid and the rectangle split."""
    key = I * n + J
    order = np.argsort(key, kind="stable")
    I, J, V = I[order], J[order], V[order]
    if np.any(np.diff(key[order]) == 0):
        raise RuntimeError("generator produced a duplicate position")
    if rpntr is None:
        rpntr = _grid_from_rects(n, rects, 0)
    if cpntr is None:
        cpntr = _grid_from_rects(n, rects, 1)
    in_rect = _in_rect_cells(I, J, rpntr, cpntr, rects)
    return Synth(name=name, nrows=n, ncols=n, dtype=dtype, delta=delta,
                 rpntr=np.asarray(rpntr, np.int32), cpntr=np.asarray(cpntr, np.int32),
                 rects=np.asarray(rects, dtype=np.int64).reshape(-1, 4), I=I, J=J, V=V,
                 x=x, in_rect=in_rect, iterations=iterations, meta=meta or {})


# ---------------------------------------------------------------------------
# C1..C5


def make_c1(seed: int = 1, scale: float = 1.0) -> Synth:
    """BASELINE.json configs[0]: fp32 2000x2000, 12 blocks h,w ~ U{8..64},
    fill U[0.7,1.0], 0.2% scatter, values and x U[-1,1], delta=50."""
    n = 2000
    gp, gf, gs, gv = rng(seed, PLACE), rng(seed, FILL), rng(seed, SCATTER), rng(seed, VALUES)
    occ = _Occupancy(64)
    rects = _place_random(gp, n, occ, 12, lambda: (int(gp.integers(8, 65)), int(gp.integers(8, 65))))
    fills = gf.uniform(0.70, 1.00, size=len(rects))
    I, J = _fill_rects(gf, rects, fills)
    taken = np.unique(I * n + J)
    sc = _scatter(gs, n, n, int(0.002 * n * n), taken)
    I = np.concatenate([I, sc // n])
    J = np.concatenate([J, sc % n])
    V = _values(gv, "u11", len(I), np.float32)
    x = _values(rng(seed + 100, XSTREAM), "u11", n, np.float32)
    return _finish("c1", n, np.float32, 50, rects, I, J, V, x)


def make_c2(seed: int = 2, scale: float = 1.0) -> Synth:
    """configs[1]: fp32 200,000^2 block-diagonal-plus-off-diagonal: 2,500
    diagonal squares + 2,500 off-diagonal rectangles (inv. 50/50), extents
    log-U[4,128], fill U[0.6,1.0], 1e-4 scatter, values and x N(0,1) (inv.)."""
    n = int(200_000 * scale)
    nb = max(2, int(2500 * scale))
    gp, gf, gs, gv = rng(seed, PLACE), rng(seed, FILL), rng(seed, SCATTER), rng(seed, VALUES)
    side = log_uniform_int(gp, 4, 128, nb)
    gap_total = n - int(side.sum())
    assert gap_total >= 0
    cuts = np.sort(gp.integers(0, gap_total + 1, size=nb))
    gaps = np.diff(np.concatenate([[0], cuts]))
    starts = np.cumsum(gaps) + np.concatenate([[0], np.cumsum(side)[:-1]])
    occ = _Occupancy(128)
    rects = []
    for s, st in zip(side, starts):
        rects.append((int(st), int(st), int(s), int(s)))
        occ.add(int(st), int(st), int(s), int(s))
    rects += _place_random(gp, n, occ, nb,
                           lambda: (int(log_uniform_int(gp, 4, 128, 1)[0]),
                                    int(log_uniform_int(gp, 4, 128, 1)[0])))
    fills = gf.uniform(0.6, 1.0, size=len(rects))
    I, J = _fill_rects(gf, rects, fills)
    taken = np.unique(I * n + J)
    sc = _scatter(gs, n, n, int(round(1e-4 * n * n)), taken)
    I = np.concatenate([I, sc // n])
    J = np.concatenate([J, sc % n])
    V = _values(gv, "n01", len(I), np.float32)
    x = _values(rng(seed + 100, XSTREAM), "n01", n, np.float32)
    return _finish("c2", n, np.float32, 50, rects, I, J, V, x)


def make_c3(seed: int = 3, scale: float = 1.0) -> Synth:
    """configs[2]: fp64 500,000^2 power-grid-like: block-tridiagonal with
    diagonal blocks of size U{2..16} (full) and off-diagonal blocks at fill
    U[0.5,1.0] (inv.; all entries |i-j| <= 31, "bandwidth 32"), plus 3
    long-range couplings per row at distinct columns with |i-j| > 32;
    values and x U[-1,1]."""
    n = int(500_000 * scale)
    gp, gf, gs, gv = rng(seed, PLACE), rng(seed, FILL), rng(seed, SCATTER), rng(seed, VALUES)
    sizes = gp.integers(2, 17, size=n // 2 + 2)
    ends = np.cumsum(sizes)
    k = int(np.searchsorted(ends, n))  # first block whose end reaches n
    sizes = sizes[: k + 1].copy()
    sizes[-1] -= int(ends[k] - n)
    if sizes[-1] <= 0:
        sizes = sizes[:-1]
    grid = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    nblk = len(sizes)
    rects = []
    fills = []
    for b in range(nblk):
        s0, sz = int(grid[b]), int(sizes[b])
        rects.append((s0, s0, sz, sz))
        fills.append(1.0)
    off_f = gf.uniform(0.5, 1.0, size=2 * (nblk - 1))
    for b in range(nblk - 1):
        s0, s1 = int(grid[b]), int(grid[b + 1])
        rects.append((s0, s1, int(sizes[b]), int(sizes[b + 1])))   # (k, k+1)
        rects.append((s1, s0, int(sizes[b + 1]), int(sizes[b])))   # (k+1, k)
        fills.append(off_f[2 * b])
        fills.append(off_f[2 * b + 1])
    I, J = _fill_rects(gf, rects, fills)
    # long-range couplings: 3 per row, distinct, |i - j| > 32
    rows = np.repeat(np.arange(n, dtype=np.int64), 3)
    cols = gs.integers(0, n, size=len(rows), dtype=np.int64)
    while True:
        c3 = cols.reshape(n, 3)
        bad = np.abs(rows.reshape(n, 3) - c3) <= 32
        bad[:, 1] |= c3[:, 1] == c3[:, 0]
        bad[:, 2] |= (c3[:, 2] == c3[:, 0]) | (c3[:, 2] == c3[:, 1])
        bad = bad.ravel()
        if not bad.any():
            break
        cols[bad] = gs.integers(0, n, size=int(bad.sum()), dtype=np.int64)
    I = np.concatenate([I, rows])
    J = np.concatenate([J, cols])
    V = _values(gv, "u11", len(I), np.float64)
    x = _values(rng(seed + 100, XSTREAM), "u11", n, np.float64)
    return _finish("c3", n, np.float64, 50, rects, I, J, V, x, rpntr=grid, cpntr=grid)


C4_KEEP_P = 1.863e-4  # reading: honour "~60M nnz"


def make_c4(seed: int = 4, scale: float = 1.0) -> Synth:
    """configs[3]: fp32 2^20 pruned-NN-like: 64x64-aligned tiles kept with
    probability p (reading: p = 1.863e-4 to honour ~60M nnz), one sub-block
    per kept tile with extents U{16..64} at a uniform offset and fill
    U[0.5,1.0]; values N(0, 0.02) (std), x N(0,1)."""
    n = int((1 << 20) * scale) // 64 * 64
    t = n // 64
    gp, gf, gv = rng(seed, PLACE), rng(seed, FILL), rng(seed, VALUES)
    kept = int(gp.binomial(t * t, C4_KEEP_P))
    picks = np.zeros(0, dtype=np.int64)
    while len(picks) < kept:
        d = gp.integers(0, t * t, size=kept - len(picks) + 16, dtype=np.int64)
        d = np.concatenate([picks, d])
        _, first = np.unique(d, return_index=True)
        picks = d[np.sort(first)][:kept]
    tr, tc = picks // t, picks % t
    h = gp.integers(16, 65, size=kept)
    w = gp.integers(16, 65, size=kept)
    ro = np.array([gp.integers(0, 64 - hh + 1) for hh in h], dtype=np.int64)
    co = np.array([gp.integers(0, 64 - ww + 1) for ww in w], dtype=np.int64)
    rects = [(int(tr[k] * 64 + ro[k]), int(tc[k] * 64 + co[k]), int(h[k]), int(w[k]))
             for k in range(kept)]
    fills = gf.uniform(0.5, 1.0, size=kept)
    I, J = _fill_rects(gf, rects, fills)
    V = _values(gv, "n002", len(I), np.float32)
    x = _values(rng(seed + 100, XSTREAM), "n01", n, np.float32)
    return _finish("c4", n, np.float32, 50, rects, I, J, V, x,
                   meta=dict(keep_p=C4_KEEP_P))


def make_c4a(seed: int = 4, scale: float = 1.0) -> Synth:
    """The 64-aligned variant of configs[3] (SURVEY 8(d) C4 reading; the
    delta-stress case of SURVEY 8(f) f2): the same matrix as C4, on the
    64 x 64 tile grid instead of the union of the sub-blocks' edges, so every
    candidate cell is a whole 64 x 64 tile holding one sub-block of 16..64 x
    16..64 at fill 0.5..1 -- cell fills from 3% to 100%, where the delta rule
    decides.  The GPU input is the all-remainder split."""
    s = make_c4(seed, scale)
    n = s.nrows
    g = np.arange(0, n + 1, 64, dtype=np.int32)
    s.name, s.rpntr, s.cpntr = "c4a", g, g.copy()
    s.in_rect = np.zeros(s.nnz, dtype=bool)
    return s


C5_ALPHA = 2.5  # (inv.) power-law exponent of the remainder row degree


def c5_dmin(n: int, mean: float = 16.0, alpha: float = C5_ALPHA) -> float:
    """d_min such that E[min(floor(d_min (1-U)^(-1/(alpha-1))), n)] = mean,
    by bisection on sum_{k=1..n} min(1, (d_min/k)^(alpha-1))."""
    k = np.arange(1, n + 1, dtype=np.float64)
    lo, hi = 1.0, mean
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        e = np.minimum(1.0, (mid / k) ** (alpha - 1.0)).sum()
        lo, hi = (mid, hi) if e < mean else (lo, mid)
    return 0.5 * (lo + hi)


def make_c5(seed: int = 5, scale: float = 1.0) -> Synth:
    """configs[4]: fp32 iterated SpMV, 2^23 square: 60% of nnz in a CSR
    remainder with power-law row degree (alpha = 2.5 inv., mean 16, columns
    uniform distinct per row) and 40% in blocks with extents log-U[4,256]
    (inv.) at fill U[0.6,1.0] (inv.); values U(0,1] scaled to column sums of
    1 (column-stochastic, inv.), x0 U(0,1]; 100 iterations."""
    n = int((1 << 23) * scale)
    gp, gf, gs, gv = rng(seed, PLACE), rng(seed, FILL), rng(seed, SCATTER), rng(seed, VALUES)
    dmin = c5_dmin(n)
    u = gs.random(size=n)
    deg = np.minimum(np.floor(dmin * (1.0 - u) ** (-1.0 / (C5_ALPHA - 1.0))), n).astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    keys = rows * n + gs.integers(0, n, size=len(rows), dtype=np.int64)
    keys = np.unique(keys)
    # top up the rows that lost columns to in-row collisions (distinct
    # columns): heavy rows (deg > n / 8) are drawn without replacement, the
    # others are redrawn with oversampling until every row has its degree
    have = np.bincount(keys // n, minlength=n)
    short = np.flatnonzero(have < deg)
    if len(short):
        is_short = np.zeros(n, dtype=bool)
        is_short[short] = True
        sel = is_short[keys // n]
        sk, keys = keys[sel], keys[~sel]
        heavy = short[deg[short] > n // 8]
        light = short[deg[short] <= n // 8]
        hk = [r * n + np.sort(gs.choice(n, size=int(deg[r]), replace=False)) for r in heavy.tolist()]
        sk = sk[~np.isin(sk // n, heavy)]
        for _ in range(1000):
            need = deg[light] - np.bincount(sk // n, minlength=n)[light]
            todo = need > 0
            if not todo.any():
                break
            r = np.repeat(light[todo], 2 * need[todo] + 4)
            new = r * n + gs.integers(0, n, size=len(r), dtype=np.int64)
            # keep every old key and, per row, the first new distinct keys in
            # draw order (not value order) up to the row's degree
            new, first_pos = np.unique(new, return_index=True)
            new_keep = ~np.isin(new, sk, assume_unique=True)
            new, first_pos = new[new_keep], first_pos[new_keep]
            order = np.argsort(first_pos, kind="stable")  # draw order
            new = new[order]
            nr_ = new // n
            o2 = np.argsort(nr_, kind="stable")  # group by row, draw order within
            new, nr_ = new[o2], nr_[o2]
            start = np.searchsorted(nr_, nr_, side="left")
            rank = np.arange(len(new)) - start
            have_r = np.bincount(sk // n, minlength=n)
            sk = np.sort(np.concatenate([sk, new[rank < (deg[nr_] - have_r[nr_])]]))
        keys = np.sort(np.concatenate([keys, sk] + hk))
    rem_nnz = len(keys)
    target = 0.4 / 0.6 * rem_nnz
    occ = _Occupancy(256)
    rects, fills, block_nnz = [], [], 0.0
    while block_nnz < target:
        batch = _place_random(gp, n, occ, 256,
                              lambda: (int(log_uniform_int(gp, 4, 256, 1)[0]),
                                       int(log_uniform_int(gp, 4, 256, 1)[0])))
        f = gf.uniform(0.6, 1.0, size=len(batch))
        for rr, ff in zip(batch, f):
            if block_nnz >= target:
                break
            rects.append(rr)
            fills.append(ff)
            block_nnz += max(1, round(ff * rr[2] * rr[3]))
    Ib, Jb = _fill_rects(gf, rects, fills)
    bkeys = np.unique(Ib * n + Jb)
    keys = keys[~np.isin(keys, bkeys, assume_unique=True)]  # one value per position
    allk = np.concatenate([bkeys, keys])
    I, J = allk // n, allk % n
    del allk, keys, bkeys, Ib, Jb
    u = _values(gv, "u01", len(I), np.float64)
    colsum = np.bincount(J, weights=u, minlength=n)
    V = (u / colsum[J]).astype(np.float32)
    z = V == 0
    if z.any():  # underflow guard; never expected for U(0,1] / O(10)
        V[z] = np.float32(np.finfo(np.float32).tiny)
    x = _values(rng(seed + 100, XSTREAM), "u01", n, np.float32)
    return _finish("c5", n, np.float32, 50, rects, I, J, V, x, iterations=100,
                   meta=dict(dmin=dmin, alpha=C5_ALPHA))


CONFIGS = {"c1": make_c1, "c2": make_c2, "c3": make_c3, "c4": make_c4, "c5": make_c5,
           "c4a": make_c4a}


def make(name: str, scale: float = 1.0, seed: int | None = None) -> Synth:
    """Build config `name` (c1..c5); `scale` < 1 shrinks n for parity tests."""
    f = CONFIGS[name]
    return f(seed=seed, scale=scale) if seed is not None else f(scale=scale)


# ---------------------------------------------------------------------------
# small random cases for parity and property tests


def random_small(seed: int, nrows: int, ncols: int, nbr: int, nbc: int,
                 dtype=np.float32, density: float = 0.3, dense_cells: float = 0.3,
                 values: str = "u11", delta: int = 50) -> Synth:
    """A random grid with nbr x nbc cells; a fraction `dense_cells` of the
    cells is filled at U[0.5,1] and the rest at `density` * U[0,1]."""
    g = rng(seed, EXTRA)
    rc = np.sort(g.choice(np.arange(1, nrows), size=min(nbr - 1, nrows - 1), replace=False))
    cc = np.sort(g.choice(np.arange(1, ncols), size=min(nbc - 1, ncols - 1), replace=False))
    rpntr = np.concatenate([[0], rc, [nrows]]).astype(np.int32)
    cpntr = np.concatenate([[0], cc, [ncols]]).astype(np.int32)
    nbr, nbc = len(rpntr) - 1, len(cpntr) - 1
    dens = np.where(g.random((nbr, nbc)) < dense_cells, g.uniform(0.5, 1.0, (nbr, nbc)),
                    density * g.random((nbr, nbc)))
    h = np.diff(rpntr)[:, None]
    w = np.diff(cpntr)[None, :]
    p = np.repeat(np.repeat(dens, h.ravel(), axis=0), w.ravel(), axis=1)
    mask = g.random((nrows, ncols)) < p
    I, J = np.nonzero(mask)
    if values == "int":  # small integers: exact in fp32 and fp64
        V = g.integers(-8, 9, size=len(I)).astype(dtype)
        V[V == 0] = 1
        x = g.integers(-8, 9, size=ncols).astype(dtype)
    else:
        V = _values(g, values, len(I), dtype)
        x = _values(g, values, ncols, dtype)
    # rectangles = the cells chosen dense, so the "rect" split is meaningful
    cells = np.argwhere(dens >= 0.5)
    rects = [(int(rpntr[a]), int(cpntr[b]), int(rpntr[a + 1] - rpntr[a]),
              int(cpntr[b + 1] - cpntr[b])) for a, b in cells]
    I = I.astype(np.int64)
    J = J.astype(np.int64)
    s = Synth(name=f"rand{seed}", nrows=nrows, ncols=ncols, dtype=dtype, delta=delta,
              rpntr=rpntr, cpntr=cpntr, rects=np.asarray(rects, np.int64).reshape(-1, 4),
              I=I, J=J, V=V, x=x, in_rect=np.zeros(len(I), bool))
    if len(rects):
        s.in_rect = _in_rect_cells(I, J, rpntr, cpntr, rects)
    return s
