"""Seeded matrices for the per-shape delta calibration and the sparsity
ablation -- drawing only, no method arithmetic.

* `shape_grid(h, w, fill, area)`: the Fig. 7 heatmap workload:
  a uniform grid of h x w cells, `area` matrix elements' worth of blocks of
  that one shape, each entry of a block non-zero with probability `fill`
  (Bernoulli; at least one per block), 8 blocks per block row at distinct
  random block columns among 64.
* `fig10(sparsity)`: the Fig. 10 ablation: a 10000 x 10000
  matrix overlaid with 50 x 50 splits (a 200 x 200 grid of 50 x 50 cells), 500
  blocks at distinct random cells, each with `sparsity` of its entries zero.

Both return the VBR input of gen/encode.py's layout (every block a stored
VBR block: the inspector's delta decides dense tile or remainder), plus the
sorted COO triples for the oracle, as a gen.Synth.
"""
from __future__ import annotations

import numpy as np

from .configs import FILL, PLACE, VALUES, XSTREAM, Synth, _values, rng


def _assemble(name, nrows, ncols, h, w, br, bc, masks, vals, x, delta=50):
    """Blocks (br[k], bc[k]) sorted by (br, bc), masks (nb, h*w) column-major
    in-block positions -> Synth with the COO triples and the grid."""
    nb = len(br)
    k, pos = np.nonzero(masks)
    I = br[k].astype(np.int64) * h + pos % h
    J = bc[k].astype(np.int64) * w + pos // h
    V = vals[: len(I)]
    order = np.lexsort((J, I))
    rpntr = np.arange(0, nrows + 1, h, dtype=np.int32)
    cpntr = np.arange(0, ncols + 1, w, dtype=np.int32)
    s = Synth(name=name, nrows=nrows, ncols=ncols, dtype=np.float32, delta=delta,
              rpntr=rpntr, cpntr=cpntr,
              rects=np.stack([br * h, bc * w, np.full(nb, h), np.full(nb, w)], 1).astype(np.int64),
              I=I[order], J=J[order], V=V[order], x=x, in_rect=np.ones(len(I), bool))
    return s


def shape_grid(h: int, w: int, fill: float, area: int = 1 << 23, seed: int = 7,
               per_row: int = 8, ncb: int = 64) -> Synth:
    nb = max(per_row, area // (h * w))
    nbr = -(-nb // per_row)
    nb = nbr * per_row
    gp, gf, gv, gx = rng(seed, PLACE), rng(seed, FILL), rng(seed, VALUES), rng(seed, XSTREAM)
    bc = np.sort(np.argsort(gp.random((nbr, ncb)), axis=1)[:, :per_row], axis=1).ravel()
    br = np.repeat(np.arange(nbr), per_row)
    masks = gf.random((nb, h * w)) < fill
    empty = ~masks.any(axis=1)
    masks[empty, gf.integers(0, h * w, int(empty.sum()))] = True
    vals = _values(gv, "u11", int(masks.sum()), np.float32)
    x = _values(gx, "u11", ncb * w, np.float32)
    return _assemble(f"shape{h}x{w}_f{fill:.2f}", nbr * h, ncb * w, h, w, br, bc, masks, vals, x)


def fig10(sparsity: float, seed: int = 10, n: int = 10000, split: int = 50,
          blocks: int = 500) -> Synth:
    g = n // split
    gp, gf, gv, gx = rng(seed, PLACE), rng(seed, FILL), rng(seed, VALUES), rng(seed, XSTREAM)
    cells = np.sort(gp.choice(g * g, size=blocks, replace=False))
    br, bc = cells // g, cells % g
    area = split * split
    k = max(1, int(round((1.0 - sparsity) * area)))
    keys = gf.random((blocks, area))
    masks = np.zeros((blocks, area), bool)
    np.put_along_axis(masks, np.argsort(keys, axis=1)[:, :k], True, axis=1)
    vals = _values(gv, "u11", int(masks.sum()), np.float32)
    x = _values(gx, "u11", n, np.float32)
    return _assemble(f"fig10_s{sparsity:.2f}", n, n, split, split, br, bc, masks, vals, x)
