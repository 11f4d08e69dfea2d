/*
 * sable_oracle.c -- plain, slow, obviously-correct CPU oracle for the SABLE
 * VBR SpMV hot path (arXiv 2407.00829).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2407_00829_b200/) never links, imports or calls it,
 * and this file includes no header of the product path (they share no code).
 *
 * What it computes (every step cites the passage it follows; "PAPER.md:L" is
 * a line of /root/reference/PAPER.md, "SURVEY 8(c)" is the reading table of
 * SURVEY.md section 8(c), restated in DESIGN.md "Readings"):
 *
 *   oracle_normalize  -- COO triples -> sorted (i,j), duplicates rejected,
 *                        zeros dropped (reading R4: v != 0 in IEEE).
 *   oracle_partition  -- COO + row/column cut grid + delta ->
 *                        (i)   candidate cells {br, bc, cnt, dense}
 *                              (a cell is a block iff it
 *                              holds >= 1 non-zero),
 *                        (ii)  dense tiles, column-major, zero-filled
 *                              (Fig. 2 "Val ... column-major", PAPER.md:221;
 *                              Listing 1; Listing 2)
 *                              with dense-only offsets (reading R7),
 *                        (iii) ublocks = ordinals of non-dense cells
 *                              (Fig. 3),
 *                        (iv)  the CSR remainder of the non-dense cells,
 *                              row-major (Fig. 3; reading R6).
 *                        delta-dense: "the percentage of non-zero elements is
 *                        at least delta %", evaluated in
 *                        integers as 100*cnt >= delta*h*w (readings R1, R3).
 *   oracle_spmv       -- y_i = sum_j A_ij x_j row by row in
 *                        fp64 over the triples in increasing j, plus the
 *                        tolerance scale s_i = sum_j |A_ij| |x_j|.
 *
 * Precision: the paper states none (reading R11); the oracle is fp64
 * throughout.  Compile with -O2 -ffp-contract=off so that no FMA contraction
 * changes the plain left-to-right sums.
 *
 * Parity pins (tests/test_oracle.py, run with -m "not gpu"): Fig. 2 arrays
 * verbatim, Fig. 3 VBR-C arrays at delta=75, Fig. 4a/Fig. 6 tile offsets,
 * Listing 2 offset arithmetic, brute-force cell slicing of dense matrices,
 * scipy CSR matvec at delta=101, closed-form y on the worked examples, and
 * the invariants of BASELINE.json north_star s10.  Every exported function
 * below is pinned; none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- error codes returned through *err -------------------------------- */
enum {
  OR_OK = 0,
  OR_E_RANGE = 1,     /* index outside [0,nrows) x [0,ncols) */
  OR_E_DUPLICATE = 2, /* the same (i,j) twice */
  OR_E_GRID = 3,      /* rpntr/cpntr not 0 = p0 < p1 < ... = n */
  OR_E_OOM = 4,
  OR_E_ARG = 5
};

/* ---- normalisation -------------------------------- */

typedef struct {
  int64_t i, j;
  double v;
} or_triple;

static int cmp_triple(const void *a, const void *b) {
  const or_triple *x = (const or_triple *)a, *y = (const or_triple *)b;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  if (x->j != y->j) return x->j < y->j ? -1 : 1;
  return 0;
}

/* Normalise nnz COO triples in place into (I,J,V): reject out-of-range
 * indices, sort by (i,j), reject duplicates, drop v == 0 (so +0 and -0 are
 * dropped; NaN is kept because NaN == 0 is false).  Returns the kept count
 * or -1 with *err set. */
int64_t oracle_normalize(int64_t nrows, int64_t ncols, int64_t nnz,
                         int64_t *I, int64_t *J, double *V, int *err) {
  *err = OR_OK;
  int sorted = 1;
  for (int64_t k = 0; k < nnz; ++k) {
    if (I[k] < 0 || I[k] >= nrows || J[k] < 0 || J[k] >= ncols) {
      *err = OR_E_RANGE;
      return -1;
    }
    if (k > 0 && (I[k] < I[k - 1] || (I[k] == I[k - 1] && J[k] <= J[k - 1])))
      sorted = 0;
  }
  if (!sorted) {
    or_triple *t = (or_triple *)malloc(sizeof(or_triple) * (size_t)(nnz ? nnz : 1));
    if (!t) {
      *err = OR_E_OOM;
      return -1;
    }
    for (int64_t k = 0; k < nnz; ++k) {
      t[k].i = I[k];
      t[k].j = J[k];
      t[k].v = V[k];
    }
    qsort(t, (size_t)nnz, sizeof(or_triple), cmp_triple);
    for (int64_t k = 0; k < nnz; ++k) {
      I[k] = t[k].i;
      J[k] = t[k].j;
      V[k] = t[k].v;
    }
    free(t);
  }
  int64_t out = 0;
  for (int64_t k = 0; k < nnz; ++k) {
    if (k > 0 && I[k] == I[k - 1] && J[k] == J[k - 1]) {
      *err = OR_E_DUPLICATE;
      return -1;
    }
    if (V[k] == 0.0) continue; /* explicit zeros are not non-zeros */
    I[out] = I[k];
    J[out] = J[k];
    V[out] = V[k];
    ++out;
  }
  return out;
}

/* ---- the partition ----------------------------- */

void oracle_rowptr(int64_t nrows, int64_t nnz, const int64_t *I, int64_t *rowptr);

typedef struct {
  /* sizes */
  int64_t n_cells;    /* candidate cells (cnt >= 1) in block rows [a0,a1) */
  int64_t n_dense;    /* delta-dense cells = tiles */
  int64_t tile_elems; /* sum of dense areas */
  int64_t rem_nnz;    /* non-zeros of non-dense cells */
  int64_t nnz;        /* non-zeros in rows of block rows [a0,a1) */
  int64_t row_begin, row_end;
  /* (i) cells in (br, bc) order */
  int32_t *cell_br, *cell_bc;
  int64_t *cell_cnt;
  uint8_t *cell_dense;
  /* (ii) dense tiles: dense-only offsets and column-major zero-filled values */
  int64_t *tile_off; /* n_dense + 1 */
  double *tile_val;  /* tile_elems */
  /* (iii) ordinals (relative to the first cell of the range) of non-dense cells */
  int64_t *ublocks; /* n_cells - n_dense */
  /* (iv) remainder CSR over rows [row_begin,row_end) */
  int64_t *rem_indptr; /* (row_end-row_begin)+1, starts at 0 */
  int32_t *rem_indices;
  double *rem_val;
} oracle_partition_t;

void oracle_partition_free(oracle_partition_t *p) {
  if (!p) return;
  free(p->cell_br);
  free(p->cell_bc);
  free(p->cell_cnt);
  free(p->cell_dense);
  free(p->tile_off);
  free(p->tile_val);
  free(p->ublocks);
  free(p->rem_indptr);
  free(p->rem_indices);
  free(p->rem_val);
  free(p);
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static int grid_ok(int32_t nb, const int32_t *p, int64_t n) {
  if (nb < 1 || p[0] != 0 || p[nb] != n) return 0;
  for (int32_t a = 0; a < nb; ++a)
    if (p[a + 1] <= p[a]) return 0;
  return 1;
}

/*
 * Partition the normalised COO (sorted by (i,j), no duplicates, no zeros)
 * over the cut grid rpntr/cpntr, restricted to block rows [a0, a1).
 * Readings applied: candidate cells are all cells with >= 1 non-zero,
 * whatever array carried them (R5); dense <=> 100*cnt >= delta*h*w in int64
 * (R1, R3); delta in 0..101.
 *
 * Two sweeps over the block rows: sweep 1 sizes the outputs, sweep 2 fills
 * them.  Both sweeps run the same per-block-row count (count_block_row).
 */

/* Step 4 for one block row: cnt[b] = number of triples of rows
 * [r0, r0+h) in block column b; touched[0..nt) = the b with cnt[b] > 0 in
 * increasing order.  Returns nt. */
static int32_t count_block_row(int64_t k0, int64_t k1, const int64_t *J,
                               const int32_t *col2bc, int64_t *cnt,
                               int32_t *touched) {
  int32_t nt = 0;
  for (int64_t k = k0; k < k1; ++k) {
    const int32_t b = col2bc[J[k]];
    if (cnt[b]++ == 0) touched[nt++] = b;
  }
  qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
  return nt;
}

/* Step 5: the delta-dense rule, in integers.  With a
 * per-shape policy (reading R22: the B200
 * replacement of the paper's per-block classifier):
 * a cell of h x w is dense iff h*w >= min_area and
 * 100*cnt >= delta(h, w)*h*w, where delta(h, w) is the delta of the first
 * rule with h_min <= h <= h_max and w_min <= w <= w_max, else the default.
 * rules holds n_rules records of 5 int32: h_min, h_max, w_min, w_max, delta. */
typedef struct {
  int32_t delta;
  int64_t min_area;
  int32_t n_rules;
  const int32_t *rules;
} policy_t;

static int32_t delta_for(const policy_t *pol, int64_t h, int64_t w) {
  for (int32_t k = 0; k < pol->n_rules; ++k) {
    const int32_t *r = pol->rules + 5 * k;
    if (h >= r[0] && h <= r[1] && w >= r[2] && w <= r[3]) return r[4];
  }
  return pol->delta;
}

static int is_dense(int64_t cnt, int64_t h, int64_t w, const policy_t *pol) {
  if (h * w < pol->min_area) return 0;
  return 100 * cnt >= (int64_t)delta_for(pol, h, w) * h * w;
}

static oracle_partition_t *partition_impl(int64_t nrows, int64_t ncols, int64_t nnz,
                                          const int64_t *I, const int64_t *J,
                                          const double *V, int32_t nbr,
                                          const int32_t *rpntr, int32_t nbc,
                                          const int32_t *cpntr, const policy_t *pol,
                                          int32_t a0, int32_t a1, int *err);

oracle_partition_t *oracle_partition(int64_t nrows, int64_t ncols, int64_t nnz,
                                     const int64_t *I, const int64_t *J,
                                     const double *V, int32_t nbr,
                                     const int32_t *rpntr, int32_t nbc,
                                     const int32_t *cpntr, int32_t delta,
                                     int32_t a0, int32_t a1, int *err) {
  const policy_t pol = {delta, 0, 0, NULL};
  return partition_impl(nrows, ncols, nnz, I, J, V, nbr, rpntr, nbc, cpntr, &pol, a0, a1, err);
}

/* The same partition under a per-shape policy (see is_dense). */
oracle_partition_t *oracle_partition_policy(int64_t nrows, int64_t ncols, int64_t nnz,
                                            const int64_t *I, const int64_t *J,
                                            const double *V, int32_t nbr,
                                            const int32_t *rpntr, int32_t nbc,
                                            const int32_t *cpntr, int32_t delta,
                                            int64_t min_area, int32_t n_rules,
                                            const int32_t *rules, int32_t a0, int32_t a1,
                                            int *err) {
  *err = OR_OK;
  if (min_area < 0 || n_rules < 0 || (n_rules > 0 && !rules)) {
    *err = OR_E_ARG;
    return NULL;
  }
  for (int32_t k = 0; k < n_rules; ++k)
    if (rules[5 * k + 4] < 0 || rules[5 * k + 4] > 101) {
      *err = OR_E_ARG;
      return NULL;
    }
  const policy_t pol = {delta, min_area, n_rules, rules};
  return partition_impl(nrows, ncols, nnz, I, J, V, nbr, rpntr, nbc, cpntr, &pol, a0, a1, err);
}

static oracle_partition_t *partition_impl(int64_t nrows, int64_t ncols, int64_t nnz,
                                          const int64_t *I, const int64_t *J,
                                          const double *V, int32_t nbr,
                                          const int32_t *rpntr, int32_t nbc,
                                          const int32_t *cpntr, const policy_t *pol,
                                          int32_t a0, int32_t a1, int *err) {
  *err = OR_OK;
  const int32_t delta = pol->delta;
  if (delta < 0 || delta > 101 || a0 < 0 || a1 > nbr || a0 > a1) {
    *err = OR_E_ARG;
    return NULL;
  }
  if (!grid_ok(nbr, rpntr, nrows) || !grid_ok(nbc, cpntr, ncols)) {
    *err = OR_E_GRID;
    return NULL;
  }
  oracle_partition_t *p = (oracle_partition_t *)calloc(1, sizeof(*p));
  int32_t *col2bc = (int32_t *)malloc(sizeof(int32_t) * (size_t)ncols);
  int64_t *rowptr = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nrows + 1));
  int64_t *cnt = (int64_t *)calloc((size_t)nbc, sizeof(int64_t));
  int64_t *tile_of = (int64_t *)malloc(sizeof(int64_t) * (size_t)nbc);
  int32_t *touched = (int32_t *)malloc(sizeof(int32_t) * (size_t)nbc);
  if (!p || !col2bc || !rowptr || !cnt || !tile_of || !touched) goto oom;

  /* Step 3: col2bc by a linear sweep over cpntr.  Block row a owns rows
   * rpntr[a] .. rpntr[a+1]-1, so row2br is not materialised. */
  for (int32_t b = 0; b < nbc; ++b)
    for (int32_t j = cpntr[b]; j < cpntr[b + 1]; ++j) col2bc[j] = b;
  oracle_rowptr(nrows, nnz, I, rowptr);

  p->row_begin = rpntr[a0];
  p->row_end = rpntr[a1];
  p->nnz = rowptr[p->row_end] - rowptr[p->row_begin];

  /* Sweep 1: sizes. */
  for (int32_t a = a0; a < a1; ++a) {
    const int64_t h = rpntr[a + 1] - rpntr[a];
    const int32_t nt = count_block_row(rowptr[rpntr[a]], rowptr[rpntr[a + 1]], J,
                                       col2bc, cnt, touched);
    for (int32_t t = 0; t < nt; ++t) {
      const int32_t b = touched[t];
      const int64_t w = cpntr[b + 1] - cpntr[b];
      p->n_cells++;
      if (is_dense(cnt[b], h, w, pol)) {
        p->n_dense++;
        p->tile_elems += h * w;
      } else {
        p->rem_nnz += cnt[b];
      }
      cnt[b] = 0;
    }
  }

  const int64_t nloc = p->row_end - p->row_begin;
  p->cell_br = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p->n_cells + 1));
  p->cell_bc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p->n_cells + 1));
  p->cell_cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p->n_cells + 1));
  p->cell_dense = (uint8_t *)malloc((size_t)(p->n_cells + 1));
  p->tile_off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p->n_dense + 1));
  p->tile_val = (double *)calloc((size_t)(p->tile_elems + 1), sizeof(double)); /* zero fill */
  p->ublocks = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p->n_cells - p->n_dense + 1));
  p->rem_indptr = (int64_t *)calloc((size_t)nloc + 1, sizeof(int64_t));
  p->rem_indices = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p->rem_nnz + 1));
  p->rem_val = (double *)malloc(sizeof(double) * (size_t)(p->rem_nnz + 1));
  if (!p->cell_br || !p->cell_bc || !p->cell_cnt || !p->cell_dense || !p->tile_off ||
      !p->tile_val || !p->ublocks || !p->rem_indptr || !p->rem_indices || !p->rem_val)
    goto oom;

  /* Sweep 2: fill. */
  int64_t c_i = 0, t_i = 0, u_i = 0, r_i = 0, off = 0;
  p->tile_off[0] = 0;
  for (int32_t a = a0; a < a1; ++a) {
    const int64_t r0 = rpntr[a], h = rpntr[a + 1] - rpntr[a];
    const int64_t k0 = rowptr[r0], k1 = rowptr[r0 + h];
    const int32_t nt = count_block_row(k0, k1, J, col2bc, cnt, touched);
    /* Steps 5-6(i),(iii): cells in (a, b) order; tiles at dense-only offsets. */
    for (int32_t t = 0; t < nt; ++t) {
      const int32_t b = touched[t];
      const int64_t w = cpntr[b + 1] - cpntr[b];
      const int dense = is_dense(cnt[b], h, w, pol);
      p->cell_br[c_i] = a;
      p->cell_bc[c_i] = b;
      p->cell_cnt[c_i] = cnt[b];
      p->cell_dense[c_i] = (uint8_t)dense;
      if (dense) {
        tile_of[b] = off;
        off += h * w;
        p->tile_off[++t_i] = off;
      } else {
        tile_of[b] = -1;
        p->ublocks[u_i++] = c_i; /* ordinal relative to the range's first cell */
      }
      c_i++;
    }
    /* Steps 6(ii),(iv): every triple of the block row, in (i, j) order, goes
     * either into its tile (column-major, val[off + (j-c0)*h + (i-r0)],
     * PAPER.md:602) or to the remainder CSR. */
    for (int64_t k = k0; k < k1; ++k) {
      const int32_t b = col2bc[J[k]];
      if (tile_of[b] >= 0) {
        p->tile_val[tile_of[b] + (J[k] - cpntr[b]) * h + (I[k] - r0)] = V[k];
      } else {
        p->rem_indices[r_i] = (int32_t)J[k];
        p->rem_val[r_i] = V[k];
        r_i++;
        p->rem_indptr[I[k] - p->row_begin + 1]++;
      }
    }
    for (int32_t t = 0; t < nt; ++t) cnt[touched[t]] = 0;
  }
  for (int64_t i = 0; i < nloc; ++i) p->rem_indptr[i + 1] += p->rem_indptr[i];

  free(col2bc);
  free(rowptr);
  free(cnt);
  free(tile_of);
  free(touched);
  return p;
oom:
  *err = OR_E_OOM;
  free(col2bc);
  free(rowptr);
  free(cnt);
  free(tile_of);
  free(touched);
  oracle_partition_free(p);
  return NULL;
}

/* ---- y = A x ------------------------- */

/* Rows are taken from the normalised COO; y and s must hold nrows doubles. */
void oracle_spmv(int64_t nrows, int64_t nnz, const int64_t *I, const int64_t *J,
                 const double *V, const double *x, double *y, double *s) {
  for (int64_t i = 0; i < nrows; ++i) {
    y[i] = 0.0;
    s[i] = 0.0;
  }
  int64_t k = 0;
  for (int64_t i = 0; i < nrows; ++i) {
    double acc = 0.0, sc = 0.0;
    while (k < nnz && I[k] == i) {
      acc += V[k] * x[J[k]];
      sc += fabs(V[k]) * fabs(x[J[k]]);
      ++k;
    }
    y[i] = acc;
    s[i] = sc;
  }
}

/* The same definition evaluated for a sample of rows only (for full-size
 * configurations): rowptr is the COO row pointer (nrows+1). */
void oracle_spmv_rows(const int64_t *rowptr, const int64_t *J, const double *V,
                      const double *x, int64_t nsample, const int64_t *rows,
                      double *y, double *s) {
  for (int64_t t = 0; t < nsample; ++t) {
    const int64_t i = rows[t];
    double acc = 0.0, sc = 0.0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      acc += V[k] * x[J[k]];
      sc += fabs(V[k]) * fabs(x[J[k]]);
    }
    y[t] = acc;
    s[t] = sc;
  }
}

/* The same definition for rows [0, nrows) split across `nthreads` OpenMP
 * threads (row-parallel; every row keeps its own order, so y and s are
 * bitwise those of oracle_spmv_rows).  Used only to time the oracle on all
 * host cores (bench.py's cpu_baseline). */
void oracle_spmv_csr_mt(const int64_t *rowptr, const int64_t *J, const double *V,
                        const double *x, int64_t nrows, int32_t nthreads, double *y,
                        double *s) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < nrows; ++i) {
    double acc = 0.0, sc = 0.0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      acc += V[k] * x[J[k]];
      sc += fabs(V[k]) * fabs(x[J[k]]);
    }
    y[i] = acc;
    s[i] = sc;
  }
}

/* COO row pointer of the normalised triples (a counting pass). */
void oracle_rowptr(int64_t nrows, int64_t nnz, const int64_t *I, int64_t *rowptr) {
  for (int64_t i = 0; i <= nrows; ++i) rowptr[i] = 0;
  for (int64_t k = 0; k < nnz; ++k) rowptr[I[k] + 1]++;
  for (int64_t i = 0; i < nrows; ++i) rowptr[i + 1] += rowptr[i];
}

/* ---- Alg. 1 "Matrix Partitioning" ---------------------
 *
 * PAPER.md:381-416 (Section 5, Algorithm 1), similarity Eq. 1
 * PAPER.md:358-362 and Eq. 2, over the non-zero PATTERN of
 * the rows (columns): u.v counts the positions non-zero in both.
 *
 *   i <- 0
 *   while i < n - 1:
 *     if row i is empty:
 *       while i < n - 1 and row i+1 is empty: i <- i + 1
 *       cuts.append(i + 1)
 *     elif similarity(row i, row i+1) < cut_threshold:
 *       cuts.append(i + 1)
 *     i <- i + 1
 *   cuts.append(n)
 *
 * Readings (R17 and R19-R20): Eq. 2's ">>" / "<<"
 * shift u by one position right / left (column j -> j +- 1, positions
 * leaving [0, n) dropped) and the similarity takes the maximum of the three
 * dot products; the threshold is the rational t_num / t_den and the test
 * "S < t" is evaluated exactly as dot * t_den < t_num * max(nnz u, nnz v);
 * a cut equal to the previous one (the final append after an empty run that
 * reaches the last row) is not repeated.  The grid is 0 followed by the cuts.
 *
 * The pattern of the "columns" partition is the transpose: call this on the
 * CSR of A^T.  rowptr/J describe a CSR pattern with columns strictly
 * increasing per row; cuts receives up to n values; returns their count.
 */
static int64_t dot_shift(const int64_t *a, int64_t na, const int64_t *b, int64_t nb,
                         int64_t shift) {
  /* #{ j in a : j + shift in b }, both sorted ascending */
  int64_t i = 0, k = 0, c = 0;
  while (i < na && k < nb) {
    const int64_t v = a[i] + shift;
    if (v < b[k]) ++i;
    else if (v > b[k]) ++k;
    else { ++c; ++i; ++k; }
  }
  return c;
}

static int below(const int64_t *rowptr, const int64_t *J, int64_t r, int32_t shifts,
                 uint32_t t_num, uint32_t t_den) {
  const int64_t *a = J + rowptr[r], *b = J + rowptr[r + 1];
  const int64_t na = rowptr[r + 1] - rowptr[r], nb = rowptr[r + 2] - rowptr[r + 1];
  int64_t dot = dot_shift(a, na, b, nb, 0);
  if (shifts) {
    const int64_t dr = dot_shift(a, na, b, nb, 1), dl = dot_shift(a, na, b, nb, -1);
    if (dr > dot) dot = dr;
    if (dl > dot) dot = dl;
  }
  const int64_t mx = na > nb ? na : nb;
  return dot * (int64_t)t_den < (int64_t)t_num * mx;
}

int64_t oracle_alg1(int64_t n, const int64_t *rowptr, const int64_t *J, uint32_t t_num,
                    uint32_t t_den, int32_t shifts, int32_t *cuts) {
  int64_t m = 0;
  int64_t i = 0;
#define EMPTY(r) (rowptr[(r) + 1] == rowptr[(r)])
#define APPEND(v) do { if (m == 0 || cuts[m - 1] != (int32_t)(v)) cuts[m++] = (int32_t)(v); } while (0)
  while (i < n - 1) {
    if (EMPTY(i)) {
      while (i < n - 1 && EMPTY(i + 1)) ++i;
      APPEND(i + 1);
    } else if (below(rowptr, J, i, shifts, t_num, t_den)) {
      APPEND(i + 1);
    }
    ++i;
  }
  APPEND(n);
#undef EMPTY
#undef APPEND
  return m;
}
