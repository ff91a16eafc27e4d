/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU reference for the
 * MaxK-GNN layer hot path (arXiv 2312.08656).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code, header or helper with the
 * CUDA path (paper_2312_08656_b200/), and neither side includes the other.
 *
 * Every function writes out the plain definition the method reaches:
 *   oracle_topk_cbsr    Eq. 1 (§3.1): keep the k largest entries of each row.
 *                       Ordering (value desc, column asc); IEEE compare so -0.0 == +0.0; NaN rejected.
 *                       Output in CBSR form (§3.2): k values + k ascending column indices.
 *   oracle_densify      the dense N x H matrix a CBSR block stands for (zero off the pattern).
 *   oracle_spmm_rows    X_l[i,:] = sum_j A[i,j] * h(X_{l-1})[j,:]  (§3.2 / Eq. 3 left,
 *                       PAPER.md:320) on a DENSE right operand, accumulated in fp64 in CSR order.
 *   oracle_transpose    CSR of A^T by a stable counting sort (the CSC view of A, PAPER.md:281/430/443).
 *   oracle_sspmm_rows   dL/dh = A^T * dL/dX_l  (Eq. 3 right; outer-product form Eq. 4,
 *                       PAPER.md:341-343) computed as a FULL dense row of A^T*dY in fp64, then sampled
 *                       at the forward pattern sp_index ("known output sparse pattern").
 *
 * Pins: see tests/test_oracle.py (brute force on tiny inputs, library cross-checks at k=H, closed forms
 * A=I, hand-worked example tests/golden/worked_example.json, adjointness).  No function here is
 * "parity unpinned".
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------------------------------- */
/* Eq. 1 — top-k of one row by the total order "a before b  iff  v[a] > v[b] or (v[a] == v[b] and a < b)". */
/* The paper leaves ties unspecified; lower index wins (reading R2).                       */

static int before(const float* v, int32_t a, int32_t b) {
  if (v[a] > v[b]) return 1;
  if (v[a] == v[b] && a < b) return 1;
  return 0;
}

/* library sort (glibc qsort_r) with the explicit rank comparator; the order is total on NaN-free
   input, so stability is irrelevant */
static int cmp_rank(const void* pa, const void* pb, void* arg) {
  const float* v = (const float*)arg;
  int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  if (before(v, a, b)) return -1;
  if (before(v, b, a)) return 1;
  return 0;
}

static int cmp_int(const void* pa, const void* pb) {
  int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  return (a > b) - (a < b);
}

static void sort_by_rank(const float* v, int32_t* order, int32_t h) {
  qsort_r(order, (size_t)h, sizeof(int32_t), cmp_rank, (void*)v);
}

static void sort_ascending(int32_t* a, int32_t n) { qsort(a, (size_t)n, sizeof(int32_t), cmp_int); }

/*
 * Returns 0 on success, -1 on invalid arguments (k < 1, k > h, ld < h), -2 if any input is NaN
 * (NaN input is a precondition violation, reading R4).
 */
int oracle_topk_cbsr(const float* x, int64_t n, int32_t h, int64_t ldx, int32_t k,
                     float* data, int32_t* idx) {
  if (n < 0 || h < 1 || k < 1 || k > h || ldx < h) return -1;
  int bad = 0;
  #pragma omp parallel
  {
    int32_t* order = (int32_t*)malloc((size_t)h * sizeof(int32_t));
    #pragma omp for schedule(dynamic, 64)
    for (int64_t r = 0; r < n; ++r) {
      const float* v = x + r * ldx;
      for (int32_t c = 0; c < h; ++c) {
        if (isnan(v[c])) bad = 1;
        order[c] = c;
      }
      sort_by_rank(v, order, h);          /* rank all columns */
      sort_ascending(order, k);           /* the first k, in ascending column order (CBSR canonical) */
      for (int32_t t = 0; t < k; ++t) {
        idx[r * k + t] = order[t];
        memcpy(&data[r * k + t], &v[order[t]], sizeof(float));  /* bit copy, keeps -0.0 */
      }
    }
    free(order);
  }
  return bad ? -2 : 0;
}

/* densify: out[r, idx[r,t]] = data[r,t]; zero elsewhere (out is n x h fp64, row-major) */
void oracle_densify(int64_t n, int32_t h, int32_t k, const float* data, const int32_t* idx, double* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    double* o = out + r * (int64_t)h;
    for (int32_t c = 0; c < h; ++c) o[c] = 0.0;
    for (int32_t t = 0; t < k; ++t) o[idx[r * k + t]] = (double)data[r * k + t];
  }
}

/*
 * Y[s, :] = sum over edges e of row rows[s]:  val[e] * D[col[e], :]     (fp64, CSR order)
 * rows == NULL means rows[s] = s for s in [0, n_sel).  D is n_cols x h fp64.  Y is n_sel x h fp64.
 * row_ptr is indexed absolutely (row_ptr[0] may be nonzero).
 */
void oracle_spmm_rows(const int64_t* row_ptr, const int32_t* col, const float* val,
                      const int64_t* rows, int64_t n_sel, const double* D, int32_t h, double* Y) {
  #pragma omp parallel for schedule(dynamic, 16)
  for (int64_t s = 0; s < n_sel; ++s) {
    int64_t i = rows ? rows[s] : s;
    double* y = Y + s * (int64_t)h;
    for (int32_t c = 0; c < h; ++c) y[c] = 0.0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const double a = (double)val[e];
      const double* d = D + (int64_t)col[e] * h;
      for (int32_t c = 0; c < h; ++c) y[c] += a * d[c];
    }
  }
}

/*
 * CSR of A^T (equivalently CSC of A): t_ptr [n_cols+1], t_row [nnz], t_val [nnz].  Stable counting
 * sort: within column j, entries appear in increasing source row i.  Returns -1 on a col >= n_cols.
 */
int oracle_transpose(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n_rows,
                     int64_t n_cols, int64_t* t_ptr, int32_t* t_row, float* t_val) {
  const int64_t base = row_ptr[0];
  for (int64_t j = 0; j <= n_cols; ++j) t_ptr[j] = 0;
  for (int64_t e = base; e < row_ptr[n_rows]; ++e) {
    if (col[e] < 0 || col[e] >= n_cols) return -1;
    t_ptr[col[e] + 1] += 1;
  }
  for (int64_t j = 0; j < n_cols; ++j) t_ptr[j + 1] += t_ptr[j];
  int64_t* fill = (int64_t*)malloc((size_t)(n_cols > 0 ? n_cols : 1) * sizeof(int64_t));
  for (int64_t j = 0; j < n_cols; ++j) fill[j] = t_ptr[j];
  for (int64_t i = 0; i < n_rows; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      int64_t p = fill[col[e]]++;
      t_row[p] = (int32_t)i;
      t_val[p] = val[e];
    }
  free(fill);
  return 0;
}

/*
 * dXs[s, t] = G[j, idx[j, t]]  with  G[j, :] = sum_{(i, a) in column j of A} a * dY[i, :]   (fp64)
 * j = rows[s] (rows == NULL: j = s).  (t_ptr, t_row, t_val) from oracle_transpose.  dY has row
 * stride ld_dy.  idx is n_cols x k int32 (the forward pattern).  Output n_sel x k fp64.
 */
void oracle_sspmm_rows(const int64_t* t_ptr, const int32_t* t_row, const float* t_val,
                       const float* dy, int64_t ld_dy, int32_t h, const int32_t* idx, int32_t k,
                       const int64_t* rows, int64_t n_sel, double* dxs) {
  #pragma omp parallel
  {
    double* g = (double*)malloc((size_t)h * sizeof(double));
    #pragma omp for schedule(dynamic, 16)
    for (int64_t s = 0; s < n_sel; ++s) {
      int64_t j = rows ? rows[s] : s;
      for (int32_t c = 0; c < h; ++c) g[c] = 0.0;                 /* full dense row of A^T dY */
      for (int64_t p = t_ptr[j]; p < t_ptr[j + 1]; ++p) {
        const double a = (double)t_val[p];
        const float* d = dy + (int64_t)t_row[p] * ld_dy;
        for (int32_t c = 0; c < h; ++c) g[c] += a * (double)d[c];
      }
      for (int32_t t = 0; t < k; ++t) dxs[s * k + t] = g[idx[j * k + t]];  /* sampled at the mask */
    }
    free(g);
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
