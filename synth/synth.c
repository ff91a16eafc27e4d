/*
 * synth.c — seeded synthetic INPUT generators shared by the CUDA path's tests/bench and the oracle.
 *
 * This module holds none of the method's arithmetic (no top-k, no aggregation, no gradient): it only
 * draws graphs and feature matrices.  It is the one piece of code both sides may use.
 *
 * Recipe (DESIGN.md §3 "Input recipe"):
 *   - Graph: directed Chung–Lu power law.  Rank r in [0,N) has weight w_r = (r + r0)^(-1/(gamma-1)),
 *     scaled by s = nnz / sum_r w_r so the expected degree sum is nnz.  r0 is found by bisection so that
 *     the expected maximum degree s*w_0 equals d_max (default min(N-1, ceil(2*sqrt(nnz)))).
 *     The paper states only N, nnz (Table 1) and "power-law distributed non-zero
 *     elements"; gamma, d_max and the Chung–Lu model are our reading.
 *   - Row degree d_r = floor(s*w_r) + Bernoulli(frac(s*w_r)), capped at N-1.
 *   - Columns: d_r DISTINCT columns drawn with probability proportional to the same weights (alias
 *     table), duplicates re-drawn, then sorted ascending.
 *   - A seeded permutation pi relabels nodes (rows and columns alike) so hubs are scattered.
 *   - Values 1/deg(row) (GraphSAGE mean aggregator, §3.2, §5.1).
 *   - Features: iid N(0,1) fp32 ("follows a normal distribution", §5.3), Box–Muller.
 *
 * Every random number is a pure function of (seed, stream, counter) — splitmix64 — so the output is
 * bit-identical for any OpenMP thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* counter-based generator: independent streams keyed by (seed, stream), indexed by ctr */
static inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return mix64(mix64(seed ^ mix64(stream * 0xD1B54A32D192ED03ull)) ^ ctr);
}

static inline double u01(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

enum { STREAM_DEG = 1, STREAM_PERM = 2, STREAM_COL = 3, STREAM_NORMAL = 4 };

/* deterministic (thread-count independent) sum of (r + r0)^(-alpha), r in [0, n) */
static double weight_sum(int64_t n, double r0, double alpha) {
  const int64_t CH = 1 << 16;
  int64_t nch = (n + CH - 1) / CH;
  double* part = (double*)calloc((size_t)(nch > 0 ? nch : 1), sizeof(double));
  #pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nch; ++c) {
    int64_t b = c * CH, e = b + CH < n ? b + CH : n;
    double s = 0.0;
    for (int64_t r = b; r < e; ++r) s += pow((double)r + r0, -alpha);
    part[c] = s;
  }
  double tot = 0.0;
  for (int64_t c = 0; c < nch; ++c) tot += part[c];
  free(part);
  return tot;
}

/*
 * synth_degrees: degree sequence and node weights of the Chung–Lu graph.
 *   deg_out[v]    : out-degree of node v (int64, length n)
 *   weight_out[v] : column-sampling weight of node v (double, length n)
 *   perm_out[r]   : node id of rank r (int64, length n) — may be NULL
 * Returns 0 on success, -1 on bad arguments.
 */
int synth_degrees(int64_t n, int64_t nnz_target, double gamma, int64_t d_max, uint64_t seed,
                  int64_t* deg_out, double* weight_out, int64_t* perm_out) {
  if (n <= 0 || nnz_target < 0 || gamma <= 1.0 || !deg_out || !weight_out) return -1;
  const double alpha = 1.0 / (gamma - 1.0);
  if (d_max <= 0) {
    d_max = (int64_t)ceil(2.0 * sqrt((double)nnz_target));
    if (d_max > n - 1) d_max = n - 1;
  }
  if (d_max < 1) d_max = 1;
  /* bisection on log r0: f(r0) = s(r0) * r0^-alpha - d_max is decreasing in r0 */
  double lo = -12.0, hi = log((double)n) + 30.0;
  for (int it = 0; it < 60; ++it) {
    double mid = 0.5 * (lo + hi), r0 = exp(mid);
    double s = (double)nnz_target / weight_sum(n, r0, alpha);
    double dmax_exp = s * pow(r0, -alpha);
    if (dmax_exp > (double)d_max) lo = mid; else hi = mid;
  }
  const double r0 = exp(0.5 * (lo + hi));
  const double s = (double)nnz_target / weight_sum(n, r0, alpha);

  /* seeded Fisher–Yates permutation of node ids (sequential, O(n)) */
  int64_t* perm = perm_out ? perm_out : (int64_t*)malloc((size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)(rng(seed, STREAM_PERM, (uint64_t)i) % (uint64_t)(i + 1));
    int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  #pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    double w = pow((double)r + r0, -alpha);
    double e = s * w;
    int64_t d = (int64_t)floor(e);
    if (u01(rng(seed, STREAM_DEG, (uint64_t)r)) < e - (double)d) d += 1;
    if (d > n - 1) d = n - 1;
    if (d < 0) d = 0;
    deg_out[perm[r]] = d;
    weight_out[perm[r]] = w;
  }
  if (!perm_out) free(perm);
  return 0;
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/*
 * synth_columns: for each node v, deg(v) = row_ptr[v+1]-row_ptr[v] distinct columns drawn with
 * probability proportional to weight[] (Vose alias table), sorted ascending, written to col_out.
 * Returns 0 on success, -1 on bad arguments, -2 on allocation failure.
 */
int synth_columns(int64_t n, const int64_t* row_ptr, const double* weight, uint64_t seed, int32_t* col_out) {
  if (n <= 0 || !row_ptr || !weight || !col_out) return -1;
  if (n > 2147483647LL) return -1;
  double* prob = (double*)malloc((size_t)n * sizeof(double));
  int32_t* alias = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int32_t* small = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int32_t* large = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  if (!prob || !alias || !small || !large) { free(prob); free(alias); free(small); free(large); return -2; }
  double tot = 0.0;
  for (int64_t v = 0; v < n; ++v) tot += weight[v];
  int64_t ns = 0, nl = 0;
  for (int64_t v = 0; v < n; ++v) {
    prob[v] = weight[v] * (double)n / tot;
    alias[v] = (int32_t)v;
    if (prob[v] < 1.0) small[ns++] = (int32_t)v; else large[nl++] = (int32_t)v;
  }
  while (ns > 0 && nl > 0) {
    int32_t sm = small[--ns], lg = large[--nl];
    alias[sm] = lg;
    prob[lg] = (prob[lg] + prob[sm]) - 1.0;
    if (prob[lg] < 1.0) small[ns++] = lg; else large[nl++] = lg;
  }
  while (nl > 0) prob[large[--nl]] = 1.0;
  while (ns > 0) prob[small[--ns]] = 1.0;
  free(small); free(large);

  int fail = 0;
  #pragma omp parallel
  {
    int64_t cap = 0;
    int32_t* buf = NULL;
    #pragma omp for schedule(dynamic, 256)
    for (int64_t v = 0; v < n; ++v) {
      int64_t d = row_ptr[v + 1] - row_ptr[v];
      if (d <= 0) continue;
      if (2 * d + 64 > cap) {
        cap = 2 * d + 64;
        int32_t* nb = (int32_t*)realloc(buf, (size_t)cap * sizeof(int32_t));
        if (!nb) { fail = 1; continue; }
        buf = nb;
      }
      int64_t have = 0;
      uint64_t ctr = 0;
      for (int round = 0; round < 64 && have < d; ++round) {
        int64_t want = d - have;
        for (int64_t t = 0; t < want; ++t) {
          uint64_t r = rng(seed ^ (uint64_t)v * 0x9E3779B97F4A7C15ull, STREAM_COL, ctr++);
          int64_t b = (int64_t)((r >> 32) % (uint64_t)n);
          double coin = (double)(r & 0xFFFFFFFFull) * 0x1.0p-32;
          buf[have + t] = coin < prob[b] ? (int32_t)b : alias[b];
        }
        have += want;
        qsort(buf, (size_t)have, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t t = 0; t < have; ++t)
          if (u == 0 || buf[t] != buf[u - 1]) buf[u++] = buf[t];
        have = u;
      }
      if (have < d) {
        /* deterministic fill with the smallest unused columns (only for near-complete rows) */
        int64_t add = 0;
        int32_t* extra = buf + have;
        int64_t p = 0;
        for (int32_t c = 0; c < (int32_t)n && have + add < d; ++c) {
          while (p < have && buf[p] < c) ++p;
          if (p < have && buf[p] == c) continue;
          extra[add++] = c;
        }
        have += add;
        qsort(buf, (size_t)have, sizeof(int32_t), cmp_i32);
      }
      memcpy(col_out + row_ptr[v], buf, (size_t)d * sizeof(int32_t));
    }
    free(buf);
  }
  free(prob); free(alias);
  return fail ? -2 : 0;
}

/* val[e] = 1/deg(row) for every edge of every row (mean aggregator) */
void synth_mean_values(int64_t n, const int64_t* row_ptr, float* val) {
  #pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    int64_t b = row_ptr[v], e = row_ptr[v + 1];
    float x = e > b ? (float)(1.0 / (double)(e - b)) : 0.0f;
    for (int64_t t = b; t < e; ++t) val[t] = x;
  }
}

/* iid N(0,1) fp32, Box–Muller on counter pairs: global element e = start + i takes z0 (e even) or z1
   (e odd) of pair e/2, so any slice [start, start+count) equals the same slice of the whole matrix */
void synth_normal_f32(uint64_t seed, int64_t start, int64_t count, float* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const int64_t e = start + i, p = e >> 1;
    uint64_t a = rng(seed, STREAM_NORMAL, 2 * (uint64_t)p), b = rng(seed, STREAM_NORMAL, 2 * (uint64_t)p + 1);
    double u1 = ((double)(a >> 11) + 0.5) * 0x1.0p-53;   /* (0,1) */
    double u2 = (double)(b >> 11) * 0x1.0p-53;
    double rad = sqrt(-2.0 * log(u1));
    double ang = 6.283185307179586 * u2;
    out[i] = (float)((e & 1) ? rad * sin(ang) : rad * cos(ang));
  }
}

int synth_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
